// C ABI over the taskmap C++ API (include/taskmap_b200.h).  No exception
// crosses this boundary: every entry point maps taskmap::Error to a status
// code and stores the message for tm_last_error().
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "json.hpp"
#include "plan.hpp"
#include "taskmap/ir.hpp"
#include "taskmap/schedule.hpp"
#include "taskmap_b200.h"
#include "tune.hpp"

using namespace taskmap;

struct tm_plan {
  std::unique_ptr<tmb::Plan> p;
};
struct tm_exec {
  std::unique_ptr<tmb::Exec> e;
};
struct tm_mapping {
  TaskMapping m;
};

namespace {
thread_local std::string g_err;

// taskmap::Error and its typed refinements (taskmap/ir.hpp) -> tm_status; the
// message goes to tm_last_error().  The exception type decides the code.
template <class F>
tm_status guarded(F&& f) {
  try {
    g_err.clear();
    return f();
  } catch (const CorrectnessError& e) {
    g_err = e.what();
    return TM_ERR_CORRECTNESS;
  } catch (const UnsupportedError& e) {
    g_err = e.what();
    return TM_ERR_UNSUPPORTED;
  } catch (const CudaError& e) {
    g_err = e.what();
    return TM_ERR_CUDA;
  } catch (const Error& e) {
    g_err = e.what();
    return TM_ERR_USAGE;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return TM_ERR_USAGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TM_ERR_USAGE;
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

ScheduleConfig from_c(const tm_schedule_config* c) {
  ScheduleConfig s;
  if (!c) return s;
  s.block_m = c->block_m ? c->block_m : 128;
  s.block_n = c->block_n ? c->block_n : 128;
  s.block_k = c->block_k ? c->block_k : 64;
  s.warp_m = c->warp_m;
  s.warp_n = c->warp_n;
  s.threads_per_block = c->threads_per_block;
  s.pipeline = c->pipeline != 0;
  s.split_k = c->split_k ? c->split_k : 1;
  s.stages = c->stages;
  s.raster = c->raster;
  s.grid = c->grid;
  static const char* maths[] = {"auto", "bf16", "tf32", "fp32_simt", "halo"};
  s.math = maths[(c->math >= 0 && c->math <= 4) ? c->math : 0];
  if (!s.pipeline) s.stages = 2;
  return s;
}

void to_c(const ScheduleConfig& s, tm_schedule_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->block_m = s.block_m;
  c->block_n = s.block_n;
  c->block_k = s.block_k;
  c->warp_m = s.warp_m;
  c->warp_n = s.warp_n;
  c->threads_per_block = s.threads_per_block;
  c->pipeline = s.pipeline;
  c->split_k = s.split_k;
  c->stages = s.stages;
  c->raster = s.raster;
  c->grid = s.grid;
  c->math = s.math == "bf16" ? 1 : s.math == "tf32" ? 2 : s.math == "fp32_simt" ? 3 : s.math == "halo" ? 4 : 0;
}
}  // namespace

extern "C" {

const char* tm_last_error(void) { return g_err.c_str(); }
const char* tm_version(void) { return "taskmap_b200 0.1 (sm_100a)"; }
void tm_free(void* p) { std::free(p); }

// ------------------------------------------------------------ mappings --
tm_status tm_mapping_parse(const char* text, tm_mapping** out) {
  return guarded([&] {
    if (!text || !out) fail("null argument");
    *out = new tm_mapping{parse_mapping(text)};
    return TM_OK;
  });
}

void tm_mapping_free(tm_mapping* m) { delete m; }

tm_status tm_mapping_info(const tm_mapping* m, uint64_t* nw, uint64_t* dim, uint64_t* tpw, uint64_t* shape) {
  return guarded([&] {
    if (!m) fail("null mapping");
    if (nw) *nw = m->m.num_workers();
    if (dim) *dim = m->m.task_dim();
    if (tpw) *tpw = m->m.tasks_per_worker();
    if (shape)
      for (size_t i = 0; i < m->m.task_dim(); ++i) shape[i] = m->m.task_shape()[i];
    return TM_OK;
  });
}

tm_status tm_mapping_assign(const tm_mapping* m, uint64_t worker, uint64_t* buf, size_t cap, size_t* n) {
  return guarded([&] {
    if (!m) fail("null mapping");
    const auto tasks = m->m.assign(worker);
    const size_t dim = m->m.task_dim();
    if (n) *n = tasks.size();
    if (tasks.size() * dim > cap) fail("buffer too small: need ", tasks.size() * dim);
    for (size_t i = 0; i < tasks.size(); ++i)
      for (size_t d = 0; d < dim; ++d) buf[i * dim + d] = tasks[i][d];
    return TM_OK;
  });
}

tm_status tm_mapping_text(const tm_mapping* m, int visualize, char** out) {
  return guarded([&] {
    if (!m || !out) fail("null argument");
    *out = dup(visualize ? m->m.visualize() : m->m.to_text());
    return TM_OK;
  });
}

tm_status tm_mapping_lowered_assign(const tm_mapping* m, uint64_t worker, uint64_t* buf, size_t cap,
                                    size_t* n) {
  return guarded([&] {
    if (!m) fail("null mapping");
    const auto atoms = m->m.atoms();
    if (atoms.size() > static_cast<size_t>(tmb::tm::kMaxAtoms)) fail("too many atoms for DevMapping");
    const size_t dim = m->m.task_dim();
    if (dim > static_cast<size_t>(tmb::tm::kMaxRank)) fail("task dimension too large for DevMapping");
    tmb::tm::DevMapping d{};
    d.n_atoms = static_cast<int32_t>(atoms.size());
    d.rank = static_cast<int32_t>(dim);
    d.workers = 1;
    d.tasks = 1;
    for (size_t a = 0; a < atoms.size(); ++a) {
      d.is_spatial[a] = atoms[a].spatial;
      uint64_t vol = 1;
      for (size_t i = 0; i < dim; ++i) {
        d.dims[a][i] = static_cast<int32_t>(atoms[a].dims[i]);
        vol *= atoms[a].dims[i];
      }
      (atoms[a].spatial ? d.workers : d.tasks) *= static_cast<uint32_t>(vol);
    }
    if (worker >= d.workers) fail("worker id ", worker, " out of range for ", d.workers, " workers");
    if (n) *n = d.tasks;
    if (d.tasks * dim > cap) fail("buffer too small");
    for (uint32_t i = 0; i < d.tasks; ++i) {
      int32_t c[tmb::tm::kMaxRank];
      tmb::tm::dev_task(d, static_cast<uint32_t>(worker), i, c);
      for (size_t k = 0; k < dim; ++k) buf[i * dim + k] = static_cast<uint64_t>(c[k]);
    }
    return TM_OK;
  });
}

tm_status tm_kernel_mapping_assign(int32_t which, uint64_t worker, uint64_t* buf, size_t cap, size_t* n) {
  return guarded([&] {
    std::vector<int> tmp(4096);
    const int k = tmb::kernel_mapping_assign(which, static_cast<uint32_t>(worker), tmp.data(), 4096);
    if (k < 0) fail("bad kernel mapping id or worker");
    if (static_cast<size_t>(2 * k) > cap) fail("buffer too small");
    for (int i = 0; i < 2 * k; ++i) buf[i] = static_cast<uint64_t>(tmp[i]);
    if (n) *n = static_cast<size_t>(k);
    return TM_OK;
  });
}

// ----------------------------------------------------------------- DAG --
tm_status tm_classify(const char* dag_json, const char* node, int32_t* cls) {
  return guarded([&] {
    ComputeDAG d = dag_from_json(dag_json);
    *cls = static_cast<int32_t>(classify(d, d.at(node)));
    return TM_OK;
  });
}

tm_status tm_partition(const char* dag_json, char** out) {
  return guarded([&] {
    ComputeDAG d = dag_from_json(dag_json);
    std::string s = "[";
    bool first = true;
    for (const auto& sg : partition(d)) {
      s += first ? "{" : ",{";
      first = false;
      s += "\"anchor\":" + tmjson::quote(sg.anchor) + ",\"prologue\":[";
      for (size_t i = 0; i < sg.prologue.size(); ++i) s += (i ? "," : "") + tmjson::quote(sg.prologue[i]);
      s += "],\"epilogue\":[";
      for (size_t i = 0; i < sg.epilogue.size(); ++i) s += (i ? "," : "") + tmjson::quote(sg.epilogue[i]);
      s += "],\"output\":" + tmjson::quote(sg.output) + "}";
    }
    *out = dup(s + "]");
    return TM_OK;
  });
}

// kind / args:
//   matmul        m, n, k, dtype(0 f32, 1 i32)
//   conv2d_im2col n, c, h, w, f, kh, kw, stride, pad, dtype
//   batchnorm     n, c, h, w, dtype
//   transpose     dtype, rank, shape..., perm...
//   reshape       dtype, rank_in, in..., rank_out, out...
tm_status tm_build_dag(const char* kind, const int64_t* a, int32_t n, char** out) {
  return guarded([&] {
    const std::string k = kind;
    auto dt = [&](int64_t v) { return v ? DType::I32 : DType::F32; };
    auto need = [&](int32_t m) { if (n < m) fail("tm_build_dag(", k, "): expected at least ", m, " args"); };
    ComputeDAG d;
    if (k == "matmul") {
      need(4);
      d = matmul_dag(a[0], a[1], a[2], dt(a[3]));
    } else if (k == "conv2d_im2col") {
      need(10);
      d = conv2d_im2col_dag(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], dt(a[9]));
    } else if (k == "batchnorm") {
      need(5);
      d = batchnorm_inference_dag(a[0], a[1], a[2], a[3], dt(a[4]));
    } else if (k == "transpose") {
      need(2);
      const int64_t r = a[1];
      need(static_cast<int32_t>(2 + 2 * r));
      std::vector<int64_t> shape(a + 2, a + 2 + r);
      std::vector<size_t> perm(a + 2 + r, a + 2 + 2 * r);
      d = transpose_dag(shape, perm, dt(a[0]));
    } else if (k == "reshape") {
      need(2);
      const int64_t ri = a[1];
      need(static_cast<int32_t>(3 + ri));
      std::vector<int64_t> in(a + 2, a + 2 + ri);
      const int64_t ro = a[2 + ri];
      need(static_cast<int32_t>(3 + ri + ro));
      std::vector<int64_t> o(a + 3 + ri, a + 3 + ri + ro);
      d = reshape_dag(in, o, dt(a[0]));
    } else {
      fail("unknown builder '", k, "'");
    }
    *out = dup(dag_to_json(d));
    return TM_OK;
  });
}

// ---------------------------------------------------------- scheduling --
tm_status tm_schedule_space(const char* op_kind, tm_schedule_config* buf, int32_t cap, int32_t* n) {
  return guarded([&] {
    const auto sp = schedule_space(op_kind);
    if (n) *n = static_cast<int32_t>(sp.size());
    for (int32_t i = 0; i < cap && i < static_cast<int32_t>(sp.size()); ++i) to_c(sp[i], &buf[i]);
    return TM_OK;
  });
}

tm_status tm_plan_create(const char* dag_json, const tm_schedule_config* cfg, int32_t device, tm_plan** out) {
  return guarded([&] {
    if (!dag_json || !out) fail("null argument");
    ComputeDAG d = dag_from_json(dag_json);
    *out = new tm_plan{tmb::build_plan(d, from_c(cfg), device)};
    return TM_OK;
  });
}

void tm_plan_destroy(tm_plan* p) { delete p; }

tm_status tm_plan_describe(const tm_plan* p, char** out) {
  return guarded([&] {
    std::string s = "{\"config\":" + p->p->cfg.to_json() + ",\"kernels\":[";
    for (size_t i = 0; i < p->p->kernels.size(); ++i) s += (i ? "," : "") + p->p->kernels[i].describe();
    s += "],\"intermediates\":[";
    for (size_t i = 0; i < p->p->intermediates.size(); ++i) s += (i ? "," : "") + tmjson::quote(p->p->intermediates[i]);
    *out = dup(s + "]}");
    return TM_OK;
  });
}

tm_status tm_exec_create(const tm_plan* p, const tm_tensor* in, int32_t n_in, const tm_tensor* out, int32_t n_out,
                         tm_exec** ex) {
  return guarded([&] {
    if (!p || !ex) fail("null argument");
    if (cudaSetDevice(p->p->device) != cudaSuccess) fail_cuda("cudaSetDevice failed");
    *ex = new tm_exec{tmb::bind_plan(*p->p, in, n_in, out, n_out)};
    return TM_OK;
  });
}

void tm_exec_destroy(tm_exec* e) { delete e; }

tm_status tm_exec_launch(const tm_exec* e, void* stream) {
  return guarded([&] {
    if (!e) fail("null exec");
    for (const auto& k : e->e->kernels) tmb::launch_bound(k, stream);
    return TM_OK;
  });
}

int32_t tm_exec_num_launches(const tm_exec* e) { return e ? static_cast<int32_t>(e->e->kernels.size()) : 0; }

tm_status tm_exec_kernel_info(const tm_exec* e, int32_t index, int32_t* grid, int32_t* cg, int32_t* bn, int32_t* sk,
                              int32_t* al, int32_t* bl) {
  return guarded([&] {
    if (!e || index < 0 || index >= static_cast<int32_t>(e->e->kernels.size())) fail("bad kernel index");
    const auto& k = e->e->kernels[index];
    if (grid) *grid = k.grid;
    if (cg) *cg = k.cg;
    if (bn) *bn = k.bn;
    if (sk) *sk = k.p.split_k;
    if (al) *al = k.p.a_loader;
    if (bl) *bl = k.p.b_loader;
    return TM_OK;
  });
}

tm_status tm_exec_kernel_kind(const tm_exec* e, int32_t index, int32_t* kind) {
  return guarded([&] {
    if (!e || index < 0 || index >= static_cast<int32_t>(e->e->kernels.size())) fail("bad kernel index");
    if (!kind) fail("null kind pointer");
    const auto& k = e->e->kernels[index];
    *kind = k.rule ? (k.rfn ? TM_KIND_RULE_GENERATED : TM_KIND_RULE_INTERP)
            : k.simt ? TM_KIND_SIMT
            : k.rowband == 2 ? TM_KIND_HALO
            : k.rowband ? TM_KIND_ROWBAND
                        : TM_KIND_GEMM;
    return TM_OK;
  });
}

tm_status tm_exec_trace(const tm_exec* e, int32_t index, int64_t* buf, size_t cap) {
  return guarded([&] {
    if (!e || index < 0 || index >= static_cast<int32_t>(e->e->kernels.size())) fail("bad kernel index");
    const auto& k = e->e->kernels[index];
    if (!k.p.trace) fail("exec was not created with TMB_TRACE set");
    const size_t n = size_t(k.grid) * tmb::kTraceTiles * tmb::kTraceEvents;
    if (cap < n) fail("trace buffer too small: need ", n);
    if (cudaMemcpy(buf, k.p.trace, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) fail_cuda("cuda memcpy failed");
    return TM_OK;
  });
}

// ---- CUDA graphs: a sequence of bound execs replayed with one launch ----
struct tm_graph {
  cudaGraphExec_t exec = nullptr;
  std::vector<cudaEvent_t> marks;  // timed graphs: one event before each exec + one at the end
  ~tm_graph() {
    if (exec) cudaGraphExecDestroy(exec);
    for (auto ev : marks) cudaEventDestroy(ev);
  }
};

tm_status tm_graph_create(const tm_exec* const* execs, int32_t n, int32_t timed, tm_graph** out) {
  return guarded([&] {
    if (!out || n < 0 || (n > 0 && !execs)) fail("tm_graph_create: bad arguments");
    auto g = std::make_unique<tm_graph>();
    auto ck = [](cudaError_t e, const char* what) {
      if (e != cudaSuccess) fail_cuda(what, " failed: cuda error ", cudaGetErrorString(e));
    };
    if (timed) {
      g->marks.resize(static_cast<size_t>(n) + 1);
      for (auto& ev : g->marks) ck(cudaEventCreate(&ev), "cudaEventCreate");
    }
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    cudaGraph_t graph = nullptr;
    ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    try {
      for (int32_t i = 0; i < n; ++i) {
        if (!execs[i]) fail("tm_graph_create: null exec");
        if (timed) ck(cudaEventRecordWithFlags(g->marks[i], s, cudaEventRecordExternal), "cudaEventRecord");
        for (const auto& k : execs[i]->e->kernels) tmb::launch_bound(k, s);
      }
      if (timed) ck(cudaEventRecordWithFlags(g->marks[n], s, cudaEventRecordExternal), "cudaEventRecord");
    } catch (...) {
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      cudaStreamDestroy(s);
      throw;
    }
    ck(cudaStreamEndCapture(s, &graph), "cudaStreamEndCapture");
    const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(s);
    ck(ie, "cudaGraphInstantiate");
    *out = g.release();
    return TM_OK;
  });
}

tm_status tm_graph_launch(const tm_graph* g, void* stream) {
  return guarded([&] {
    if (!g) fail("null graph");
    const cudaError_t e = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) fail_cuda("cudaGraphLaunch failed: cuda error ", cudaGetErrorString(e));
    return TM_OK;
  });
}

tm_status tm_graph_exec_ms(const tm_graph* g, float* ms, int32_t n) {
  return guarded([&] {
    if (!g || g->marks.empty()) fail("tm_graph_exec_ms: graph was not created with timed = 1");
    if (!ms || n != static_cast<int32_t>(g->marks.size()) - 1) fail("tm_graph_exec_ms: n must equal the exec count");
    for (int32_t i = 0; i < n; ++i) {
      const cudaError_t e = cudaEventElapsedTime(&ms[i], g->marks[i], g->marks[i + 1]);
      if (e != cudaSuccess) fail_cuda("cudaEventElapsedTime failed: cuda error ", cudaGetErrorString(e));
    }
    return TM_OK;
  });
}

void tm_graph_destroy(tm_graph* g) { delete g; }

tm_status tm_plan_launch(const tm_plan* p, const tm_tensor* in, int32_t n_in, const tm_tensor* out, int32_t n_out,
                         void* stream) {
  return guarded([&] {
    auto e = tmb::bind_plan(*p->p, in, n_in, out, n_out);
    for (const auto& k : e->kernels) tmb::launch_bound(k, stream);
    if (!e->scratch.empty() && cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess)
      fail_cuda("cuda stream synchronize failed");
    return TM_OK;
  });
}

// tune: see tune.cpp.  The TuneReport is returned through
// *report also when the gate fails (status TM_ERR_CORRECTNESS).
tm_status tm_tune(const char* dag_json, const tm_tensor* in, int32_t n_in, const tm_tensor* out, int32_t n_out,
                  int32_t device, int32_t reps, tm_schedule_config* best, char** report) {
  return guarded([&] {
    if (!dag_json) fail("null argument");
    ComputeDAG d = dag_from_json(dag_json);
    tmb::TuneOutcome r = tmb::tune(d, in, n_in, out, n_out, device, reps);
    if (report) *report = dup(r.report);
    if (!r.ok) {
      if (r.unsupported) fail_unsupported(r.error);
      fail_as<CorrectnessError>(r.error);
    }
    if (best) to_c(r.best, best);
    return TM_OK;
  });
}

// Device DAG interpreter (reference_eval semantics, dev_eval.hpp): evaluates
// the DAG and writes its outputs, rounded to each output's dtype.
tm_status tm_dag_eval(const char* dag_json, const tm_tensor* in, int32_t n_in, const tm_tensor* out, int32_t n_out,
                      int32_t device, void* stream) {
  return guarded([&] {
    if (!dag_json || (n_out > 0 && !out)) fail("null argument");
    ComputeDAG d = dag_from_json(dag_json);
    auto r = tmb::dag_eval(d, in, n_in, out, n_out, device, stream);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int i = 0; i < n_out; ++i) {
      const std::string& o = d.outputs[i];
      if (tmb::ev::numel_of(out[i]) != r->numel(o)) fail("tm_dag_eval: output '", o, "' has the wrong size");
      tmb::ev::launch_store(r->values(o), r->is_float(o), r->numel(o), out[i].data, out[i].dtype, out[i].rank,
                            tmb::ev::shape_of(out[i]), s);
    }
    tmb::sync_with_timeout(s, 60.0, "tm_dag_eval");
    return TM_OK;
  });
}

}  // extern "C"
