// TEST INFRASTRUCTURE ONLY — the oracle.  Never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/.
// It exposes:
//   ref_eval        taskmap::reference_eval (proj/src/compute_ir.cpp:418-466)
//                   on a DAG given in the repo's JSON wire form
//   ref_classify    taskmap::classify (compute_ir.cpp:222-243)
//   ref_mapping_*   TaskMapping parse/assign/text/visualize (mapping.cpp)
//   ref_random      taskmap::random_tensor with the splitmix64 Rng (tensor.cpp:42-69)
//   ref_fold_bn     fold_batchnorm_params (compute_ir.cpp:721-733)
//   ref_build       reference builders -> JSON (compute_ir.cpp:496-733)
// Only this file is ours; the reference sources are compiled where they lie.
#include <cstring>
#include <string>
#include <vector>

#include "taskmap/compute_ir.hpp"
#include "taskmap/mapping.hpp"
#include "taskmap/tensor.hpp"
#include "../paper_2210_09603_b200/csrc/host/json.hpp"

using namespace taskmap;

namespace {

void set_err(char* err, int cap, const std::string& m) {
  if (err && cap > 0) {
    std::strncpy(err, m.c_str(), cap - 1);
    err[cap - 1] = 0;
  }
}

const char* kBin[] = {"add", "sub", "mul", "div", "mod", "min", "max", "and", "or", "lt", "le", "gt", "ge", "eq", "ne"};
const char* kUn[] = {"neg", "relu", "exp", "sqrt", "f32", "i32"};

Expr to_expr(const tmjson::Value& v) {
  const auto& a = v.arr();
  const std::string& op = a.at(0).str();
  if (op == "i") return imm(a.at(1).integer());
  if (op == "f") return fimm(a.at(1).num());
  if (op == "v") return var(a.at(1).str());
  if (op == "tid") return thread_idx();
  if (op == "bid") return block_idx();
  if (op == "select") return select(to_expr(a.at(1)), to_expr(a.at(2)), to_expr(a.at(3)));
  if (op == "load") {
    std::vector<Expr> idx;
    for (size_t i = 2; i < a.size(); ++i) idx.push_back(to_expr(a[i]));
    return load(a.at(1).str(), idx);
  }
  if (op == "lookup") {
    auto t = std::make_shared<std::vector<int64_t>>();
    for (const auto& x : a.at(1).arr()) t->push_back(x.integer());
    return table_lookup(t, to_expr(a.at(2)));
  }
  for (int i = 0; i < 15; ++i)
    if (op == kBin[i]) return binary(static_cast<BinOp>(i), to_expr(a.at(1)), to_expr(a.at(2)));
  for (int i = 0; i < 6; ++i)
    if (op == kUn[i]) return unary(static_cast<UnOp>(i), to_expr(a.at(1)));
  fail("unknown op ", op);
}

std::vector<Axis> to_axes(const tmjson::Value* v) {
  std::vector<Axis> out;
  if (v)
    for (const auto& a : v->arr()) out.push_back({a.arr().at(0).str(), a.arr().at(1).integer()});
  return out;
}

ComputeDAG to_dag(const char* text) {
  const tmjson::Value root = tmjson::parse(text);
  ComputeDAG d;
  for (const auto& nv : root.at("nodes").arr()) {
    TensorNode n;
    n.name = nv.at("name").str();
    for (const auto& s : nv.at("shape").arr()) n.shape.push_back(s.integer());
    if (const auto* dt = nv.get("dtype")) n.dtype = dtype_from_name(dt->str());
    const std::string kind = nv.get("kind") ? nv.at("kind").str() : "input";
    if (kind != "input") {
      n.kind = kind == "reduce" ? NodeKind::GridReduce : NodeKind::GridCompute;
      n.axes = to_axes(nv.get("axes"));
      n.reduce_axes = to_axes(nv.get("reduce_axes"));
      if (const auto* c = nv.get("combiner")) n.combiner = combiner_from_name(c->str());
      n.value = to_expr(nv.at("value"));
    }
    d.nodes.push_back(std::move(n));
  }
  for (const auto& s : root.at("inputs").arr()) d.inputs.push_back(s.str());
  for (const auto& s : root.at("outputs").arr()) d.outputs.push_back(s.str());
  return d;
}

// JSON writer for reference-built DAGs (so the product's builders can be
// compared with the reference's, node by node).
void expr_out(std::string& o, const Expr& e) {
  switch (e->kind) {
    case ExprKind::IntImm: o += "[\"i\"," + std::to_string(e->ival) + "]"; return;
    case ExprKind::FloatImm: { char b[40]; std::snprintf(b, sizeof b, "%.17g", e->fval); std::string s = b;
      if (s.find_first_of(".eni") == std::string::npos) s += ".0"; o += "[\"f\"," + s + "]"; return; }
    case ExprKind::Var: o += "[\"v\"," + tmjson::quote(e->name) + "]"; return;
    case ExprKind::ThreadIdx: o += "[\"tid\"]"; return;
    case ExprKind::BlockIdx: o += "[\"bid\"]"; return;
    case ExprKind::Binary: o += std::string("[\"") + kBin[static_cast<int>(e->bop)] + "\""; break;
    case ExprKind::Unary: o += std::string("[\"") + kUn[static_cast<int>(e->uop)] + "\""; break;
    case ExprKind::Select: o += "[\"select\""; break;
    case ExprKind::Load: o += "[\"load\"," + tmjson::quote(e->name); break;
    case ExprKind::TableLookup: o += "[\"lookup\",["; for (size_t i = 0; i < e->table->size(); ++i) o += (i ? "," : "") + std::to_string((*e->table)[i]); o += "]"; break;
  }
  for (const auto& a : e->args) { o += ","; expr_out(o, a); }
  o += "]";
}

std::string dag_out(const ComputeDAG& d) {
  std::string o = "{\"nodes\":[";
  for (size_t i = 0; i < d.nodes.size(); ++i) {
    const auto& n = d.nodes[i];
    o += (i ? ",{" : "{");
    o += "\"name\":" + tmjson::quote(n.name) + ",\"shape\":[";
    for (size_t j = 0; j < n.shape.size(); ++j) o += (j ? "," : "") + std::to_string(n.shape[j]);
    o += std::string("],\"dtype\":\"") + dtype_name(n.dtype) + "\"";
    if (n.kind == NodeKind::Input) { o += ",\"kind\":\"input\"}"; continue; }
    o += n.kind == NodeKind::GridReduce ? ",\"kind\":\"reduce\"" : ",\"kind\":\"compute\"";
    auto ax = [&](const char* k, const std::vector<Axis>& v) {
      o += std::string(",\"") + k + "\":[";
      for (size_t j = 0; j < v.size(); ++j) o += (j ? "," : "") + std::string("[") + tmjson::quote(v[j].name) + "," + std::to_string(v[j].extent) + "]";
      o += "]";
    };
    ax("axes", n.axes);
    if (n.kind == NodeKind::GridReduce) { ax("reduce_axes", n.reduce_axes); o += std::string(",\"combiner\":\"") + combiner_name(n.combiner) + "\""; }
    o += ",\"value\":";
    expr_out(o, n.value);
    o += "}";
  }
  o += "],\"inputs\":[";
  for (size_t i = 0; i < d.inputs.size(); ++i) o += (i ? "," : "") + tmjson::quote(d.inputs[i]);
  o += "],\"outputs\":[";
  for (size_t i = 0; i < d.outputs.size(); ++i) o += (i ? "," : "") + tmjson::quote(d.outputs[i]);
  return o + "]}";
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

// Evaluates dag with reference_eval.  Inputs/outputs are row-major doubles in
// the DAG's logical shapes (i32 tensors converted exactly).  Returns 0 on
// success, 1 on a reference error (message in err).
int ref_eval(const char* dag_json, int n_in, const char** in_names, const double** in_data, int n_out,
             const char** out_names, double** out_data, char* err, int errcap) {
  try {
    ComputeDAG d = to_dag(dag_json);
    TensorMap inputs;
    for (int i = 0; i < n_in; ++i) {
      const TensorNode& n = d.at(in_names[i]);
      Tensor t = Tensor::zeros(n.dtype, n.shape);
      const int64_t sz = t.size();
      if (t.is_float()) for (int64_t j = 0; j < sz; ++j) t.fdata[j] = in_data[i][j];
      else for (int64_t j = 0; j < sz; ++j) t.idata[j] = static_cast<int64_t>(in_data[i][j]);
      inputs[in_names[i]] = std::move(t);
    }
    ComputeDAG dd = d;
    dd.outputs.clear();
    for (int i = 0; i < n_out; ++i) dd.outputs.push_back(out_names[i]);
    TensorMap res = reference_eval(dd, inputs);
    for (int i = 0; i < n_out; ++i) {
      const Tensor& t = res.at(out_names[i]);
      const int64_t sz = t.size();
      if (t.is_float()) for (int64_t j = 0; j < sz; ++j) out_data[i][j] = t.fdata[j];
      else for (int64_t j = 0; j < sz; ++j) out_data[i][j] = static_cast<double>(t.idata[j]);
    }
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

int ref_classify(const char* dag_json, const char* node, int* out, char* err, int errcap) {
  try {
    ComputeDAG d = to_dag(dag_json);
    *out = static_cast<int>(classify(d, d.at(node)));
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

int ref_validate(const char* dag_json, char* err, int errcap) {
  try {
    to_dag(dag_json).validate();
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

int ref_mapping_info(const char* text, uint64_t* workers, uint64_t* dim, uint64_t* tpw, uint64_t* shape,
                     char* err, int errcap) {
  try {
    TaskMapping m = parse_mapping(text);
    *workers = m.num_workers();
    *dim = m.task_dim();
    *tpw = m.tasks_per_worker();
    for (size_t i = 0; i < m.task_dim(); ++i) shape[i] = m.task_shape()[i];
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

int ref_mapping_assign(const char* text, uint64_t worker, uint64_t* buf, uint64_t cap, uint64_t* n,
                       char* err, int errcap) {
  try {
    TaskMapping m = parse_mapping(text);
    auto tasks = m.assign(worker);
    *n = tasks.size();
    const size_t dim = m.task_dim();
    if (tasks.size() * dim > cap) { set_err(err, errcap, "buffer too small"); return 2; }
    for (size_t i = 0; i < tasks.size(); ++i)
      for (size_t k = 0; k < dim; ++k) buf[i * dim + k] = tasks[i][k];
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

int ref_mapping_text(const char* text, int visualize, char* buf, int cap, char* err, int errcap) {
  try {
    TaskMapping m = parse_mapping(text);
    const std::string s = visualize ? m.visualize() : m.to_text();
    if (static_cast<int>(s.size()) + 1 > cap) { set_err(err, errcap, "buffer too small"); return 2; }
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

// compose() of two parsed mappings (exercises the rank-mismatch error path)
int ref_mapping_compose_text(const char* a, const char* b, char* buf, int cap, char* err, int errcap) {
  try {
    TaskMapping m = TaskMapping::compose(parse_mapping(a), parse_mapping(b));
    const std::string s = m.to_text();
    if (static_cast<int>(s.size()) + 1 > cap) return 2;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

// random_tensor(f32 -> U(-1,1), i32 -> U{-8..8}) from Rng(seed), continuing
// the stream across calls via *state (pass the seed-initialised state first).
void ref_rng_init(uint64_t seed, uint64_t* state) { *state = Rng(seed).state; }

void ref_random(uint64_t* state, int is_int, int64_t n, double* out) {
  Rng r(1);
  r.state = *state;
  Tensor t = random_tensor(is_int ? DType::I32 : DType::F32, {n}, r);
  for (int64_t i = 0; i < n; ++i) out[i] = is_int ? static_cast<double>(t.idata[i]) : t.fdata[i];
  *state = r.state;
}

void ref_fold_bn(int64_t c, const double* gamma, const double* beta, const double* mean, const double* var_,
                 double eps, double* scale, double* shift) {
  auto mk = [&](const double* p) {
    Tensor t = Tensor::zeros(DType::F32, {c});
    for (int64_t i = 0; i < c; ++i) t.fdata[i] = p[i];
    return t;
  };
  auto [s, h] = fold_batchnorm_params(mk(gamma), mk(beta), mk(mean), mk(var_), eps);
  for (int64_t i = 0; i < c; ++i) {
    scale[i] = s.fdata[i];
    shift[i] = h.fdata[i];
  }
}

// Reference builders -> JSON (same argument layout as tm_build_dag).
int ref_build(const char* kind, const int64_t* a, int n, char* buf, int cap, char* err, int errcap) {
  try {
    const std::string k = kind;
    auto dt = [&](int64_t v) { return v ? DType::I32 : DType::F32; };
    ComputeDAG d;
    if (k == "matmul") d = matmul_dag(a[0], a[1], a[2], dt(a[3]));
    else if (k == "conv2d_im2col") d = conv2d_im2col_dag(a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], dt(a[9]));
    else if (k == "batchnorm") d = batchnorm_inference_dag(a[0], a[1], a[2], a[3], dt(a[4]));
    else if (k == "transpose") {
      const int64_t r = a[1];
      d = transpose_dag(std::vector<int64_t>(a + 2, a + 2 + r), std::vector<size_t>(a + 2 + r, a + 2 + 2 * r), dt(a[0]));
    } else if (k == "reshape") {
      const int64_t ri = a[1], ro = a[2 + ri];
      d = reshape_dag(std::vector<int64_t>(a + 2, a + 2 + ri), std::vector<int64_t>(a + 3 + ri, a + 3 + ri + ro), dt(a[0]));
    } else { set_err(err, errcap, "unknown builder"); return 1; }
    (void)n;
    const std::string s = dag_out(d);
    if (static_cast<int>(s.size()) + 1 > cap) { set_err(err, errcap, "buffer too small"); return 2; }
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errcap, e.what());
    return 1;
  }
}

}  // extern "C"
#pragma GCC visibility pop
