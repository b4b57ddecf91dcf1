/* taskmap_b200 — C ABI of the B200 task-mapping tensor-program library.
 *
 * The reference (arXiv 2210.09603 re-creation, /root/reference/proj) exposes
 * only a C++ header API in namespace taskmap and has no FFI.  This header is
 * the thin C layer the north star asks for underneath that API: plain
 * pointers, sizes and status codes, no exceptions and no torch types.  Each
 * entry point names the reference interface (file:line) or spec operation it
 * stands for.
 *
 * Status codes mirror the spec CLI's exit codes: 0 ok,
 * 1 correctness failure, 2 usage error; plus CUDA and "unsupported".
 * Messages are retrieved with tm_last_error() (thread-local), the analogue of
 * taskmap::Error::what() (proj/include/taskmap/common.hpp:10-19).
 */
#ifndef TASKMAP_B200_H_
#define TASKMAP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TM_OK = 0,
  TM_ERR_CORRECTNESS = 1,
  TM_ERR_USAGE = 2,
  TM_ERR_CUDA = 3,
  TM_ERR_UNSUPPORTED = 4
} tm_status;

/* Physical element types of bound tensors. */
typedef enum { TM_F32 = 0, TM_BF16 = 1, TM_F16 = 2 } tm_dtype;

#define TM_MAX_RANK 8

/* A strided tensor view: element (i0..i_{r-1}) lives at
 * data + sum_d i_d * stride[d] elements.  Logical shape follows the DAG node
 * (e.g. NCHW for conv inputs); strides may describe any physical layout
 * (channels-last etc.). `data` is a device pointer for launches. */
typedef struct {
  void* data;
  int32_t dtype;
  int32_t rank;
  int64_t shape[TM_MAX_RANK];
  int64_t stride[TM_MAX_RANK];
} tm_tensor;

/* ScheduleConfig + Blackwell fields; see taskmap/schedule.hpp. */
typedef struct {
  int32_t block_m, block_n, block_k, warp_m, warp_n, threads_per_block;
  int32_t pipeline, split_k;
  int32_t stages, raster, grid;
  int32_t math; /* 0 auto, 1 bf16 (tcgen05 kind::f16), 2 tf32 (kind::tf32), 3 fp32 SIMT, 4 halo conv family */
} tm_schedule_config;

typedef struct tm_plan tm_plan;       /* compiled fused subgraphs of one DAG */
typedef struct tm_exec tm_exec;       /* a plan bound to concrete tensors */
typedef struct tm_mapping tm_mapping; /* a TaskMapping value */

const char* tm_last_error(void);
const char* tm_version(void);
void tm_free(void* p); /* frees strings returned through char** */

/* ---- task mappings: TaskMapping (proj/include/taskmap/mapping.hpp:38-90) ---- */
/* parse_mapping (mapping.hpp:88-90) */
tm_status tm_mapping_parse(const char* text, tm_mapping** out);
void tm_mapping_free(tm_mapping* m);
/* num_workers / task_dim / tasks_per_worker / task_shape (mapping.hpp:50-61) */
tm_status tm_mapping_info(const tm_mapping* m, uint64_t* num_workers, uint64_t* task_dim,
                          uint64_t* tasks_per_worker, uint64_t* shape /* >= task_dim */);
/* assign (mapping.hpp:57): row-major [n_tasks][task_dim] into buf */
tm_status tm_mapping_assign(const tm_mapping* m, uint64_t worker, uint64_t* buf, size_t cap,
                            size_t* n_tasks);
/* to_text / visualize (mapping.hpp:73-77); *out freed with tm_free */
tm_status tm_mapping_text(const tm_mapping* m, int visualize, char** out);
/* Closed-form lowering used by the kernels (device DevMapping), evaluated on
 * the host: must equal tm_mapping_assign bit for bit. */
tm_status tm_mapping_lowered_assign(const tm_mapping* m, uint64_t worker, uint64_t* buf,
                                    size_t cap, size_t* n_tasks);

/* Task lists of the compile-time mappings compiled into the fp32 CUDA-core
 * kernel (0: compute spatial(4,2)*repeat(2,2)*spatial(4,8)*repeat(4,4),
 * 1: A-tile load repeat(4,1)*spatial(32,8), 2: B-tile load
 * repeat(1,4)*spatial(8,32)), evaluated on the host. */
tm_status tm_kernel_mapping_assign(int32_t which, uint64_t worker, uint64_t* buf, size_t cap, size_t* n_tasks);

/* ---- compute DAG: ComputeDAG / classify (compute_ir.hpp:39-56) ---- */
/* classify (compute_ir.hpp:56): 0 reduction, 1 injective, 2 bijective */
tm_status tm_classify(const char* dag_json, const char* node, int32_t* op_class);
/* partition: JSON list of fused subgraphs */
tm_status tm_partition(const char* dag_json, char** out_json);
/* builders (compute_ir.hpp:92-114) -> DAG JSON; kind in {matmul, conv2d_im2col,
 * batchnorm, transpose, reshape}; args documented in capi.cpp */
tm_status tm_build_dag(const char* kind, const int64_t* args, int32_t n_args, char** out_json);

/* ---- scheduling / fusion / execution ---- */
/* schedule_space: writes up to cap configs, *n = space size */
tm_status tm_schedule_space(const char* op_kind, tm_schedule_config* buf, int32_t cap,
                            int32_t* n);
/* Partition + fuse the DAG into tcgen05 kernels (matmul_template +
 * fuse_prologue/fuse_epilogue). cfg NULL = default. */
tm_status tm_plan_create(const char* dag_json, const tm_schedule_config* cfg, int32_t device,
                         tm_plan** out);
void tm_plan_destroy(tm_plan* p);
/* JSON description of the fused kernels (loaders, epilogue ops, remaps). */
tm_status tm_plan_describe(const tm_plan* p, char** out_json);
/* Bind device tensors (order = dag.inputs, dag.outputs); allocates
 * intermediates, builds TMA descriptors and the kernels' parameter blocks. */
tm_status tm_exec_create(const tm_plan* p, const tm_tensor* inputs, int32_t n_in,
                         const tm_tensor* outputs, int32_t n_out, tm_exec** out);
void tm_exec_destroy(tm_exec* e);
/* Launch all fused kernels of the bound plan on a CUDA stream. */
tm_status tm_exec_launch(const tm_exec* e, void* cuda_stream);
/* Number of kernel launches per tm_exec_launch. */
int32_t tm_exec_num_launches(const tm_exec* e);
/* Launch geometry of kernel `index`: grid size, CTAs per MMA (1/2), tile N, split-K. */
tm_status tm_exec_kernel_info(const tm_exec* e, int32_t index, int32_t* grid, int32_t* cta_group,
                              int32_t* block_n, int32_t* split_k, int32_t* a_loader, int32_t* b_loader);
/* Which kernel family launch `index` runs: TM_KIND_* below. */
enum { TM_KIND_GEMM = 0, TM_KIND_SIMT = 1, TM_KIND_ROWBAND = 2, TM_KIND_HALO = 3, TM_KIND_RULE_INTERP = 4,
       TM_KIND_RULE_GENERATED = 5 };
tm_status tm_exec_kernel_kind(const tm_exec* e, int32_t index, int32_t* kind);
/* Per-tile role timeline of kernel `index` (exec created with TMB_TRACE=1 in the
 * environment): [grid][64 tiles][16 events] int64 clock64 deltas; see TraceEv. */
tm_status tm_exec_trace(const tm_exec* e, int32_t index, int64_t* buf, size_t cap);
/* bind + launch (+ destroy) in one call. */
tm_status tm_plan_launch(const tm_plan* p, const tm_tensor* inputs, int32_t n_in,
                         const tm_tensor* outputs, int32_t n_out, void* cuda_stream);

/* CUDA graph of a sequence of bound execs (e.g. every layer of a network), replayed
 * with one launch: removes the per-kernel host launch cost. The execs must outlive
 * the graph (it references their buffers). timed != 0 records an event before each
 * exec and after the last, read back with tm_graph_exec_ms (per-exec ms of the most
 * recent launch, after the stream is synchronised). */
typedef struct tm_graph tm_graph;
tm_status tm_graph_create(const tm_exec* const* execs, int32_t n, int32_t timed, tm_graph** out);
tm_status tm_graph_launch(const tm_graph* g, void* cuda_stream);
tm_status tm_graph_exec_ms(const tm_graph* g, float* ms, int32_t n);
void tm_graph_destroy(tm_graph* g);

/* tune: enumerate schedule_space; verify every config on two
 * fixed seeded inputs (integer U{-8..8}: bit-exact where the DAG keeps integers
 * exact; dyadic k/256: within tolerance) against the device DAG interpreter
 * (tm_dag_eval); time the config on the bound tensors with CUDA events; pick
 * the fastest correct one (ties: space order).  Correctness is a hard gate: any
 * incorrect config aborts with TM_ERR_CORRECTNESS.  The TuneReport JSON
 * is returned through *report_json in both cases. */
tm_status tm_tune(const char* dag_json, const tm_tensor* inputs, int32_t n_in,
                  const tm_tensor* outputs, int32_t n_out, int32_t device, int32_t reps,
                  tm_schedule_config* best, char** report_json);

/* reference_eval (proj/include/taskmap/compute_ir.hpp:60) re-run on the device:
 * every node of the DAG evaluated element by element with the reference
 * interpreter's semantics (fp64 / int64 values, row-major reductions from the
 * combiner identity, short-circuit select).  Independent of the tensor
 * programs; it is the tuner's correctness reference.  Outputs are written
 * rounded to their dtype; synchronous on `cuda_stream`. */
tm_status tm_dag_eval(const char* dag_json, const tm_tensor* inputs, int32_t n_in,
                      const tm_tensor* outputs, int32_t n_out, int32_t device, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* TASKMAP_B200_H_ */
