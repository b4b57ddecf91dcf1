// Internal planner types: a DAG partitioned into fused subgraphs, each lowered
// to one task-mapped GEMM launch with prologue loaders and an epilogue program.
#pragma once
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../device/gemm_params.h"
#include "../device/rule.h"
#include "taskmap/ir.hpp"
#include "taskmap/schedule.hpp"
#include "taskmap_b200.h"

namespace tmb {

// Integer index program compiled from an Expr (postfix), evaluated at plan
// bind time to fit operand/output address maps.  Variables: slot 0 = GEMM
// row, 1 = GEMM col (or K for operands), 2 = batch.
struct IndexProgram {
  struct Ins {
    int op;  // 0 imm, 1 var, 2 binary, 3 neg, 4 select
    int64_t v;
    taskmap::BinOp bop;
  };
  std::vector<Ins> code;
  static IndexProgram compile(const taskmap::Expr& e, const std::vector<std::string>& slots);
  int64_t eval(const int64_t* vars) const;
};

// physical tensor address as sum_d stride_d * idx_d(row, x, batch)
struct AddrExpr {
  std::string tensor;                    // bound tensor name
  std::vector<taskmap::Expr> idx;        // per tensor dim, in slot vars
  std::vector<IndexProgram> prog;        // compiled idx
};

struct ConvInfo {
  int64_t n, c, h, w, f, kh, kw, stride, pad, ho, wo;
  std::string x_tensor, w_tensor;
};

struct EpiStep {
  int32_t kind;   // tmb::EpiKind
  float c = 0.f;
  int side = -1;  // index into SubgraphPlan::sides for *_T kinds
};

struct OperandPlan {
  enum Kind { Strided, Im2col, ConvFilter } kind = Strided;
  AddrExpr addr;  // Strided: physical idx in (row, k, batch)
  ConvInfo conv;  // Im2col / ConvFilter
  std::vector<EpiStep> pre;  // arithmetic prologue (constant operands only), applied per loaded element
};

struct SubgraphPlan {
  // Gemm: the task-mapped tcgen05 / CUDA-core matmul template with fused
  // prologue loaders and epilogue program.  Rule: a rule-based injective kernel
  // or, when the root is a non-matmul reduction, the reduce template
  // (rule_kernels.cu); the root's expression has every inlined producer spliced in.
  enum Kind { Gemm, Rule } kind = Gemm;
  std::string rule_node;       // Rule: the root node (written to its tensor)
  taskmap::Expr rule_expr;     // Rule: root value with inlined producers substituted
  taskmap::FusedSubgraph sg;
  int64_t M = 0, N = 0, K = 0, batch = 1;
  OperandPlan a, b;                 // A provides rows, B provides cols
  std::vector<EpiStep> ops;
  std::vector<AddrExpr> sides;      // side operands, idx in (row, col, batch)
  AddrExpr out;                     // output address, idx in (row, col, batch)
  std::string describe() const;
};

struct Plan {
  taskmap::ComputeDAG dag;
  taskmap::ScheduleConfig cfg;
  int device = 0;
  std::vector<SubgraphPlan> kernels;
  std::vector<std::string> intermediates;  // materialised between kernels
};

std::unique_ptr<Plan> build_plan(const taskmap::ComputeDAG& dag, const taskmap::ScheduleConfig& cfg,
                                 int device);

// A plan bound to tensors: fully formed kernel parameter blocks.
struct BoundKernel {
  GemmParams p;
  int bn = 128, stages = 4, tf32 = 0, grid = 148, simt = 0, cg = 1;
  int generic = 1;  // 0: compact instantiation (TMA loaders + canonical epilogue only)
  int rowband = 0;  // 1: tm_rowband_kernel (conv_rowband.cuh), 2: tm_halo_kernel (conv_halo.cuh); smem = its layout
  int rule = 0;     // 1: rule-based / reduce-template kernel (rule_kernels.cu) running `rj`
  int rule_threads = 128;
  RuleJob rj{};
  void* rfn = nullptr;  // generated rule kernel (rule_codegen.hpp); nullptr: the bytecode interpreter runs rj
  RulePtrs rp{};
  unsigned rgrid = 0, rblock = 0;
  int smem = 0;
  alignas(64) unsigned char tma_a[128];
  alignas(64) unsigned char tma_b[128];
  alignas(64) unsigned char tma_c[128];  // output map (row-major outputs, TMA-store epilogue)
};

struct Exec {
  std::vector<BoundKernel> kernels;
  std::vector<void*> scratch;  // device buffers owned by the exec
  ~Exec();
};

std::unique_ptr<Exec> bind_plan(const Plan& plan, const tm_tensor* inputs, int n_in,
                                const tm_tensor* outputs, int n_out);

// kernel launcher (gemm_launch.cu)
int num_sms(int device);
void launch_bound(const BoundKernel& k, void* stream);
int kernel_stages(const BoundKernel& k);  // ring depth of the instantiation launch_bound will pick
void pack_filter(const ConvGeom& g, int kp, void* out, int out_dtype);  // bf16/fp16 [f][kp] in the GEMM K order
// filter image of the row-band kernel: [kh][steps][bn/8][2][8][8] 16-bit, K order (fw + shift, c < cpad)
void pack_rowband_filter(const ConvGeom& g, int cpad, int shift, int steps, int bn, void* out, int out_dtype);
int rowband_smem(int rows, int rowb, int bbytes, int bn);
int halo_smem(int band_bytes, int stage_bytes, int stages, int bn, int nbands = 2);
// storage dtype of materialised intermediates for these inputs: f32 if any input
// is f32, fp16 if the 16-bit inputs are all fp16, else bf16
int intermediate_dtype(const tm_tensor* inputs, int n_in);
void launch_simt(const BoundKernel& k, void* stream);   // fp32 CUDA-core kernel (simt_fp32.cu)
void launch_rule(const RuleJob& j, int threads, int sms, void* stream);  // rule_kernels.cu
// grid and CTA width launch_rule uses for `j` (the generated kernels launch the same shape)
void rule_launch_shape(const RuleJob& j, int threads, int sms, unsigned* grid, unsigned* block);
void launch_rule_compiled(void* fn, const RulePtrs& ptrs, unsigned grid, unsigned block, void* stream);
int kernel_mapping_assign(int which, uint32_t worker, int* buf, int cap);
unsigned long long device_mismatch(const void* a, const void* b, size_t bytes, void* stream);
float device_max_rel_error(const void* a, const void* b, size_t n, int dtype, void* stream);
// swizzle: smem swizzle span in bytes (0 = none, 64, 128), or kSwizzle128Atom32: the
// 128-byte span with 32-byte atoms (MN-major kind::tf32 operands; UMMA layout type
// SWIZZLE_128B_BASE32B, 4-row K groups)
constexpr int kSwizzle128Atom32 = 129;
void make_tma_2d3d(void* map, const void* ptr, int dtype, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, int swizzle = 128);
void make_tma_im2col(void* map, const void* ptr, int dtype, const uint64_t* dims_cwhn,
                     const uint64_t* strides_bytes, int pad_lo, int pad_hi_corner, int stride,
                     uint32_t channels, uint32_t pixels, bool swizzle128 = true);

}  // namespace tmb
