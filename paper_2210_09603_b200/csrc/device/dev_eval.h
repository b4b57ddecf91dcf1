// Device DAG interpreter: the reference's reference_eval semantics
// (proj/src/compute_ir.cpp:250-466) executed on the GPU, node by node, one
// thread per output element.  It is the tuner's correctness gate (SPEC.md:483:
// "verifies correctness against reference_eval on a fixed seeded input") and
// shares nothing with the tcgen05 tensor programs it checks: no planner, no
// loaders, no TMA, no epilogue op list -- it walks the DAG's own expression
// trees, compiled to a small stack bytecode.
//
// Semantics kept from eval_expr (compute_ir.cpp:277-366): f32 values are
// doubles, i32 values int64; a binary op is float if either side is; integer
// div/mod floor; select short-circuits; reductions accumulate in declared
// reduce-axis row-major order starting from the combiner identity
// (compute_ir.cpp:368-396, :444-459).
#pragma once
#include <cstdint>

namespace tmb {
namespace ev {

enum Op : int32_t {
  OP_PUSH_I = 0,  // push int  i
  OP_PUSH_F,      // push float f
  OP_VAR,         // push int  vars[a]
  OP_LOAD,        // pop b indices, push tensors[a][idx]
  OP_BIN,         // pop y, x; push x (BinOp a) y
  OP_UN,          // pop x; push (UnOp a) x
  OP_JZ,          // pop c; if !truthy(c) pc = a
  OP_JMP,         // pc = a
  OP_TABLE        // pop i; push tables[a + i] (0 <= i < b)
};

// same numbering as taskmap::BinOp / UnOp
enum BinOpCode : int32_t { B_ADD = 0, B_SUB, B_MUL, B_DIV, B_MOD, B_MIN, B_MAX, B_AND, B_OR, B_LT, B_LE, B_GT, B_GE, B_EQ, B_NE };
enum UnOpCode : int32_t { U_NEG = 0, U_RELU, U_EXP, U_SQRT, U_CASTF, U_CASTI };

struct Ins {
  int32_t op;
  int32_t a;
  int32_t b;
  int32_t pad_;
  int64_t i;
  double f;
};

constexpr int kMaxRank = 8;
constexpr int kMaxStack = 32;
constexpr int kMaxVars = 16;

// storage kinds a Load can read
enum Store : int32_t { ST_DENSE8 = 0, ST_F32 = 1, ST_BF16 = 2, ST_F16 = 3 };

struct TensorRef {
  const void* ptr;
  int32_t store;     // Store
  int32_t is_float;  // the DAG node's dtype (F32 -> float values, I32 -> int values)
  int32_t rank;
  int32_t pad_;
  int64_t shape[kMaxRank];
  int64_t stride[kMaxRank];  // elements (dense intermediates: row-major)
};

// rounding applied when a computed node is stored (models the product's
// storage dtype of materialised intermediates; 0 = none, the reference's fp64)
enum Round : int32_t { RD_NONE = 0, RD_F32 = 1, RD_BF16 = 2, RD_F16 = 3 };

struct NodeJob {
  const Ins* code;
  int32_t n_code;
  int32_t n_axes;
  int32_t n_red;
  int32_t combiner;  // 0 sum, 1 max, 2 min (taskmap::Combiner)
  int32_t is_float;
  int32_t round;
  int32_t reduce;    // GridReduce node
  int32_t pad_;
  int64_t ext[kMaxRank];
  int64_t red[kMaxRank];
  int64_t numel;
  const TensorRef* tensors;
  const int64_t* tables;
  void* out;  // dense 8-byte row-major: double (float nodes) or int64 (int nodes)
};

}  // namespace ev
}  // namespace tmb
