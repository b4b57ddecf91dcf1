// Parameter block of the rule-based and reduce kernels (kernels/rule_kernels.cu):
// the spec's rule_based_schedule for anchor-free injective
// subgraphs and reduce_template for reductions that are not
// matrix products (softmax max/sum, pooling, norms).
//
// A fused subgraph's root expression -- with every inlined producer spliced in
// by rewrite_loads -- is compiled to the stack bytecode of dev_eval.h and run by
// one of two kernels:
//   RULE  : output elements distributed over threads by a spatial mapping
//           (grid-stride); reduce axes, if any, as a sequential loop in declared
//           row-major order (the spec's SeqFor for small reductions);
//   TREE  : one CTA per output element (grid-stride over outputs); each thread
//           folds a strided slice of the reduce domain, then a shared-memory /
//           warp-shuffle tree combines the CTA's partials.
// Float values are fp32 (the product's arithmetic), integer values int64 (the
// reference's index semantics); the result is stored through the bound output's
// strides in its dtype.
#pragma once
#include <cstdint>

#include "dev_eval.h"

namespace tmb {

constexpr int kMaxRuleTensors = 15;  // generated kernels: loaded tensors (+ the output) by pointer

// argument block of a generated (NVRTC) rule kernel (host/rule_codegen.hpp)
struct RulePtrs {
  const void* p[kMaxRuleTensors + 1];  // tensors in source order, the output last
};

enum RuleMode : int32_t { RULE_ELEM = 0, RULE_TREE = 1 };

struct RuleJob {
  const ev::Ins* code;
  const ev::TensorRef* tensors;
  const int64_t* tables;
  int32_t n_code;
  int32_t n_axes;
  int32_t n_red;
  int32_t combiner;  // 0 sum, 1 max, 2 min (taskmap::Combiner)
  int32_t is_float;  // the root node's dtype is F32
  int32_t mode;      // RuleMode
  int64_t ext[ev::kMaxRank];
  int64_t red[ev::kMaxRank];
  int64_t numel;      // output elements
  int64_t red_numel;  // reduce-domain size (1 without reduce axes)
  ev::TensorRef out;  // bound output (strided; store F32 / BF16 / F16)
};

}  // namespace tmb
