// Source generation and NVRTC compilation of the rule-based / reduce kernels
// (SPEC.md:282-290, :300-308).  The reference lowers an anchor-free subgraph to
// CUDA source and compiles it (the ir_to_cuda path of codegen); the product does
// the same at bind time: the fused root expression -- inlined producers already
// spliced in -- becomes straight-line C with every extent, stride and storage
// type a literal, compiled once per distinct source by NVRTC for the device's
// sm_100a and launched through the driver API (capturable in CUDA graphs).
//
// Numerics follow the bytecode interpreter of rule_kernels.cu exactly: fp32 /
// int64 values with the interpreter's promotion rules, no FMA contraction
// (--fmad=false), the same reduction order.  Expressions the generator does not
// type statically (a select whose branches differ in type, a float index) keep
// the interpreter.
#pragma once
#include <string>
#include <vector>

#include "../device/dev_eval.h"
#include "../device/rule.h"
#include "taskmap/ir.hpp"

namespace tmb {

struct RuleSourceSpec {
  taskmap::Expr expr;
  std::vector<std::string> vars;  // spatial axes, then reduce axes
  std::vector<int64_t> ext, red;  // spatial / reduce extents
  std::vector<std::string> tensor_names;
  std::vector<ev::TensorRef> tensors;  // shape / stride / store / is_float (pointers unused)
  ev::TensorRef out;
  int combiner = 0;   // 0 sum, 1 max, 2 min
  bool is_float = true;  // the root node's dtype
  int mode = 0;          // GenMode
  int threads = 256;     // CTA width (tree / split)
  int group = 1;         // GEN_GROUP: lanes per output (power of two <= 32)
  int splits = 1;        // GEN_SPLIT: CTAs per output
};

// Kernel shapes of the generated code.  ELEM and TREE restate the interpreter's
// two kernels (bit-identical results); GROUP and SPLIT exist only generated:
//   GROUP: short reductions over many outputs -- `group` adjacent lanes per
//          output stride the reduce domain (coalesced when the reduced axis is
//          the contiguous one), then a shuffle tree inside the group;
//   SPLIT: long reductions over fewer outputs than SMs -- `splits` CTAs per
//          output fold contiguous chunks, write partials to a scratch block
//          (pointer slot = number of loaded tensors), and the last CTA to
//          arrive (atomic ticket, self-resetting) combines them in chunk order.
// Float sums under GROUP / SPLIT associate differently from the sequential /
// single-CTA order (deterministic from launch to launch).
enum GenMode : int { GEN_ELEM = 0, GEN_TREE = 1, GEN_GROUP = 2, GEN_SPLIT = 3 };

// Returns false (and leaves `src` empty) when the expression needs the
// interpreter; otherwise the complete translation unit with entry "tmb_rule".
bool emit_rule_source(const RuleSourceSpec& s, std::string& src, std::string& why);

// Compiled entry point for `src` on the current device (cached per device and
// source); nullptr with `why` set when NVRTC or the driver is unavailable or
// the compile fails.
void* compile_rule_source(const std::string& src, std::string& why);

// cuLaunchKernel of a compiled entry with the pointer block as its one argument.
void launch_rule_compiled(void* fn, const RulePtrs& ptrs, unsigned grid, unsigned block, void* stream);

}  // namespace tmb
