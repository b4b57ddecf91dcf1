// Scheduling, post-scheduling fusion and tuning API of the B200 build.
//
// These are the spec-only parts of the reference (no code exists there):
//   ScheduleConfig / schedule_space  <- SPEC.md:276-279, :309-317
//   FusedSubgraph / partition        <- SPEC.md:355-369
//   fuse_prologue / fuse_epilogue    <- SPEC.md:370-387 (realised as operand
//                                       loaders and the TMEM-drain epilogue)
//   tune / TuneReport                <- SPEC.md:474-488
// re-designed for sm_100a: the schedule space enumerates tcgen05 tile widths,
// pipeline depths and CTA->tile task mappings, and tuning times candidates on
// the device with CUDA events.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "taskmap/ir.hpp"

namespace taskmap {

// One point of the hardware-centric schedule space.  The spec fields
// (block_m .. split_k) keep their meaning; the Blackwell fields select the
// tcgen05 tile (block_n = UMMA N, block_m = 128 TMEM lanes), the depth of the
// TMA/mbarrier ring (stages; pipeline=false means 2 stages, i.e. the paper's
// double buffer) and the CTA->tile task mapping (raster).
struct ScheduleConfig {
  int block_m = 128;
  int block_n = 128;
  int block_k = 64;
  int warp_m = 4;   // epilogue warps along M (TMEM lane groups)
  int warp_n = 1;
  int threads_per_block = 288;
  bool pipeline = true;
  int split_k = 1;
  int stages = 0;   // 0 = deepest ring that fits shared memory
  int raster = 0;   // 0: repeat(r) * spatial(g) (waves sweep tile blocks); 1: spatial(g) * repeat(r)
  int grid = 0;     // 0 = number of SMs
  std::string math = "auto";  // auto | bf16 | tf32 | fp32_simt
  std::string to_json() const;
  static ScheduleConfig from_json(const std::string& text);
  std::string key() const;
};

// Input-size-agnostic space: identical list for every problem shape (§4.3).
std::vector<ScheduleConfig> schedule_space(const std::string& op_kind);

struct FusedSubgraph {
  std::string anchor;                       // the GridReduce node
  std::vector<std::string> prologue;        // injective producers folded into loads
  std::vector<std::string> epilogue;        // bijective consumers, in order
  std::string output;                       // tensor this kernel writes
};

// Greedy anchor partition: each reduction anchors a
// subgraph; single-use injective producers become prologues, single-use
// bijective consumers become the epilogue chain; first reduction wins.
std::vector<FusedSubgraph> partition(const ComputeDAG& dag);

}  // namespace taskmap
