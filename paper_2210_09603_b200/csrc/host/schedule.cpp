// Hardware-centric schedule space for the sm_100a GEMM template
// (§4.3: "agnostic to input size", < 200 schedules).
#include <sstream>

#include "json.hpp"
#include "taskmap/schedule.hpp"

namespace taskmap {

std::string ScheduleConfig::to_json() const {
  std::ostringstream o;
  o << "{\"block_m\":" << block_m << ",\"block_n\":" << block_n << ",\"block_k\":" << block_k
    << ",\"warp_m\":" << warp_m << ",\"warp_n\":" << warp_n << ",\"threads_per_block\":" << threads_per_block
    << ",\"pipeline\":" << (pipeline ? "true" : "false") << ",\"split_k\":" << split_k
    << ",\"stages\":" << stages << ",\"raster\":" << raster << ",\"grid\":" << grid
    << ",\"math\":" << tmjson::quote(math) << "}";
  return o.str();
}

ScheduleConfig ScheduleConfig::from_json(const std::string& text) {
  ScheduleConfig c;
  tmjson::Value v;
  try {
    v = tmjson::parse(text);
  } catch (const std::exception& e) {
    fail(e.what());
  }
  auto geti = [&](const char* k, int& dst) {
    if (const auto* x = v.get(k)) dst = static_cast<int>(x->integer());
  };
  geti("block_m", c.block_m);
  geti("block_n", c.block_n);
  geti("block_k", c.block_k);
  geti("warp_m", c.warp_m);
  geti("warp_n", c.warp_n);
  geti("threads_per_block", c.threads_per_block);
  geti("split_k", c.split_k);
  geti("stages", c.stages);
  geti("raster", c.raster);
  geti("grid", c.grid);
  if (const auto* x = v.get("pipeline")) c.pipeline = x->type == tmjson::Value::Bool ? x->b : x->integer() != 0;
  if (const auto* x = v.get("math")) c.math = x->str();
  return c;
}

std::string ScheduleConfig::key() const {
  std::ostringstream o;
  o << "bn" << block_n << (pipeline ? "_deep" : "_db") << "_r" << raster << "_sk" << split_k << "_" << math;
  return o.str();
}

// The space: UMMA N (tile width; M is fixed at 128 TMEM lanes per CTA) x ring
// depth (paper double buffer = 2 stages, or the deepest ring that fits 227 KB)
// x split-K x CTA->tile task mapping (repeat*spatial vs spatial*repeat), for
// single-SM tiles, SM-pair tiles (tcgen05 cta_group::2, 256 x N) and half-size
// persistent grids.  The same list is returned for every problem shape; tails
// are handled by TMA zero fill and predicated gathers/stores, never by
// shrinking the space.  (Round 1 kept split-K 4, BN=64 split-K and pair BN=128
// out of the tuned space after intermittent hangs; the cause -- loader warps
// polling ring slots they did not own, and a missing producer tail -- is fixed
// in gemm_sm100.cuh, and every point is back.)
std::vector<ScheduleConfig> schedule_space(const std::string& op_kind) {
  std::vector<ScheduleConfig> out;
  if (op_kind == "reduce") {
    // reduce_template: CTA width of the block-level tree
    // reduction (one CTA per output element); the rule-based form of short
    // reductions ignores it
    for (int t : {128, 256, 512, 64, 32}) {
      ScheduleConfig c;
      c.threads_per_block = t;
      out.push_back(c);
    }
    return out;
  }
  if (op_kind != "matmul" && op_kind != "conv2d" && op_kind != "batch_matmul")
    fail("unknown op kind '", op_kind, "' for schedule_space");
  // single-SM tiles (128 x N)
  for (int bn : {128, 256, 192, 64, 96})
    for (int sk : {1, 2, 4})
      for (bool deep : {true, false})
        for (int raster : {0, 1}) {
          ScheduleConfig c;
          c.block_n = bn;
          c.split_k = sk;
          c.pipeline = deep;
          c.stages = deep ? 0 : 2;
          c.raster = raster;
          out.push_back(c);
        }
  // half-size persistent grids (74 CTAs, two SMs' worth of tiles each): L2 reuse
  // across a CTA's consecutive tiles against fewer SMs in flight
  for (int bn : {128, 256, 192, 64, 96})
    for (int raster : {0, 1}) {
      ScheduleConfig c;
      c.block_n = bn;
      c.raster = raster;
      c.grid = 74;
      out.push_back(c);
    }
  // SM-pair tiles (256 x N, tcgen05.mma.cta_group::2), deep ring
  for (int bn : {256, 128, 64})
    for (int sk : {1, 2, 4})
      for (int raster : {0, 1}) {
        ScheduleConfig c;
        c.block_m = 256;
        c.block_n = bn;
        c.split_k = sk;
        c.raster = raster;
        out.push_back(c);
      }
  // conv2d: the halo kernel family (conv_halo.cuh) as one more point; it applies
  // to stride-1 channels-last convs with C % 64 == 0 and falls back to the
  // default K3 form elsewhere
  if (op_kind == "conv2d") {
    ScheduleConfig c;
    c.math = "halo";
    out.push_back(c);
  }
  return out;
}

}  // namespace taskmap
