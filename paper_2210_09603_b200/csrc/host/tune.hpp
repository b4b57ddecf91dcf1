// Tuner and device evaluation entry points (see tune.cpp).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>

#include "dev_eval.hpp"
#include "taskmap/ir.hpp"
#include "taskmap/schedule.hpp"
#include "taskmap_b200.h"

namespace tmb {

struct TuneOutcome {
  bool ok = false;           // a correct best configuration was found
  bool unsupported = false;  // no configuration of the space can bind this problem
  taskmap::ScheduleConfig best;
  std::string report;  // TuneReport JSON, also when !ok
  std::string error;   // why !ok
};

TuneOutcome tune(const taskmap::ComputeDAG& d, const tm_tensor* in, int n_in, const tm_tensor* out, int n_out,
                 int device, int reps);

// The DAG evaluated by the device interpreter (no storage rounding).
std::unique_ptr<ev::DagEval> dag_eval(const taskmap::ComputeDAG& d, const tm_tensor* in, int n_in,
                                      const tm_tensor* out, int n_out, int device, void* stream);

// cudaStreamSynchronize with a watchdog: a launch that makes no progress for
// `seconds` raises CudaError instead of blocking the caller forever.
void sync_with_timeout(cudaStream_t s, double seconds, const char* what);

}  // namespace tmb
