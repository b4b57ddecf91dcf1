// Host side of the device DAG interpreter (device/dev_eval.h): compiles each
// computed node's expression tree to the stack bytecode, evaluates the DAG
// node by node on the GPU, and compares tensor-program outputs with it.  This
// is the correctness gate of tm_tune and the engine behind the
// tm_dag_eval C entry point.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../device/dev_eval.h"
#include "taskmap/ir.hpp"
#include "taskmap_b200.h"

namespace tmb {
namespace ev {

struct TensorShape {
  int64_t shape[kMaxRank];
  int64_t stride[kMaxRank];
};

// kernels (dev_eval.cu)
void launch_eval_node(const NodeJob& j, int* err, cudaStream_t s);
void launch_fill(void* p, int32_t dt, int32_t rank, const TensorShape& s, int64_t span, uint64_t key, int32_t mode,
                 cudaStream_t st);
void launch_fill_nan(void* p, int32_t dt, int64_t span, cudaStream_t st);
// dense fp64 values -> a strided tensor of any float dtype (round to nearest)
// (int64 values when !is_float: an i32 node of the DAG)
void launch_store(const void* v, bool is_float, int64_t n, void* p, int32_t dt, int32_t rank, const TensorShape& s,
                  cudaStream_t st);
// host3 = {max error, #bit mismatches vs the rounded reference, scale (rms of the reference)}
void launch_compare(const void* cand, int32_t dt, int32_t rank, const TensorShape& s, const void* ref, bool is_float,
                    int64_t n, double* tmp3, double* host3, cudaStream_t st);

// Owns device memory released on destruction (RAII for the tuner's buffers).
struct DeviceBuffer {
  void* p = nullptr;
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes);
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p(o.p) { o.p = nullptr; }
  ~DeviceBuffer();
};

// The whole DAG evaluated on the device.  `round` maps node names to the
// storage rounding (Round) applied when that node is stored, so a materialised
// bf16 intermediate of the product can be modelled; every other value is fp64
// / int64 like reference_eval.
class DagEval {
 public:
  DagEval(const taskmap::ComputeDAG& dag, const tm_tensor* inputs, int n_in, const std::map<std::string, int>& round,
          cudaStream_t s);
  // dense row-major values of a computed node: double (float nodes) or int64 (i32 nodes)
  const void* values(const std::string& node) const;
  int64_t numel(const std::string& node) const;
  bool is_float(const std::string& node) const;

 private:
  std::map<std::string, std::pair<std::shared_ptr<DeviceBuffer>, int64_t>> dense_;
  std::map<std::string, bool> float_;
  std::vector<std::shared_ptr<DeviceBuffer>> keep_;
};

// Stack bytecode of one expression tree; variable slot i is var_names[i], load
// slot j reads tensors[j].  Shared by this interpreter and the product's
// rule-based / reduce kernels (rule.cpp).
struct Program {
  std::vector<Ins> code;
  std::vector<std::string> tensors;
  std::vector<int64_t> tables;
};
Program compile_program(const taskmap::Expr& e, const std::vector<std::string>& var_names);

// True when every computed node keeps integer-valued inputs exact in fp32
// (no exp/sqrt/float division, float constants exact in bf16): the integer
// verification trial then requires bit-identical outputs.
bool dag_integer_exact(const taskmap::ComputeDAG& dag);

TensorShape shape_of(const tm_tensor& t);
int64_t span_of(const tm_tensor& t);  // elements covered by the strided view
int64_t numel_of(const tm_tensor& t);

}  // namespace ev
}  // namespace tmb
