// taskmap IR for the B200 build: task mappings, scalar expressions and the
// operator DAG, with the same public names and semantics as the reference's
// C++ API so code written against `taskmap::` keeps compiling:
//   TaskMapping / TaskShape / parse_mapping   <- proj/include/taskmap/mapping.hpp:15-90
//   Expr builders / substitute / rewrite_loads <- proj/include/taskmap/expr.hpp:15-95
//   ComputeDAG / classify / builders          <- proj/include/taskmap/compute_ir.hpp:13-119
// The reference's reference_eval / Tensor oracle is intentionally NOT part of
// this library (it lives under oracle/ as test infrastructure only).
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace taskmap {

// ------------------------------------------------------------------ common --
struct Error : std::runtime_error {
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};

template <class... Args>
[[noreturn]] void fail(Args&&... args) {
  std::ostringstream os;
  (os << ... << args);
  throw Error(os.str());
}

// Typed refinements of Error for the C ABI's status codes (tm_status): the
// boundary maps the exception type, never the message text, to a code.
struct UnsupportedError : Error {  // TM_ERR_UNSUPPORTED: valid input outside what the device path implements
  using Error::Error;
};
struct CudaError : Error {  // TM_ERR_CUDA: a CUDA runtime / driver call failed
  using Error::Error;
};
struct CorrectnessError : Error {  // TM_ERR_CORRECTNESS: a result failed its correctness gate
  using Error::Error;
};

template <class E, class... Args>
[[noreturn]] void fail_as(Args&&... args) {
  std::ostringstream os;
  (os << ... << args);
  throw E(os.str());
}
template <class... Args>
[[noreturn]] void fail_unsupported(Args&&... args) {
  fail_as<UnsupportedError>(std::forward<Args>(args)...);
}
template <class... Args>
[[noreturn]] void fail_cuda(Args&&... args) {
  fail_as<CudaError>(std::forward<Args>(args)...);
}

enum class DType { F32, I32 };
const char* dtype_name(DType t);
DType dtype_from_name(const std::string& s);
inline bool is_float_dtype(DType t) { return t == DType::F32; }

// floor semantics (Python-style) used by all index arithmetic
int64_t floordiv(int64_t a, int64_t b);
int64_t floormod(int64_t a, int64_t b);

// ------------------------------------------------------------ task mapping --
using Task = std::vector<uint64_t>;

class TaskShape {
 public:
  TaskShape() = default;
  TaskShape(std::initializer_list<uint64_t> d) : TaskShape(std::vector<uint64_t>(d)) {}
  explicit TaskShape(std::vector<uint64_t> dims);
  const std::vector<uint64_t>& dims() const { return dims_; }
  size_t rank() const { return dims_.size(); }
  uint64_t operator[](size_t i) const { return dims_[i]; }
  uint64_t total() const { return volume_; }
  TaskShape elementwise_mul(const TaskShape& o) const;
  bool operator==(const TaskShape& o) const { return dims_ == o.dims_; }

 private:
  std::vector<uint64_t> dims_;
  uint64_t volume_ = 1;
};

class TaskMapping {
 public:
  enum class Kind { Repeat, Spatial, Custom, Compose };

  static TaskMapping repeat(TaskShape shape);
  static TaskMapping spatial(TaskShape shape);
  static TaskMapping custom(uint64_t num_workers, TaskShape shape,
                            std::vector<std::vector<Task>> table);
  static TaskMapping compose(const TaskMapping& outer, const TaskMapping& inner);

  Kind kind() const;
  uint64_t num_workers() const;
  const TaskShape& task_shape() const;
  size_t task_dim() const { return task_shape().rank(); }
  uint64_t tasks_per_worker() const;
  std::vector<Task> assign(uint64_t worker) const;
  TaskMapping lhs() const;
  TaskMapping rhs() const;
  const std::vector<std::vector<Task>>& table() const;
  std::string to_text() const;
  std::string visualize() const;
  bool operator==(const TaskMapping& o) const;

  // Flattened left-to-right atom chain (Custom atoms unsupported); the form
  // lowered to device index arithmetic (tmb::tm::DevMapping).
  struct Atom {
    bool spatial;
    std::vector<uint64_t> dims;
  };
  std::vector<Atom> atoms() const;

 private:
  struct Rep;
  explicit TaskMapping(std::shared_ptr<const Rep> r) : rep_(std::move(r)) {}
  std::shared_ptr<const Rep> rep_;
};

TaskMapping operator*(const TaskMapping& a, const TaskMapping& b);
TaskMapping parse_mapping(const std::string& text);

// -------------------------------------------------------------- expressions --
enum class BinOp { Add, Sub, Mul, Div, Mod, Min, Max, And, Or, Lt, Le, Gt, Ge, Eq, Ne };
enum class UnOp { Neg, Relu, Exp, Sqrt, CastF32, CastI32 };
enum class ExprKind { IntImm, FloatImm, Var, ThreadIdx, BlockIdx, Binary, Unary, Select, Load, TableLookup };

struct ExprNode;
using Expr = std::shared_ptr<const ExprNode>;
using IndexTable = std::shared_ptr<const std::vector<int64_t>>;

struct ExprNode {
  ExprKind kind;
  int64_t ival = 0;
  double fval = 0.0;
  std::string name;
  BinOp bop = BinOp::Add;
  UnOp uop = UnOp::Neg;
  std::vector<Expr> args;
  IndexTable table;
  bool is_const_int(int64_t v) const { return kind == ExprKind::IntImm && ival == v; }
};

Expr imm(int64_t v);
Expr fimm(double v);
Expr var(const std::string& name);
Expr thread_idx();
Expr block_idx();
Expr binary(BinOp op, Expr a, Expr b);
Expr unary(UnOp op, Expr a);
Expr select(Expr cond, Expr then_val, Expr else_val);
Expr load(const std::string& buffer, std::vector<Expr> indices);
Expr table_lookup(IndexTable table, Expr index);

inline Expr add(Expr a, Expr b) { return binary(BinOp::Add, std::move(a), std::move(b)); }
inline Expr sub(Expr a, Expr b) { return binary(BinOp::Sub, std::move(a), std::move(b)); }
inline Expr mul(Expr a, Expr b) { return binary(BinOp::Mul, std::move(a), std::move(b)); }
inline Expr div(Expr a, Expr b) { return binary(BinOp::Div, std::move(a), std::move(b)); }
inline Expr mod(Expr a, Expr b) { return binary(BinOp::Mod, std::move(a), std::move(b)); }
inline Expr min(Expr a, Expr b) { return binary(BinOp::Min, std::move(a), std::move(b)); }
inline Expr max(Expr a, Expr b) { return binary(BinOp::Max, std::move(a), std::move(b)); }
inline Expr land(Expr a, Expr b) { return binary(BinOp::And, std::move(a), std::move(b)); }
inline Expr lor(Expr a, Expr b) { return binary(BinOp::Or, std::move(a), std::move(b)); }
inline Expr lt(Expr a, Expr b) { return binary(BinOp::Lt, std::move(a), std::move(b)); }
inline Expr le(Expr a, Expr b) { return binary(BinOp::Le, std::move(a), std::move(b)); }
inline Expr gt(Expr a, Expr b) { return binary(BinOp::Gt, std::move(a), std::move(b)); }
inline Expr ge(Expr a, Expr b) { return binary(BinOp::Ge, std::move(a), std::move(b)); }
inline Expr eq(Expr a, Expr b) { return binary(BinOp::Eq, std::move(a), std::move(b)); }
inline Expr ne(Expr a, Expr b) { return binary(BinOp::Ne, std::move(a), std::move(b)); }
inline Expr neg(Expr a) { return unary(UnOp::Neg, std::move(a)); }
inline Expr relu(Expr a) { return unary(UnOp::Relu, std::move(a)); }
inline Expr zero_of(DType t) { return t == DType::F32 ? fimm(0.0) : imm(0); }

// tanh-form GELU written with Exp/Div only (the reference IR has no tanh/erf,
// expr.hpp:16): 0.5*x*(1 + (1 - 2/(exp(2*c*(x + 0.044715*x^3)) + 1))).
Expr gelu_tanh(Expr x);

Expr substitute(const Expr& e, const std::map<std::string, Expr>& vars);
Expr rewrite_loads(const Expr& e, const std::function<std::optional<Expr>(const ExprNode&)>& fn);
Expr fold(const Expr& e);
bool expr_equal(const Expr& a, const Expr& b);
bool uses_thread_idx(const Expr& e);
void collect_vars(const Expr& e, std::vector<std::string>& out);
void collect_loads(const Expr& e, std::vector<Expr>& out);
std::string expr_to_text(const Expr& e);
const char* binop_name(BinOp op);
const char* unop_name(UnOp op);

// ---------------------------------------------------------------- the DAG --
struct Axis {
  std::string name;
  int64_t extent;
};

enum class Combiner { Sum, Max, Min };
const char* combiner_name(Combiner c);
Combiner combiner_from_name(const std::string& s);

enum class NodeKind { Input, GridCompute, GridReduce };

struct TensorNode {
  std::string name;
  std::vector<int64_t> shape;
  DType dtype = DType::F32;
  NodeKind kind = NodeKind::Input;
  std::vector<Axis> axes;
  std::vector<Axis> reduce_axes;
  Combiner combiner = Combiner::Sum;
  Expr value;
  bool is_computed() const { return kind != NodeKind::Input; }
};

struct ComputeDAG {
  std::vector<TensorNode> nodes;
  std::vector<std::string> inputs;
  std::vector<std::string> outputs;
  const TensorNode* find(const std::string& name) const;
  const TensorNode& at(const std::string& name) const;
  void validate() const;
};

enum class OpClass { Reduction, Injective, Bijective };
const char* opclass_name(OpClass c);
OpClass classify(const ComputeDAG& dag, const TensorNode& node);

struct AffineTerm {
  size_t axis;
  int64_t coeff;
};
struct AffineIndex {
  std::vector<AffineTerm> terms;
  int64_t offset = 0;
};
std::optional<std::vector<AffineIndex>> analyze_affine_access(const Expr& load_node,
                                                              const std::vector<Axis>& axes);
bool affine_access_injective(const std::vector<AffineIndex>& access, const std::vector<Axis>& axes);
bool affine_access_bijective(const std::vector<AffineIndex>& access, const std::vector<Axis>& axes,
                             const std::vector<int64_t>& input_shape);

// builders (same DAG structure as the reference builders so that DAGs built
// on either side are interchangeable)
ComputeDAG matmul_dag(int64_t m, int64_t n, int64_t k, DType dtype);
ComputeDAG conv2d_im2col_dag(int64_t n, int64_t c, int64_t h, int64_t w, int64_t f, int64_t kh,
                             int64_t kw, int64_t stride, int64_t pad, DType dtype);
ComputeDAG elementwise_unary_dag(UnOp op, std::vector<int64_t> shape, DType dtype);
ComputeDAG elementwise_binary_dag(BinOp op, std::vector<int64_t> shape, DType dtype);
ComputeDAG reshape_dag(std::vector<int64_t> in_shape, std::vector<int64_t> out_shape, DType dtype);
ComputeDAG transpose_dag(std::vector<int64_t> shape, std::vector<size_t> perm, DType dtype);
ComputeDAG batchnorm_inference_dag(int64_t n, int64_t c, int64_t h, int64_t w, DType dtype);
inline int64_t conv_out_extent(int64_t in, int64_t kernel, int64_t stride, int64_t pad) {
  return (in + 2 * pad - kernel) / stride + 1;
}

// JSON wire form of a DAG (the spec's DAG JSON): used by the C ABI.
ComputeDAG dag_from_json(const std::string& text);
std::string dag_to_json(const ComputeDAG& dag);

}  // namespace taskmap
