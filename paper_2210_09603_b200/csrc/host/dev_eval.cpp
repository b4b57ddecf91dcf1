// Device DAG interpreter, host side: bytecode compilation of the reference
// expression trees and node-by-node evaluation (see dev_eval.hpp).
#include "dev_eval.hpp"

#include <cmath>
#include <cstring>

namespace tmb {
namespace ev {

using namespace taskmap;

DeviceBuffer::DeviceBuffer(size_t bytes) {
  if (bytes == 0) bytes = 8;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    p = nullptr;
    fail_cuda("cudaMalloc of ", bytes, " bytes failed in the device evaluator");
  }
}
DeviceBuffer::~DeviceBuffer() {
  if (p) cudaFree(p);
}

TensorShape shape_of(const tm_tensor& t) {
  TensorShape s{};
  for (int d = 0; d < t.rank && d < kMaxRank; ++d) {
    s.shape[d] = t.shape[d];
    s.stride[d] = t.stride[d];
  }
  return s;
}

int64_t numel_of(const tm_tensor& t) {
  int64_t n = 1;
  for (int d = 0; d < t.rank; ++d) n *= t.shape[d];
  return n;
}

int64_t span_of(const tm_tensor& t) {
  int64_t s = 1;
  for (int d = 0; d < t.rank; ++d) {
    if (t.shape[d] == 0) return 0;
    s += (t.shape[d] - 1) * std::abs(t.stride[d]);
  }
  return s;
}

struct Compiler {
  std::map<std::string, int> vars;       // axis name -> var slot
  std::map<std::string, int> tensor_ix;  // tensor name -> TensorRef slot
  std::vector<std::string> tensors;
  std::vector<Ins> code;
  std::vector<int64_t> tables;
  int depth = 0, max_depth = 0;

  void push(int n = 1) {
    depth += n;
    if (depth > max_depth) max_depth = depth;
  }
  void emit(int32_t op, int32_t a = 0, int32_t b = 0, int64_t i = 0, double f = 0.0) {
    Ins in{};
    in.op = op;
    in.a = a;
    in.b = b;
    in.i = i;
    in.f = f;
    code.push_back(in);
  }

  void compile(const Expr& e) {
    switch (e->kind) {
      case ExprKind::IntImm: emit(OP_PUSH_I, 0, 0, e->ival); push(); return;
      case ExprKind::FloatImm: emit(OP_PUSH_F, 0, 0, 0, e->fval); push(); return;
      case ExprKind::Var: {
        auto it = vars.find(e->name);
        if (it == vars.end()) fail("device evaluator: unbound axis '", e->name, "'");
        emit(OP_VAR, it->second);
        push();
        return;
      }
      case ExprKind::ThreadIdx:
      case ExprKind::BlockIdx: fail("thread/block index in a computation definition");
      case ExprKind::Binary:
        compile(e->args[0]);
        compile(e->args[1]);
        emit(OP_BIN, static_cast<int32_t>(e->bop));
        depth -= 1;
        return;
      case ExprKind::Unary:
        compile(e->args[0]);
        emit(OP_UN, static_cast<int32_t>(e->uop));
        return;
      case ExprKind::Select: {
        compile(e->args[0]);
        const size_t jz = code.size();
        emit(OP_JZ);
        depth -= 1;
        compile(e->args[1]);
        const size_t jmp = code.size();
        emit(OP_JMP);
        depth -= 1;  // only one branch's value is on the stack at run time
        code[jz].a = static_cast<int32_t>(code.size());
        compile(e->args[2]);
        code[jmp].a = static_cast<int32_t>(code.size());
        return;
      }
      case ExprKind::Load: {
        auto it = tensor_ix.find(e->name);
        int slot;
        if (it == tensor_ix.end()) {
          slot = static_cast<int>(tensors.size());
          tensor_ix[e->name] = slot;
          tensors.push_back(e->name);
        } else {
          slot = it->second;
        }
        for (const auto& a : e->args) compile(a);
        emit(OP_LOAD, slot, static_cast<int32_t>(e->args.size()));
        depth -= static_cast<int>(e->args.size());
        push();
        return;
      }
      case ExprKind::TableLookup: {
        compile(e->args[0]);
        emit(OP_TABLE, static_cast<int32_t>(tables.size()), static_cast<int32_t>(e->table->size()));
        tables.insert(tables.end(), e->table->begin(), e->table->end());
        return;
      }
    }
    fail("device evaluator: unknown expression kind");
  }
};

Program compile_program(const Expr& e, const std::vector<std::string>& var_names) {
  Compiler c;
  for (size_t i = 0; i < var_names.size(); ++i) c.vars[var_names[i]] = static_cast<int>(i);
  c.compile(e);
  if (c.max_depth > kMaxStack) fail_unsupported("expression is too deep for the device interpreter (stack ", c.max_depth, ")");
  Program p;
  p.code = std::move(c.code);
  p.tensors = std::move(c.tensors);
  p.tables = std::move(c.tables);
  return p;
}

namespace {

int store_of(int32_t dt) { return dt == TM_F32 ? ST_F32 : dt == TM_BF16 ? ST_BF16 : ST_F16; }

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail_cuda(what, ": ", cudaGetErrorString(e));
}

// value type of an expression under the interpreter's promotion rules
// (compute_ir.cpp:277-366): float if a float immediate / f32 tensor / exp /
// sqrt / cast feeds it through arithmetic; comparisons and logic are int
bool expr_is_float(const ComputeDAG& dag, const Expr& e) {
  switch (e->kind) {
    case ExprKind::FloatImm: return true;
    case ExprKind::IntImm:
    case ExprKind::Var:
    case ExprKind::ThreadIdx:
    case ExprKind::BlockIdx:
    case ExprKind::TableLookup: return false;
    case ExprKind::Load: {
      const TensorNode* t = dag.find(e->name);
      return t != nullptr && t->dtype == DType::F32;
    }
    case ExprKind::Unary:
      if (e->uop == UnOp::Exp || e->uop == UnOp::Sqrt || e->uop == UnOp::CastF32) return true;
      if (e->uop == UnOp::CastI32) return false;
      return expr_is_float(dag, e->args[0]);
    case ExprKind::Select: return expr_is_float(dag, e->args[1]) || expr_is_float(dag, e->args[2]);
    case ExprKind::Binary:
      switch (e->bop) {
        case BinOp::And: case BinOp::Or: case BinOp::Lt: case BinOp::Le: case BinOp::Gt: case BinOp::Ge:
        case BinOp::Eq: case BinOp::Ne: return false;
        default: return expr_is_float(dag, e->args[0]) || expr_is_float(dag, e->args[1]);
      }
  }
  return false;
}

bool expr_integer_exact(const ComputeDAG& dag, const Expr& e) {
  switch (e->kind) {
    case ExprKind::FloatImm: {
      // exact in bf16 (8 significant bits): products with integers stay exact in fp32
      const double v = e->fval;
      if (!std::isfinite(v)) return false;
      int ex;
      const double m = std::frexp(v, &ex);
      return std::ldexp(m, 8) == std::floor(std::ldexp(m, 8));
    }
    case ExprKind::Unary:
      if (e->uop == UnOp::Exp || e->uop == UnOp::Sqrt) return false;
      break;
    case ExprKind::Binary:  // float division (integer index division floors exactly)
      if (e->bop == BinOp::Div && expr_is_float(dag, e)) return false;
      break;
    default: break;
  }
  for (const auto& a : e->args)
    if (!expr_integer_exact(dag, a)) return false;
  return true;
}

}  // namespace

bool dag_integer_exact(const ComputeDAG& dag) {
  for (const auto& n : dag.nodes)
    if (n.is_computed() && !expr_integer_exact(dag, n.value)) return false;
  return true;
}

DagEval::DagEval(const ComputeDAG& dag, const tm_tensor* inputs, int n_in, const std::map<std::string, int>& round,
                 cudaStream_t s) {
  dag.validate();
  if (n_in != static_cast<int>(dag.inputs.size())) fail("expected ", dag.inputs.size(), " input tensors, got ", n_in);
  std::map<std::string, TensorRef> env;
  for (int i = 0; i < n_in; ++i) {
    const TensorNode& node = dag.at(dag.inputs[i]);
    const tm_tensor& t = inputs[i];
    if (t.rank != static_cast<int>(node.shape.size()) || t.rank > kMaxRank) fail("input '", node.name, "' has wrong rank");
    TensorRef r{};
    r.ptr = t.data;
    r.store = store_of(t.dtype);
    r.is_float = node.dtype == DType::F32;
    r.rank = t.rank;
    for (int d = 0; d < t.rank; ++d) {
      if (t.shape[d] != node.shape[d]) fail("input '", node.name, "' has wrong shape at dim ", d);
      r.shape[d] = t.shape[d];
      r.stride[d] = t.stride[d];
    }
    env[node.name] = r;
    float_[node.name] = r.is_float;
  }
  DeviceBuffer errbuf(sizeof(int));
  check(cudaMemsetAsync(errbuf.p, 0, sizeof(int), s), "cudaMemsetAsync");
  for (const TensorNode& node : dag.nodes) {
    if (!node.is_computed()) {
      if (!env.count(node.name)) fail("input '", node.name, "' is not bound");
      continue;
    }
    if (node.axes.size() + node.reduce_axes.size() > static_cast<size_t>(kMaxVars) ||
        node.axes.size() > static_cast<size_t>(kMaxRank) || node.reduce_axes.size() > static_cast<size_t>(kMaxRank))
      fail_unsupported("device evaluator: node '", node.name, "' has too many axes");
    Compiler c;
    for (size_t i = 0; i < node.axes.size(); ++i) c.vars[node.axes[i].name] = static_cast<int>(i);
    for (size_t i = 0; i < node.reduce_axes.size(); ++i)
      c.vars[node.reduce_axes[i].name] = static_cast<int>(node.axes.size() + i);
    c.compile(node.value);
    if (c.max_depth > kMaxStack) fail_unsupported("device evaluator: expression of '", node.name, "' is too deep");
    std::vector<TensorRef> refs;
    for (const auto& name : c.tensors) {
      auto it = env.find(name);
      if (it == env.end()) fail("device evaluator: '", node.name, "' reads unknown tensor '", name, "'");
      refs.push_back(it->second);
    }
    int64_t numel = 1;
    for (const auto& a : node.axes) numel *= a.extent;
    auto out = std::make_shared<DeviceBuffer>(static_cast<size_t>(numel) * 8);
    // program blob: code | tensor refs | tables
    const size_t code_b = c.code.size() * sizeof(Ins), refs_b = refs.size() * sizeof(TensorRef),
                 tab_b = c.tables.size() * sizeof(int64_t);
    auto blob = std::make_shared<DeviceBuffer>(code_b + refs_b + tab_b + 64);
    std::vector<unsigned char> host(code_b + refs_b + tab_b + 64, 0);
    std::memcpy(host.data(), c.code.data(), code_b);
    std::memcpy(host.data() + code_b, refs.data(), refs_b);
    if (tab_b) std::memcpy(host.data() + code_b + refs_b, c.tables.data(), tab_b);
    check(cudaMemcpyAsync(blob->p, host.data(), host.size(), cudaMemcpyHostToDevice, s), "cudaMemcpyAsync");
    NodeJob j{};
    j.code = static_cast<const Ins*>(blob->p);
    j.n_code = static_cast<int32_t>(c.code.size());
    j.tensors = reinterpret_cast<const TensorRef*>(static_cast<unsigned char*>(blob->p) + code_b);
    j.tables = reinterpret_cast<const int64_t*>(static_cast<unsigned char*>(blob->p) + code_b + refs_b);
    j.n_axes = static_cast<int32_t>(node.axes.size());
    j.n_red = static_cast<int32_t>(node.reduce_axes.size());
    j.combiner = static_cast<int32_t>(node.combiner);
    j.is_float = node.dtype == DType::F32;
    j.reduce = node.kind == NodeKind::GridReduce;
    for (size_t i = 0; i < node.axes.size(); ++i) j.ext[i] = node.axes[i].extent;
    for (size_t i = 0; i < node.reduce_axes.size(); ++i) j.red[i] = node.reduce_axes[i].extent;
    j.numel = numel;
    auto rit = round.find(node.name);
    j.round = rit == round.end() ? RD_NONE : rit->second;
    j.out = out->p;
    launch_eval_node(j, static_cast<int*>(errbuf.p), s);
    TensorRef r{};
    r.ptr = out->p;
    r.store = ST_DENSE8;
    r.is_float = j.is_float;
    r.rank = static_cast<int32_t>(node.axes.size());
    int64_t st = 1;
    for (int d = r.rank - 1; d >= 0; --d) {
      r.shape[d] = node.axes[d].extent;
      r.stride[d] = st;
      st *= node.axes[d].extent;
    }
    env[node.name] = r;
    float_[node.name] = j.is_float;
    dense_[node.name] = {out, numel};
    keep_.push_back(blob);
  }
  int err = 0;
  check(cudaMemcpyAsync(&err, errbuf.p, sizeof(int), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
  check(cudaStreamSynchronize(s), "device evaluator");
  if (err == 1) fail("device evaluator: an expression failed (out-of-bounds load, division by zero or float modulo)");
  if (err == 2) fail("device evaluator: float value stored to an i32 tensor");
}

const void* DagEval::values(const std::string& node) const {
  auto it = dense_.find(node);
  if (it == dense_.end()) fail("device evaluator: '", node, "' is not a computed node");
  return it->second.first->p;
}

int64_t DagEval::numel(const std::string& node) const {
  auto it = dense_.find(node);
  if (it == dense_.end()) fail("device evaluator: '", node, "' is not a computed node");
  return it->second.second;
}

bool DagEval::is_float(const std::string& node) const {
  auto it = float_.find(node);
  return it != float_.end() && it->second;
}

}  // namespace ev
}  // namespace tmb
