// taskmap IR: task mappings, expressions, DAG validation, fusion classifier,
// builders and the JSON wire form.  Semantics follow the reference
// (proj/src/{mapping,expr,compute_ir}.cpp); citations per function.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <set>
#include <unordered_map>

#include "json.hpp"
#include "taskmap/ir.hpp"

namespace taskmap {

// ================================================================== common ==
const char* dtype_name(DType t) { return t == DType::F32 ? "f32" : "i32"; }
DType dtype_from_name(const std::string& s) {
  if (s == "f32") return DType::F32;
  if (s == "i32") return DType::I32;
  fail("unknown dtype: ", s);
}

// common.hpp:34-44 (floor semantics)
int64_t floordiv(int64_t a, int64_t b) {
  const int64_t q = a / b, r = a % b;
  return (r != 0 && ((r < 0) != (b < 0))) ? q - 1 : q;
}
int64_t floormod(int64_t a, int64_t b) {
  const int64_t r = a % b;
  return (r != 0 && ((r < 0) != (b < 0))) ? r + b : r;
}

// ============================================================ task mapping ==
namespace {
uint64_t mul_or_fail(uint64_t a, uint64_t b, const char* what) {
  uint64_t r;
  if (__builtin_mul_overflow(a, b, &r)) fail("overflow computing ", what, ": ", a, " * ", b);
  return r;
}
}  // namespace

TaskShape::TaskShape(std::vector<uint64_t> dims) : dims_(std::move(dims)) {
  if (dims_.empty()) fail("task shape must have at least one dimension");
  for (uint64_t d : dims_) {
    if (d == 0) fail("task shape extents must be positive");
    volume_ = mul_or_fail(volume_, d, "task shape volume");
  }
}

TaskShape TaskShape::elementwise_mul(const TaskShape& o) const {
  if (rank() != o.rank())
    fail("elementwise product needs equal ranks, got ", rank(), " and ", o.rank());
  std::vector<uint64_t> out;
  out.reserve(rank());
  for (size_t i = 0; i < rank(); ++i) out.push_back(mul_or_fail(dims_[i], o.dims_[i], "task shape"));
  return TaskShape(std::move(out));
}

struct TaskMapping::Rep {
  Kind kind = Kind::Repeat;
  TaskShape shape;
  uint64_t workers = 1;
  uint64_t per_worker = 1;
  std::shared_ptr<const Rep> outer, inner;  // Compose
  std::vector<std::vector<Task>> table;     // Custom
};

TaskMapping TaskMapping::repeat(TaskShape shape) {
  auto r = std::make_shared<Rep>();
  r->kind = Kind::Repeat;
  r->per_worker = shape.total();
  r->shape = std::move(shape);
  return TaskMapping(r);
}

TaskMapping TaskMapping::spatial(TaskShape shape) {
  auto r = std::make_shared<Rep>();
  r->kind = Kind::Spatial;
  r->workers = shape.total();
  r->shape = std::move(shape);
  return TaskMapping(r);
}

// mapping.cpp:64-85
TaskMapping TaskMapping::custom(uint64_t num_workers, TaskShape shape,
                                std::vector<std::vector<Task>> table) {
  if (num_workers == 0) fail("custom mapping needs at least one worker");
  if (table.size() != num_workers)
    fail("custom mapping table must list every worker: got ", table.size(), " lists for ",
         num_workers, " workers");
  for (const auto& list : table)
    for (const Task& t : list) {
      if (t.size() != shape.rank())
        fail("custom task rank ", t.size(), " does not match shape rank ", shape.rank());
      for (size_t d = 0; d < t.size(); ++d)
        if (t[d] >= shape[d]) fail("custom task coordinate ", t[d], " outside extent ", shape[d]);
    }
  auto r = std::make_shared<Rep>();
  r->kind = Kind::Custom;
  r->workers = num_workers;
  r->per_worker = table.empty() ? 0 : table.front().size();
  r->shape = std::move(shape);
  r->table = std::move(table);
  return TaskMapping(r);
}

// mapping.cpp:87-99: workers n1*n2, shape d1 (.) d2
TaskMapping TaskMapping::compose(const TaskMapping& outer, const TaskMapping& inner) {
  if (outer.task_dim() != inner.task_dim())
    fail("cannot compose mappings with task dimensions ", outer.task_dim(), " and ",
         inner.task_dim());
  auto r = std::make_shared<Rep>();
  r->kind = Kind::Compose;
  r->workers = mul_or_fail(outer.rep_->workers, inner.rep_->workers, "composed worker count");
  r->per_worker = mul_or_fail(outer.rep_->per_worker, inner.rep_->per_worker, "tasks per worker");
  r->shape = outer.task_shape().elementwise_mul(inner.task_shape());
  r->outer = outer.rep_;
  r->inner = inner.rep_;
  return TaskMapping(r);
}

TaskMapping::Kind TaskMapping::kind() const { return rep_->kind; }
uint64_t TaskMapping::num_workers() const { return rep_->workers; }
const TaskShape& TaskMapping::task_shape() const { return rep_->shape; }

uint64_t TaskMapping::tasks_per_worker() const {
  if (rep_->kind == Kind::Custom)
    for (const auto& l : rep_->table)
      if (l.size() != rep_->per_worker) fail("custom mapping has non-uniform per-worker task counts");
  return rep_->per_worker;
}

TaskMapping TaskMapping::lhs() const {
  if (rep_->kind != Kind::Compose) fail("lhs() requires a composed mapping");
  return TaskMapping(rep_->outer);
}
TaskMapping TaskMapping::rhs() const {
  if (rep_->kind != Kind::Compose) fail("rhs() requires a composed mapping");
  return TaskMapping(rep_->inner);
}
const std::vector<std::vector<Task>>& TaskMapping::table() const {
  if (rep_->kind != Kind::Custom) fail("table() requires a custom mapping");
  return rep_->table;
}

namespace {
// row-major coordinates of `flat` inside `shape`
Task delinearize(uint64_t flat, const TaskShape& shape) {
  Task t(shape.rank());
  for (size_t d = shape.rank(); d-- > 0;) {
    t[d] = flat % shape[d];
    flat /= shape[d];
  }
  return t;
}
}  // namespace

// mapping.cpp:155-188 (repeat: row-major domain; spatial: delinearised
// worker id; compose: t1 (.) d2 + t2 with the outer list as the outer loop).
std::vector<Task> TaskMapping::assign(uint64_t worker) const {
  const Rep& r = *rep_;
  if (worker >= r.workers)
    fail("worker id ", worker, " out of range for ", r.workers, " workers");
  std::vector<Task> out;
  switch (r.kind) {
    case Kind::Repeat:
      out.reserve(r.shape.total());
      for (uint64_t f = 0; f < r.shape.total(); ++f) out.push_back(delinearize(f, r.shape));
      return out;
    case Kind::Spatial:
      out.push_back(delinearize(worker, r.shape));
      return out;
    case Kind::Custom:
      return r.table[worker];
    case Kind::Compose: {
      const TaskMapping o(r.outer), in(r.inner);
      const uint64_t n_in = in.num_workers();
      const auto outer_tasks = o.assign(worker / n_in);
      const auto inner_tasks = in.assign(worker % n_in);
      const auto& d2 = in.task_shape();
      out.reserve(outer_tasks.size() * inner_tasks.size());
      for (const Task& a : outer_tasks)
        for (const Task& b : inner_tasks) {
          Task t(a.size());
          for (size_t d = 0; d < t.size(); ++d) t[d] = a[d] * d2[d] + b[d];
          out.push_back(std::move(t));
        }
      return out;
    }
  }
  fail("unreachable mapping kind");
}

namespace {
std::string dims_text(const TaskShape& s) {
  std::string o;
  for (size_t i = 0; i < s.rank(); ++i) o += (i ? ", " : "") + std::to_string(s[i]);
  return o;
}
}  // namespace

// mapping.cpp:190-231
std::string TaskMapping::to_text() const {
  const Rep& r = *rep_;
  switch (r.kind) {
    case Kind::Repeat: return "repeat(" + dims_text(r.shape) + ")";
    case Kind::Spatial: return "spatial(" + dims_text(r.shape) + ")";
    case Kind::Compose: return TaskMapping(r.outer).to_text() + " * " + TaskMapping(r.inner).to_text();
    case Kind::Custom: {
      std::string o = "custom(workers=" + std::to_string(r.workers) + ", shape=(" + dims_text(r.shape) + "), table=[";
      for (size_t w = 0; w < r.table.size(); ++w) {
        o += w ? ", [" : "[";
        for (size_t j = 0; j < r.table[w].size(); ++j) {
          o += j ? ", (" : "(";
          for (size_t d = 0; d < r.table[w][j].size(); ++d)
            o += (d ? ", " : "") + std::to_string(r.table[w][j][d]);
          o += ")";
        }
        o += "]";
      }
      return o + "])";
    }
  }
  fail("unreachable mapping kind");
}

// mapping.cpp:233-265 (cells "w{id}:{order}", left-aligned, padded to the widest)
std::string TaskMapping::visualize() const {
  const size_t dim = task_dim();
  if (dim > 2) fail("visualize supports task dimension <= 2, got ", dim);
  const uint64_t rows = dim == 2 ? task_shape()[0] : 1;
  const uint64_t cols = dim == 2 ? task_shape()[1] : task_shape()[0];
  std::vector<std::string> cell(rows * cols);
  for (uint64_t w = 0; w < num_workers(); ++w) {
    const auto tasks = assign(w);
    for (size_t k = 0; k < tasks.size(); ++k) {
      const uint64_t rr = dim == 2 ? tasks[k][0] : 0, cc = dim == 2 ? tasks[k][1] : tasks[k][0];
      std::string& s = cell[rr * cols + cc];
      const std::string lab = "w" + std::to_string(w) + ":" + std::to_string(k);
      s = s.empty() ? lab : s + "," + lab;
    }
  }
  size_t width = 1;
  for (auto& s : cell) {
    if (s.empty()) s = "-";
    width = std::max(width, s.size());
  }
  std::string out;
  for (uint64_t rr = 0; rr < rows; ++rr) {
    for (uint64_t cc = 0; cc < cols; ++cc) {
      const std::string& s = cell[rr * cols + cc];
      if (cc) out += ' ';
      out += s;
      if (cc + 1 < cols) out.append(width - s.size(), ' ');
    }
    out += '\n';
  }
  return out;
}

bool TaskMapping::operator==(const TaskMapping& o) const {
  if (rep_ == o.rep_) return true;
  const Rep &a = *rep_, &b = *o.rep_;
  if (a.kind != b.kind || !(a.shape == b.shape) || a.workers != b.workers) return false;
  if (a.kind == Kind::Custom) return a.table == b.table;
  if (a.kind == Kind::Compose)
    return TaskMapping(a.outer) == TaskMapping(b.outer) && TaskMapping(a.inner) == TaskMapping(b.inner);
  return true;
}

std::vector<TaskMapping::Atom> TaskMapping::atoms() const {
  const Rep& r = *rep_;
  switch (r.kind) {
    case Kind::Repeat: return {Atom{false, r.shape.dims()}};
    case Kind::Spatial: return {Atom{true, r.shape.dims()}};
    case Kind::Compose: {
      auto a = TaskMapping(r.outer).atoms();
      auto b = TaskMapping(r.inner).atoms();
      a.insert(a.end(), b.begin(), b.end());
      return a;
    }
    case Kind::Custom: fail("custom mappings have no closed-form atom chain");
  }
  fail("unreachable mapping kind");
}

TaskMapping operator*(const TaskMapping& a, const TaskMapping& b) { return TaskMapping::compose(a, b); }

// Canonical text grammar (mapping.cpp:292-402): atoms joined left-associatively by '*'.
namespace {
class MappingReader {
 public:
  explicit MappingReader(const std::string& s) : s_(s) {}
  TaskMapping chain() {
    TaskMapping m = atom();
    while (take('*')) m = m * atom();
    return m;
  }
  void finish() {
    space();
    if (i_ != s_.size()) fail("mapping parse error: trailing input at offset ", i_);
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  void space() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool take(char c) {
    space();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  void need(char c) {
    if (!take(c)) fail("mapping parse error at offset ", i_, ": expected '", c, "'");
  }
  bool word(const std::string& w) {
    space();
    if (s_.compare(i_, w.size(), w) == 0) {
      i_ += w.size();
      return true;
    }
    return false;
  }
  uint64_t number() {
    space();
    const size_t b = i_;
    while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
    if (b == i_) fail("mapping parse error at offset ", i_, ": expected integer");
    return std::stoull(s_.substr(b, i_ - b));
  }
  std::vector<uint64_t> tuple() {
    need('(');
    std::vector<uint64_t> v{number()};
    while (take(',')) v.push_back(number());
    need(')');
    return v;
  }
  TaskMapping atom() {
    space();
    if (word("repeat")) return TaskMapping::repeat(TaskShape(tuple()));
    if (word("spatial")) return TaskMapping::spatial(TaskShape(tuple()));
    if (word("custom")) {
      need('(');
      if (!word("workers")) fail("custom mapping: expected workers=");
      need('=');
      const uint64_t n = number();
      need(',');
      if (!word("shape")) fail("custom mapping: expected shape=");
      need('=');
      TaskShape shape(tuple());
      need(',');
      if (!word("table")) fail("custom mapping: expected table=");
      need('=');
      need('[');
      std::vector<std::vector<Task>> table;
      if (!take(']')) {
        do {
          need('[');
          std::vector<Task> list;
          if (!take(']')) {
            do list.push_back(Task(tuple()));
            while (take(','));
            need(']');
          }
          table.push_back(std::move(list));
        } while (take(','));
        need(']');
      }
      need(')');
      return TaskMapping::custom(n, shape, std::move(table));
    }
    if (take('(')) {
      TaskMapping m = chain();
      need(')');
      return m;
    }
    fail("mapping parse error at offset ", i_, ": expected repeat/spatial/custom");
  }
};
}  // namespace

TaskMapping parse_mapping(const std::string& text) {
  MappingReader r(text);
  TaskMapping m = r.chain();
  r.finish();
  return m;
}

// ============================================================= expressions ==
namespace {
Expr node(ExprNode n) { return std::make_shared<const ExprNode>(std::move(n)); }
Expr leaf(ExprKind k) {
  ExprNode n;
  n.kind = k;
  return node(std::move(n));
}
}  // namespace

Expr imm(int64_t v) { ExprNode n; n.kind = ExprKind::IntImm; n.ival = v; return node(std::move(n)); }
Expr fimm(double v) { ExprNode n; n.kind = ExprKind::FloatImm; n.fval = v; return node(std::move(n)); }
Expr var(const std::string& name) { ExprNode n; n.kind = ExprKind::Var; n.name = name; return node(std::move(n)); }
Expr thread_idx() { return leaf(ExprKind::ThreadIdx); }
Expr block_idx() { return leaf(ExprKind::BlockIdx); }

// expr.cpp:48-56: div/mod by the constant 0 is a construction error
Expr binary(BinOp op, Expr a, Expr b) {
  if ((op == BinOp::Div || op == BinOp::Mod) && b->is_const_int(0)) fail("division/modulo by zero constant");
  ExprNode n;
  n.kind = ExprKind::Binary;
  n.bop = op;
  n.args = {std::move(a), std::move(b)};
  return node(std::move(n));
}
Expr unary(UnOp op, Expr a) {
  ExprNode n;
  n.kind = ExprKind::Unary;
  n.uop = op;
  n.args = {std::move(a)};
  return node(std::move(n));
}
Expr select(Expr c, Expr t, Expr e) {
  ExprNode n;
  n.kind = ExprKind::Select;
  n.args = {std::move(c), std::move(t), std::move(e)};
  return node(std::move(n));
}
Expr load(const std::string& buffer, std::vector<Expr> idx) {
  ExprNode n;
  n.kind = ExprKind::Load;
  n.name = buffer;
  n.args = std::move(idx);
  return node(std::move(n));
}
Expr table_lookup(IndexTable table, Expr index) {
  if (!table || table->empty()) fail("table lookup needs a non-empty table");
  ExprNode n;
  n.kind = ExprKind::TableLookup;
  n.table = std::move(table);
  n.args = {std::move(index)};
  return node(std::move(n));
}

Expr gelu_tanh(Expr x) {
  // u = 2 * sqrt(2/pi) * (x + 0.044715 * x^3); tanh(v) = 1 - 2 / (exp(2v) + 1)
  Expr x3 = mul(mul(x, x), x);
  Expr inner = mul(fimm(0.7978845608028654), add(x, mul(fimm(0.044715), x3)));
  Expr t = sub(fimm(1.0), div(fimm(2.0), add(unary(UnOp::Exp, mul(fimm(2.0), inner)), fimm(1.0))));
  return mul(mul(fimm(0.5), x), add(fimm(1.0), t));
}

namespace {
template <class F>
Expr rebuild(const Expr& e, F&& f) {
  if (e->args.empty()) return e;
  std::vector<Expr> kids;
  kids.reserve(e->args.size());
  bool same = true;
  for (const Expr& a : e->args) {
    kids.push_back(f(a));
    same = same && kids.back() == a;
  }
  if (same) return e;
  ExprNode n = *e;
  n.args = std::move(kids);
  return node(std::move(n));
}
}  // namespace

Expr substitute(const Expr& e, const std::map<std::string, Expr>& vars) {
  if (e->kind == ExprKind::Var) {
    auto it = vars.find(e->name);
    return it == vars.end() ? e : it->second;
  }
  return rebuild(e, [&](const Expr& a) { return substitute(a, vars); });
}

Expr rewrite_loads(const Expr& e, const std::function<std::optional<Expr>(const ExprNode&)>& fn) {
  Expr m = rebuild(e, [&](const Expr& a) { return rewrite_loads(a, fn); });
  if (m->kind == ExprKind::Load)
    if (auto r = fn(*m)) return *r;
  return m;
}

namespace {
bool no_memory(const Expr& e) {
  if (e->kind == ExprKind::Load || e->kind == ExprKind::TableLookup) return false;
  return std::all_of(e->args.begin(), e->args.end(), no_memory);
}
bool is_compare(BinOp op) {
  return op == BinOp::Lt || op == BinOp::Le || op == BinOp::Gt || op == BinOp::Ge || op == BinOp::Eq || op == BinOp::Ne;
}
bool is_logic(BinOp op) { return op == BinOp::And || op == BinOp::Or; }
int64_t int_op(BinOp op, int64_t a, int64_t b) {
  switch (op) {
    case BinOp::Add: return a + b;
    case BinOp::Sub: return a - b;
    case BinOp::Mul: return a * b;
    case BinOp::Div: return floordiv(a, b);
    case BinOp::Mod: return floormod(a, b);
    case BinOp::Min: return std::min(a, b);
    case BinOp::Max: return std::max(a, b);
    case BinOp::And: return (a != 0 && b != 0) ? 1 : 0;
    case BinOp::Or: return (a != 0 || b != 0) ? 1 : 0;
    case BinOp::Lt: return a < b;
    case BinOp::Le: return a <= b;
    case BinOp::Gt: return a > b;
    case BinOp::Ge: return a >= b;
    case BinOp::Eq: return a == b;
    case BinOp::Ne: return a != b;
  }
  fail("unreachable binop");
}
double real_op(BinOp op, double a, double b) {
  switch (op) {
    case BinOp::Add: return a + b;
    case BinOp::Sub: return a - b;
    case BinOp::Mul: return a * b;
    case BinOp::Div: return a / b;
    case BinOp::Min: return std::min(a, b);
    case BinOp::Max: return std::max(a, b);
    default: fail("binop ", binop_name(op), " not foldable on floats here");
  }
}
}  // namespace

// expr.cpp:175-264 — constant folding + identities that only drop pure scalars
Expr fold(const Expr& e) {
  Expr m = rebuild(e, [](const Expr& a) { return fold(a); });
  if (m->kind == ExprKind::Binary) {
    const Expr &a = m->args[0], &b = m->args[1];
    const BinOp op = m->bop;
    const bool ai = a->kind == ExprKind::IntImm, bi = b->kind == ExprKind::IntImm;
    const bool af = a->kind == ExprKind::FloatImm, bf = b->kind == ExprKind::FloatImm;
    const bool arith = !is_compare(op) && !is_logic(op) && op != BinOp::Mod;
    if (ai && bi) return imm(int_op(op, a->ival, b->ival));
    if (af && bf && arith) return fimm(real_op(op, a->fval, b->fval));
    if (ai && bf && arith && op != BinOp::Div) return fimm(real_op(op, static_cast<double>(a->ival), b->fval));
    if (af && bi && arith && op != BinOp::Div) return fimm(real_op(op, a->fval, static_cast<double>(b->ival)));
    switch (op) {
      case BinOp::Add:
        if (a->is_const_int(0)) return b;
        if (b->is_const_int(0)) return a;
        break;
      case BinOp::Sub:
        if (b->is_const_int(0)) return a;
        break;
      case BinOp::Mul:
        if (a->is_const_int(1)) return b;
        if (b->is_const_int(1)) return a;
        if ((a->is_const_int(0) && no_memory(b)) || (b->is_const_int(0) && no_memory(a))) return imm(0);
        break;
      case BinOp::Div:
        if (b->is_const_int(1)) return a;
        break;
      case BinOp::Mod:
        if (b->is_const_int(1) && no_memory(a)) return imm(0);
        break;
      case BinOp::And:
        if (a->is_const_int(1)) return b;
        if (b->is_const_int(1)) return a;
        break;
      default: break;
    }
    return m;
  }
  if (m->kind == ExprKind::Unary) {
    const Expr& a = m->args[0];
    if (a->kind == ExprKind::IntImm) {
      switch (m->uop) {
        case UnOp::Neg: return imm(-a->ival);
        case UnOp::Relu: return imm(std::max<int64_t>(a->ival, 0));
        case UnOp::CastI32: return a;
        case UnOp::CastF32: return fimm(static_cast<double>(a->ival));
        default: break;
      }
    } else if (a->kind == ExprKind::FloatImm) {
      switch (m->uop) {
        case UnOp::Neg: return fimm(-a->fval);
        case UnOp::Relu: return fimm(std::max(a->fval, 0.0));
        case UnOp::Exp: return fimm(std::exp(a->fval));
        case UnOp::Sqrt: return fimm(std::sqrt(a->fval));
        case UnOp::CastF32: return a;
        case UnOp::CastI32: return imm(static_cast<int64_t>(a->fval));
      }
    }
    return m;
  }
  if (m->kind == ExprKind::Select && m->args[0]->kind == ExprKind::IntImm)
    return m->args[0]->ival != 0 ? m->args[1] : m->args[2];
  if (m->kind == ExprKind::TableLookup && m->args[0]->kind == ExprKind::IntImm) {
    const int64_t i = m->args[0]->ival;
    if (i < 0 || static_cast<size_t>(i) >= m->table->size()) fail("constant table lookup out of range: ", i);
    return imm((*m->table)[i]);
  }
  return m;
}

bool expr_equal(const Expr& a, const Expr& b) {
  if (a == b) return true;
  if (a->kind != b->kind || a->args.size() != b->args.size()) return false;
  switch (a->kind) {
    case ExprKind::IntImm: return a->ival == b->ival;
    case ExprKind::FloatImm: return a->fval == b->fval;
    case ExprKind::Var: return a->name == b->name;
    case ExprKind::ThreadIdx:
    case ExprKind::BlockIdx: return true;
    case ExprKind::Binary: if (a->bop != b->bop) return false; break;
    case ExprKind::Unary: if (a->uop != b->uop) return false; break;
    case ExprKind::Load: if (a->name != b->name) return false; break;
    case ExprKind::TableLookup: if (a->table != b->table && *a->table != *b->table) return false; break;
    case ExprKind::Select: break;
  }
  for (size_t i = 0; i < a->args.size(); ++i)
    if (!expr_equal(a->args[i], b->args[i])) return false;
  return true;
}

bool uses_thread_idx(const Expr& e) {
  if (e->kind == ExprKind::ThreadIdx) return true;
  return std::any_of(e->args.begin(), e->args.end(), uses_thread_idx);
}
void collect_vars(const Expr& e, std::vector<std::string>& out) {
  if (e->kind == ExprKind::Var) out.push_back(e->name);
  for (const Expr& a : e->args) collect_vars(a, out);
}
void collect_loads(const Expr& e, std::vector<Expr>& out) {
  if (e->kind == ExprKind::Load) out.push_back(e);
  for (const Expr& a : e->args) collect_loads(a, out);
}

const char* binop_name(BinOp op) {
  static const char* n[] = {"+", "-", "*", "/", "%", "min", "max", "&&", "||", "<", "<=", ">", ">=", "==", "!="};
  return n[static_cast<int>(op)];
}
const char* unop_name(UnOp op) {
  static const char* n[] = {"-", "relu", "exp", "sqrt", "f32", "i32"};
  return n[static_cast<int>(op)];
}

namespace {
int prec_of(BinOp op) {
  switch (op) {
    case BinOp::Or: return 1;
    case BinOp::And: return 2;
    case BinOp::Add: case BinOp::Sub: return 4;
    case BinOp::Mul: case BinOp::Div: case BinOp::Mod: return 5;
    case BinOp::Min: case BinOp::Max: return 9;
    default: return 3;  // comparisons
  }
}
std::string real_text(double v) {
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".e") == std::string::npos) s += ".0";
  return s;
}
void emit(std::string& o, const Expr& e, int ctx) {
  switch (e->kind) {
    case ExprKind::IntImm: o += e->ival < 0 ? "(" + std::to_string(e->ival) + ")" : std::to_string(e->ival); return;
    case ExprKind::FloatImm: { std::string s = real_text(e->fval); o += s[0] == '-' ? "(" + s + ")" : s; return; }
    case ExprKind::Var: o += e->name; return;
    case ExprKind::ThreadIdx: o += "threadIdx"; return;
    case ExprKind::BlockIdx: o += "blockIdx"; return;
    case ExprKind::Binary: {
      if (e->bop == BinOp::Min || e->bop == BinOp::Max) {
        o += e->bop == BinOp::Min ? "min(" : "max(";
        emit(o, e->args[0], 0);
        o += ", ";
        emit(o, e->args[1], 0);
        o += ")";
        return;
      }
      const int p = prec_of(e->bop);
      if (p < ctx) o += "(";
      emit(o, e->args[0], p);
      o += std::string(" ") + binop_name(e->bop) + " ";
      emit(o, e->args[1], p + 1);
      if (p < ctx) o += ")";
      return;
    }
    case ExprKind::Unary:
      if (e->uop == UnOp::Neg) { o += "-"; emit(o, e->args[0], 8); return; }
      o += std::string(unop_name(e->uop)) + "(";
      emit(o, e->args[0], 0);
      o += ")";
      return;
    case ExprKind::Select:
      o += "select(";
      for (int i = 0; i < 3; ++i) { if (i) o += ", "; emit(o, e->args[i], 0); }
      o += ")";
      return;
    case ExprKind::Load:
      o += e->name + "[";
      for (size_t i = 0; i < e->args.size(); ++i) { if (i) o += ", "; emit(o, e->args[i], 0); }
      o += "]";
      return;
    case ExprKind::TableLookup:
      o += "lookup([";
      for (size_t i = 0; i < e->table->size(); ++i) o += (i ? ", " : "") + std::to_string((*e->table)[i]);
      o += "], ";
      emit(o, e->args[0], 0);
      o += ")";
      return;
  }
}
}  // namespace

std::string expr_to_text(const Expr& e) {
  std::string o;
  emit(o, e, 0);
  return o;
}

// ==================================================================== DAG ==
const char* combiner_name(Combiner c) {
  return c == Combiner::Sum ? "sum" : c == Combiner::Max ? "max" : "min";
}
Combiner combiner_from_name(const std::string& s) {
  if (s == "sum") return Combiner::Sum;
  if (s == "max") return Combiner::Max;
  if (s == "min") return Combiner::Min;
  fail("unknown combiner: ", s);
}
const char* opclass_name(OpClass c) {
  return c == OpClass::Reduction ? "reduction" : c == OpClass::Injective ? "injective" : "bijective";
}

const TensorNode* ComputeDAG::find(const std::string& name) const {
  for (const auto& n : nodes)
    if (n.name == name) return &n;
  return nullptr;
}
const TensorNode& ComputeDAG::at(const std::string& name) const {
  if (const TensorNode* n = find(name)) return *n;
  fail("no tensor named '", name, "' in DAG");
}

// compute_ir.cpp:48-101 — same checks, same messages
void ComputeDAG::validate() const {
  std::set<std::string> names;
  for (size_t idx = 0; idx < nodes.size(); ++idx) {
    const TensorNode& n = nodes[idx];
    if (n.name.empty()) fail("tensor node with empty name");
    if (!names.insert(n.name).second) fail("duplicate tensor name '", n.name, "'");
    if (n.shape.empty()) fail("tensor '", n.name, "' has empty shape");
    for (int64_t d : n.shape)
      if (d <= 0) fail("tensor '", n.name, "' has non-positive extent");
    if (!n.is_computed()) continue;
    if (!n.value) fail("computed tensor '", n.name, "' has no value expression");
    if (n.axes.size() != n.shape.size()) fail("tensor '", n.name, "': spatial axis count does not match shape rank");
    for (size_t i = 0; i < n.axes.size(); ++i)
      if (n.axes[i].extent != n.shape[i]) fail("tensor '", n.name, "': axis extent mismatch at dim ", i);
    if (n.kind == NodeKind::GridReduce && n.reduce_axes.empty()) fail("reduce tensor '", n.name, "' has no reduce axes");
    if (n.kind == NodeKind::GridCompute && !n.reduce_axes.empty()) fail("grid compute '", n.name, "' cannot have reduce axes");
    std::set<std::string> bound;
    for (const Axis& a : n.axes) bound.insert(a.name);
    for (const Axis& a : n.reduce_axes)
      if (!bound.insert(a.name).second) fail("duplicate axis '", a.name, "'");
    std::vector<std::string> vs;
    collect_vars(n.value, vs);
    for (const auto& v : vs)
      if (!bound.count(v)) fail("tensor '", n.name, "' uses undeclared axis '", v, "'");
    std::vector<Expr> ls;
    collect_loads(n.value, ls);
    for (const Expr& l : ls) {
      const TensorNode* src = nullptr;
      for (size_t j = 0; j < idx; ++j)
        if (nodes[j].name == l->name) { src = &nodes[j]; break; }
      if (!src) fail("tensor '", n.name, "' reads '", l->name, "' which is not defined before it");
      if (l->args.size() != src->shape.size()) fail("access to '", l->name, "' in '", n.name, "' has wrong rank");
    }
  }
  for (const auto& i : inputs) {
    const TensorNode* n = find(i);
    if (!n || n->kind != NodeKind::Input) fail("declared input '", i, "' is not an input node");
  }
  for (const auto& o : outputs) {
    const TensorNode* n = find(o);
    if (!n || !n->is_computed()) fail("declared output '", o, "' is not a computed node");
  }
}

// ---------------------------------------------------- affine access + classify
namespace {
// Linear form of an index expression over the node's spatial axes; only
// +, -, unary -, and multiplication by an integer constant are affine
// (compute_ir.cpp:119-151).
bool linearize(const Expr& e, int64_t scale, const std::vector<Axis>& axes, AffineIndex& out) {
  switch (e->kind) {
    case ExprKind::IntImm:
      out.offset += scale * e->ival;
      return true;
    case ExprKind::Var:
      for (size_t i = 0; i < axes.size(); ++i)
        if (axes[i].name == e->name) {
          out.terms.push_back({i, scale});
          return true;
        }
      return false;
    case ExprKind::Unary:
      return e->uop == UnOp::Neg && linearize(e->args[0], -scale, axes, out);
    case ExprKind::Binary: {
      const Expr &a = e->args[0], &b = e->args[1];
      if (e->bop == BinOp::Add) return linearize(a, scale, axes, out) && linearize(b, scale, axes, out);
      if (e->bop == BinOp::Sub) return linearize(a, scale, axes, out) && linearize(b, -scale, axes, out);
      if (e->bop == BinOp::Mul) {
        if (a->kind == ExprKind::IntImm) return linearize(b, scale * a->ival, axes, out);
        if (b->kind == ExprKind::IntImm) return linearize(a, scale * b->ival, axes, out);
      }
      return false;
    }
    default:
      return false;
  }
}
}  // namespace

std::optional<std::vector<AffineIndex>> analyze_affine_access(const Expr& ld, const std::vector<Axis>& axes) {
  if (ld->kind != ExprKind::Load) fail("analyze_affine_access expects a Load");
  std::vector<AffineIndex> res;
  for (const Expr& ix : ld->args) {
    AffineIndex raw;
    if (!linearize(ix, 1, axes, raw)) return std::nullopt;
    // merge repeated axes; drop zero coefficients and unit-extent axes (:155-164)
    std::vector<int64_t> c(axes.size(), 0);
    for (const auto& t : raw.terms) c[t.axis] += t.coeff;
    AffineIndex norm;
    norm.offset = raw.offset;
    for (size_t a = 0; a < axes.size(); ++a)
      if (c[a] != 0 && axes[a].extent != 1) norm.terms.push_back({a, c[a]});
    res.push_back(std::move(norm));
  }
  return res;
}

// compute_ir.cpp:182-203: each non-unit axis used exactly once, and within each
// index the terms pack mixed-radix: |c_t| >= |c_{t+1}| * e_{t+1}.
bool affine_access_injective(const std::vector<AffineIndex>& acc, const std::vector<Axis>& axes) {
  std::vector<int> used(axes.size(), 0);
  for (const auto& ix : acc)
    for (const auto& t : ix.terms) ++used[t.axis];
  for (size_t a = 0; a < axes.size(); ++a)
    if (axes[a].extent != 1 && used[a] != 1) return false;
  for (const auto& ix : acc) {
    auto ts = ix.terms;
    std::stable_sort(ts.begin(), ts.end(), [](const AffineTerm& x, const AffineTerm& y) {
      return std::llabs(x.coeff) > std::llabs(y.coeff);
    });
    for (size_t i = 1; i < ts.size(); ++i)
      if (std::llabs(ts[i - 1].coeff) < std::llabs(ts[i].coeff) * axes[ts[i].axis].extent) return false;
  }
  return true;
}

// compute_ir.cpp:205-220: additionally each index covers exactly [0, extent).
bool affine_access_bijective(const std::vector<AffineIndex>& acc, const std::vector<Axis>& axes,
                             const std::vector<int64_t>& shape) {
  if (acc.size() != shape.size() || !affine_access_injective(acc, axes)) return false;
  for (size_t d = 0; d < acc.size(); ++d) {
    int64_t lo = acc[d].offset, hi = acc[d].offset, cnt = 1;
    for (const auto& t : acc[d].terms) {
      const int64_t span = t.coeff * (axes[t.axis].extent - 1);
      (span < 0 ? lo : hi) += span;
      cnt *= axes[t.axis].extent;
    }
    if (lo != 0 || hi != shape[d] - 1 || cnt != shape[d]) return false;
  }
  return true;
}

// compute_ir.cpp:222-243
OpClass classify(const ComputeDAG& dag, const TensorNode& n) {
  if (!n.is_computed()) fail("classify expects a computed node");
  if (n.kind == NodeKind::GridReduce) return OpClass::Reduction;
  std::vector<Expr> ls;
  collect_loads(n.value, ls);
  std::vector<std::pair<std::string, Expr>> uniq;  // first access per tensor
  for (const Expr& l : ls) {
    auto it = std::find_if(uniq.begin(), uniq.end(), [&](const auto& p) { return p.first == l->name; });
    if (it == uniq.end()) uniq.emplace_back(l->name, l);
    else if (!expr_equal(it->second, l)) return OpClass::Injective;
  }
  bool any_bij = false;
  for (const auto& [name, l] : uniq) {
    const auto acc = analyze_affine_access(l, n.axes);
    if (!acc) return OpClass::Injective;
    const TensorNode* src = dag.find(name);
    if (!src) return OpClass::Injective;
    any_bij = any_bij || affine_access_bijective(*acc, n.axes, src->shape);
  }
  return any_bij ? OpClass::Bijective : OpClass::Injective;
}

// =============================================================== builders ==
namespace {
TensorNode placeholder(const std::string& name, std::vector<int64_t> shape, DType dt) {
  TensorNode t;
  t.name = name;
  t.shape = std::move(shape);
  t.dtype = dt;
  return t;
}
TensorNode grid(const std::string& name, std::vector<Axis> axes, DType dt, Expr value) {
  TensorNode t;
  t.name = name;
  t.kind = NodeKind::GridCompute;
  t.dtype = dt;
  for (const auto& a : axes) t.shape.push_back(a.extent);
  t.axes = std::move(axes);
  t.value = std::move(value);
  return t;
}
std::vector<Axis> numbered_axes(const std::vector<int64_t>& shape) {
  std::vector<Axis> v;
  for (size_t i = 0; i < shape.size(); ++i) v.push_back({"i" + std::to_string(i), shape[i]});
  return v;
}
std::vector<Expr> as_vars(const std::vector<Axis>& axes) {
  std::vector<Expr> v;
  for (const auto& a : axes) v.push_back(var(a.name));
  return v;
}
ComputeDAG finish(ComputeDAG d, std::vector<std::string> in, std::vector<std::string> out) {
  d.inputs = std::move(in);
  d.outputs = std::move(out);
  d.validate();
  return d;
}
}  // namespace

// compute_ir.cpp:496-515
ComputeDAG matmul_dag(int64_t m, int64_t n, int64_t k, DType dt) {
  if (m <= 0 || n <= 0 || k <= 0) fail("matmul extents must be positive");
  ComputeDAG d;
  d.nodes.push_back(placeholder("A", {m, k}, dt));
  d.nodes.push_back(placeholder("B", {k, n}, dt));
  TensorNode c = grid("C", {{"i", m}, {"j", n}}, dt,
                      mul(load("A", {var("i"), var("k")}), load("B", {var("k"), var("j")})));
  c.kind = NodeKind::GridReduce;
  c.reduce_axes = {{"k", k}};
  d.nodes.push_back(std::move(c));
  return finish(std::move(d), {"A", "B"}, {"C"});
}

// compute_ir.cpp:517-597: im2col gather -> GEMM anchor -> NCHW reshape
ComputeDAG conv2d_im2col_dag(int64_t n, int64_t c, int64_t h, int64_t w, int64_t f, int64_t kh,
                             int64_t kw, int64_t stride, int64_t pad, DType dt) {
  if (n <= 0 || c <= 0 || h <= 0 || w <= 0 || f <= 0 || kh <= 0 || kw <= 0) fail("conv extents must be positive");
  if (stride <= 0 || pad < 0) fail("invalid conv stride/padding");
  if (kh > h + 2 * pad || kw > w + 2 * pad) fail("conv kernel larger than padded input");
  const int64_t ho = conv_out_extent(h, kh, stride, pad), wo = conv_out_extent(w, kw, stride, pad);
  const int64_t gk = c * kh * kw, gn = n * ho * wo;
  auto tap = [&](const Expr& r) {  // r -> (channel, fh, fw)
    return std::vector<Expr>{div(r, imm(kh * kw)), mod(div(r, imm(kw)), imm(kh)), mod(r, imm(kw))};
  };
  ComputeDAG d;
  d.nodes.push_back(placeholder("X", {n, c, h, w}, dt));
  d.nodes.push_back(placeholder("W", {f, c, kh, kw}, dt));
  {
    const Expr r = var("r"), s = var("s");
    const auto t = tap(r);
    const Expr img = div(s, imm(ho * wo)), oh = mod(div(s, imm(wo)), imm(ho)), ow = mod(s, imm(wo));
    const Expr ih = add(sub(mul(oh, imm(stride)), imm(pad)), t[1]);
    const Expr iw = add(sub(mul(ow, imm(stride)), imm(pad)), t[2]);
    Expr v = load("X", {img, t[0], ih, iw});
    if (pad > 0)
      v = select(land(land(ge(ih, imm(0)), lt(ih, imm(h))), land(ge(iw, imm(0)), lt(iw, imm(w)))), v, zero_of(dt));
    d.nodes.push_back(grid("Col", {{"r", gk}, {"s", gn}}, dt, v));
  }
  {
    const auto t = tap(var("r"));
    d.nodes.push_back(grid("Wf", {{"p", f}, {"r", gk}}, dt, load("W", {var("p"), t[0], t[1], t[2]})));
  }
  {
    TensorNode y = grid("Y", {{"p", f}, {"s", gn}}, dt,
                        mul(load("Wf", {var("p"), var("r")}), load("Col", {var("r"), var("s")})));
    y.kind = NodeKind::GridReduce;
    y.reduce_axes = {{"r", gk}};
    d.nodes.push_back(std::move(y));
  }
  d.nodes.push_back(grid("Out", {{"n", n}, {"p", f}, {"oh", ho}, {"ow", wo}}, dt,
                         load("Y", {var("p"), add(mul(add(mul(var("n"), imm(ho)), var("oh")), imm(wo)), var("ow"))})));
  return finish(std::move(d), {"X", "W"}, {"Out"});
}

// compute_ir.cpp:599-616
ComputeDAG elementwise_unary_dag(UnOp op, std::vector<int64_t> shape, DType dt) {
  if ((op == UnOp::Exp || op == UnOp::Sqrt) && dt != DType::F32) fail("exp/sqrt require f32 tensors");
  ComputeDAG d;
  d.nodes.push_back(placeholder("X", shape, dt));
  auto ax = numbered_axes(shape);
  d.nodes.push_back(grid("Y", ax, dt, unary(op, load("X", as_vars(ax)))));
  return finish(std::move(d), {"X"}, {"Y"});
}

// compute_ir.cpp:618-634
ComputeDAG elementwise_binary_dag(BinOp op, std::vector<int64_t> shape, DType dt) {
  ComputeDAG d;
  d.nodes.push_back(placeholder("X0", shape, dt));
  d.nodes.push_back(placeholder("X1", shape, dt));
  auto ax = numbered_axes(shape);
  d.nodes.push_back(grid("Y", ax, dt, binary(op, load("X0", as_vars(ax)), load("X1", as_vars(ax)))));
  return finish(std::move(d), {"X0", "X1"}, {"Y"});
}

// compute_ir.cpp:636-672 (flat index folded, then split by input strides)
ComputeDAG reshape_dag(std::vector<int64_t> in_shape, std::vector<int64_t> out_shape, DType dt) {
  int64_t nin = 1, nout = 1;
  for (auto v : in_shape) nin *= v;
  for (auto v : out_shape) nout *= v;
  if (nin != nout) fail("reshape must preserve element count");
  auto ax = numbered_axes(out_shape);
  Expr flat = imm(0);
  for (size_t i = 0; i < ax.size(); ++i) flat = add(mul(flat, imm(out_shape[i])), var(ax[i].name));
  flat = fold(flat);
  std::vector<Expr> idx;
  if (in_shape.size() == 1) {
    idx.push_back(flat);
  } else {
    int64_t stride = nin;
    for (size_t i = 0; i < in_shape.size(); ++i) {
      stride /= in_shape[i];
      Expr e = div(flat, imm(stride));
      if (i > 0) e = mod(e, imm(in_shape[i]));
      idx.push_back(fold(e));
    }
  }
  ComputeDAG d;
  d.nodes.push_back(placeholder("X", in_shape, dt));
  d.nodes.push_back(grid("Y", ax, dt, load("X", std::move(idx))));
  return finish(std::move(d), {"X"}, {"Y"});
}

// compute_ir.cpp:674-699
ComputeDAG transpose_dag(std::vector<int64_t> shape, std::vector<size_t> perm, DType dt) {
  if (perm.size() != shape.size()) fail("transpose permutation rank mismatch");
  std::vector<bool> hit(shape.size(), false);
  for (size_t p : perm) {
    if (p >= shape.size() || hit[p]) fail("invalid transpose permutation");
    hit[p] = true;
  }
  std::vector<int64_t> out_shape;
  for (size_t p : perm) out_shape.push_back(shape[p]);
  auto ax = numbered_axes(out_shape);
  std::vector<Expr> idx(shape.size());
  for (size_t i = 0; i < perm.size(); ++i) idx[perm[i]] = var(ax[i].name);
  ComputeDAG d;
  d.nodes.push_back(placeholder("X", shape, dt));
  d.nodes.push_back(grid("Y", ax, dt, load("X", std::move(idx))));
  return finish(std::move(d), {"X"}, {"Y"});
}

// compute_ir.cpp:701-719
ComputeDAG batchnorm_inference_dag(int64_t n, int64_t c, int64_t h, int64_t w, DType dt) {
  ComputeDAG d;
  d.nodes.push_back(placeholder("X", {n, c, h, w}, dt));
  d.nodes.push_back(placeholder("Scale", {c}, dt));
  d.nodes.push_back(placeholder("Shift", {c}, dt));
  const Expr x = load("X", {var("n"), var("c"), var("h"), var("w")});
  d.nodes.push_back(grid("Y", {{"n", n}, {"c", c}, {"h", h}, {"w", w}}, dt,
                         add(mul(x, load("Scale", {var("c")})), load("Shift", {var("c")}))));
  return finish(std::move(d), {"X", "Scale", "Shift"}, {"Y"});
}

// ================================================================== JSON ==
// Expression wire form: prefix arrays, e.g. ["mul", ["load","A",["v","i"],["v","k"]], ["f",2.0]]
namespace {
const char* kBinNames[] = {"add", "sub", "mul", "div", "mod", "min", "max", "and", "or", "lt", "le", "gt", "ge", "eq", "ne"};
const char* kUnNames[] = {"neg", "relu", "exp", "sqrt", "f32", "i32"};

Expr expr_from(const tmjson::Value& v) {
  const auto& a = v.arr();
  if (a.empty()) fail("empty expression array");
  const std::string& op = a[0].str();
  if (op == "i") return imm(a.at(1).integer());
  if (op == "f") return fimm(a.at(1).num());
  if (op == "v") return var(a.at(1).str());
  if (op == "tid") return thread_idx();
  if (op == "bid") return block_idx();
  if (op == "select") return select(expr_from(a.at(1)), expr_from(a.at(2)), expr_from(a.at(3)));
  if (op == "load") {
    std::vector<Expr> idx;
    for (size_t i = 2; i < a.size(); ++i) idx.push_back(expr_from(a[i]));
    return load(a.at(1).str(), std::move(idx));
  }
  if (op == "lookup") {
    auto t = std::make_shared<std::vector<int64_t>>();
    for (const auto& x : a.at(1).arr()) t->push_back(x.integer());
    return table_lookup(t, expr_from(a.at(2)));
  }
  for (int i = 0; i < 15; ++i)
    if (op == kBinNames[i]) return binary(static_cast<BinOp>(i), expr_from(a.at(1)), expr_from(a.at(2)));
  for (int i = 0; i < 6; ++i)
    if (op == kUnNames[i]) return unary(static_cast<UnOp>(i), expr_from(a.at(1)));
  fail("unknown expression operator '", op, "'");
}

void expr_json(std::string& o, const Expr& e) {
  switch (e->kind) {
    case ExprKind::IntImm: o += "[\"i\"," + std::to_string(e->ival) + "]"; return;
    case ExprKind::FloatImm: {
      char buf[40];
      std::snprintf(buf, sizeof buf, "%.17g", e->fval);
      std::string s = buf;
      if (s.find_first_of(".eni") == std::string::npos) s += ".0";
      o += "[\"f\"," + s + "]";
      return;
    }
    case ExprKind::Var: o += "[\"v\"," + tmjson::quote(e->name) + "]"; return;
    case ExprKind::ThreadIdx: o += "[\"tid\"]"; return;
    case ExprKind::BlockIdx: o += "[\"bid\"]"; return;
    case ExprKind::Binary: o += std::string("[\"") + kBinNames[static_cast<int>(e->bop)] + "\""; break;
    case ExprKind::Unary: o += std::string("[\"") + kUnNames[static_cast<int>(e->uop)] + "\""; break;
    case ExprKind::Select: o += "[\"select\""; break;
    case ExprKind::Load: o += "[\"load\"," + tmjson::quote(e->name); break;
    case ExprKind::TableLookup: {
      o += "[\"lookup\",[";
      for (size_t i = 0; i < e->table->size(); ++i) o += (i ? "," : "") + std::to_string((*e->table)[i]);
      o += "]";
      break;
    }
  }
  for (const Expr& x : e->args) {
    o += ",";
    expr_json(o, x);
  }
  o += "]";
}

std::vector<Axis> axes_from(const tmjson::Value* v) {
  std::vector<Axis> out;
  if (!v) return out;
  for (const auto& a : v->arr()) out.push_back({a.arr().at(0).str(), a.arr().at(1).integer()});
  return out;
}
}  // namespace

ComputeDAG dag_from_json(const std::string& text) {
  tmjson::Value root;
  try {
    root = tmjson::parse(text);
  } catch (const std::exception& e) {
    fail(e.what());
  }
  ComputeDAG d;
  for (const auto& nv : root.at("nodes").arr()) {
    TensorNode n;
    n.name = nv.at("name").str();
    for (const auto& s : nv.at("shape").arr()) n.shape.push_back(s.integer());
    if (const auto* dt = nv.get("dtype")) n.dtype = dtype_from_name(dt->str());
    const std::string kind = nv.get("kind") ? nv.at("kind").str() : "input";
    if (kind == "input") {
      n.kind = NodeKind::Input;
    } else {
      n.kind = kind == "reduce" ? NodeKind::GridReduce : kind == "compute" ? NodeKind::GridCompute
                                                                          : (fail("unknown node kind '", kind, "'"), NodeKind::Input);
      n.axes = axes_from(nv.get("axes"));
      n.reduce_axes = axes_from(nv.get("reduce_axes"));
      if (const auto* c = nv.get("combiner")) n.combiner = combiner_from_name(c->str());
      n.value = expr_from(nv.at("value"));
    }
    d.nodes.push_back(std::move(n));
  }
  for (const auto& s : root.at("inputs").arr()) d.inputs.push_back(s.str());
  for (const auto& s : root.at("outputs").arr()) d.outputs.push_back(s.str());
  d.validate();
  return d;
}

std::string dag_to_json(const ComputeDAG& d) {
  std::string o = "{\"nodes\":[";
  for (size_t i = 0; i < d.nodes.size(); ++i) {
    const auto& n = d.nodes[i];
    if (i) o += ",";
    o += "{\"name\":" + tmjson::quote(n.name) + ",\"shape\":[";
    for (size_t j = 0; j < n.shape.size(); ++j) o += (j ? "," : "") + std::to_string(n.shape[j]);
    o += std::string("],\"dtype\":\"") + dtype_name(n.dtype) + "\"";
    if (n.kind == NodeKind::Input) {
      o += ",\"kind\":\"input\"}";
      continue;
    }
    o += n.kind == NodeKind::GridReduce ? ",\"kind\":\"reduce\"" : ",\"kind\":\"compute\"";
    auto axes = [&](const char* key, const std::vector<Axis>& ax) {
      o += std::string(",\"") + key + "\":[";
      for (size_t j = 0; j < ax.size(); ++j) o += (j ? "," : "") + std::string("[") + tmjson::quote(ax[j].name) + "," + std::to_string(ax[j].extent) + "]";
      o += "]";
    };
    axes("axes", n.axes);
    if (n.kind == NodeKind::GridReduce) {
      axes("reduce_axes", n.reduce_axes);
      o += std::string(",\"combiner\":\"") + combiner_name(n.combiner) + "\"";
    }
    o += ",\"value\":";
    expr_json(o, n.value);
    o += "}";
  }
  o += "],\"inputs\":[";
  for (size_t i = 0; i < d.inputs.size(); ++i) o += (i ? "," : "") + tmjson::quote(d.inputs[i]);
  o += "],\"outputs\":[";
  for (size_t i = 0; i < d.outputs.size(); ++i) o += (i ? "," : "") + tmjson::quote(d.outputs[i]);
  return o + "]}";
}

}  // namespace taskmap
