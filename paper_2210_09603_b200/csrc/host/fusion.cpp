// Post-scheduling fusion for the B200 build (Hidet §4.2 / §5.2).
//
// partition()   groups the DAG around reduction anchors.
// build_plan()  lowers each FusedSubgraph onto the task-mapped tcgen05 GEMM:
//   * prologue  -> operand loader: direct/strided loads, pure re-index
//                 prologues (the filter flatten Wf, transposes, Fig. 11's
//                 A[99-i]) composed symbolically by substitution, and the
//                 im2col gather recognised structurally (compute_ir.cpp:532-557);
//   * epilogue  -> an op program run on the TMEM accumulator in registers plus
//                 an output address map obtained by inverting each bijective
//                 access (the "index remap" of fuse_epilogue).
// bind_plan()   evaluates the symbolic address maps on the bound tensors'
//               strides and fits them to the kernel's canonical Addr form.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <mutex>
#include <cstring>
#include <cstdlib>
#include <cstdio>
#include <random>
#include <set>

#include "json.hpp"
#include "plan.hpp"
#include "dev_eval.hpp"
#include "rule_codegen.hpp"

namespace tmb {

using namespace taskmap;

// ============================================================ partition ==
namespace {
std::map<std::string, std::vector<std::string>> consumers_of(const ComputeDAG& dag) {
  std::map<std::string, std::vector<std::string>> c;
  for (const auto& n : dag.nodes) {
    if (!n.is_computed()) continue;
    std::vector<Expr> ls;
    collect_loads(n.value, ls);
    std::set<std::string> seen;
    for (const auto& l : ls)
      if (seen.insert(l->name).second) c[l->name].push_back(n.name);
  }
  return c;
}

bool is_output(const ComputeDAG& dag, const std::string& n) {
  return std::find(dag.outputs.begin(), dag.outputs.end(), n) != dag.outputs.end();
}

// The single distinct access pattern with which `reader` loads `src` (nullptr
// when it is read through two different index expressions).
Expr unique_access(const TensorNode& reader, const std::string& src) {
  std::vector<Expr> ls;
  collect_loads(reader.value, ls);
  Expr first;
  for (const auto& l : ls) {
    if (l->name != src) continue;
    if (!first) first = l;
    else if (!expr_equal(first, l)) return nullptr;
  }
  return first;
}
}  // namespace

}  // namespace tmb

std::vector<taskmap::FusedSubgraph> taskmap::partition(const taskmap::ComputeDAG& dag) {
  using namespace tmb;
  dag.validate();
  auto cons = consumers_of(dag);
  std::set<std::string> taken;
  std::vector<FusedSubgraph> out;
  auto single_use = [&](const std::string& n) { return cons[n].size() == 1 && !is_output(dag, n); };
  for (const auto& r : dag.nodes) {
    if (r.kind != NodeKind::GridReduce || taken.count(r.name)) continue;
    FusedSubgraph sg;
    sg.anchor = r.name;
    taken.insert(r.name);
    // prologues: injective, single-use producers of the anchor's operands
    std::vector<Expr> ls;
    collect_loads(r.value, ls);
    std::set<std::string> seen;
    for (const auto& l : ls) {
      if (!seen.insert(l->name).second) continue;
      const TensorNode& s = dag.at(l->name);
      if (s.kind == NodeKind::GridCompute && !taken.count(s.name) && single_use(s.name) &&
          classify(dag, s) != OpClass::Reduction) {
        sg.prologue.push_back(s.name);
        taken.insert(s.name);
      }
    }
    // epilogue: chain of single-use consumers that read the chain bijectively
    std::string cur = r.name;
    for (;;) {
      if (!single_use(cur)) break;
      const TensorNode& e = dag.at(cons[cur][0]);
      if (e.kind != NodeKind::GridCompute || taken.count(e.name)) break;
      if (classify(dag, e) != OpClass::Bijective) break;
      Expr acc = unique_access(e, cur);
      if (!acc) break;
      auto aff = analyze_affine_access(acc, e.axes);
      if (!aff || !affine_access_bijective(*aff, e.axes, dag.at(cur).shape)) break;
      sg.epilogue.push_back(e.name);
      taken.insert(e.name);
      cur = e.name;
    }
    sg.output = cur;
    out.push_back(std::move(sg));
  }
  // anchor-free remainder: rule-based injective kernels.  A
  // remainder node used once, by another remainder node, and not a DAG output is
  // inlined into its consumer (listed as that subgraph's prologue); every other
  // remainder node roots one kernel.
  std::set<std::string> rem;
  for (const auto& n : dag.nodes)
    if (n.kind == NodeKind::GridCompute && !taken.count(n.name)) rem.insert(n.name);
  auto inlined = [&](const std::string& n) {
    return rem.count(n) && single_use(n) && rem.count(cons[n][0]);
  };
  for (const auto& n : dag.nodes) {
    if (!rem.count(n.name) || inlined(n.name)) continue;
    FusedSubgraph sg;
    // producers spliced into this root, innermost first
    std::vector<std::string> stack = {n.name}, order;
    std::set<std::string> seen;
    while (!stack.empty()) {
      const std::string cur = stack.back();
      stack.pop_back();
      std::vector<Expr> ls;
      collect_loads(dag.at(cur).value, ls);
      for (const auto& l : ls)
        if (inlined(l->name) && seen.insert(l->name).second) {
          order.push_back(l->name);
          stack.push_back(l->name);
        }
    }
    for (auto it = order.rbegin(); it != order.rend(); ++it) sg.prologue.push_back(*it);
    sg.epilogue.push_back(n.name);
    sg.output = n.name;
    out.push_back(std::move(sg));
  }
  return out;
}

namespace tmb {

// ========================================================= IndexProgram ==
IndexProgram IndexProgram::compile(const Expr& e, const std::vector<std::string>& slots) {
  IndexProgram p;
  std::function<void(const Expr&)> go = [&](const Expr& x) {
    switch (x->kind) {
      case ExprKind::IntImm: p.code.push_back({0, x->ival, BinOp::Add}); return;
      case ExprKind::Var: {
        auto it = std::find(slots.begin(), slots.end(), x->name);
        if (it == slots.end()) fail("index expression uses unbound variable '", x->name, "'");
        p.code.push_back({1, it - slots.begin(), BinOp::Add});
        return;
      }
      case ExprKind::Binary:
        go(x->args[0]);
        go(x->args[1]);
        p.code.push_back({2, 0, x->bop});
        return;
      case ExprKind::Unary:
        if (x->uop == UnOp::Neg) { go(x->args[0]); p.code.push_back({3, 0, BinOp::Add}); return; }
        if (x->uop == UnOp::CastI32) { go(x->args[0]); return; }
        break;
      case ExprKind::Select:
        go(x->args[0]); go(x->args[1]); go(x->args[2]);
        p.code.push_back({4, 0, BinOp::Add});
        return;
      default: break;
    }
    fail_unsupported("unsupported construct in an index expression: ", expr_to_text(x));
  };
  go(e);
  // static stack depth (eval keeps a fixed 64-slot stack): reject deeper programs here
  int depth = 0, max_depth = 0;
  for (const auto& in : p.code) {
    depth += in.op <= 1 ? 1 : in.op == 2 ? -1 : in.op == 4 ? -2 : 0;
    max_depth = std::max(max_depth, depth);
  }
  if (max_depth > 60) fail_unsupported("index expression too deep (", max_depth, " stack slots, at most 60)");
  return p;
}

int64_t IndexProgram::eval(const int64_t* vars) const {
  int64_t st[64];
  int sp = 0;
  for (const auto& in : code) {
    switch (in.op) {
      case 0: st[sp++] = in.v; break;
      case 1: st[sp++] = vars[in.v]; break;
      case 3: st[sp - 1] = -st[sp - 1]; break;
      case 4: { const int64_t e = st[--sp], t = st[--sp], c = st[--sp]; st[sp++] = c ? t : e; break; }
      default: {
        const int64_t b = st[--sp], a = st[--sp];
        int64_t r = 0;
        switch (in.bop) {
          case BinOp::Add: r = a + b; break;
          case BinOp::Sub: r = a - b; break;
          case BinOp::Mul: r = a * b; break;
          case BinOp::Div: if (!b) fail("integer division by zero in index"); r = floordiv(a, b); break;
          case BinOp::Mod: if (!b) fail("integer modulo by zero in index"); r = floormod(a, b); break;
          case BinOp::Min: r = std::min(a, b); break;
          case BinOp::Max: r = std::max(a, b); break;
          case BinOp::And: r = a && b; break;
          case BinOp::Or: r = a || b; break;
          case BinOp::Lt: r = a < b; break;
          case BinOp::Le: r = a <= b; break;
          case BinOp::Gt: r = a > b; break;
          case BinOp::Ge: r = a >= b; break;
          case BinOp::Eq: r = a == b; break;
          case BinOp::Ne: r = a != b; break;
        }
        st[sp++] = r;
      }
    }
    if (sp >= 63) fail("index expression too deep");
  }
  return st[0];
}

// ============================================================ lowering ==
namespace {
const char* kRow = "__row";
const char* kCol = "__col";
const char* kBat = "__bat";

bool contains_var(const Expr& e, const std::string& v) {
  std::vector<std::string> vs;
  collect_vars(e, vs);
  return std::find(vs.begin(), vs.end(), v) != vs.end();
}

// Recognise the reference's im2col gather node (compute_ir.cpp:532-557) by
// rebuilding candidates with our builder and comparing expressions.
bool match_im2col(const ComputeDAG& dag, const TensorNode& col, ConvInfo& ci) {
  if (col.axes.size() != 2) return false;
  std::vector<Expr> ls;
  collect_loads(col.value, ls);
  if (ls.empty()) return false;
  const std::string xname = ls[0]->name;
  const TensorNode* x = dag.find(xname);
  if (!x || x->kind != NodeKind::Input || x->shape.size() != 4) return false;
  const int64_t n = x->shape[0], c = x->shape[1], h = x->shape[2], w = x->shape[3];
  const int64_t gk = col.shape[0], gn = col.shape[1];
  if (gk % c) return false;
  const int64_t taps = gk / c;
  for (int64_t kh = 1; kh <= taps; ++kh) {
    if (taps % kh) continue;
    const int64_t kw = taps / kh;
    for (int64_t stride = 1; stride <= 8; ++stride)
      for (int64_t pad = 0; pad <= std::max(kh, kw); ++pad) {
        if (kh > h + 2 * pad || kw > w + 2 * pad) continue;
        const int64_t ho = conv_out_extent(h, kh, stride, pad), wo = conv_out_extent(w, kw, stride, pad);
        if (ho <= 0 || wo <= 0 || n * ho * wo != gn) continue;
        ComputeDAG ref = conv2d_im2col_dag(n, c, h, w, 1, kh, kw, stride, pad, x->dtype);
        const TensorNode& rc = ref.at("Col");
        Expr cand = substitute(rc.value, {{"r", var(col.axes[0].name)}, {"s", var(col.axes[1].name)}});
        cand = rewrite_loads(cand, [&](const ExprNode& l) -> std::optional<Expr> {
          return load(xname, l.args);
        });
        if (expr_equal(cand, col.value)) {
          ci = ConvInfo{n, c, h, w, 0, kh, kw, stride, pad, ho, wo, xname, ""};
          return true;
        }
      }
  }
  return false;
}

// The filter flatten Wf[p, r] = W[p, r/(kh kw), (r/kw)%kh, r%kw] (compute_ir.cpp:558-569).
bool match_filter(const ComputeDAG& dag, const TensorNode& wf, const ConvInfo& ci, std::string& wname) {
  if (wf.value->kind != ExprKind::Load || wf.axes.size() != 2) return false;
  const TensorNode* w = dag.find(wf.value->name);
  if (!w || w->kind != NodeKind::Input || w->shape.size() != 4) return false;
  ComputeDAG ref = conv2d_im2col_dag(ci.n, ci.c, ci.h, ci.w, w->shape[0], ci.kh, ci.kw, ci.stride, ci.pad, w->dtype);
  Expr cand = substitute(ref.at("Wf").value, {{"p", var(wf.axes[0].name)}, {"r", var(wf.axes[1].name)}});
  cand = rewrite_loads(cand, [&](const ExprNode& l) -> std::optional<Expr> { return load(w->name, l.args); });
  if (!expr_equal(cand, wf.value)) return false;
  wname = w->name;
  return true;
}

// Inverse of an affine bijective access: expressions for the reader's axes in
// terms of the source coordinates `src` (already in slot variables).
std::map<std::string, Expr> invert_access(const TensorNode& reader, const std::vector<AffineIndex>& acc,
                                          const std::vector<Expr>& src) {
  std::map<std::string, Expr> m;
  for (const auto& a : reader.axes) m[a.name] = imm(0);  // unit axes
  for (size_t d = 0; d < acc.size(); ++d) {
    int64_t lo = acc[d].offset;
    for (const auto& t : acc[d].terms)
      if (t.coeff < 0) lo += t.coeff * (reader.axes[t.axis].extent - 1);
    Expr v = fold(sub(src[d], imm(lo)));
    for (const auto& t : acc[d].terms) {
      const int64_t e = reader.axes[t.axis].extent, c = std::llabs(t.coeff);
      Expr x = fold(mod(fold(div(v, imm(c))), imm(e)));
      if (t.coeff < 0) x = fold(sub(imm(e - 1), x));
      m[reader.axes[t.axis].name] = x;
    }
  }
  return m;
}

struct EpiBuilder {
  const ComputeDAG& dag;
  SubgraphPlan& sp;
  std::map<std::string, Expr> coords;  // current level axes -> slot exprs
  const std::string* pred = nullptr;   // tensor holding the accumulator value

  bool has_acc(const Expr& e) {
    if (e->kind == ExprKind::Load && e->name == *pred) return true;
    return std::any_of(e->args.begin(), e->args.end(), [&](const Expr& a) { return has_acc(a); });
  }

  // wildcard match against gelu_tanh(__x__)
  bool match_gelu(const Expr& e, Expr& x) {
    static const Expr tmpl = gelu_tanh(var("__gelu_x__"));
    Expr bound;
    std::function<bool(const Expr&, const Expr&)> m = [&](const Expr& t, const Expr& s) -> bool {
      if (t->kind == ExprKind::Var && t->name == "__gelu_x__") {
        if (!bound) { bound = s; return true; }
        return expr_equal(bound, s);
      }
      if (t->kind != s->kind || t->args.size() != s->args.size()) return false;
      if (t->kind == ExprKind::FloatImm && t->fval != s->fval) return false;
      if (t->kind == ExprKind::IntImm && t->ival != s->ival) return false;
      if (t->kind == ExprKind::Binary && t->bop != s->bop) return false;
      if (t->kind == ExprKind::Unary && t->uop != s->uop) return false;
      if (t->kind == ExprKind::Var || t->kind == ExprKind::Load) return false;
      for (size_t i = 0; i < t->args.size(); ++i)
        if (!m(t->args[i], s->args[i])) return false;
      return true;
    };
    if (!m(tmpl, e)) return false;
    x = bound;
    return true;
  }

  int side_of(const Expr& ld) {
    const TensorNode* t = dag.find(ld->name);
    if (!t) fail("epilogue reads unknown tensor '", ld->name, "'");
    AddrExpr a;
    a.tensor = ld->name;
    for (const auto& ix : ld->args) a.idx.push_back(fold(substitute(ix, coords)));
    sp.sides.push_back(std::move(a));
    return static_cast<int>(sp.sides.size()) - 1;
  }

  void walk(const Expr& e) {
    if (e->kind == ExprKind::Load && e->name == *pred) return;  // the accumulator
    Expr gx;
    if (match_gelu(e, gx) && has_acc(gx)) {
      walk(gx);
      sp.ops.push_back({EPI_GELU_TANH});
      return;
    }
    if (e->kind == ExprKind::Unary) {
      walk(e->args[0]);
      switch (e->uop) {
        case UnOp::Relu: sp.ops.push_back({EPI_RELU}); return;
        case UnOp::Neg: sp.ops.push_back({EPI_NEG}); return;
        case UnOp::Exp: sp.ops.push_back({EPI_EXP}); return;
        case UnOp::Sqrt: sp.ops.push_back({EPI_SQRT}); return;
        case UnOp::CastF32: return;
        default: fail_unsupported("epilogue op ", unop_name(e->uop), " is not supported on the device");
      }
    }
    if (e->kind == ExprKind::Binary) {
      const bool l = has_acc(e->args[0]), r = has_acc(e->args[1]);
      if (l == r) fail_unsupported("epilogue expression is not a single-use chain of the accumulator: ", expr_to_text(e));
      const Expr& spine = l ? e->args[0] : e->args[1];
      const Expr side = fold(l ? e->args[1] : e->args[0]);
      walk(spine);
      EpiStep st{0};
      const bool is_const = side->kind == ExprKind::FloatImm || side->kind == ExprKind::IntImm;
      if (is_const) st.c = static_cast<float>(side->kind == ExprKind::FloatImm ? side->fval : static_cast<double>(side->ival));
      else if (side->kind == ExprKind::Load) st.side = side_of(side);
      else fail_unsupported("epilogue side operand must be a constant or a tensor element: ", expr_to_text(side));
      const int t = is_const ? 0 : (EPI_ADD_T - EPI_ADD_C);
      switch (e->bop) {
        case BinOp::Add: st.kind = EPI_ADD_C + t; break;
        case BinOp::Sub: st.kind = (l ? EPI_SUB_C : EPI_RSUB_C) + t; break;
        case BinOp::Mul: st.kind = EPI_MUL_C + t; break;
        case BinOp::Div: st.kind = (l ? EPI_DIV_C : EPI_RDIV_C) + t; break;
        case BinOp::Max: st.kind = EPI_MAX_C + t; break;
        case BinOp::Min: st.kind = EPI_MIN_C + t; break;
        default: fail_unsupported("epilogue operator ", binop_name(e->bop), " is not supported on the device");
      }
      sp.ops.push_back(st);
      return;
    }
    fail_unsupported("unsupported epilogue expression: ", expr_to_text(e));
  }
};

SubgraphPlan lower_subgraph(const ComputeDAG& dag, const FusedSubgraph& sg) {
  SubgraphPlan sp;
  sp.sg = sg;
  if (sg.anchor.empty())
    fail_unsupported("subgraph '", sg.output, "' has no reduction anchor; rule-based injective kernels are out of scope");
  const TensorNode& r = dag.at(sg.anchor);
  if (r.combiner != Combiner::Sum) fail_unsupported("anchor '", r.name, "': only sum reductions lower to tcgen05");
  if (r.reduce_axes.size() != 1) fail_unsupported("anchor '", r.name, "': exactly one reduce axis is supported");
  if (r.axes.size() != 2 && r.axes.size() != 3) fail_unsupported("anchor '", r.name, "': 2 or 3 spatial axes expected");
  Expr v = r.value;
  if (v->kind != ExprKind::Binary || v->bop != BinOp::Mul || v->args[0]->kind != ExprKind::Load ||
      v->args[1]->kind != ExprKind::Load)
    fail_unsupported("anchor '", r.name, "': value must be the product of two tensor elements");
  const std::string kname = r.reduce_axes[0].name;
  Expr L[2] = {v->args[0], v->args[1]};
  auto uses = [&](const Expr& l, const std::string& ax) {
    return std::any_of(l->args.begin(), l->args.end(), [&](const Expr& i) { return contains_var(i, ax); });
  };
  std::string own[2], batch;
  for (const auto& ax : r.axes) {
    const bool u0 = uses(L[0], ax.name), u1 = uses(L[1], ax.name);
    if (u0 && u1) {
      if (!batch.empty()) fail_unsupported("anchor '", r.name, "': at most one batch axis");
      batch = ax.name;
    } else if (u0 || u1) {
      std::string& slot = own[u0 ? 0 : 1];
      if (!slot.empty()) fail_unsupported("anchor '", r.name, "': operand owns two spatial axes");
      slot = ax.name;
    } else {
      fail_unsupported("anchor '", r.name, "': axis '", ax.name, "' unused by the operands");
    }
  }
  if (own[0].empty() || own[1].empty()) fail_unsupported("anchor '", r.name, "': not a matrix product");
  if (!uses(L[0], kname) || !uses(L[1], kname)) fail_unsupported("anchor '", r.name, "': reduce axis missing from an operand");

  const bool pro0 = std::find(sg.prologue.begin(), sg.prologue.end(), L[0]->name) != sg.prologue.end();
  const bool pro1 = std::find(sg.prologue.begin(), sg.prologue.end(), L[1]->name) != sg.prologue.end();
  ConvInfo ci{};
  int im2col_side = -1;
  if (pro0 && match_im2col(dag, dag.at(L[0]->name), ci)) im2col_side = 0;
  else if (pro1 && match_im2col(dag, dag.at(L[1]->name), ci)) im2col_side = 1;
  // orientation: im2col operand provides the rows (pixels on TMEM lanes);
  // otherwise the operand owning the first non-batch anchor axis
  int ia = 0;
  if (im2col_side >= 0) ia = im2col_side;
  else {
    for (const auto& ax : r.axes)
      if (ax.name == own[0] || ax.name == own[1]) { ia = ax.name == own[0] ? 0 : 1; break; }
  }
  const int ib = 1 - ia;
  auto extent = [&](const std::string& n) {
    for (const auto& ax : r.axes) if (ax.name == n) return ax.extent;
    return int64_t(1);
  };
  sp.M = extent(own[ia]);
  sp.N = extent(own[ib]);
  sp.K = r.reduce_axes[0].extent;
  sp.batch = batch.empty() ? 1 : extent(batch);

  // operand address maps: rename anchor axes to slot vars
  auto lower_operand = [&](int which, OperandPlan& op) {
    const Expr& ld = L[which];
    std::map<std::string, Expr> ren = {{own[which], var(kRow)}, {kname, var(kCol)}};
    if (!batch.empty()) ren[batch] = var(kBat);
    std::vector<Expr> idx;
    for (const auto& i : ld->args) idx.push_back(substitute(i, ren));
    const TensorNode& s = dag.at(ld->name);
    const bool is_pro = (which == 0 ? pro0 : pro1);
    // Pure re-index prologue (value = Load of a graph input): compose its
    // index expressions with the anchor's access by substitution.  Kept even
    // for recognised conv operands: when the bound strides make it a plain
    // TMA tile (1x1 stride-1 conv on channels-last data) it beats im2col.
    auto reindex = [&](AddrExpr& out) {
      if (s.value->kind != ExprKind::Load || dag.at(s.value->name).kind != NodeKind::Input) return false;
      std::map<std::string, Expr> sub_map;
      for (size_t d = 0; d < s.axes.size(); ++d) sub_map[s.axes[d].name] = idx[d];
      out.tensor = s.value->name;
      for (const auto& i : s.value->args) out.idx.push_back(fold(substitute(i, sub_map)));
      return true;
    };
    if (which == im2col_side) {
      // the anchor must read Col[k, pixel] directly
      if (idx.size() != 2 || !expr_equal(idx[0], var(kCol)) || !expr_equal(idx[1], var(kRow)))
        fail_unsupported("anchor reads the im2col node through a non-identity index");
      op.kind = OperandPlan::Im2col;
      op.conv = ci;
      reindex(op.addr);
      return;
    }
    if (!is_pro) {
      // a graph input, or a tensor materialised by an earlier fused kernel
      op.kind = OperandPlan::Strided;
      op.addr.tensor = s.name;
      op.addr.idx = idx;
      return;
    }
    // prologue node
    if (im2col_side >= 0) {
      std::string wname;
      if (match_filter(dag, s, ci, wname) && idx.size() == 2 && expr_equal(idx[0], var(kRow)) &&
          expr_equal(idx[1], var(kCol))) {
        op.kind = OperandPlan::ConvFilter;
        op.conv = ci;
        op.conv.w_tensor = wname;
        op.conv.f = dag.at(wname).shape[0];
        reindex(op.addr);
        return;
      }
    }
    op.kind = OperandPlan::Strided;
    if (reindex(op.addr)) return;
    // Arithmetic prologue (Fig. 11: A[99-i] -> C[99-i]*2.0): the
    // node's value is a chain of elementwise ops over ONE element of a graph input
    // with constant side operands.  The input's index expressions are composed with
    // the anchor's access (as for a re-index) and the chain becomes the operand's
    // prologue op list, applied by the gather loader to every element it reads.
    std::vector<Expr> lds;
    collect_loads(s.value, lds);
    if (lds.size() != 1 || dag.at(lds[0]->name).kind != NodeKind::Input)
      fail_unsupported("prologue '", s.name, "' must read exactly one element of one graph input");
    const Expr src = lds[0];
    std::function<void(const Expr&)> chain = [&](const Expr& e) {
      if (e->kind == ExprKind::Load) return;  // the source element
      if (e->kind == ExprKind::Unary) {
        chain(e->args[0]);
        switch (e->uop) {
          case UnOp::Relu: op.pre.push_back({EPI_RELU}); return;
          case UnOp::Neg: op.pre.push_back({EPI_NEG}); return;
          case UnOp::Exp: op.pre.push_back({EPI_EXP}); return;
          case UnOp::Sqrt: op.pre.push_back({EPI_SQRT}); return;
          case UnOp::CastF32: return;
          default: fail_unsupported("prologue op ", unop_name(e->uop), " is not supported on the device");
        }
      }
      if (e->kind == ExprKind::Binary) {
        std::vector<Expr> l0, l1;
        collect_loads(e->args[0], l0);
        collect_loads(e->args[1], l1);
        if (l0.empty() == l1.empty())
          fail_unsupported("prologue expression is not a chain of its input element: ", expr_to_text(e));
        const bool l = !l0.empty();
        const Expr side = fold(l ? e->args[1] : e->args[0]);
        if (side->kind != ExprKind::FloatImm && side->kind != ExprKind::IntImm)
          fail_unsupported("prologue side operands must be constants: ", expr_to_text(side));
        chain(l ? e->args[0] : e->args[1]);
        EpiStep st{0};
        st.c = static_cast<float>(side->kind == ExprKind::FloatImm ? side->fval : static_cast<double>(side->ival));
        switch (e->bop) {
          case BinOp::Add: st.kind = EPI_ADD_C; break;
          case BinOp::Sub: st.kind = l ? EPI_SUB_C : EPI_RSUB_C; break;
          case BinOp::Mul: st.kind = EPI_MUL_C; break;
          case BinOp::Div: st.kind = l ? EPI_DIV_C : EPI_RDIV_C; break;
          case BinOp::Max: st.kind = EPI_MAX_C; break;
          case BinOp::Min: st.kind = EPI_MIN_C; break;
          default: fail_unsupported("prologue operator ", binop_name(e->bop), " is not supported on the device");
        }
        op.pre.push_back(st);
        return;
      }
      fail_unsupported("unsupported prologue expression: ", expr_to_text(e));
    };
    chain(s.value);
    if (op.pre.size() > static_cast<size_t>(kMaxPreOps))
      fail_unsupported("prologue '", s.name, "' has more than ", kMaxPreOps, " ops");
    std::map<std::string, Expr> sub_map;
    for (size_t d = 0; d < s.axes.size(); ++d) sub_map[s.axes[d].name] = idx[d];
    op.addr.tensor = src->name;
    op.addr.idx.clear();
    for (const auto& i : src->args) op.addr.idx.push_back(fold(substitute(i, sub_map)));
  };
  lower_operand(ia, sp.a);
  lower_operand(ib, sp.b);
  if (sp.a.kind == OperandPlan::Im2col && sp.b.kind == OperandPlan::Strided) {
    // keep as strided filter (e.g. an already-flattened weight input)
  }

  // epilogue chain: accumulate coordinate maps level by level
  EpiBuilder eb{dag, sp, {}, nullptr};
  {
    std::map<std::string, Expr> m = {{own[ia], var(kRow)}, {own[ib], var(kCol)}};
    if (!batch.empty()) m[batch] = var(kBat);
    eb.coords = m;
  }
  std::string pred = r.name;
  std::vector<Expr> pred_coords;  // predecessor coords in slot vars (in its axis order)
  for (const auto& ax : r.axes) pred_coords.push_back(eb.coords.at(ax.name));
  for (const auto& en : sg.epilogue) {
    const TensorNode& e = dag.at(en);
    Expr acc = unique_access(e, pred);
    auto aff = analyze_affine_access(acc, e.axes);
    std::map<std::string, Expr> inv = invert_access(e, *aff, pred_coords);
    eb.coords = inv;
    eb.pred = &pred;
    eb.walk(e.value);
    pred = en;
    pred_coords.clear();
    for (const auto& ax : e.axes) pred_coords.push_back(eb.coords.at(ax.name));
  }
  sp.out.tensor = sg.output;
  sp.out.idx = pred_coords;
  return sp;
}
}  // namespace

std::string SubgraphPlan::describe() const {
  std::ostringstream o;
  if (kind == Rule) {
    o << "{\"kind\":" << tmjson::quote(sg.anchor.empty() ? "rule" : "reduce") << ",\"root\":" << tmjson::quote(rule_node)
      << ",\"elements\":" << M << ",\"reduce\":" << K << ",\"inlined\":[";
    for (size_t i = 0; i < sg.prologue.size(); ++i) o << (i ? "," : "") << tmjson::quote(sg.prologue[i]);
    o << "],\"expr\":" << tmjson::quote(expr_to_text(rule_expr)) << "}";
    return o.str();
  }
  auto idxs = [](const AddrExpr& a) {
    std::string s = a.tensor + "[";
    for (size_t i = 0; i < a.idx.size(); ++i) s += (i ? ", " : "") + expr_to_text(a.idx[i]);
    return s + "]";
  };
  auto opd = [&](const OperandPlan& p) {
    if (p.kind == OperandPlan::Im2col) return std::string("im2col(") + p.conv.x_tensor + ")";
    if (p.kind == OperandPlan::ConvFilter) return std::string("filter(") + p.conv.w_tensor + ")";
    std::string s = idxs(p.addr);
    for (const auto& st : p.pre) s += " |> op" + std::to_string(st.kind) + "(" + std::to_string(st.c) + ")";
    return s;
  };
  o << "{\"kind\":\"gemm\",\"anchor\":" << tmjson::quote(sg.anchor) << ",\"M\":" << M << ",\"N\":" << N << ",\"K\":" << K
    << ",\"batch\":" << batch << ",\"A\":" << tmjson::quote(opd(a)) << ",\"B\":" << tmjson::quote(opd(b))
    << ",\"prologue\":[";
  for (size_t i = 0; i < sg.prologue.size(); ++i) o << (i ? "," : "") << tmjson::quote(sg.prologue[i]);
  o << "],\"epilogue\":[";
  for (size_t i = 0; i < sg.epilogue.size(); ++i) o << (i ? "," : "") << tmjson::quote(sg.epilogue[i]);
  o << "],\"ops\":[";
  for (size_t i = 0; i < ops.size(); ++i) {
    o << (i ? "," : "") << "{\"kind\":" << ops[i].kind << ",\"c\":" << ops[i].c;
    if (ops[i].side >= 0) o << ",\"side\":" << tmjson::quote(idxs(sides[ops[i].side]));
    o << "}";
  }
  o << "],\"out\":" << tmjson::quote(idxs(out)) << "}";
  return o.str();
}

namespace {

// The reduction anchor is a matrix product the GEMM templates lower (one sum
// axis over the product of two loads, each operand owning one spatial axis, at
// most one shared batch axis): the checks lower_subgraph enforces.
bool matmul_anchor(const TensorNode& r) {
  if (r.combiner != Combiner::Sum || r.reduce_axes.size() != 1 || (r.axes.size() != 2 && r.axes.size() != 3)) return false;
  const Expr& v = r.value;
  if (v->kind != ExprKind::Binary || v->bop != BinOp::Mul || v->args[0]->kind != ExprKind::Load ||
      v->args[1]->kind != ExprKind::Load)
    return false;
  auto uses = [&](const Expr& l, const std::string& ax) {
    return std::any_of(l->args.begin(), l->args.end(), [&](const Expr& i) { return contains_var(i, ax); });
  };
  int own0 = 0, own1 = 0, bat = 0;
  for (const auto& ax : r.axes) {
    const bool u0 = uses(v->args[0], ax.name), u1 = uses(v->args[1], ax.name);
    if (u0 && u1) ++bat;
    else if (u0) ++own0;
    else if (u1) ++own1;
    else return false;
  }
  const std::string k = r.reduce_axes[0].name;
  return own0 == 1 && own1 == 1 && bat <= 1 && uses(v->args[0], k) && uses(v->args[1], k);
}

// A prologue node the operand loaders can apply: a pure re-index of a graph
// input, or an elementwise chain over one element of one graph input with
// constant side operands (lower_subgraph's arithmetic prologue).
bool loader_prologue(const ComputeDAG& dag, const TensorNode& s) {
  if (s.value->kind == ExprKind::Load) return dag.at(s.value->name).kind == NodeKind::Input;
  std::vector<Expr> lds;
  collect_loads(s.value, lds);
  if (lds.size() != 1 || dag.at(lds[0]->name).kind != NodeKind::Input) return false;
  std::function<bool(const Expr&)> chain = [&](const Expr& e) -> bool {
    if (e->kind == ExprKind::Load) return true;
    if (e->kind == ExprKind::Unary)
      return e->uop != UnOp::CastI32 && chain(e->args[0]);
    if (e->kind == ExprKind::Binary) {
      std::vector<Expr> l0, l1;
      collect_loads(e->args[0], l0);
      collect_loads(e->args[1], l1);
      if (l0.empty() == l1.empty()) return false;
      const Expr side = fold(l0.empty() ? e->args[0] : e->args[1]);
      if (side->kind != ExprKind::FloatImm && side->kind != ExprKind::IntImm) return false;
      switch (e->bop) {
        case BinOp::Add: case BinOp::Sub: case BinOp::Mul: case BinOp::Div: case BinOp::Max: case BinOp::Min: break;
        default: return false;
      }
      return chain(l0.empty() ? e->args[1] : e->args[0]);
    }
    return false;
  };
  if (!chain(s.value)) return false;
  int ops = 0;  // the loader applies at most kMaxPreOps ops
  std::function<void(const Expr&)> count = [&](const Expr& e) {
    if (e->kind == ExprKind::Unary && e->uop != UnOp::CastF32) ++ops;
    if (e->kind == ExprKind::Binary) ++ops;
    for (const auto& a : e->args)
      if (a->kind != ExprKind::Load) count(a);
  };
  count(s.value);
  return ops <= kMaxPreOps;
}

// rule_based_schedule / reduce_template lowering:
// the root's value with the inlined producers spliced in (rewrite_loads, the
// fuse_prologue primitive).
SubgraphPlan lower_rule(const ComputeDAG& dag, const std::string& root, const std::vector<std::string>& inlined) {
  SubgraphPlan sp;
  sp.kind = SubgraphPlan::Rule;
  sp.rule_node = root;
  sp.sg.output = root;
  sp.sg.prologue = inlined;
  const TensorNode& n = dag.at(root);
  if (n.axes.size() > static_cast<size_t>(ev::kMaxRank) || n.reduce_axes.size() > static_cast<size_t>(ev::kMaxRank) ||
      n.axes.size() + n.reduce_axes.size() > static_cast<size_t>(ev::kMaxVars))
    fail_unsupported("rule kernel '", n.name, "': more than ", ev::kMaxRank, " axes");
  if (n.kind == NodeKind::GridReduce) sp.sg.anchor = root;
  else sp.sg.epilogue.push_back(root);
  const std::set<std::string> inl(inlined.begin(), inlined.end());
  Expr e = n.value;
  for (int round = 0; round < 256; ++round) {
    bool changed = false;
    e = rewrite_loads(e, [&](const ExprNode& ld) -> std::optional<Expr> {
      if (!inl.count(ld.name)) return std::nullopt;
      const TensorNode& p = dag.at(ld.name);
      if (p.kind != NodeKind::GridCompute) fail("rule kernel: cannot inline reduction '", p.name, "'");
      std::map<std::string, Expr> m;
      for (size_t d = 0; d < p.axes.size(); ++d) m[p.axes[d].name] = ld.args[d];
      changed = true;
      return substitute(p.value, m);
    });
    if (!changed) break;
  }
  sp.rule_expr = fold(e);
  int64_t m = 1;
  for (const auto& a : n.axes) m *= a.extent;
  sp.M = m;
  sp.N = 1;
  sp.K = 1;
  for (const auto& a : n.reduce_axes) sp.K *= a.extent;
  return sp;
}

}  // namespace

std::unique_ptr<Plan> build_plan(const ComputeDAG& dag, const ScheduleConfig& cfg, int device) {
  auto plan = std::make_unique<Plan>();
  plan->dag = dag;
  plan->cfg = cfg;
  plan->device = device;
  std::set<std::string> produced;
  for (const auto& sg0 : partition(dag)) {
    FusedSubgraph sg = sg0;
    if (sg.anchor.empty()) {
      // anchor-free: one rule-based kernel, the prologue nodes inlined
      plan->kernels.push_back(lower_rule(dag, sg.output, sg.prologue));
      produced.insert(sg.output);
      continue;
    }
    const TensorNode& r = dag.at(sg.anchor);
    if (!matmul_anchor(r)) {
      // reduce template for the anchor (its injective prologues inlined), then the
      // epilogue chain as one rule-based kernel reading the materialised reduction
      plan->kernels.push_back(lower_rule(dag, sg.anchor, sg.prologue));
      produced.insert(sg.anchor);
      if (!sg.epilogue.empty()) {
        std::vector<std::string> chain(sg.epilogue.begin(), sg.epilogue.end() - 1);
        plan->kernels.push_back(lower_rule(dag, sg.output, chain));
        produced.insert(sg.output);
      }
      continue;
    }
    // matrix-product anchor: prologue nodes the loaders cannot apply (they read
    // intermediates or several tensors) are materialised by rule kernels first
    bool conv = false;
    for (const auto& pn : sg.prologue) {
      ConvInfo ci{};
      conv = conv || match_im2col(dag, dag.at(pn), ci);
    }
    if (!conv) {
      std::vector<std::string> keep;
      for (const auto& pn : sg.prologue) {
        if (loader_prologue(dag, dag.at(pn))) {
          keep.push_back(pn);
        } else {
          plan->kernels.push_back(lower_rule(dag, pn, {}));
          produced.insert(pn);
        }
      }
      sg.prologue = keep;
    }
    // an epilogue chain the register program cannot express is cut where it
    // stops lowering; the cut-off consumers run as rule-based kernels
    std::vector<std::string> cut;
    for (;;) {
      try {
        plan->kernels.push_back(lower_subgraph(dag, sg));
        break;
      } catch (const UnsupportedError&) {
        if (sg.epilogue.empty()) throw;
        cut.insert(cut.begin(), sg.epilogue.back());
        sg.epilogue.pop_back();
        sg.output = sg.epilogue.empty() ? sg.anchor : sg.epilogue.back();
      }
    }
    produced.insert(sg.output);
    if (!cut.empty()) {
      std::vector<std::string> chain(cut.begin(), cut.end() - 1);
      plan->kernels.push_back(lower_rule(dag, cut.back(), chain));
      produced.insert(cut.back());
    }
  }
  // kernels in dependency order: anchors come out of partition first and the
  // anchor-free (rule) kernels after them, but a reduction may read an
  // anchor-free node (softmax: sum_j exp(S - max)); stable topological order
  {
    std::vector<SubgraphPlan> todo = std::move(plan->kernels), sorted;
    std::set<std::string> done;
    for (const auto& n : dag.nodes)
      if (n.kind == NodeKind::Input) done.insert(n.name);
    auto reads = [&](const SubgraphPlan& sp) {
      std::set<std::string> mem, out;
      if (!sp.sg.anchor.empty()) mem.insert(sp.sg.anchor);
      for (const auto& x : sp.sg.prologue) mem.insert(x);
      for (const auto& x : sp.sg.epilogue) mem.insert(x);
      if (!sp.rule_node.empty()) mem.insert(sp.rule_node);
      for (const auto& m : mem) {
        std::vector<Expr> ls;
        collect_loads(dag.at(m).value, ls);
        for (const auto& l : ls)
          if (!mem.count(l->name)) out.insert(l->name);
      }
      return out;
    };
    while (!todo.empty()) {
      size_t pick = todo.size();
      for (size_t i = 0; i < todo.size() && pick == todo.size(); ++i) {
        const auto r = reads(todo[i]);
        if (std::all_of(r.begin(), r.end(), [&](const std::string& x) { return done.count(x) > 0; })) pick = i;
      }
      if (pick == todo.size()) fail("fused kernels have a cyclic dependency");
      done.insert(todo[pick].sg.output);
      sorted.push_back(std::move(todo[pick]));
      todo.erase(todo.begin() + static_cast<std::ptrdiff_t>(pick));
    }
    plan->kernels = std::move(sorted);
  }
  for (const auto& o : dag.outputs)
    if (!produced.count(o)) fail("output '", o, "' is not produced by a fused kernel");
  for (const auto& s : produced)
    if (!is_output(dag, s)) plan->intermediates.push_back(s);
  return plan;
}

// ================================================================ binding ==
namespace {
struct Bound {
  tm_tensor t;
};

// Fitted canonical form of addr(x0, x1, x2) = sum_d stride_d * idx_d.
struct Fit {
  int64_t P, hi, lo, c1, c2, off;
};

bool fit_address_uncached(const AddrExpr& a, const tm_tensor& t, int64_t n0, int64_t n1, int64_t n2, Fit& f,
                          std::string& why);

// Fits depend only on the index expressions, the tensor's shape/strides and
// the GEMM extents, never on the schedule: memoised so that tuning a shape
// over the whole space pays for each fit once.
bool fit_address(const AddrExpr& a, const tm_tensor& t, int64_t n0, int64_t n1, int64_t n2, Fit& f,
                 std::string& why) {
  static std::mutex mu;
  static std::map<std::string, std::pair<bool, Fit>> cache;
  std::string key;
  for (const auto& e : a.idx) key += expr_to_text(e) + ";";
  for (int d = 0; d < t.rank; ++d) key += std::to_string(t.shape[d]) + "/" + std::to_string(t.stride[d]) + ",";
  key += "|" + std::to_string(n0) + "," + std::to_string(n1) + "," + std::to_string(n2);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      f = it->second.second;
      if (!it->second.first) why = "cached: address map does not fit";
      return it->second.first;
    }
  }
  const bool ok = fit_address_uncached(a, t, n0, n1, n2, f, why);
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = {ok, f};
  return ok;
}

bool fit_address_uncached(const AddrExpr& a, const tm_tensor& t, int64_t n0, int64_t n1, int64_t n2, Fit& f,
                          std::string& why) {
  if (static_cast<int>(a.idx.size()) != t.rank) { why = "rank mismatch"; return false; }
  std::vector<IndexProgram> progs;
  for (const auto& e : a.idx) progs.push_back(IndexProgram::compile(e, {kRow, kCol, kBat}));
  auto addr = [&](int64_t x0, int64_t x1, int64_t x2, bool& oob) {
    const int64_t v[3] = {x0, x1, x2};
    int64_t s = 0;
    for (int d = 0; d < t.rank; ++d) {
      const int64_t i = progs[d].eval(v);
      if (i < 0 || i >= t.shape[d]) oob = true;
      s += i * t.stride[d];
    }
    return s;
  };
  bool oob = false;
  f.off = addr(0, 0, 0, oob);
  f.c1 = n1 > 1 ? addr(0, 1, 0, oob) - f.off : 0;
  f.c2 = n2 > 1 ? addr(0, 0, 1, oob) - f.off : 0;
  for (int64_t x = 0; x < n1; ++x)
    if (addr(0, x, 0, oob) != f.off + x * f.c1) { why = "not affine along the column/K axis"; return false; }
  for (int64_t x = 0; x < n2; ++x)
    if (addr(0, 0, x, oob) != f.off + x * f.c2) { why = "not affine along the batch axis"; return false; }
  f.lo = n0 > 1 ? addr(1, 0, 0, oob) - f.off : 0;
  f.P = std::max<int64_t>(n0, 1);
  f.hi = 0;
  for (int64_t x = 1; x < n0; ++x)
    if (addr(x, 0, 0, oob) - f.off != x * f.lo) { f.P = x; f.hi = addr(x, 0, 0, oob) - f.off; break; }
  for (int64_t x = 0; x < n0; ++x)
    if (addr(x, 0, 0, oob) - f.off != (x / f.P) * f.hi + (x % f.P) * f.lo) {
      why = "row map is not of the form (r/P)*a + (r%P)*b";
      return false;
    }
  std::mt19937_64 rng(1234);
  for (int s = 0; s < 512; ++s) {
    const int64_t x0 = s < 8 ? ((s & 1) ? n0 - 1 : 0) : static_cast<int64_t>(rng() % n0);
    const int64_t x1 = s < 8 ? ((s & 2) ? n1 - 1 : 0) : static_cast<int64_t>(rng() % n1);
    const int64_t x2 = s < 8 ? ((s & 4) ? n2 - 1 : 0) : static_cast<int64_t>(rng() % n2);
    if (addr(x0, x1, x2, oob) != f.off + (x0 / f.P) * f.hi + (x0 % f.P) * f.lo + x1 * f.c1 + x2 * f.c2) {
      why = "address map is not separable";
      return false;
    }
  }
  if (oob) { why = "index out of bounds"; return false; }
  return true;
}

int esize(int dt) { return dt == TM_F32 ? 4 : 2; }

Addr to_addr(const Fit& f) { return Addr{f.P, f.hi, f.lo, f.c1, f.c2, f.off}; }

const tm_tensor& lookup(const std::map<std::string, tm_tensor>& env, const std::string& n) {
  auto it = env.find(n);
  if (it == env.end()) fail("tensor '", n, "' is not bound");
  return it->second;
}

// CTA -> tile task mapping over the (batch, tiles_m, tiles_n) domain:
// raster 0: repeat(r) * spatial(g)  (each wave sweeps a g-block of tiles)
// raster 1: spatial(g) * repeat(r)  (each CTA owns a contiguous r-block)
tm::DevMapping tile_mapping(int64_t B, int64_t TM, int64_t TN, int grid, int raster, int& used) {
  const int64_t dom[3] = {B, TM, TN};
  int64_t best_cost = INT64_MAX, bg[3] = {1, 1, 1};
  for (int64_t gb = 1; gb <= std::min<int64_t>(B, grid); ++gb)
    for (int64_t gm = 1; gm <= std::min<int64_t>(TM, grid / gb); ++gm) {
      const int64_t gn = std::min<int64_t>(TN, grid / (gb * gm));
      if (gn < 1) continue;
      const int64_t g[3] = {gb, gm, gn};
      int64_t waves = 1;
      for (int d = 0; d < 3; ++d) waves *= (dom[d] + g[d] - 1) / g[d];
      // primary: fewest tile rounds; secondary: more CTAs (less per-CTA work)
      const int64_t cost = waves * 4096 - gb * gm * gn;
      if (cost < best_cost) { best_cost = cost; bg[0] = gb; bg[1] = gm; bg[2] = gn; }
    }
  tm::DevMapping m{};
  m.rank = 3;
  m.n_atoms = 2;
  const int rep = raster == 0 ? 0 : 1, spa = 1 - rep;
  m.is_spatial[rep] = 0;
  m.is_spatial[spa] = 1;
  m.workers = 1;
  m.tasks = 1;
  for (int d = 0; d < 3; ++d) {
    const int64_t r = (dom[d] + bg[d] - 1) / bg[d];
    m.dims[rep][d] = static_cast<int32_t>(r);
    m.dims[spa][d] = static_cast<int32_t>(bg[d]);
    m.tasks *= static_cast<uint32_t>(r);
    m.workers *= static_cast<uint32_t>(bg[d]);
    m.shape[d] = static_cast<int32_t>(r * bg[d]);
  }
  used = static_cast<int>(m.workers);
  return m;
}

// MN-major fp32 B for kind::tf32 (TMB_TF32_MN=0 restores the gather loader)
bool tf32_mn_ok() {
  static const bool on = [] { const char* e = std::getenv("TMB_TF32_MN"); return !(e && e[0] == '0'); }();
  return on;
}

// TMA tile views are {K, rows, batch} (K-major) or {rows, K, batch} (MN-major)
// with strides {row, batch}: the batch stride is encoded as given, so a batch
// whose stride is below one batch's row span (e.g. heads interleaved inside a
// row, [H,S,D] with strides (D, H*D, 1)) cannot be a TMA view and falls back to
// the predicated gather loader / direct stores.  With batch == 1 the stride is
// unused (and encoded as the row span).
bool batch_ok(int64_t c2, int64_t span, int64_t batch) { return batch <= 1 || c2 >= span; }

bool tma_ok_kmajor(const Fit& f, const tm_tensor& t, int64_t rows, int want_dt, int64_t batch) {
  const int es = esize(t.dtype);
  if (t.dtype != want_dt) return false;
  if (f.c1 != 1 || f.P < rows) return false;
  if (!batch_ok(f.c2, f.lo * rows, batch)) return false;
  if ((f.lo * es) % 16 || (f.c2 * es) % 16 || f.lo <= 0) return false;
  const uintptr_t base = reinterpret_cast<uintptr_t>(t.data) + f.off * es;
  return base % 16 == 0;
}

bool tma_ok_mnmajor(const Fit& f, const tm_tensor& t, int64_t rows, int64_t k, int64_t batch, int want_dt) {
  if (t.dtype != want_dt) return false;
  const int es = esize(t.dtype);
  if (f.lo != 1 || f.P < rows || f.c1 <= 0) return false;
  if (!batch_ok(f.c2, f.c1 * k, batch)) return false;
  if ((f.c1 * es) % 16 || (f.c2 * es) % 16) return false;
  return (reinterpret_cast<uintptr_t>(t.data) + f.off * es) % 16 == 0;
}

// Halo implicit GEMM (conv_halo.cuh) for a stride-1 conv anchor with a square
// odd kernel (pad = (k - 1) / 2, so Ho = H, Wo = W), channels-last bf16/fp16 X
// with C % 64 == 0, an OHWI (K-major, K order (tap, c)) filter, W + 2 pad <= 128,
// and a canonical epilogue writing channels-last rows without a residual.
bool bind_halo(const SubgraphPlan& sp, const std::map<std::string, tm_tensor>& env, BoundKernel& k, Exec& ex,
               int want_dt, int sms) {
  GemmParams& p = k.p;
  if (std::getenv("TMB_NO_HALO")) return false;
  if (sp.a.kind != OperandPlan::Im2col || sp.b.kind != OperandPlan::ConvFilter || k.simt || k.tf32) return false;
  if (!p.canon || p.canon_res_op >= 0 || p.out_dtype != want_dt || sp.batch != 1) return false;
  const ConvInfo& c = sp.a.conv;
  const tm_tensor& x = lookup(env, c.x_tensor);
  const tm_tensor& w = lookup(env, sp.b.conv.w_tensor);
  const int64_t F = sp.N;
  // (1x1 convs are plain K-major GEMM tiles already: no tap reuse to gain)
  if (c.stride != 1 || c.kh != c.kw || c.kh < 3 || c.kh % 2 == 0 || c.pad * 2 + 1 != c.kh || c.ho != c.h ||
      c.wo != c.w)
    return false;
  if (x.dtype != want_dt || w.dtype != want_dt || c.c % 64 != 0) return false;
  // channels-last X (any 16-byte-multiple row / image strides) and OHWI filter rows
  if (x.stride[1] != 1 || x.stride[3] != c.c || (x.stride[2] * 2) % 16 || (x.stride[0] * 2) % 16 ||
      reinterpret_cast<uintptr_t>(x.data) % 16)
    return false;
  const int64_t K = c.kh * c.kw * c.c;
  if (w.stride[1] != 1 || w.stride[3] != c.c || w.stride[2] != c.kw * c.c || (w.stride[0] * 2) % 16 ||
      w.stride[0] < K || reinterpret_cast<uintptr_t>(w.data) % 16)
    return false;
  const int P = static_cast<int>(c.w + 2 * c.pad);
  if (P > 128) return false;
  const int R = static_cast<int>(std::min<int64_t>(128 / P, c.ho));
  const int kbs = static_cast<int>(K / 64);
  if (kbs > 128) return false;
  const int bn = (F > 64 && F % 128 == 0) ? 128 : 64;
  if (F % bn) return false;
  // TMEM lane utilisation: R output rows of Wo valid lanes out of 128 (l4.c2's 7x7
  // maps keep 49 of 128; the K3 kernel's split-K is faster there)
  if ((128 / P < c.ho ? 128 / P : c.ho) * c.wo < 96 || c.c / 64 > 8) return false;
  // output: rows = pixels (n, oh, ow) at a uniform 16-byte-multiple stride, columns contiguous
  const Addr& oa = p.out_a;
  if (oa.s_col != 1 || oa.P < sp.M || (oa.s_lo * 2) % 16 || (oa.offset * 2) % 16 ||
      reinterpret_cast<uintptr_t>(p.out) % 16)
    return false;
  const int rows = R + static_cast<int>(c.kh) - 1;
  const int G = rows * P * 16;
  // dead TMEM lanes (r >= R * P) read up to (128 + (kh - 1) P + kw) pixels into the
  // last channel group: slack past the band
  const int band_bytes = G * static_cast<int>(c.c / 8) + (128 + static_cast<int>(c.kh) * P + static_cast<int>(c.kw)) * 16;
  // eligibility: two bands and a 2-stage ring of single k-blocks fit
  if (halo_smem(band_bytes, bn * 128, 2, bn, 2) > kMaxSmem) return false;
  // one band buffer when no CTA gets a second tile (l3.c2 at batch 32: 128 tiles on
  // 128 CTAs) -- the second band would never be loaded; its space deepens the ring
  const int64_t tiles_total = c.n * ((c.ho + R - 1) / R) * (F / bn);
  const char* mc_env0 = std::getenv("TMB_HALO_MC");
  const bool mc_req = mc_env0 && mc_env0[0] == '2';
  const int nbands = (!mc_req && tiles_total <= sms && !std::getenv("TMB_HALO_2BANDS")) ? 1 : 2;
  // filter stages of nb k-blocks (32 KB where it fits), the deepest ring that fits
  int nb = 0, stages = 0;
  for (int cand = bn == 64 ? 4 : 2; cand >= 1 && !stages; cand /= 2)
    for (int st = 8; st >= 2 && !stages; --st)
      if (halo_smem(band_bytes, cand * bn * 128, st, bn, nbands) <= kMaxSmem) {
        stages = st;
        nb = cand;
      }
  if (!stages) return false;
  // tensor maps: the band (5-D, channel-group-major) and the filter ({64, F, K/64})
  {  // one 64-channel chunk of the band per box: {8 ch, P px, rows, 8 groups, 1 image}
    const uint64_t dims[5] = {8, (uint64_t)c.w, (uint64_t)c.h, (uint64_t)(c.c / 8), (uint64_t)c.n};
    const uint64_t strides[4] = {(uint64_t)x.stride[3] * 2, (uint64_t)x.stride[2] * 2, 16, (uint64_t)x.stride[0] * 2};
    const uint32_t box[5] = {8u, (uint32_t)P, (uint32_t)rows, 8u, 1u};
    make_tma_2d3d(k.tma_a, x.data, x.dtype, 5, dims, strides, box, 0);
  }
  // CTA pairs (clusters of 2) share every filter stage: each CTA loads half of it
  // (half the taps when a stage holds an even number, else half the filter rows) and
  // multicasts it into both, halving the filter's L2 -> SM traffic.  Opt-in
  // (TMB_HALO_MC=2): the filter stream does not bound this kernel on the ResNet
  // layers (measured: equal or slower than one CTA per stage).
  const int64_t spatial = c.n * ((c.ho + R - 1) / R);
  const char* mc_env = std::getenv("TMB_HALO_MC");
  const int mc = mc_env && mc_env[0] == '2' && std::min<int64_t>(sms, spatial * (F / bn)) >= 2 ? 2 : 1;
  {  // filter {64 c, F, C/64 blocks, taps}: a stage is nb taps of one 64-channel block
    const uint64_t taps = c.kh * c.kw;
    const uint64_t dims[4] = {64, (uint64_t)F, (uint64_t)(c.c / 64), taps};
    const uint64_t strides[3] = {(uint64_t)w.stride[0] * 2, 128, (uint64_t)(c.c / 64) * 128};
    const bool split_taps = nb % 2 == 0;
    const uint32_t box[4] = {64u, (uint32_t)(mc == 2 && !split_taps ? bn / 2 : bn), 1u,
                             (uint32_t)(mc == 2 && split_taps ? nb / 2 : nb)};
    make_tma_2d3d(k.tma_b, w.data, w.dtype, 4, dims, strides, box, 128);
    p.hb_mc = mc;
    p.hb_split = split_taps ? 1 : 0;
  }
  ConvGeom& g = p.conv;
  g.n = static_cast<int32_t>(c.n); g.c = static_cast<int32_t>(c.c); g.h = static_cast<int32_t>(c.h);
  g.w = static_cast<int32_t>(c.w); g.f = static_cast<int32_t>(F); g.kh = static_cast<int32_t>(c.kh);
  g.kw = static_cast<int32_t>(c.kw); g.stride = 1; g.pad = static_cast<int32_t>(c.pad);
  g.ho = static_cast<int32_t>(c.ho); g.wo = static_cast<int32_t>(c.wo);
  p.hb_R = R;
  p.hb_P = P;
  p.hb_rows = rows;
  p.hb_G = G;
  p.hb_band = band_bytes;
  p.hb_kb = kbs;
  p.hb_tpi = static_cast<int32_t>((c.ho + R - 1) / R);
  p.hb_ftiles = static_cast<int32_t>(F / bn);
  p.hb_total = static_cast<int32_t>(c.n * p.hb_tpi * p.hb_ftiles);
  p.hb_stages = stages;
  p.rb_steps = nb;  // k-blocks per filter stage
  p.a_loader = LD_HALO;
  p.b_loader = LD_TMA_K;
  p.split_k = 1;
  k.rowband = 2;
  k.bn = bn;
  k.cg = 1;
  p.hb_nbands = nbands;
  k.smem = halo_smem(band_bytes, nb * bn * 128, stages, bn, nbands);
  k.grid = static_cast<int>(std::min<int64_t>(sms, p.hb_total));
  if (mc == 2) k.grid = static_cast<int>(std::min<int64_t>(sms, 2 * ((spatial + 1) / 2) * p.hb_ftiles)) & ~1;
  if (std::getenv("TMB_TRACE")) {
    void* tr = nullptr;
    const size_t tb = size_t(k.grid) * kTraceTiles * kTraceEvents * 8;
    if (cudaMalloc(&tr, tb) != cudaSuccess || cudaMemset(tr, 0, tb) != cudaSuccess)
      fail_cuda("cudaMalloc failed for the trace buffer");
    ex.scratch.push_back(tr);
    p.trace = static_cast<long long*>(tr);
  }
  return true;
}

// Row-band implicit GEMM (conv_rowband.cuh) for a conv anchor whose input
// pixels are padded to cpad in {4, 8} channels (C <= cpad) with stride * cpad
// == 8, Wo <= 128, kw + shift <= 8, and a canonical epilogue storing bf16/fp16
// channels-last rows without a residual.  Called once the generic operand /
// epilogue binding is known; returns false (leaving k untouched) otherwise.
bool bind_rowband(const SubgraphPlan& sp, const std::map<std::string, tm_tensor>& env, BoundKernel& k, Exec& ex,
                  int want_dt, int sms) {
  GemmParams& p = k.p;
  if (std::getenv("TMB_NO_ROWBAND")) return false;
  if (sp.a.kind != OperandPlan::Im2col || sp.b.kind != OperandPlan::ConvFilter || k.simt || k.tf32) return false;
  if (!p.canon || p.canon_res_op >= 0 || !p.out_tma || p.out_dtype != want_dt || sp.batch != 1) return false;
  const ConvInfo& c = sp.a.conv;
  const tm_tensor& x = lookup(env, c.x_tensor);
  const tm_tensor& w = lookup(env, sp.b.conv.w_tensor);
  const int64_t cpad = x.stride[3];
  if (x.dtype != want_dt || x.stride[1] != 1 || (cpad != 4 && cpad != 8) || c.c > cpad || c.stride * cpad != 8) return false;
  if ((c.w * cpad) % 8 || x.stride[2] < c.w * cpad || x.stride[2] % 8 || x.stride[0] < c.h * x.stride[2] ||
      x.stride[0] % 8 || reinterpret_cast<uintptr_t>(x.data) % 16)
    return false;
  const int ppg = static_cast<int>(8 / cpad);  // pixels per 16-byte granule
  const int shift = static_cast<int>((ppg - c.pad % ppg) % ppg);
  const int64_t F = sp.N;  // output channels (the filter's rows)
  if (c.wo > 128 || c.kw + shift > 8 || F > 256 || c.ho < 1) return false;
  // output: rows = pixels (n, oh, ow) at stride lo, uniform across rows of pixels
  const Addr& oa = p.out_a;
  if (oa.s_col != 1 || oa.P < sp.M || oa.s_lo <= 0) return false;
  const int es = 2;
  const int bn = F <= 64 ? 64 : F <= 128 ? 128 : 256;
  const int steps = static_cast<int>(cpad / 2);  // 8 taps * cpad channels * 2 B / 32 B per K16 step
  // staged rows are loaded in 128-byte chunks when an image row is a whole
  // number of them (a TMA box with 128-byte inner rows moves ~8x fewer lines
  // than one with 16-byte granules), else in 16-byte granules; the left
  // padding (pad + shift pixels) is rounded up to whole chunks of zero fill
  const int64_t row_bytes = c.w * cpad * 2;
  const int chunk = row_bytes % 128 == 0 ? 128 : 16;
  const int64_t lp_bytes = ((c.pad + shift) * cpad * 2 + chunk - 1) / chunk * chunk;  // left zero fill
  const int off0 = static_cast<int>(lp_bytes - (c.pad + shift) * cpad * 2);  // window of ow = 0
  // (rows are whole 128-byte units: each TMA box lands 128-byte aligned)
  const int rowb = static_cast<int>((off0 + 16 * 127 + 16 * cpad + 127) / 128 * 128);
  const int bbytes = static_cast<int>(c.kh * steps * bn * 32);
  int T = 0;
  const int tmax = std::getenv("TMB_RB_T") ? std::max(1, std::atoi(std::getenv("TMB_RB_T"))) : 16;  // diagnostics
  constexpr int kBoxes = 4;  // conv_rowband.cuh kRbLoadWarps
  auto rbox_of = [&](int t) { return static_cast<int>((c.stride * (t - 1) + c.kh + kBoxes - 1) / kBoxes); };
  for (int t = tmax; t >= 1 && !T; --t)
    if (rowband_smem(kBoxes * rbox_of(t), rowb, bbytes, bn) <= kMaxSmem) T = t;
  if (!T) return false;
  // filter image, packed once at bind (an inference constant of the bound plan)
  ConvGeom& g = p.conv;
  g.n = static_cast<int32_t>(c.n); g.c = static_cast<int32_t>(c.c); g.h = static_cast<int32_t>(c.h);
  g.w = static_cast<int32_t>(c.w); g.f = static_cast<int32_t>(F); g.kh = static_cast<int32_t>(c.kh);
  g.kw = static_cast<int32_t>(c.kw); g.stride = static_cast<int32_t>(c.stride); g.pad = static_cast<int32_t>(c.pad);
  g.ho = static_cast<int32_t>(c.ho); g.wo = static_cast<int32_t>(c.wo);
  g.x = x.data; g.x_dtype = x.dtype; g.wt = w.data; g.w_dtype = w.dtype;
  for (int d = 0; d < 4; ++d) { g.sx[d] = x.stride[d]; g.sw[d] = w.stride[d]; }
  void* img = nullptr;
  if (cudaMalloc(&img, bbytes) != cudaSuccess) fail_cuda("cudaMalloc failed for the row-band filter image");
  ex.scratch.push_back(img);
  pack_rowband_filter(g, static_cast<int>(cpad), shift, steps, bn, img, want_dt);
  // staged-row view {chunk elements, chunks per row, H, N} (no swizzle); the
  // first band's box (tma_b slot) has fewer rows
  const int T0 = std::min(T, 4);
  for (int which = 0; which < 2; ++which) {
    const uint64_t dims[4] = {(uint64_t)(chunk / es), (uint64_t)(row_bytes / chunk), (uint64_t)c.h, (uint64_t)c.n};
    const uint64_t strides[3] = {(uint64_t)chunk, (uint64_t)x.stride[2] * es, (uint64_t)x.stride[0] * es};
    const int t = which == 0 ? T : T0;
    const uint32_t box[4] = {(uint32_t)(chunk / es), (uint32_t)(rowb / chunk), (uint32_t)rbox_of(t), 1u};
    make_tma_2d3d(which == 0 ? k.tma_a : k.tma_b, x.data, x.dtype, 4, dims, strides, box, 0);
  }
  // output view {F, Wo, N*Ho}: one tile = one output row, lanes >= Wo clipped
  {
    const uintptr_t base = reinterpret_cast<uintptr_t>(p.out) + oa.offset * es;
    const uint64_t dims[3] = {(uint64_t)F, (uint64_t)c.wo, (uint64_t)(c.n * c.ho)};
    const uint64_t strides[2] = {(uint64_t)(oa.s_lo * es), (uint64_t)(oa.s_lo * c.wo * es)};
    const uint32_t box[3] = {static_cast<uint32_t>(kRbOutRow / es), 32u, 1u};
    make_tma_2d3d(k.tma_c, reinterpret_cast<const void*>(base), p.out_dtype, 3, dims, strides, box, kRbOutRow);
  }
  p.rb_T = T;
  p.rb_rows = rbox_of(T);
  p.rb_rowb = rowb;
  p.rb_off0 = off0;
  p.rb_T0 = T0;
  p.rb_rows0 = rbox_of(T0);
  p.rb_steps = steps;
  p.rb_g0 = static_cast<int32_t>(-lp_bytes / chunk);
  p.rb_total = static_cast<int32_t>(c.n * c.ho);
  p.rb_cpad = static_cast<int32_t>(cpad);
  p.rb_fix = (c.c < cpad && !std::getenv("TMB_RB_NOFIX")) ? 1 : 0;  // NOFIX: diagnostics only
  if (const char* d = std::getenv("TMB_DBG")) p.dbg = std::atoi(d);  // 11-13: MMA operand-layout timing probes
  p.rb_bbytes = bbytes;
  p.rb_bimg = img;
  k.rowband = 1;
  p.a_loader = LD_ROWBAND;
  p.b_loader = LD_TMA_K;
  k.bn = bn;
  k.cg = 1;
  k.smem = rowband_smem(kBoxes * p.rb_rows, rowb, bbytes, bn);
  k.grid = static_cast<int>(std::min<int64_t>(sms, c.n * c.ho));
  p.split_k = 1;
  if (std::getenv("TMB_TRACE")) {  // per-tile role timeline (tm_exec_trace)
    void* tr = nullptr;
    const size_t tb = size_t(k.grid) * kTraceTiles * kTraceEvents * 8;
    if (cudaMalloc(&tr, tb) != cudaSuccess || cudaMemset(tr, 0, tb) != cudaSuccess)
      fail_cuda("cudaMalloc failed for the trace buffer");
    ex.scratch.push_back(tr);
    p.trace = static_cast<long long*>(tr);
  }
  return true;
}
// Rule / reduce kernel binding: bytecode + tensor references in one device
// blob owned by the exec; the output is the root node's bound (or
// plan-owned intermediate) tensor.
BoundKernel bind_rule(const Plan& plan, const SubgraphPlan& sp, const std::map<std::string, tm_tensor>& env, Exec& ex,
                      int sms) {
  const ComputeDAG& dag = plan.dag;
  const TensorNode& n = dag.at(sp.rule_node);
  if (n.axes.size() > static_cast<size_t>(ev::kMaxRank) || n.reduce_axes.size() > static_cast<size_t>(ev::kMaxRank) ||
      n.axes.size() + n.reduce_axes.size() > static_cast<size_t>(ev::kMaxVars))
    fail_unsupported("rule kernel '", n.name, "': too many axes");
  std::vector<std::string> vars;
  for (const auto& a : n.axes) vars.push_back(a.name);
  for (const auto& a : n.reduce_axes) vars.push_back(a.name);
  const ev::Program prog = ev::compile_program(sp.rule_expr, vars);
  auto ref_of = [&](const std::string& name) {
    const tm_tensor& t = lookup(env, name);
    const TensorNode& tn = dag.at(name);
    if (t.rank > ev::kMaxRank) fail_unsupported("tensor '", name, "' has too many dims for a rule kernel");
    ev::TensorRef r{};
    r.ptr = t.data;
    r.store = t.dtype == TM_F32 ? ev::ST_F32 : t.dtype == TM_BF16 ? ev::ST_BF16 : ev::ST_F16;
    r.is_float = tn.dtype == taskmap::DType::F32;
    r.rank = t.rank;
    for (int d = 0; d < t.rank; ++d) {
      r.shape[d] = t.shape[d];
      r.stride[d] = t.stride[d];
    }
    return r;
  };
  std::vector<ev::TensorRef> refs;
  for (const auto& name : prog.tensors) refs.push_back(ref_of(name));
  const size_t code_b = prog.code.size() * sizeof(ev::Ins), refs_b = refs.size() * sizeof(ev::TensorRef),
               tab_b = prog.tables.size() * sizeof(int64_t);
  std::vector<unsigned char> host(code_b + refs_b + tab_b + 64, 0);
  std::memcpy(host.data(), prog.code.data(), code_b);
  if (refs_b) std::memcpy(host.data() + code_b, refs.data(), refs_b);
  if (tab_b) std::memcpy(host.data() + code_b + refs_b, prog.tables.data(), tab_b);
  void* blob = nullptr;
  if (cudaMalloc(&blob, host.size()) != cudaSuccess ||
      cudaMemcpy(blob, host.data(), host.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    fail_cuda("cudaMalloc/cudaMemcpy failed for a rule-kernel program");
  ex.scratch.push_back(blob);
  BoundKernel k{};
  k.rule = 1;
  RuleJob& j = k.rj;
  j.code = static_cast<const ev::Ins*>(blob);
  j.tensors = reinterpret_cast<const ev::TensorRef*>(static_cast<unsigned char*>(blob) + code_b);
  j.tables = reinterpret_cast<const int64_t*>(static_cast<unsigned char*>(blob) + code_b + refs_b);
  j.n_code = static_cast<int32_t>(prog.code.size());
  j.n_axes = static_cast<int32_t>(n.axes.size());
  j.n_red = static_cast<int32_t>(n.reduce_axes.size());
  j.combiner = static_cast<int32_t>(n.combiner);
  j.is_float = n.dtype == taskmap::DType::F32;
  j.numel = 1;
  for (size_t d = 0; d < n.axes.size(); ++d) {
    j.ext[d] = n.axes[d].extent;
    j.numel *= n.axes[d].extent;
  }
  j.red_numel = 1;
  for (size_t d = 0; d < n.reduce_axes.size(); ++d) {
    j.red[d] = n.reduce_axes[d].extent;
    j.red_numel *= n.reduce_axes[d].extent;
  }
  // reduce_template (one CTA per output, tree) for long reductions or few
  // outputs; the sequential in-thread loop of rule_based_schedule for short ones
  // over many outputs (reduce extent <= 256 inlines as SeqFor)
  const bool tree = j.n_red > 0 && (j.red_numel > 256 || j.numel < int64_t(sms) * 64);
  j.mode = tree ? RULE_TREE : RULE_ELEM;
  j.out = ref_of(sp.rule_node);
  k.rule_threads = plan.cfg.threads_per_block > 0 ? plan.cfg.threads_per_block : 128;
  k.grid = sms;  // launch_rule sizes the grid from the SM count
  k.bn = 0;
  // the generated kernel (NVRTC) unless the expression needs the interpreter,
  // NVRTC is absent, or TMB_RULE_INTERP=1 forces the bytecode path
  const char* force = std::getenv("TMB_RULE_INTERP");
  if (!(force && force[0] == '1')) {
    RuleSourceSpec spec;
    spec.expr = sp.rule_expr;
    spec.vars = vars;
    for (size_t d = 0; d < n.axes.size(); ++d) spec.ext.push_back(n.axes[d].extent);
    for (size_t d = 0; d < n.reduce_axes.size(); ++d) spec.red.push_back(n.reduce_axes[d].extent);
    spec.tensor_names = prog.tensors;
    spec.tensors = refs;
    spec.out = j.out;
    spec.combiner = j.combiner;
    spec.is_float = j.is_float != 0;
    rule_launch_shape(j, k.rule_threads, sms, &k.rgrid, &k.rblock);
    spec.threads = static_cast<int>(k.rblock);
    spec.mode = tree ? GEN_TREE : GEN_ELEM;
    int64_t scratch_bytes = 0;
    if (tree && j.numel < sms && j.red_numel >= 8192) {
      // fewer outputs than SMs: split each reduction over several CTAs
      const int64_t by_sm = (8 * int64_t(sms) + j.numel - 1) / j.numel;
      const int64_t by_len = j.red_numel / (int64_t(k.rblock) * 8);
      const int64_t S = std::max<int64_t>(2, std::min(by_sm, by_len));
      spec.mode = GEN_SPLIT;
      spec.splits = static_cast<int>(S);
      k.rgrid = static_cast<unsigned>(j.numel * S);
      scratch_bytes = j.numel * S * 8 + j.numel * 4;
    } else if (j.n_red > 0 && j.red_numel >= 16 && j.red_numel <= 256) {
      // short reductions: a lane group per output
      // (about four loads per lane: independent, unrolled, still whole sectors)
      int G = 1;
      while (G * 2 <= 32 && G * 8 <= j.red_numel) G *= 2;
      spec.mode = GEN_GROUP;
      spec.group = G;
      const int64_t want = (j.numel + 256 / G - 1) / (256 / G);
      k.rgrid = static_cast<unsigned>(std::min<int64_t>(want, int64_t(sms) * 8));
      k.rblock = 256;
    }
    std::string src, why;
    if (emit_rule_source(spec, src, why)) k.rfn = compile_rule_source(src, why);
    if (k.rfn) {
      for (size_t t = 0; t < refs.size(); ++t) k.rp.p[t] = refs[t].ptr;
      k.rp.p[kMaxRuleTensors] = j.out.ptr;
      if (scratch_bytes) {
        void* scratch = nullptr;
        if (cudaMalloc(&scratch, scratch_bytes) != cudaSuccess || cudaMemset(scratch, 0, scratch_bytes) != cudaSuccess)
          fail_cuda("cudaMalloc of the split-reduction scratch failed");
        ex.scratch.push_back(scratch);
        k.rp.p[refs.size()] = scratch;
      }
    } else if (std::getenv("TMB_RULE_VERBOSE")) {
      std::fprintf(stderr, "[taskmap] rule kernel '%s' keeps the interpreter: %s\n", n.name.c_str(), why.c_str());
    }
  }
  return k;
}
}  // namespace

int intermediate_dtype(const tm_tensor* inputs, int n_in) {
  bool f32 = false, f16 = false, bf16 = false;
  for (int i = 0; i < n_in; ++i) {
    f32 = f32 || inputs[i].dtype == TM_F32;
    f16 = f16 || inputs[i].dtype == TM_F16;
    bf16 = bf16 || inputs[i].dtype == TM_BF16;
  }
  if (f32) return TM_F32;
  if (f16 && !bf16) return TM_F16;
  return TM_BF16;
}

Exec::~Exec() {
  for (void* p : scratch) cudaFree(p);
}

std::unique_ptr<Exec> bind_plan(const Plan& plan, const tm_tensor* inputs, int n_in,
                                const tm_tensor* outputs, int n_out) {
  const ComputeDAG& dag = plan.dag;
  if (n_in != static_cast<int>(dag.inputs.size()))
    fail("expected ", dag.inputs.size(), " input tensors, got ", n_in);
  if (n_out != static_cast<int>(dag.outputs.size()))
    fail("expected ", dag.outputs.size(), " output tensors, got ", n_out);
  std::map<std::string, tm_tensor> env;
  auto check = [&](const std::string& name, const tm_tensor& t) {
    const TensorNode& n = dag.at(name);
    if (t.rank != static_cast<int>(n.shape.size())) fail("tensor '", name, "' has wrong rank");
    for (int d = 0; d < t.rank; ++d)
      if (t.shape[d] != n.shape[d]) fail("tensor '", name, "' has wrong shape at dim ", d);
    if (t.dtype != TM_F32 && t.dtype != TM_BF16 && t.dtype != TM_F16) fail_unsupported("tensor '", name, "' has unsupported dtype");
    if (!t.data) fail("tensor '", name, "' has a null data pointer");
    env[name] = t;
  };
  for (int i = 0; i < n_in; ++i) check(dag.inputs[i], inputs[i]);
  for (int i = 0; i < n_out; ++i) check(dag.outputs[i], outputs[i]);
  auto ex = std::make_unique<Exec>();
  const int idt = intermediate_dtype(inputs, n_in);
  for (const auto& name : plan.intermediates) {
    const TensorNode& n = dag.at(name);
    tm_tensor t{};
    t.dtype = idt;
    t.rank = static_cast<int>(n.shape.size());
    int64_t numel = 1;
    for (int d = t.rank - 1; d >= 0; --d) {
      t.shape[d] = n.shape[d];
      t.stride[d] = numel;
      numel *= n.shape[d];
    }
    void* p = nullptr;
    if (cudaMalloc(&p, numel * esize(idt)) != cudaSuccess) fail_cuda("cudaMalloc failed for intermediate '", name, "'");
    ex->scratch.push_back(p);
    t.data = p;
    env[name] = t;
  }
  const int sms = num_sms(plan.device);
  for (const auto& sp : plan.kernels) {
    if (sp.kind == SubgraphPlan::Rule) {
      ex->kernels.push_back(bind_rule(plan, sp, env, *ex, sms));
      continue;
    }
    BoundKernel k{};
    GemmParams& p = k.p;
    p.M = static_cast<int32_t>(sp.M);
    p.N = static_cast<int32_t>(sp.N);
    p.K = static_cast<int32_t>(sp.K);
    p.batch = static_cast<int32_t>(sp.batch);
    // math kind
    std::string math = plan.cfg.math;
    const tm_tensor* opa = sp.a.kind == OperandPlan::Strided ? &lookup(env, sp.a.addr.tensor) : &lookup(env, sp.a.conv.x_tensor);
    const tm_tensor* opb = sp.b.kind == OperandPlan::Strided ? &lookup(env, sp.b.addr.tensor) : &lookup(env, sp.b.conv.w_tensor);
    // auto: bf16 operands -> tcgen05 kind::f16; fp32 operands keep fp32 semantics on
    // the CUDA-core kernel (matrix operands) or run kind::tf32 (convolutions);
    // tf32 for matrices is an explicit choice (math="tf32")
    const bool want_halo = math == "halo";  // the halo conv kernel family (bind_halo), else K3
    if (math == "halo") math = "auto";
    if (math == "auto") {
      if (opa->dtype == TM_F32 || opb->dtype == TM_F32)
        math = (sp.a.kind == OperandPlan::Strided && sp.b.kind == OperandPlan::Strided) ? "fp32_simt" : "tf32";
      else
        math = "bf16";
    }
    if (math == "fp32_simt") k.simt = 1;
    k.tf32 = math == "tf32";
    // 16-bit tensor-core path (tcgen05 kind::f16): the a/b operand format is that of
    // the operands -- fp16 when both are fp16, else bf16.  Mixed bf16/fp16 operands
    // would need a lossy conversion of one of them, which is refused.
    const bool a16 = opa->dtype == TM_F16, b16 = opb->dtype == TM_F16;
    if (!k.tf32 && !k.simt && (opa->dtype == TM_BF16 || opb->dtype == TM_BF16) && (a16 || b16))
      fail_unsupported("mixed bf16 / fp16 GEMM operands: cast one side to the other's type first");
    p.ab_f16 = (!k.tf32 && !k.simt && (a16 || b16)) ? 1 : 0;
    const int BK = k.tf32 ? 32 : 64;
    const int want_dt = k.tf32 ? TM_F32 : (p.ab_f16 ? TM_F16 : TM_BF16);
    k.bn = plan.cfg.block_n;
    if (k.bn < 16 || k.bn > 256 || k.bn % 16) fail("block_n must be 16..256 in steps of 16");
    k.stages = plan.cfg.pipeline ? plan.cfg.stages : 2;
    p.num_kb = static_cast<int32_t>((sp.K + BK - 1) / BK);
    p.tiles_n = static_cast<int32_t>((sp.N + k.bn - 1) / k.bn);
    auto strided_of = [&](const Fit& f, const tm_tensor& t, const std::vector<EpiStep>& pre) {
      Strided s{};
      s.ptr = t.data;
      s.dtype = t.dtype;
      s.P = f.P; s.s_hi = f.hi; s.s_lo = f.lo; s.s_k = f.c1; s.s_batch = f.c2; s.offset = f.off;
      s.n_pre = static_cast<int32_t>(pre.size());
      for (size_t i = 0; i < pre.size() && i < static_cast<size_t>(kMaxPreOps); ++i) s.pre[i] = PreOp{pre[i].kind, pre[i].c};
      return s;
    };
    std::string why;
    // Operand loaders for a given CTA group (cg = 2: each CTA stages BN/2 rows of B).
    auto bind_operands = [&](int cg) {
    const int bn_cta = k.bn / cg;
    bool im2col_tma = false;
    // conv operands whose re-index map is a plain K-major tile (1x1 stride-1
    // conv on channels-last data) use ordinary TMA tiles instead of im2col
    bool conv_as_gemm = false;
    if (sp.a.kind == OperandPlan::Im2col && !sp.a.addr.idx.empty() && sp.b.kind == OperandPlan::ConvFilter &&
        !sp.b.addr.idx.empty()) {
      Fit fa, fb;
      std::string w2;
      conv_as_gemm = fit_address(sp.a.addr, *opa, sp.M, sp.K, sp.batch, fa, w2) && tma_ok_kmajor(fa, *opa, sp.M, want_dt, sp.batch) &&
                     fit_address(sp.b.addr, *opb, sp.N, sp.K, sp.batch, fb, w2) && tma_ok_kmajor(fb, *opb, sp.N, want_dt, sp.batch);
    }
    if (sp.a.kind == OperandPlan::Im2col && !conv_as_gemm) {
      const ConvInfo& c = sp.a.conv;
      const tm_tensor& x = *opa;
      ConvGeom& g = p.conv;
      g.n = c.n; g.c = c.c; g.h = c.h; g.w = c.w; g.kh = c.kh; g.kw = c.kw; g.stride = c.stride;
      g.pad = c.pad; g.ho = c.ho; g.wo = c.wo; g.x = x.data; g.x_dtype = x.dtype;
      for (int d = 0; d < 4; ++d) g.sx[d] = x.stride[d];
      const bool cl = x.stride[1] == 1 && x.stride[3] == c.c && x.stride[2] == c.w * c.c && x.stride[0] == c.h * c.w * c.c;
      im2col_tma = !k.tf32 && x.dtype == want_dt && cl && c.c % BK == 0 && c.stride <= 8 &&
                   c.pad <= 127 && (c.kh - 1 - c.pad) <= 128 && c.kh <= 127 && c.kw <= 127 &&
                   (reinterpret_cast<uintptr_t>(x.data) % 16 == 0) &&
                   sp.b.kind == OperandPlan::ConvFilter && plan.cfg.split_k >= 1;
      // C <= 8 stored 16-byte padded channels-last (pixel stride 8): one im2col box per tap
      const bool cl8 = x.stride[1] == 1 && x.stride[3] == 8 && x.stride[2] == c.w * 8 && x.stride[0] == c.h * c.w * 8;
      const bool tma8 = !im2col_tma && !k.tf32 && cg == 1 && x.dtype == want_dt && c.c <= 8 && cl8 &&
                        c.stride <= 8 && c.pad <= 127 && (reinterpret_cast<uintptr_t>(x.data) % 16 == 0) &&
                        sp.b.kind == OperandPlan::ConvFilter;
      g.korder = (im2col_tma || tma8) ? 1 : 0;
      g.cpad = tma8 ? 8 : static_cast<int32_t>(c.c);
      // small C: 16-byte-per-(pixel, tap) LSU gather (LD_IM2COL_G8) -- a TMA box per
      // tap (LD_IM2COL_TMA8) costs ~600 clk of TMA issue each, 49 of them per tile
      p.a_loader = im2col_tma ? LD_IM2COL_TMA : tma8 ? LD_IM2COL_G8 : LD_IM2COL_GATHER;
      if (tma8) {
        p.K = static_cast<int32_t>(c.kh * c.kw * 8);  // K order (tap, 8 channels)
        p.num_kb = (p.K + BK - 1) / BK;
      }
      if (im2col_tma) {
        const uint64_t dims[4] = {(uint64_t)c.c, (uint64_t)c.w, (uint64_t)c.h, (uint64_t)c.n};
        const uint64_t strides[3] = {(uint64_t)x.stride[3] * 2, (uint64_t)x.stride[2] * 2, (uint64_t)x.stride[0] * 2};
        make_tma_im2col(k.tma_a, x.data, x.dtype, dims, strides, static_cast<int>(c.pad),
                        static_cast<int>(c.pad - (c.kh - 1)), static_cast<int>(c.stride), BK, 128);
      }
    } else {
      Fit f;
      if (!fit_address(sp.a.addr, *opa, sp.M, sp.K, sp.batch, f, why)) fail_unsupported("operand A '", sp.a.addr.tensor, "': ", why);
      p.a = strided_of(f, *opa, sp.a.pre);
      if (sp.a.pre.empty() && tma_ok_kmajor(f, *opa, sp.M, want_dt, sp.batch)) {
        p.a_loader = LD_TMA_K;
        const uint64_t dims[3] = {(uint64_t)sp.K, (uint64_t)sp.M, (uint64_t)sp.batch};
        const uint64_t strides[2] = {(uint64_t)(f.lo * esize(opa->dtype)),
                                     (uint64_t)(std::max<int64_t>(f.c2, f.lo * sp.M) * esize(opa->dtype))};
        const uint32_t box[3] = {(uint32_t)BK, 128u, 1u};
        make_tma_2d3d(k.tma_a, static_cast<const char*>(opa->data) + f.off * esize(opa->dtype), opa->dtype, 3, dims, strides, box);
      } else {
        p.a_loader = LD_GATHER;
      }
    }
    // ---- operand B
    if (sp.b.kind == OperandPlan::ConvFilter && !conv_as_gemm) {
      const tm_tensor& w = *opb;
      ConvGeom& g = p.conv;
      g.f = static_cast<int32_t>(sp.N);
      g.wt = w.data;
      g.w_dtype = w.dtype;
      for (int d = 0; d < 4; ++d) g.sw[d] = w.stride[d];
      const ConvInfo& c = sp.b.conv;
      // K-major filter view: korder 0 needs OIHW-contiguous, korder 1 needs OHWI
      const bool oihw = w.stride[3] == 1 && w.stride[2] == c.kw && w.stride[1] == c.kh * c.kw;
      const bool ohwi = w.stride[1] == 1 && w.stride[3] == c.c && w.stride[2] == c.kw * c.c;
      const bool lin = g.korder == 0 ? oihw : ohwi;
      const int64_t row_stride = w.stride[0];
      if (lin && w.dtype == want_dt && (row_stride * esize(w.dtype)) % 16 == 0 &&
          reinterpret_cast<uintptr_t>(w.data) % 16 == 0) {
        p.b_loader = LD_TMA_K;
        const uint64_t dims[3] = {(uint64_t)p.K, (uint64_t)sp.N, 1};
        const uint64_t strides[2] = {(uint64_t)(row_stride * esize(w.dtype)), (uint64_t)(row_stride * sp.N * esize(w.dtype))};
        const uint32_t box[3] = {(uint32_t)BK, (uint32_t)bn_cta, 1u};
        make_tma_2d3d(k.tma_b, w.data, w.dtype, 3, dims, strides, box);
      } else if (!k.tf32) {
        // Filter layout not TMA-describable in this K order (e.g. the padded
        // (tap, 8-channel) order of LD_IM2COL_TMA8): repack it once, at bind
        // time, into a K-major [F, K'] bf16 buffer owned by the exec -- the
        // filter is an inference constant of the bound plan (re-bind after
        // changing weights).
        const int kp = (p.K + 7) / 8 * 8;
        void* packed = nullptr;
        if (cudaMalloc(&packed, size_t(sp.N) * kp * 2) != cudaSuccess) fail_cuda("cudaMalloc failed for the filter repack");
        ex->scratch.push_back(packed);
        pack_filter(g, kp, packed, want_dt);
        p.b_loader = LD_TMA_K;
        const uint64_t dims[3] = {(uint64_t)p.K, (uint64_t)sp.N, 1};
        const uint64_t strides[2] = {(uint64_t)kp * 2, (uint64_t)kp * 2 * sp.N};
        const uint32_t box[3] = {(uint32_t)BK, (uint32_t)bn_cta, 1u};
        make_tma_2d3d(k.tma_b, packed, want_dt, 3, dims, strides, box);
      } else {
        p.b_loader = LD_FILTER_GATHER;
      }
    } else {
      if (sp.b.addr.idx.empty()) fail("operand B must be a strided tensor or a conv filter");
      Fit f;
      if (!fit_address(sp.b.addr, *opb, sp.N, sp.K, sp.batch, f, why)) fail_unsupported("operand B '", sp.b.addr.tensor, "': ", why);
      p.b = strided_of(f, *opb, sp.b.pre);
      if (sp.b.pre.empty() && tma_ok_kmajor(f, *opb, sp.N, want_dt, sp.batch)) {
        p.b_loader = LD_TMA_K;
        const uint64_t dims[3] = {(uint64_t)sp.K, (uint64_t)sp.N, (uint64_t)sp.batch};
        const uint64_t strides[2] = {(uint64_t)(f.lo * esize(opb->dtype)),
                                     (uint64_t)(std::max<int64_t>(f.c2, f.lo * sp.N) * esize(opb->dtype))};
        const uint32_t box[3] = {(uint32_t)BK, (uint32_t)bn_cta, 1u};
        make_tma_2d3d(k.tma_b, static_cast<const char*>(opb->data) + f.off * esize(opb->dtype), opb->dtype, 3, dims, strides, box);
      } else if ((!k.tf32 || tf32_mn_ok()) && sp.b.pre.empty() && bn_cta % (128 / esize(want_dt)) == 0 &&
                 tma_ok_mnmajor(f, *opb, sp.N, sp.K, sp.batch, want_dt)) {
        // MN-major B (N contiguous): SWIZZLE_128B rows of MNB = 128 B / element
        // (64 16-bit or 32 fp32 elements) along N, BK k-rows per block.  The SS
        // form of kind::tf32 takes an MN-major B like the 16-bit kinds (only the
        // TMEM-A forms require K-major), so row-major fp32 B is TMA-fed too.
        p.b_loader = LD_TMA_MN;
        const int bes = esize(want_dt);
        const uint64_t mnb = 128 / bes;
        if (sp.N % mnb == 0 && !std::getenv("TMB_NO_MN4D")) {
          // {MNB n, K, N/MNB n-blocks, batch}: one box per slot lands the BN/MNB column
          // blocks at BK*128-byte strides, the layout the per-block boxes produced
          p.b_mn4d = 1;
          const uint64_t dims[4] = {mnb, (uint64_t)sp.K, (uint64_t)(sp.N / mnb), (uint64_t)sp.batch};
          const uint64_t strides[3] = {(uint64_t)(f.c1 * bes), 128,
                                       (uint64_t)(std::max<int64_t>(f.c2, f.c1 * sp.K) * bes)};
          const uint32_t box[4] = {(uint32_t)mnb, (uint32_t)BK, (uint32_t)(bn_cta / mnb), 1u};
          make_tma_2d3d(k.tma_b, static_cast<const char*>(opb->data) + f.off * bes, opb->dtype, 4, dims, strides, box,
                        k.tf32 ? kSwizzle128Atom32 : 128);
        } else {
          p.b_mn4d = 0;
          const uint64_t dims[3] = {(uint64_t)sp.N, (uint64_t)sp.K, (uint64_t)sp.batch};
          const uint64_t strides[2] = {(uint64_t)(f.c1 * bes), (uint64_t)(std::max<int64_t>(f.c2, f.c1 * sp.K) * bes)};
          const uint32_t box[3] = {(uint32_t)mnb, (uint32_t)BK, 1u};
          make_tma_2d3d(k.tma_b, static_cast<const char*>(opb->data) + f.off * bes, opb->dtype, 3, dims, strides, box,
                        k.tf32 ? kSwizzle128Atom32 : 128);
        }
      } else {
        p.b_loader = LD_GATHER;
      }
    }
    const bool a_tma = p.a_loader == LD_TMA_K || p.a_loader == LD_IM2COL_TMA;
    const bool b_tma = p.b_loader == LD_TMA_K || p.b_loader == LD_TMA_MN;
    return a_tma && b_tma;
    };
    // SM-pair (cta_group::2, 256-row tiles) when requested and every operand is TMA-fed
    k.cg = 1;
    if (!k.simt && plan.cfg.block_m == 256 && (k.bn == 64 || k.bn == 128 || k.bn == 256) && bind_operands(2)) k.cg = 2;
    else bind_operands(1);
    p.tiles_m = static_cast<int32_t>((sp.M + 128 * k.cg - 1) / (128 * k.cg));
    if (k.simt) {
      // fp32 CUDA-core kernel (simt_fp32.cu): 128x128 tiles, strided predicated loads
      if (p.a_loader == LD_IM2COL_GATHER || p.a_loader == LD_IM2COL_TMA || p.a_loader == LD_IM2COL_TMA8 ||
          p.a_loader == LD_IM2COL_G8 ||
          p.b_loader == LD_FILTER_GATHER || sp.b.kind == OperandPlan::ConvFilter)
        fail_unsupported("math=fp32_simt supports matrix operands only (conv im2col is not supported on this path)");
      // 128x128 tiles (the paper's mapping), or 128x64 when block_n asks for it
      k.bn = plan.cfg.block_n <= 64 ? 64 : 128;
      k.stages = plan.cfg.block_k == 16 ? 16 : 8;  // K-tile depth: the spec's block_k 16, else the paper's 8
      p.tiles_n = static_cast<int32_t>((sp.N + k.bn - 1) / k.bn);
      p.tiles_m = static_cast<int32_t>((sp.M + 127) / 128);
    }
    // ---- epilogue
    if (sp.ops.size() > static_cast<size_t>(kMaxEpiOps)) fail_unsupported("epilogue longer than ", kMaxEpiOps, " ops");
    p.n_ops = static_cast<int32_t>(sp.ops.size());
    int mat_slots = 0;
    for (size_t i = 0; i < sp.ops.size(); ++i) {
      EpiOp& o = p.ops[i];
      o.kind = sp.ops[i].kind;
      o.c = sp.ops[i].c;
      o.a = Addr{1, 0, 0, 0, 0, 0};
      if (sp.ops[i].side >= 0) {
        const AddrExpr& ae = sp.sides[sp.ops[i].side];
        const tm_tensor& t = lookup(env, ae.tensor);
        Fit f;
        if (!fit_address(ae, t, sp.M, sp.N, sp.batch, f, why)) fail_unsupported("epilogue operand '", ae.tensor, "': ", why);
        o.ptr = t.data;
        o.dtype = t.dtype;
        o.a = to_addr(f);
        // where the epilogue keeps it (see SideKind)
        if (o.a.s_col == 0) {
          o.side = SIDE_ROW;
        } else if (o.a.s_hi == 0 && o.a.s_lo == 0) {
          o.side = SIDE_COL;
        } else {
          if (mat_slots >= kMaxMatOps) fail_unsupported("epilogue has more than ", kMaxMatOps, " full-tile side operands (unsupported)");
          o.side = SIDE_MAT;
          o.slot = mat_slots++;
          p.has_mat = 1;
        }
      }
    }
    // canonical epilogue v = act(acc * S[c] + T[c]) (+ R): [MUL s]? [ADD|SUB t]? [RELU|GELU]? [ADD residual]?
    {
      int i = 0;
      const int n = p.n_ops;
      p.canon_s = 1.f;
      p.canon_t = 0.f;
      p.canon_s_op = p.canon_t_op = p.canon_res_slot = p.canon_res_op = -1;
      p.canon_res_pre = 0;
      auto is = [&](int kind) { return i < n && p.ops[i].kind == kind; };
      if (is(EPI_MUL_C)) { p.canon_s = p.ops[i].c; ++i; }
      else if (is(EPI_MUL_T) && p.ops[i].side == SIDE_COL) { p.canon_s_op = i; ++i; }
      if (is(EPI_ADD_C)) { p.canon_t = p.ops[i].c * (p.canon_s_op < 0 ? 1.f : 1.f); ++i; }
      else if (is(EPI_SUB_C)) { p.canon_t = -p.ops[i].c; ++i; }
      else if (is(EPI_ADD_T) && p.ops[i].side == SIDE_COL) { p.canon_t_op = i; ++i; }
      // residual before the activation (ResNet's relu(bn(conv) + identity)) or after it
      if (is(EPI_ADD_T) && p.ops[i].side == SIDE_MAT) {
        p.canon_res_slot = p.ops[i].slot;
        p.canon_res_op = i;
        p.canon_res_pre = 1;
        ++i;
      }
      if (is(EPI_RELU)) { p.canon_act = 1; ++i; }
      else if (is(EPI_GELU_TANH)) { p.canon_act = 2; ++i; }
      if (p.canon_res_op < 0 && is(EPI_ADD_T) && p.ops[i].side == SIDE_MAT) {
        p.canon_res_slot = p.ops[i].slot;
        p.canon_res_op = i;
        ++i;
      }
      // a residual before "no activation" is the same sum as after it; GELU(x + R)
      // is left to the generic epilogue (the compact drains instantiate ReLU only)
      if (p.canon_res_pre && p.canon_act == 0) p.canon_res_pre = 0;
      const bool pre_ok = !p.canon_res_pre || p.canon_act == 1;
      p.canon = (i == n && pre_ok && !std::getenv("TMB_NO_CANON")) ? 1 : 0;
    }
    {
      const tm_tensor& t = lookup(env, sp.out.tensor);
      Fit f;
      if (!fit_address(sp.out, t, sp.M, sp.N, sp.batch, f, why)) fail_unsupported("output '", sp.out.tensor, "': ", why);
      p.out = t.data;
      p.out_dtype = t.dtype;
      p.out_a = to_addr(f);
      // Row-major (channels-last, [M,N]) outputs: each epilogue warp stages a
      // 32-row x (64 or 128 byte) column group in swizzled smem and TMA-stores
      // it (coalesced, off the LSU).  Outputs whose rows are the contiguous
      // dimension (NCHW) keep direct stores, which are already coalesced (lanes
      // = consecutive pixels).
      const int es = esize(t.dtype);
      const uintptr_t base = reinterpret_cast<uintptr_t>(t.data) + f.off * es;
      if (f.c1 == 1 && f.P >= sp.M && f.lo > 0 && (f.lo * es) % 16 == 0 && (f.c2 * es) % 16 == 0 && base % 16 == 0 &&
          batch_ok(f.c2, f.lo * sp.M, sp.batch) &&
          (t.dtype == TM_BF16 || t.dtype == TM_F32) && !std::getenv("TMB_NO_TMA_STORE")) {
        p.out_tma = 1;
        const uint64_t dims[3] = {(uint64_t)sp.N, (uint64_t)sp.M, (uint64_t)sp.batch};
        const uint64_t strides[2] = {(uint64_t)(f.lo * es), (uint64_t)(std::max<int64_t>(f.c2, f.lo * sp.M) * es)};
        const int rb = out_stage_row_bytes(k.bn, k.cg);
        const uint32_t box[3] = {static_cast<uint32_t>(rb / es), 32u, 1u};
        make_tma_2d3d(k.tma_c, reinterpret_cast<const void*>(base), t.dtype, 3, dims, strides, box, rb);
      }
    }
    {
      // compact instantiation (drain_fast): TMA-fed operands, canonical epilogue,
      // bf16 TMA-stored output, residual absent or bf16 / contiguous / 16-byte
      // aligned rows with N % 32 == 0
      const bool a_t = p.a_loader == LD_TMA_K || p.a_loader == LD_IM2COL_TMA || p.a_loader == LD_IM2COL_TMA8;
      const bool b_t = p.b_loader == LD_TMA_K || p.b_loader == LD_TMA_MN;
      bool res_ok = true;
      if (p.canon && p.canon_res_op >= 0) {
        const EpiOp& r = p.ops[p.canon_res_op];
        const Addr& a = r.a;
        res_ok = r.dtype == DT_BF16 && a.s_col == 1 && p.N % 32 == 0 &&
                 reinterpret_cast<uintptr_t>(r.ptr) % 16 == 0 && (a.s_hi * 2) % 16 == 0 &&
                 (a.s_lo * 2) % 16 == 0 && (a.s_batch * 2) % 16 == 0 && (a.offset * 2) % 16 == 0;
      }
      p.epi_fast = (p.canon && !k.tf32 && p.out_tma && p.out_dtype == DT_BF16 && res_ok &&
                    !std::getenv("TMB_GENERIC"))
                       ? 1
                       : 0;
      k.generic = (a_t && b_t && p.epi_fast) ? 0 : 1;
      // direct register -> global stores for the lean drain: opt-in (TMB_OUT_DIRECT=1); measured
      // slower than smem staging + TMA store on every sweep shape
      {
        const Addr& a = p.out_a;
        p.out_direct = (p.epi_fast && a.s_col == 1 && p.N % 8 == 0 && reinterpret_cast<uintptr_t>(p.out) % 16 == 0 &&
                        (a.s_hi * 2) % 16 == 0 && (a.s_lo * 2) % 16 == 0 && (a.s_batch * 2) % 16 == 0 &&
                        (a.offset * 2) % 16 == 0 && std::getenv("TMB_OUT_DIRECT"))
                           ? 1
                           : 0;
      }
    }
    p.fast_math = p.out_dtype != TM_F32;  // approximate tanh only where the output rounding dominates
    if (bind_rowband(sp, env, k, *ex, want_dt, sms) || (want_halo && bind_halo(sp, env, k, *ex, want_dt, sms))) {
      ex->kernels.push_back(k);
      continue;
    }
    if (const char* sw = std::getenv("TMB_MN_SWAP")) p.mn_lbo_sbo_swap = std::atoi(sw);
    // fault injection for the tuner-gate test (tests/test_gpu_tuner.py): every kernel
    // silently drops its last k-block, so every schedule computes a wrong result
    if (std::getenv("TMB_FAULT_SKIP_KBLOCK") && p.num_kb > 1) {
      p.num_kb -= 1;
      p.K = p.num_kb * BK;
    }
    // split-K: every split gets a non-empty k-block range
    {
      int s = k.simt ? 1 : std::max(1, std::min(plan.cfg.split_k, p.num_kb));
      p.kb_per_split = (p.num_kb + s - 1) / s;
      p.split_k = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
      // fp32 output rows through the lean drain too (identity / ReLU epilogue, no
      // residual, 128-column single-CTA tiles, no split-K): the op-interpreter drain
      // took ~13k clk per 128x128 fp32 tile against ~2k for the lean one
      if (!k.simt && p.out_dtype == DT_F32 && p.canon && p.out_tma && !p.out_direct && p.canon_res_op < 0 &&
          p.canon_act <= 1 && k.cg == 1 && k.bn == 128 && p.split_k == 1 && !std::getenv("TMB_GENERIC") &&
          !std::getenv("TMB_NO_F32_LEAN")) {
        const bool a_t = p.a_loader == LD_TMA_K || p.a_loader == LD_IM2COL_TMA || p.a_loader == LD_IM2COL_TMA8;
        const bool b_t = p.b_loader == LD_TMA_K || p.b_loader == LD_TMA_MN;
        p.epi_fast = 1;
        k.generic = (a_t && b_t && !k.tf32) ? 0 : 1;  // the compact instantiation is bf16/fp16-operand only
      }
      if (p.split_k > 1) {
        const int64_t tiles = int64_t(sp.batch) * p.tiles_m * p.tiles_n * k.cg;
        void* ws = nullptr;
        void* cnt = nullptr;
        if (cudaMalloc(&ws, tiles * p.split_k * 128 * int64_t(k.bn) * 4) != cudaSuccess ||
            cudaMalloc(&cnt, tiles * 8) != cudaSuccess || cudaMemset(cnt, 0, tiles * 8) != cudaSuccess)
          fail_cuda("cudaMalloc failed for the split-K workspace");
        ex->scratch.push_back(ws);
        ex->scratch.push_back(cnt);
        p.workspace = static_cast<float*>(ws);
        p.counters = static_cast<int32_t*>(cnt);
      }
    }
    int grid = plan.cfg.grid > 0 ? std::min(plan.cfg.grid, sms * 4) : sms;
    int used = grid / k.cg;
    p.tile_map = tile_mapping(int64_t(sp.batch) * p.split_k, p.tiles_m, p.tiles_n, grid / k.cg, plan.cfg.raster, used);
    k.grid = used * k.cg;  // workers of the tile mapping are CTA pairs when cg == 2
    // split-K reduction spread over the tile's units when they are all resident
    // (2 or 4 splits: the 8 / split_k reducing warps' slabs, split_k x 32 rows x BN/2
    // fp32 each, fill 8 * 32 * BN/2 * 4 bytes of the idle ring, which must hold them:
    // not the 2-stage double-buffer rings of the wide tiles)
    const int64_t ring_bytes = int64_t(kernel_stages(k)) * (128 + k.bn) * 128;
    p.sk_spin = (p.split_k > 1 && (p.split_k == 2 || p.split_k == 4) && k.cg == 1 && k.bn % 64 == 0 &&
                 p.tile_map.tasks == 1 && int64_t(512) * k.bn <= ring_bytes && !std::getenv("TMB_NO_SK_SPIN"))
                    ? 1
                    : 0;
    // per-worker task lists, decoded once here instead of in every CTA of every launch
    if (p.tile_map.tasks <= 128 && p.tiles_m < 65536 && p.tiles_n < 65536 && !std::getenv("TMB_NO_TILE_TAB")) {
      const uint32_t workers = p.tile_map.workers, tasks = p.tile_map.tasks;
      std::vector<uint32_t> tab(size_t(workers) * tasks * 2, 0u);
      for (uint32_t w = 0; w < workers; ++w)
        for (uint32_t i = 0; i < tasks; ++i) {
          int32_t c[tm::kMaxRank];
          tm::dev_task_fixed<2, 3>(p.tile_map, w, i, c);
          const int b = c[0] / p.split_k, ks = c[0] % p.split_k;
          if (b < p.batch && c[1] < p.tiles_m && c[2] < p.tiles_n) {
            const size_t e = (size_t(w) * tasks + i) * 2;
            tab[e] = static_cast<uint32_t>(c[1]) | (static_cast<uint32_t>(c[2]) << 16);
            tab[e + 1] = (static_cast<uint32_t>(b * p.split_k + ks) << 1) | 1u;
          }
        }
      void* d = nullptr;
      if (cudaMalloc(&d, tab.size() * 4) != cudaSuccess ||
          cudaMemcpy(d, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        fail_cuda("cudaMalloc/cudaMemcpy failed for the tile table");
      ex->scratch.push_back(d);
      p.tile_tab = static_cast<const uint32_t*>(d);
    }
    {
      const int st = kernel_stages(k);
      p.b_resident = (!k.simt && p.tiles_n == 1 && sp.batch == 1 && p.split_k == 1 && p.num_kb <= st &&
                      !std::getenv("TMB_NO_BRES"))
                         ? 1
                         : 0;
      p.ring = p.b_resident ? (st / p.num_kb) * p.num_kb : 0;
    }
    if (const char* d = std::getenv("TMB_DBG")) p.dbg = std::atoi(d);
    if (const char* d = std::getenv("TMB_SKIP")) p.dbg_skip = std::atoi(d);
    if (std::getenv("TMB_TRACE")) {  // per-tile role timeline (tm_exec_trace)
      void* tr = nullptr;
      const size_t bytes = size_t(k.grid) * kTraceTiles * kTraceEvents * 8;
      if (cudaMalloc(&tr, bytes) != cudaSuccess || cudaMemset(tr, 0, bytes) != cudaSuccess)
        fail_cuda("cudaMalloc failed for the trace buffer");
      ex->scratch.push_back(tr);
      p.trace = static_cast<long long*>(tr);
    }
    ex->kernels.push_back(k);
  }
  return ex;
}

}  // namespace tmb
