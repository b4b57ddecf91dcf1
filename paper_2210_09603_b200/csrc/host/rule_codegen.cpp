// Rule / reduce kernel source generation and NVRTC compilation (see
// rule_codegen.hpp).  The generated kernels restate rule_kernels.cu's
// interpreter loops with the program inlined: rule_elem_kernel (grid-stride
// over outputs, reduce axes as a sequential row-major loop) and
// rule_tree_kernel (one CTA per output, strided partials, warp-shuffle and
// shared-memory tree).
#include "rule_codegen.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

namespace tmb {

using namespace taskmap;

namespace {

struct Unsupported {
  std::string why;
};

std::string hex_i64(int64_t v) {
  char b[40];
  std::snprintf(b, sizeof b, "((ix)0x%016" PRIx64 "ULL)", static_cast<uint64_t>(v));
  return b;
}
std::string f32_lit(double v) {
  const float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  char b[40];
  std::snprintf(b, sizeof b, "__int_as_float(0x%08x)", u);
  return b;
}
std::string as_f(const std::string& x, bool isf) { return isf ? x : "((float)(" + x + "))"; }
std::string truthy(const std::string& x, bool isf) { return "(" + x + (isf ? " != 0.f)" : " != 0)"); }
const char* elem_type(int32_t store) { return store == ev::ST_F32 ? "float" : "unsigned short"; }

struct Gen {
  const RuleSourceSpec& s;
  std::map<std::string, int> var_ix;
  std::map<std::string, int> tensor_ix;
  std::ostringstream helpers;
  int n_helpers = 0;

  explicit Gen(const RuleSourceSpec& spec) : s(spec) {
    for (size_t i = 0; i < s.vars.size(); ++i) var_ix[s.vars[i]] = static_cast<int>(i);
    for (size_t i = 0; i < s.tensor_names.size(); ++i) tensor_ix[s.tensor_names[i]] = static_cast<int>(i);
  }

  // A load becomes one helper taking the evaluated indices: bounds check
  // (out of range yields NaN like the interpreter), strided offset with the
  // literal strides, conversion of the storage type to fp32.
  std::string load_helper(int t, size_t rank) {
    const ev::TensorRef& r = s.tensors[t];
    if (static_cast<int>(rank) != r.rank) throw Unsupported{"load rank differs from the bound tensor"};
    const int h = n_helpers++;
    helpers << "__device__ __forceinline__ float ld" << h << "(const Ptrs& P";
    for (size_t d = 0; d < rank; ++d) helpers << ", ix x" << d;
    helpers << ") {\n  if (!(true";
    for (size_t d = 0; d < rank; ++d) helpers << " && x" << d << " >= 0 && x" << d << " < " << r.shape[d];
    helpers << ")) return __int_as_float(0x7fffffff);\n  const ix off = 0";
    for (size_t d = 0; d < rank; ++d) helpers << " + x" << d << " * " << hex_i64(r.stride[d]);
    helpers << ";\n  const " << elem_type(r.store) << "* p = (const " << elem_type(r.store) << "*)P.p[" << t << "];\n";
    if (r.store == ev::ST_F32) helpers << "  return __ldg(p + off);\n";
    else if (r.store == ev::ST_BF16) helpers << "  return bf2f(__ldg(p + off));\n";
    else helpers << "  return h2f(__ldg(p + off));\n";
    helpers << "}\n";
    return "ld" + std::to_string(h);
  }

  std::string table_helper(const std::vector<int64_t>& tab) {
    const int h = n_helpers++;
    helpers << "__device__ const ix tab" << h << "[" << (tab.empty() ? 1 : tab.size()) << "] = {";
    for (size_t i = 0; i < tab.size(); ++i) helpers << (i ? ", " : "") << hex_i64(tab[i]);
    if (tab.empty()) helpers << "0";
    helpers << "};\n__device__ __forceinline__ ix lut" << h << "(ix x) { return (x < 0 || x >= " << tab.size()
            << "LL) ? 0 : tab" << h << "[x]; }\n";
    return "lut" + std::to_string(h);
  }

  // C expression and static type (interpreter promotion rules, rule_kernels.cu run())
  std::string emit(const Expr& e, bool& isf) {
    switch (e->kind) {
      case ExprKind::IntImm: isf = false; return hex_i64(e->ival);
      case ExprKind::FloatImm: isf = true; return f32_lit(e->fval);
      case ExprKind::Var: {
        auto it = var_ix.find(e->name);
        if (it == var_ix.end()) throw Unsupported{"unbound axis " + e->name};
        isf = false;
        return "v" + std::to_string(it->second);
      }
      case ExprKind::ThreadIdx:
      case ExprKind::BlockIdx: throw Unsupported{"thread/block index in a computation"};
      case ExprKind::Binary: {
        bool fa, fb;
        const std::string a = emit(e->args[0], fa), b = emit(e->args[1], fb);
        if (fa || fb) {
          const std::string x = as_f(a, fa), y = as_f(b, fb);
          isf = true;
          switch (e->bop) {
            case BinOp::Add: return "(" + x + " + " + y + ")";
            case BinOp::Sub: return "(" + x + " - " + y + ")";
            case BinOp::Mul: return "(" + x + " * " + y + ")";
            case BinOp::Div: return "(" + x + " / " + y + ")";
            case BinOp::Min: return "fminf(" + x + ", " + y + ")";
            case BinOp::Max: return "fmaxf(" + x + ", " + y + ")";
            case BinOp::Mod: return "__int_as_float(0x7fffffff)";
            default: break;
          }
          isf = false;
          switch (e->bop) {
            case BinOp::And: return "((ix)((" + x + " != 0.f) & (" + y + " != 0.f)))";
            case BinOp::Or: return "((ix)((" + x + " != 0.f) | (" + y + " != 0.f)))";
            case BinOp::Lt: return "((ix)(" + x + " < " + y + "))";
            case BinOp::Le: return "((ix)(" + x + " <= " + y + "))";
            case BinOp::Gt: return "((ix)(" + x + " > " + y + "))";
            case BinOp::Ge: return "((ix)(" + x + " >= " + y + "))";
            case BinOp::Eq: return "((ix)(" + x + " == " + y + "))";
            default: return "((ix)(" + x + " != " + y + "))";
          }
        }
        isf = false;
        switch (e->bop) {
          case BinOp::Add: return "(" + a + " + " + b + ")";
          case BinOp::Sub: return "(" + a + " - " + b + ")";
          case BinOp::Mul: return "(" + a + " * " + b + ")";
          case BinOp::Div: return "ifloordiv(" + a + ", " + b + ")";
          case BinOp::Mod: return "ifloormod(" + a + ", " + b + ")";
          case BinOp::Min: return "imin(" + a + ", " + b + ")";
          case BinOp::Max: return "imax(" + a + ", " + b + ")";
          case BinOp::And: return "((ix)((" + a + " != 0) & (" + b + " != 0)))";
          case BinOp::Or: return "((ix)((" + a + " != 0) | (" + b + " != 0)))";
          case BinOp::Lt: return "((ix)(" + a + " < " + b + "))";
          case BinOp::Le: return "((ix)(" + a + " <= " + b + "))";
          case BinOp::Gt: return "((ix)(" + a + " > " + b + "))";
          case BinOp::Ge: return "((ix)(" + a + " >= " + b + "))";
          case BinOp::Eq: return "((ix)(" + a + " == " + b + "))";
          default: return "((ix)(" + a + " != " + b + "))";
        }
      }
      case ExprKind::Unary: {
        bool fa;
        const std::string a = emit(e->args[0], fa);
        switch (e->uop) {
          case UnOp::Neg: isf = fa; return "(-" + a + ")";
          case UnOp::Relu: isf = fa; return fa ? "fmaxf(" + a + ", 0.f)" : "imax(" + a + ", 0)";
          case UnOp::Exp: isf = true; return "expf(" + as_f(a, fa) + ")";
          case UnOp::Sqrt: isf = true; return "sqrtf(" + as_f(a, fa) + ")";
          case UnOp::CastF32: isf = true; return as_f(a, fa);
          case UnOp::CastI32: isf = false; return fa ? "((ix)(" + a + "))" : a;
        }
        throw Unsupported{"unknown unary op"};
      }
      case ExprKind::Select: {
        bool fc, ft, fe;
        const std::string c = emit(e->args[0], fc), t = emit(e->args[1], ft), f = emit(e->args[2], fe);
        if (ft != fe) throw Unsupported{"select branches of different types"};
        isf = ft;
        return "(" + truthy(c, fc) + " ? " + t + " : " + f + ")";
      }
      case ExprKind::Load: {
        auto it = tensor_ix.find(e->name);
        if (it == tensor_ix.end()) throw Unsupported{"unbound tensor " + e->name};
        std::vector<std::string> idx;
        for (const auto& a : e->args) {
          bool fi;
          idx.push_back(emit(a, fi));
          if (fi) throw Unsupported{"float-valued index"};
        }
        std::string call = load_helper(it->second, idx.size()) + "(P";
        for (const auto& i : idx) call += ", " + i;
        call += ")";
        isf = s.tensors[it->second].is_float != 0;
        return isf ? call : "((ix)" + call + ")";
      }
      case ExprKind::TableLookup: {
        bool fi;
        const std::string x = emit(e->args[0], fi);
        if (fi) throw Unsupported{"float-valued table index"};
        isf = false;
        return table_helper(*e->table) + "(" + x + ")";
      }
    }
    throw Unsupported{"unknown expression kind"};
  }
};

// Interval of every integer-valued subexpression, from the axis extents and the
// literal constants.  When all of them -- and every offset, extent and integer
// accumulation -- fit in 32 bits, the generated code computes indices in `int`
// (half the instructions of 64-bit integer math) with the same results as the
// interpreter's int64.
struct Range {
  bool ok = true;
  __int128 lo = 0, hi = 0;
};
constexpr __int128 kI32Max = 2147483647;
Range mk(__int128 lo, __int128 hi) {
  Range r;
  r.lo = lo;
  r.hi = hi;
  r.ok = lo >= -kI32Max && hi <= kI32Max;
  return r;
}
Range bad() {
  Range r;
  r.ok = false;
  return r;
}

Range int_range(const Expr& e, const RuleSourceSpec& s, const std::map<std::string, int>& var_ix) {
  switch (e->kind) {
    case ExprKind::IntImm: return mk(e->ival, e->ival);
    case ExprKind::FloatImm: return mk(0, 0);  // float: no integer range needed
    case ExprKind::Var: {
      auto it = var_ix.find(e->name);
      if (it == var_ix.end()) return bad();
      const int v = it->second;
      const int nsp = static_cast<int>(s.ext.size());
      const int64_t ext = v < nsp ? s.ext[v] : s.red[v - nsp];
      return mk(0, ext - 1);
    }
    case ExprKind::Load: {
      for (const auto& a : e->args)
        if (!int_range(a, s, var_ix).ok) return bad();
      // an integer tensor's values are data: unbounded; a float load has no integer range
      for (size_t t = 0; t < s.tensor_names.size(); ++t)
        if (s.tensor_names[t] == e->name) return s.tensors[t].is_float ? mk(0, 0) : bad();
      return bad();
    }
    case ExprKind::TableLookup: {
      if (!int_range(e->args[0], s, var_ix).ok) return bad();
      int64_t lo = 0, hi = 0;
      for (int64_t v : *e->table) {
        lo = std::min(lo, v);
        hi = std::max(hi, v);
      }
      return mk(lo, hi);
    }
    case ExprKind::Unary: {
      const Range a = int_range(e->args[0], s, var_ix);
      if (!a.ok) return bad();
      switch (e->uop) {
        case UnOp::Neg: return mk(-a.hi, -a.lo);
        case UnOp::Relu: return mk(a.lo > 0 ? a.lo : 0, a.hi > 0 ? a.hi : 0);
        case UnOp::CastI32: return bad();  // float -> int: unbounded
        default: return mk(0, 0);          // float-valued
      }
    }
    case ExprKind::Select: {
      const Range c = int_range(e->args[0], s, var_ix), t = int_range(e->args[1], s, var_ix),
                  f = int_range(e->args[2], s, var_ix);
      if (!c.ok || !t.ok || !f.ok) return bad();
      return mk(std::min(t.lo, f.lo), std::max(t.hi, f.hi));
    }
    case ExprKind::Binary: {
      const Range a = int_range(e->args[0], s, var_ix), b = int_range(e->args[1], s, var_ix);
      if (!a.ok || !b.ok) return bad();
      switch (e->bop) {
        case BinOp::Add: return mk(a.lo + b.lo, a.hi + b.hi);
        case BinOp::Sub: return mk(a.lo - b.hi, a.hi - b.lo);
        case BinOp::Mul: {
          const __int128 c[4] = {a.lo * b.lo, a.lo * b.hi, a.hi * b.lo, a.hi * b.hi};
          return mk(std::min(std::min(c[0], c[1]), std::min(c[2], c[3])),
                    std::max(std::max(c[0], c[1]), std::max(c[2], c[3])));
        }
        case BinOp::Div:
        case BinOp::Mod: {
          const __int128 m = std::max(a.hi < 0 ? -a.hi : a.hi, a.lo < 0 ? -a.lo : a.lo);
          const __int128 d = std::max(b.hi < 0 ? -b.hi : b.hi, b.lo < 0 ? -b.lo : b.lo);
          return e->bop == BinOp::Div ? mk(-m, m) : mk(-d, d);
        }
        case BinOp::Min: return mk(std::min(a.lo, b.lo), std::min(a.hi, b.hi));
        case BinOp::Max: return mk(std::max(a.lo, b.lo), std::max(a.hi, b.hi));
        default: return mk(0, 1);  // comparisons, logic
      }
    }
    default: return bad();
  }
}

int64_t span_elems(const ev::TensorRef& t) {
  int64_t s = 1;
  for (int d = 0; d < t.rank; ++d) s += (t.shape[d] - 1) * (t.stride[d] < 0 ? -t.stride[d] : t.stride[d]);
  return s;
}

const char* kPrelude = R"(typedef long long i64;
struct Ptrs { const void* p[16]; };
__device__ __forceinline__ float bf2f(unsigned short h) { return __int_as_float(((unsigned)h) << 16); }
__device__ __forceinline__ float h2f(unsigned short h) { float f; asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h)); return f; }
__device__ __forceinline__ unsigned short f2bf(float f) { unsigned short h; asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(h) : "f"(f)); return h; }
__device__ __forceinline__ unsigned short f2h(float f) { unsigned short h; asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(f)); return h; }
__device__ __forceinline__ ix imin(ix a, ix b) { return a < b ? a : b; }
__device__ __forceinline__ ix imax(ix a, ix b) { return a > b ? a : b; }
__device__ __forceinline__ ix ifloordiv(ix a, ix b) {
  if (b == 0) return 0;
  ix q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__device__ __forceinline__ ix ifloormod(ix a, ix b) { return b == 0 ? 0 : a - ifloordiv(a, b) * b; }
)";

// decomposition of `flat` over `dims` = (variable slot, extent), outermost
// first: the last entry varies fastest
void decompose(std::ostringstream& o, const char* flat, const std::vector<std::pair<int, int64_t>>& dims,
               const char* ind) {
  // 32-bit division by the literal extents when the domain fits (mul-hi sequences)
  int64_t total = 1;
  for (const auto& d : dims) total *= d.second;
  const bool narrow = total < (int64_t(1) << 31);
  o << ind << "{\n" << ind << "  " << (narrow ? "unsigned rem = (unsigned)" : "ix rem = ") << flat << ";\n";
  for (int d = static_cast<int>(dims.size()) - 1; d >= 0; --d) {
    if (d == 0) {
      o << ind << "  v" << dims[d].first << " = rem;\n";
    } else {
      o << ind << "  v" << dims[d].first << " = rem % " << dims[d].second << (narrow ? "u" : "LL") << "; rem /= "
        << dims[d].second << (narrow ? "u" : "LL") << ";\n";
    }
  }
  o << ind << "}\n";
}

}  // namespace

bool emit_rule_source(const RuleSourceSpec& s, std::string& src, std::string& why) {
  src.clear();
  if (s.tensors.size() + (s.mode == GEN_SPLIT ? 1 : 0) > static_cast<size_t>(kMaxRuleTensors)) {
    why = "more than " + std::to_string(kMaxRuleTensors) + " tensors";
    return false;
  }
  Gen g(s);
  bool vf;
  std::string val;
  try {
    val = g.emit(s.expr, vf);
  } catch (const Unsupported& u) {
    why = u.why;
    return false;
  }
  const int nsp = static_cast<int>(s.ext.size()), nred = static_cast<int>(s.red.size());
  int64_t numel = 1, red_numel = 1;
  for (auto e : s.ext) numel *= e;
  for (auto e : s.red) red_numel *= e;
  // accumulator type: float when the node or any reduced value is float
  const bool af = nred > 0 ? (s.is_float || vf) : vf;
  const std::string at = af ? "float" : "ix";
  std::string ident, comb_body;
  if (s.combiner == 0) ident = af ? "0.f" : "0LL";
  else if (s.combiner == 1) ident = s.is_float ? "__int_as_float(0xff800000)" : (af ? "(-2147483648.f)" : "(-2147483648LL)");
  else ident = s.is_float ? "__int_as_float(0x7f800000)" : (af ? "2147483647.f" : "2147483647LL");
  if (s.combiner == 0) comb_body = "a + b";
  else if (s.combiner == 1) comb_body = af ? "fmaxf(a, b)" : "imax(a, b)";
  else comb_body = af ? "fminf(a, b)" : "imin(a, b)";

  // 32-bit index arithmetic when every integer value provably fits (see Range)
  bool narrow = numel < (int64_t(1) << 31) && red_numel < (int64_t(1) << 31) && !std::getenv("TMB_RULE_WIDE");
  const Range vr = int_range(s.expr, s, g.var_ix);
  narrow = narrow && vr.ok && span_elems(s.out) < (int64_t(1) << 31);
  for (const auto& t : s.tensors) narrow = narrow && span_elems(t) < (int64_t(1) << 31);
  for (const auto& t : s.tensors)
    for (int d = 0; d < t.rank; ++d) narrow = narrow && t.stride[d] < (int64_t(1) << 31) && t.stride[d] > -(int64_t(1) << 31);
  if (nred > 0 && !af) {  // an integer accumulation: |value| * reduce extent must fit too
    const __int128 m = std::max(vr.hi < 0 ? -vr.hi : vr.hi, vr.lo < 0 ? -vr.lo : vr.lo);
    narrow = narrow && m * red_numel <= kI32Max && red_numel <= kI32Max;
  }
  std::ostringstream o;
  o << (narrow ? "typedef int ix;\n" : "typedef long long ix;\n") << kPrelude;
  o << "__device__ __forceinline__ " << at << " comb(" << at << " a, " << at << " b) { return " << comb_body << "; }\n";
  o << g.helpers.str();
  // output store through the bound strides in the output's storage type
  const ev::TensorRef& out = s.out;
  o << "__device__ __forceinline__ void put(const Ptrs& P, const ix* v, float x) {\n  const ix off = 0";
  for (int d = 0; d < nsp; ++d) o << " + v[" << d << "] * " << hex_i64(out.stride[d]);
  o << ";\n";
  if (out.store == ev::ST_F32) o << "  ((float*)P.p[15])[off] = x;\n";
  else if (out.store == ev::ST_BF16) o << "  ((unsigned short*)P.p[15])[off] = f2bf(x);\n";
  else o << "  ((unsigned short*)P.p[15])[off] = f2h(x);\n";
  o << "}\n";
  const std::string vdecl = "ix v[" + std::to_string(nsp + nred > 0 ? nsp + nred : 1) + "];";
  // the value expression reads v<i>; alias them onto the array
  std::ostringstream alias;
  for (int i = 0; i < nsp + nred; ++i) alias << "#define v" << i << " v[" << i << "]\n";
  o << alias.str();
  const std::string valc = af && !vf ? as_f(val, false) : val;
  // outputs are visited in the output tensor's memory order (axes by decreasing
  // stride), so consecutive threads store -- and, for same-layout inputs such as
  // channels-last pooling, load -- consecutive addresses; values do not depend
  // on the visiting order
  std::vector<std::pair<int, int64_t>> sp_dims, red_dims;
  for (int d = 0; d < nsp; ++d) sp_dims.push_back({d, s.ext[d]});
  std::stable_sort(sp_dims.begin(), sp_dims.end(), [&](const auto& a, const auto& b) {
    const int64_t sa = s.out.stride[a.first] < 0 ? -s.out.stride[a.first] : s.out.stride[a.first];
    const int64_t sb = s.out.stride[b.first] < 0 ? -s.out.stride[b.first] : s.out.stride[b.first];
    return sa > sb;
  });
  for (int d = 0; d < nred; ++d) red_dims.push_back({nsp + d, s.red[d]});
  if (s.mode == GEN_ELEM) {
    o << "extern \"C\" __global__ void __launch_bounds__(256) tmb_rule(const Ptrs P) {\n"
      << "  const i64 step = (i64)gridDim.x * 256;\n"
      << "  for (i64 flat = (i64)blockIdx.x * 256 + threadIdx.x; flat < " << numel << "LL; flat += step) {\n"
      << "    " << vdecl << "\n";
    decompose(o, "flat", sp_dims, "    ");
    if (nred == 0) {
      o << "    const float x = " << as_f(val, vf) << ";\n";
    } else {
      o << "    " << at << " acc = " << ident << ";\n";
      std::string ind = "    ";
      for (int d = 0; d < nred; ++d) {
        o << ind << "for (v" << nsp + d << " = 0; v" << nsp + d << " < " << s.red[d] << "LL; ++v" << nsp + d << ") {\n";
        ind += "  ";
      }
      o << ind << "acc = comb(acc, " << valc << ");\n";
      for (int d = nred - 1; d >= 0; --d) {
        ind.resize(ind.size() - 2);
        o << ind << "}\n";
      }
      o << "    const float x = " << as_f("acc", af) << ";\n";
    }
    o << "    put(P, v, x);\n  }\n}\n";
  } else if (s.mode == GEN_TREE) {
    const int T = s.threads;
    o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") tmb_rule(const Ptrs P) {\n"
      << "  __shared__ " << at << " sh[" << T / 32 << "];\n"
      << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
      << "  for (i64 o = blockIdx.x; o < " << numel << "LL; o += gridDim.x) {\n"
      << "    " << vdecl << "\n";
    decompose(o, "o", sp_dims, "    ");
    o << "    " << at << " acc = " << ident << ";\n"
      << "#pragma unroll 4\n    for (i64 r = threadIdx.x; r < " << red_numel << "LL; r += " << T << ") {\n";
    decompose(o, "r", red_dims, "      ");
    o << "      acc = comb(acc, " << valc << ");\n"
      << "    }\n"
      << "#pragma unroll\n    for (int sft = 16; sft >= 1; sft >>= 1) acc = comb(acc, __shfl_xor_sync(0xffffffffu, acc, sft));\n"
      << "    if (lane == 0) sh[warp] = acc;\n    __syncthreads();\n"
      << "    if (threadIdx.x == 0) {\n      " << at << " t = sh[0];\n"
      << "      for (int w = 1; w < " << T / 32 << "; ++w) t = comb(t, sh[w]);\n"
      << "      put(P, v, " << as_f("t", af) << ");\n    }\n    __syncthreads();\n  }\n}\n";
  } else if (s.mode == GEN_GROUP) {
    const int G = s.group, per = 256 / G;
    o << "extern \"C\" __global__ void __launch_bounds__(256) tmb_rule(const Ptrs P) {\n"
      << "  const int g = threadIdx.x & " << G - 1 << ";\n"
      << "  const i64 gid = threadIdx.x / " << G << ";\n"
      << "  for (i64 base = (i64)blockIdx.x * " << per << "; base < " << numel << "LL; base += (i64)gridDim.x * " << per
      << ") {\n"
      << "    const i64 o = base + gid;\n"
      << "    " << vdecl << "\n"
      << "    " << at << " acc = " << ident << ";\n"
      << "    if (o < " << numel << "LL) {\n";
    decompose(o, "o", sp_dims, "      ");
    o << "#pragma unroll 4\n      for (i64 r = g; r < " << red_numel << "LL; r += " << G << ") {\n";
    decompose(o, "r", red_dims, "        ");
    o << "        acc = comb(acc, " << valc << ");\n      }\n    }\n";
    if (G > 1)
      o << "#pragma unroll\n    for (int sft = " << G / 2
        << "; sft >= 1; sft >>= 1) acc = comb(acc, __shfl_xor_sync(0xffffffffu, acc, sft));\n";
    o << "    if (g == 0 && o < " << numel << "LL) put(P, v, " << as_f("acc", af) << ");\n  }\n}\n";
  } else {
    const int T = s.threads, S = s.splits;
    const int slot = static_cast<int>(s.tensors.size());
    const int64_t chunk = (red_numel + S - 1) / S;
    o << "extern \"C\" __global__ void __launch_bounds__(" << T << ") tmb_rule(const Ptrs P) {\n"
      << "  __shared__ " << at << " sh[" << T / 32 << "];\n"
      << "  __shared__ int last;\n"
      << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
      << "  " << at << "* part = (" << at << "*)P.p[" << slot << "];\n"
      << "  unsigned* ticket = (unsigned*)(part + " << numel * S << "LL);\n"
      << "  const i64 o = blockIdx.x / " << S << ";\n"
      << "  const int sidx = blockIdx.x % " << S << ";\n"
      << "  " << vdecl << "\n";
    decompose(o, "o", sp_dims, "  ");
    o << "  " << at << " acc = " << ident << ";\n"
      << "  const i64 lo = (i64)sidx * " << chunk << "LL;\n"
      << "  const i64 hi = lo + " << chunk << "LL < " << red_numel << "LL ? lo + " << chunk << "LL : " << red_numel
      << "LL;\n"
      << "#pragma unroll 4\n  for (i64 r = lo + threadIdx.x; r < hi; r += " << T << ") {\n";
    decompose(o, "r", red_dims, "    ");
    o << "    acc = comb(acc, " << valc << ");\n  }\n"
      << "#pragma unroll\n  for (int sft = 16; sft >= 1; sft >>= 1) acc = comb(acc, __shfl_xor_sync(0xffffffffu, acc, sft));\n"
      << "  if (lane == 0) sh[warp] = acc;\n  __syncthreads();\n"
      << "  if (threadIdx.x == 0) {\n    " << at << " t = sh[0];\n"
      << "    for (int w = 1; w < " << T / 32 << "; ++w) t = comb(t, sh[w]);\n"
      << "    part[o * " << S << " + sidx] = t;\n    __threadfence();\n"
      << "    last = atomicAdd(ticket + o, 1u) == " << S - 1 << "u;\n  }\n  __syncthreads();\n"
      << "  if (last && threadIdx.x == 0) {\n    __threadfence();\n"
      << "    const volatile " << at << "* pv = part + o * " << S << ";\n"
      << "    " << at << " u = pv[0];\n"
      << "    for (int k = 1; k < " << S << "; ++k) u = comb(u, pv[k]);\n"
      << "    put(P, v, " << as_f("u", af) << ");\n    ticket[o] = 0u;\n  }\n}\n";
  }
  src = o.str();
  return true;
}

namespace {

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  std::string error;
};

const Nvrtc& nvrtc() {
  static const Nvrtc lib = [] {
    Nvrtc n;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) {
      n.error = "libnvrtc.so.12 not found";
      return n;
    }
    n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
    n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
    n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    n.log_size = reinterpret_cast<decltype(n.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    if (!n.create || !n.compile || !n.cubin_size || !n.cubin || !n.log_size || !n.log || !n.destroy)
      n.error = "libnvrtc lacks the CUBIN entry points";
    return n;
  }();
  return lib;
}

template <class F>
F drv(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess) return nullptr;
  return reinterpret_cast<F>(fn);
}

using ModuleLoadData = CUresult (*)(CUmodule*, const void*);
using ModuleGetFunction = CUresult (*)(CUfunction*, CUmodule, const char*);
using LaunchKernel = CUresult (*)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                  CUstream, void**, void**);

}  // namespace

// compile to CUBIN for the current device's "a" target; the CUBIN is cached
// per (architecture, source) and loaded once per device
void* compile_rule_source(const std::string& src, std::string& why) {
  static std::mutex mu;
  static std::map<std::string, std::vector<char>> cubins;
  static std::map<std::pair<int, std::string>, CUfunction> fns;
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess) {
    why = "no CUDA device";
    return nullptr;
  }
  const std::string arch = "--gpu-architecture=sm_" + std::to_string(major * 10 + minor) + "a";
  std::lock_guard<std::mutex> lock(mu);
  auto fit = fns.find({dev, src});
  if (fit != fns.end()) return fit->second;
  const std::string key = arch + "\n" + src;
  auto cit = cubins.find(key);
  if (cit == cubins.end()) {
    const Nvrtc& n = nvrtc();
    if (!n.error.empty()) {
      why = n.error;
      return nullptr;
    }
    nvrtcProgram prog;
    if (n.create(&prog, src.c_str(), "tmb_rule.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
      why = "nvrtcCreateProgram failed";
      return nullptr;
    }
    const char* opts[] = {arch.c_str(), "--fmad=false", "--std=c++17", "-default-device"};
    const nvrtcResult r = n.compile(prog, 4, opts);
    if (r != NVRTC_SUCCESS) {
      size_t ls = 0;
      n.log_size(prog, &ls);
      std::string log(ls, '\0');
      if (ls) n.log(prog, log.data());
      why = "NVRTC compile failed: " + log;
      n.destroy(&prog);
      return nullptr;
    }
    size_t sz = 0;
    n.cubin_size(prog, &sz);
    std::vector<char> bin(sz);
    n.cubin(prog, bin.data());
    n.destroy(&prog);
    cit = cubins.emplace(key, std::move(bin)).first;
  }
  static const auto load = drv<ModuleLoadData>("cuModuleLoadData");
  static const auto getf = drv<ModuleGetFunction>("cuModuleGetFunction");
  if (!load || !getf) {
    why = "driver module entry points unavailable";
    return nullptr;
  }
  CUmodule mod;
  CUfunction fn;
  if (load(&mod, cit->second.data()) != CUDA_SUCCESS || getf(&fn, mod, "tmb_rule") != CUDA_SUCCESS) {
    why = "cuModuleLoadData / cuModuleGetFunction failed";
    return nullptr;
  }
  fns[{dev, src}] = fn;
  return fn;
}

void launch_rule_compiled(void* fn, const RulePtrs& ptrs, unsigned grid, unsigned block, void* stream) {
  static const auto launch = drv<LaunchKernel>("cuLaunchKernel");
  if (!launch) fail_cuda("cuLaunchKernel entry point unavailable");
  RulePtrs p = ptrs;
  void* args[] = {&p};
  const CUresult r = launch(static_cast<CUfunction>(fn), grid, 1, 1, block, 1, 1, 0, static_cast<CUstream>(stream),
                            args, nullptr);
  if (r != CUDA_SUCCESS) fail_cuda("cuLaunchKernel of a generated rule kernel failed with CUresult ", static_cast<int>(r));
}

}  // namespace tmb
