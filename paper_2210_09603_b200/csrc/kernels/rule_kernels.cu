// Rule-based (injective) and reduce-template kernels of the product
// (device/rule.h): the bytecode of a fused anchor-free subgraph, evaluated in
// fp32 / int64 and stored through the bound output's strides.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "../device/rule.h"
#include "../host/plan.hpp"

namespace tmb {
namespace {

using ev::Ins;
using ev::TensorRef;

struct RVal {
  float f;
  long long i;
  int isf;
};

__device__ __forceinline__ float as_f(const RVal& v) { return v.isf ? v.f : static_cast<float>(v.i); }
__device__ __forceinline__ bool truthy(const RVal& v) { return v.isf ? v.f != 0.f : v.i != 0; }
__device__ __forceinline__ RVal fv(float x) { return RVal{x, 0, 1}; }
__device__ __forceinline__ RVal iv(long long x) { return RVal{0.f, x, 0}; }

__device__ __forceinline__ long long floordiv_r(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

__device__ __forceinline__ float load_f(const TensorRef& t, int64_t off) {
  switch (t.store) {
    case ev::ST_F32: return __ldg(reinterpret_cast<const float*>(t.ptr) + off);
    case ev::ST_BF16: return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(t.ptr)[off]);
    default: return __half2float(reinterpret_cast<const __half*>(t.ptr)[off]);
  }
}

// Runs the program at coordinates `vars` (spatial, then reduce).  A failed
// evaluation (out-of-bounds load, integer division by zero -- which a valid
// DAG's guards exclude) yields NaN.
__device__ RVal run(const RuleJob& j, const long long* vars) {
  RVal st[ev::kMaxStack];
  int sp = 0, pc = 0;
  while (pc < j.n_code) {
    const Ins in = j.code[pc++];
    switch (in.op) {
      case ev::OP_PUSH_I: st[sp++] = iv(in.i); break;
      case ev::OP_PUSH_F: st[sp++] = fv(static_cast<float>(in.f)); break;
      case ev::OP_VAR: st[sp++] = iv(vars[in.a]); break;
      case ev::OP_LOAD: {
        const TensorRef& t = j.tensors[in.a];
        int64_t off = 0;
        sp -= in.b;
        bool ok = true;
        for (int d = 0; d < in.b; ++d) {
          const long long x = st[sp + d].isf ? -1 : st[sp + d].i;
          ok = ok && x >= 0 && x < t.shape[d];
          off += x * t.stride[d];
        }
        if (!ok) return fv(__int_as_float(0x7fffffff));
        const float x = load_f(t, off);
        st[sp++] = t.is_float ? fv(x) : iv(static_cast<long long>(x));
        break;
      }
      case ev::OP_BIN: {
        const RVal y = st[--sp];
        const RVal x = st[sp - 1];
        RVal r;
        if (x.isf || y.isf) {
          const float a = as_f(x), b = as_f(y);
          switch (in.a) {
            case ev::B_ADD: r = fv(a + b); break;
            case ev::B_SUB: r = fv(a - b); break;
            case ev::B_MUL: r = fv(a * b); break;
            case ev::B_DIV: r = fv(a / b); break;
            case ev::B_MIN: r = fv(fminf(a, b)); break;
            case ev::B_MAX: r = fv(fmaxf(a, b)); break;
            case ev::B_AND: r = iv(a != 0.f && b != 0.f); break;
            case ev::B_OR: r = iv(a != 0.f || b != 0.f); break;
            case ev::B_LT: r = iv(a < b); break;
            case ev::B_LE: r = iv(a <= b); break;
            case ev::B_GT: r = iv(a > b); break;
            case ev::B_GE: r = iv(a >= b); break;
            case ev::B_EQ: r = iv(a == b); break;
            case ev::B_NE: r = iv(a != b); break;
            default: r = fv(__int_as_float(0x7fffffff)); break;  // float modulo
          }
        } else {
          const long long a = x.i, b = y.i;
          switch (in.a) {
            case ev::B_ADD: r = iv(a + b); break;
            case ev::B_SUB: r = iv(a - b); break;
            case ev::B_MUL: r = iv(a * b); break;
            case ev::B_DIV: r = b == 0 ? fv(__int_as_float(0x7fffffff)) : iv(floordiv_r(a, b)); break;
            case ev::B_MOD: r = b == 0 ? fv(__int_as_float(0x7fffffff)) : iv(a - floordiv_r(a, b) * b); break;
            case ev::B_MIN: r = iv(a < b ? a : b); break;
            case ev::B_MAX: r = iv(a > b ? a : b); break;
            case ev::B_AND: r = iv(a != 0 && b != 0); break;
            case ev::B_OR: r = iv(a != 0 || b != 0); break;
            case ev::B_LT: r = iv(a < b); break;
            case ev::B_LE: r = iv(a <= b); break;
            case ev::B_GT: r = iv(a > b); break;
            case ev::B_GE: r = iv(a >= b); break;
            case ev::B_EQ: r = iv(a == b); break;
            default: r = iv(a != b); break;
          }
        }
        st[sp - 1] = r;
        break;
      }
      case ev::OP_UN: {
        RVal& x = st[sp - 1];
        switch (in.a) {
          case ev::U_NEG: x = x.isf ? fv(-x.f) : iv(-x.i); break;
          case ev::U_RELU: x = x.isf ? fv(fmaxf(x.f, 0.f)) : iv(x.i > 0 ? x.i : 0); break;
          case ev::U_EXP: x = fv(expf(as_f(x))); break;
          case ev::U_SQRT: x = fv(sqrtf(as_f(x))); break;
          case ev::U_CASTF: x = fv(as_f(x)); break;
          default: x = x.isf ? iv(static_cast<long long>(x.f)) : x; break;
        }
        break;
      }
      case ev::OP_JZ: {
        const RVal c = st[--sp];
        if (!truthy(c)) pc = in.a;
        break;
      }
      case ev::OP_JMP: pc = in.a; break;
      case ev::OP_TABLE: {
        RVal& x = st[sp - 1];
        x = (x.isf || x.i < 0 || x.i >= in.b) ? fv(__int_as_float(0x7fffffff)) : iv(j.tables[in.a + x.i]);
        break;
      }
      default: return fv(__int_as_float(0x7fffffff));
    }
  }
  return st[0];
}

// combiner identity (compute_ir.cpp:368-379) and fold (:381-396)
__device__ __forceinline__ RVal identity(const RuleJob& j) {
  if (j.combiner == 0) return j.is_float ? fv(0.f) : iv(0);
  if (j.combiner == 1) return j.is_float ? fv(-INFINITY) : iv(-2147483648LL);
  return j.is_float ? fv(INFINITY) : iv(2147483647LL);
}
__device__ __forceinline__ RVal combine(const RuleJob& j, const RVal& a, const RVal& b) {
  if (a.isf || b.isf) {
    const float x = as_f(a), y = as_f(b);
    return fv(j.combiner == 0 ? x + y : j.combiner == 1 ? fmaxf(x, y) : fminf(x, y));
  }
  return iv(j.combiner == 0 ? a.i + b.i : j.combiner == 1 ? (a.i > b.i ? a.i : b.i) : (a.i < b.i ? a.i : b.i));
}

__device__ __forceinline__ void spatial_vars(const RuleJob& j, int64_t flat, long long* vars) {
  for (int d = j.n_axes - 1; d >= 0; --d) {  // row-major odometer position
    vars[d] = flat % j.ext[d];
    flat /= j.ext[d];
  }
}

__device__ __forceinline__ void store(const RuleJob& j, const long long* vars, const RVal& v) {
  int64_t off = 0;
  for (int d = 0; d < j.n_axes; ++d) off += vars[d] * j.out.stride[d];
  const float x = as_f(v);
  switch (j.out.store) {
    case ev::ST_F32: reinterpret_cast<float*>(const_cast<void*>(j.out.ptr))[off] = x; break;
    case ev::ST_BF16: reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(j.out.ptr))[off] = __float2bfloat16_rn(x); break;
    default: reinterpret_cast<__half*>(const_cast<void*>(j.out.ptr))[off] = __float2half_rn(x); break;
  }
}

// rule_based_schedule: spatial(grid * block) over output elements, reduce axes
// (extent <= the host's inline limit) as a sequential loop
__global__ void __launch_bounds__(256) rule_elem_kernel(const RuleJob j) {
  for (int64_t flat = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; flat < j.numel;
       flat += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    long long vars[ev::kMaxVars];
    spatial_vars(j, flat, vars);
    RVal acc;
    if (j.n_red == 0) {
      acc = run(j, vars);
    } else {
      acc = identity(j);
      for (int d = 0; d < j.n_red; ++d) vars[j.n_axes + d] = 0;
      for (int64_t r = 0; r < j.red_numel; ++r) {
        acc = combine(j, acc, run(j, vars));
        for (int d = j.n_red - 1; d >= 0; --d) {  // row-major advance over the reduce axes
          if (++vars[j.n_axes + d] < j.red[d]) break;
          vars[j.n_axes + d] = 0;
        }
      }
    }
    store(j, vars, acc);
  }
}

// reduce_template: one CTA per output element, block-level tree reduction
template <int THREADS>
__global__ void __launch_bounds__(THREADS) rule_tree_kernel(const RuleJob j) {
  __shared__ float sf[THREADS / 32];
  __shared__ long long si[THREADS / 32];
  __shared__ int sflt[THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t o = blockIdx.x; o < j.numel; o += gridDim.x) {
    long long vars[ev::kMaxVars];
    spatial_vars(j, o, vars);
    RVal acc = identity(j);
    for (int64_t r = threadIdx.x; r < j.red_numel; r += THREADS) {
      int64_t rem = r;
      for (int d = j.n_red - 1; d >= 0; --d) {
        vars[j.n_axes + d] = rem % j.red[d];
        rem /= j.red[d];
      }
      acc = combine(j, acc, run(j, vars));
    }
    // warp tree, then across warps
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      RVal other;
      other.f = __shfl_xor_sync(0xffffffffu, acc.f, s);
      other.i = __shfl_xor_sync(0xffffffffu, acc.i, s);
      other.isf = __shfl_xor_sync(0xffffffffu, acc.isf, s);
      acc = combine(j, acc, other);
    }
    if (lane == 0) {
      sf[warp] = acc.f;
      si[warp] = acc.i;
      sflt[warp] = acc.isf;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      RVal t = RVal{sf[0], si[0], sflt[0]};
      for (int w = 1; w < THREADS / 32; ++w) t = combine(j, t, RVal{sf[w], si[w], sflt[w]});
      store(j, vars, t);
    }
    __syncthreads();
  }
}

}  // namespace

void rule_launch_shape(const RuleJob& j, int threads, int sms, unsigned* grid, unsigned* block) {
  if (j.mode == RULE_TREE) {
    const int64_t g = j.numel < int64_t(sms) * 16 ? j.numel : int64_t(sms) * 16;
    *grid = static_cast<unsigned>(g > 0 ? g : 1);
    // CTA width: the largest of 64/128/256/512 not above threads_per_block
    *block = threads >= 512 ? 512 : threads >= 256 ? 256 : threads >= 128 ? 128 : 64;
  } else {
    const int64_t want = (j.numel + 255) / 256;
    const int64_t g = want < int64_t(sms) * 8 ? want : int64_t(sms) * 8;
    *grid = static_cast<unsigned>(g > 0 ? g : 1);
    *block = 256;
  }
}

void launch_rule(const RuleJob& j, int threads, int sms, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned grid, block;
  rule_launch_shape(j, threads, sms, &grid, &block);
  if (j.mode == RULE_TREE) {
    if (block == 512) rule_tree_kernel<512><<<grid, 512, 0, s>>>(j);
    else if (block == 256) rule_tree_kernel<256><<<grid, 256, 0, s>>>(j);
    else if (block == 128) rule_tree_kernel<128><<<grid, 128, 0, s>>>(j);
    else rule_tree_kernel<64><<<grid, 64, 0, s>>>(j);
  } else {
    rule_elem_kernel<<<grid, block, 0, s>>>(j);
  }
}

}  // namespace tmb
