// Kernels of the device DAG interpreter (dev_eval.h) and of the tuner's
// correctness gate: seeded verification inputs, node evaluation, and the
// comparison of a tensor program's output with the interpreter's.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../device/dev_eval.h"
#include "../host/dev_eval.hpp"
#include "taskmap/ir.hpp"

namespace tmb {
namespace ev {
namespace {

struct Val {
  double f;
  long long i;
  int isf;
};

__device__ __forceinline__ double as_f(const Val& v) { return v.isf ? v.f : static_cast<double>(v.i); }
__device__ __forceinline__ bool truthy(const Val& v) { return v.isf ? v.f != 0.0 : v.i != 0; }
__device__ __forceinline__ Val fv(double x) { return Val{x, 0, 1}; }
__device__ __forceinline__ Val iv(long long x) { return Val{0.0, x, 0}; }

__device__ __forceinline__ long long floordiv_d(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__device__ __forceinline__ long long floormod_d(long long a, long long b) { return a - floordiv_d(a, b) * b; }

__device__ double load_elem(const TensorRef& t, int64_t off) {
  switch (t.store) {
    case ST_F32: return static_cast<double>(reinterpret_cast<const float*>(t.ptr)[off]);
    case ST_BF16: return static_cast<double>(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(t.ptr)[off]));
    case ST_F16: return static_cast<double>(__half2float(reinterpret_cast<const __half*>(t.ptr)[off]));
    default: return reinterpret_cast<const double*>(t.ptr)[off];
  }
}

// Evaluates a node program; returns false on an evaluation error (the host
// reports it).  `vars` holds the spatial then the reduce coordinates.
__device__ bool run(const NodeJob& j, const long long* vars, Val& out) {
  Val st[kMaxStack];
  int sp = 0;
  int pc = 0;
  while (pc < j.n_code) {
    const Ins in = j.code[pc++];
    switch (in.op) {
      case OP_PUSH_I: st[sp++] = iv(in.i); break;
      case OP_PUSH_F: st[sp++] = fv(in.f); break;
      case OP_VAR: st[sp++] = iv(vars[in.a]); break;
      case OP_LOAD: {
        const TensorRef& t = j.tensors[in.a];
        int64_t off = 0;
        sp -= in.b;
        for (int d = 0; d < in.b; ++d) {
          if (st[sp + d].isf) return false;
          const long long x = st[sp + d].i;
          if (x < 0 || x >= t.shape[d]) return false;  // reference Tensor::flatten bounds check
          off += x * t.stride[d];
        }
        if (t.store == ST_DENSE8 && !t.is_float) {
          st[sp++] = iv(reinterpret_cast<const long long*>(t.ptr)[off]);
        } else {
          const double x = load_elem(t, off);
          st[sp++] = t.is_float ? fv(x) : iv(static_cast<long long>(x));
        }
        break;
      }
      case OP_BIN: {
        const Val y = st[--sp];
        const Val x = st[sp - 1];
        Val r;
        if (x.isf || y.isf) {
          const double a = as_f(x), b = as_f(y);
          switch (in.a) {
            case B_ADD: r = fv(a + b); break;
            case B_SUB: r = fv(a - b); break;
            case B_MUL: r = fv(a * b); break;
            case B_DIV: r = fv(a / b); break;
            case B_MIN: r = fv(fmin(a, b)); break;
            case B_MAX: r = fv(fmax(a, b)); break;
            case B_AND: r = iv(a != 0.0 && b != 0.0); break;
            case B_OR: r = iv(a != 0.0 || b != 0.0); break;
            case B_LT: r = iv(a < b); break;
            case B_LE: r = iv(a <= b); break;
            case B_GT: r = iv(a > b); break;
            case B_GE: r = iv(a >= b); break;
            case B_EQ: r = iv(a == b); break;
            case B_NE: r = iv(a != b); break;
            default: return false;  // float modulo
          }
        } else {
          const long long a = x.i, b = y.i;
          switch (in.a) {
            case B_ADD: r = iv(a + b); break;
            case B_SUB: r = iv(a - b); break;
            case B_MUL: r = iv(a * b); break;
            case B_DIV: if (b == 0) return false; r = iv(floordiv_d(a, b)); break;
            case B_MOD: if (b == 0) return false; r = iv(floormod_d(a, b)); break;
            case B_MIN: r = iv(a < b ? a : b); break;
            case B_MAX: r = iv(a > b ? a : b); break;
            case B_AND: r = iv(a != 0 && b != 0); break;
            case B_OR: r = iv(a != 0 || b != 0); break;
            case B_LT: r = iv(a < b); break;
            case B_LE: r = iv(a <= b); break;
            case B_GT: r = iv(a > b); break;
            case B_GE: r = iv(a >= b); break;
            case B_EQ: r = iv(a == b); break;
            default: r = iv(a != b); break;
          }
        }
        st[sp - 1] = r;
        break;
      }
      case OP_UN: {
        Val& x = st[sp - 1];
        switch (in.a) {
          case U_NEG: x = x.isf ? fv(-x.f) : iv(-x.i); break;
          case U_RELU: x = x.isf ? fv(fmax(x.f, 0.0)) : iv(x.i > 0 ? x.i : 0); break;
          case U_EXP: x = fv(exp(as_f(x))); break;
          case U_SQRT: x = fv(sqrt(as_f(x))); break;
          case U_CASTF: x = fv(as_f(x)); break;
          default: x = x.isf ? iv(static_cast<long long>(x.f)) : x; break;
        }
        break;
      }
      case OP_JZ: {
        const Val c = st[--sp];
        if (!truthy(c)) pc = in.a;
        break;
      }
      case OP_JMP: pc = in.a; break;
      case OP_TABLE: {
        Val& x = st[sp - 1];
        if (x.isf || x.i < 0 || x.i >= in.b) return false;
        x = iv(j.tables[in.a + x.i]);
        break;
      }
      default: return false;
    }
  }
  out = st[0];
  return sp == 1;
}

__device__ __forceinline__ double round_to(double x, int32_t rd) {
  switch (rd) {
    case RD_F32: return static_cast<double>(static_cast<float>(x));
    case RD_BF16: return static_cast<double>(__bfloat162float(__double2bfloat16(x)));
    case RD_F16: return static_cast<double>(__half2float(__double2half(x)));
    default: return x;
  }
}

__global__ void eval_node_kernel(const NodeJob j, int* err) {
  for (int64_t flat = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; flat < j.numel;
       flat += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    long long vars[kMaxVars];
    int64_t rem = flat;
    for (int d = j.n_axes - 1; d >= 0; --d) {  // row-major odometer position
      vars[d] = rem % j.ext[d];
      rem /= j.ext[d];
    }
    Val acc;
    bool ok = true;
    if (!j.reduce) {
      ok = run(j, vars, acc);
    } else {
      // combiner identity (compute_ir.cpp:368-379)
      if (j.combiner == 0) acc = j.is_float ? fv(0.0) : iv(0);
      else if (j.combiner == 1) acc = j.is_float ? fv(-INFINITY) : iv(-2147483648LL);
      else acc = j.is_float ? fv(INFINITY) : iv(2147483647LL);
      for (int d = 0; d < j.n_red; ++d) vars[j.n_axes + d] = 0;
      while (ok) {
        Val x;
        ok = run(j, vars, x);
        if (!ok) break;
        if (acc.isf || x.isf) {
          const double a = as_f(acc), b = as_f(x);
          acc = fv(j.combiner == 0 ? a + b : j.combiner == 1 ? fmax(a, b) : fmin(a, b));
        } else {
          acc = iv(j.combiner == 0 ? acc.i + x.i : j.combiner == 1 ? (acc.i > x.i ? acc.i : x.i) : (acc.i < x.i ? acc.i : x.i));
        }
        int d = j.n_red - 1;  // row-major advance over the reduce axes
        for (; d >= 0; --d) {
          if (++vars[j.n_axes + d] < j.red[d]) break;
          vars[j.n_axes + d] = 0;
        }
        if (d < 0) break;
      }
    }
    if (!ok) {
      atomicExch(err, 1);
      continue;
    }
    if (j.is_float) {
      reinterpret_cast<double*>(j.out)[flat] = round_to(as_f(acc), j.round);
    } else {
      if (acc.isf) atomicExch(err, 2);  // float value stored to an i32 tensor
      reinterpret_cast<long long*>(j.out)[flat] = acc.i;
    }
  }
}

// splitmix64 (the reference Rng's generator, proj/src/tensor.cpp:42-49) keyed
// by (seed, tensor, element)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void store_phys(void* p, int32_t dt, int64_t off, float x) {
  if (dt == TM_F32) reinterpret_cast<float*>(p)[off] = x;
  else if (dt == TM_BF16) reinterpret_cast<__nv_bfloat16*>(p)[off] = __float2bfloat16_rn(x);
  else reinterpret_cast<__half*>(p)[off] = __float2half_rn(x);
}

__global__ void fill_nan_kernel(void* p, int32_t dt, int64_t span) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < span;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (dt == TM_F32) reinterpret_cast<uint32_t*>(p)[i] = 0x7fc00000u;
    else reinterpret_cast<uint16_t*>(p)[i] = dt == TM_BF16 ? 0x7fc0u : 0x7e00u;
  }
}

// logical element -> value: integers U{-8..8} (mode 0, the reference's exact
// test data, tensor.cpp:66) or dyadic k/256, |k| < 256 (mode 1: exact in bf16,
// fp16 and tf32, so the float trial measures accumulation, not input rounding)
__global__ void fill_values_kernel(void* p, int32_t dt, int32_t rank, TensorShape s, uint64_t key, int32_t mode) {
  int64_t numel = 1;
  for (int d = 0; d < rank; ++d) numel *= s.shape[d];
  for (int64_t flat = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; flat < numel;
       flat += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = flat, off = 0;
    for (int d = rank - 1; d >= 0; --d) {
      off += (rem % s.shape[d]) * s.stride[d];
      rem /= s.shape[d];
    }
    const uint64_t r = mix64(key ^ (static_cast<uint64_t>(flat) * 0x2545F4914F6CDD1Dull));
    const float x = mode == 0 ? static_cast<float>(static_cast<int>(r % 17u) - 8)
                              : static_cast<float>(static_cast<int>(r % 511u) - 255) / 256.0f;
    store_phys(p, dt, off, x);
  }
}

__device__ __forceinline__ double ref_value(const void* v, int64_t i, bool is_float) {
  return is_float ? reinterpret_cast<const double*>(v)[i] : static_cast<double>(reinterpret_cast<const long long*>(v)[i]);
}

__global__ void store_kernel(const void* v, bool is_float, int64_t n, void* p, int32_t dt, int32_t rank, TensorShape s) {
  for (int64_t flat = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; flat < n;
       flat += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = flat, off = 0;
    for (int d = rank - 1; d >= 0; --d) {
      off += (rem % s.shape[d]) * s.stride[d];
      rem /= s.shape[d];
    }
    const double x = ref_value(v, flat, is_float);
    if (dt == TM_F32) reinterpret_cast<float*>(p)[off] = static_cast<float>(x);
    else if (dt == TM_BF16) reinterpret_cast<__nv_bfloat16*>(p)[off] = __double2bfloat16(x);
    else reinterpret_cast<__half*>(p)[off] = __double2half(x);
  }
}

__device__ __forceinline__ double phys_value(const void* p, int32_t dt, int64_t off, uint32_t* bits) {
  if (dt == TM_F32) {
    const uint32_t b = reinterpret_cast<const uint32_t*>(p)[off];
    *bits = b;
    return static_cast<double>(__uint_as_float(b));
  }
  const uint16_t b = reinterpret_cast<const uint16_t*>(p)[off];
  *bits = b;
  if (dt == TM_BF16) return static_cast<double>(__uint_as_float(static_cast<uint32_t>(b) << 16));
  __half h;
  *reinterpret_cast<uint16_t*>(&h) = b;
  return static_cast<double>(__half2float(h));
}

__device__ __forceinline__ uint32_t rounded_bits(double x, int32_t dt) {
  if (dt == TM_F32) return __float_as_uint(static_cast<float>(x));
  if (dt == TM_BF16) {
    const __nv_bfloat16 h = __double2bfloat16(x);
    return *reinterpret_cast<const uint16_t*>(&h);
  }
  const __half h = __double2half(x);
  return *reinterpret_cast<const uint16_t*>(&h);
}

__device__ void atomic_max_double(double* a, double v) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(a);
  unsigned long long old = *p;
  while (__longlong_as_double(static_cast<long long>(old)) < v) {
    const unsigned long long prev = atomicCAS(p, old, static_cast<unsigned long long>(__double_as_longlong(v)));
    if (prev == old) break;
    old = prev;
  }
}

__global__ void sumsq_kernel(const void* ref, bool is_float, int64_t n, double* out) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = ref_value(ref, i, is_float);
    s += x * x;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

// out[0] = max error |c - r| / max(1, |r|, scale); out[1] = #elements whose bits
// differ from the reference rounded to the output dtype (as a double)
__global__ void compare_kernel(const void* cand, int32_t dt, int32_t rank, TensorShape s, const void* ref,
                               bool is_float, double scale, double* out) {
  int64_t numel = 1;
  for (int d = 0; d < rank; ++d) numel *= s.shape[d];
  double emax = 0.0;
  double nbad = 0.0;
  for (int64_t flat = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; flat < numel;
       flat += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t rem = flat, off = 0;
    for (int d = rank - 1; d >= 0; --d) {
      off += (rem % s.shape[d]) * s.stride[d];
      rem /= s.shape[d];
    }
    uint32_t bits;
    const double c = phys_value(cand, dt, off, &bits);
    const double r = ref_value(ref, flat, is_float);
    const double den = fmax(1.0, fmax(fabs(r), scale));
    double e = fabs(c - r) / den;
    if (!(e == e)) e = INFINITY;  // NaN: never a match
    emax = fmax(emax, e);
    if (bits != rounded_bits(r, dt)) nbad += 1.0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_double(&out[0], emax);
    if (nbad > 0) atomicAdd(&out[1], nbad);
  }
}

int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return static_cast<int>(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) taskmap::fail_cuda(what, ": ", cudaGetErrorString(e));
}

}  // namespace

void launch_eval_node(const NodeJob& j, int* err, cudaStream_t s) {
  if (j.numel <= 0) return;
  eval_node_kernel<<<grid_for(j.numel), 256, 0, s>>>(j, err);
  check(cudaGetLastError(), "dev_eval node kernel launch");
}

void launch_fill(void* p, int32_t dt, int32_t rank, const TensorShape& s, int64_t span, uint64_t key, int32_t mode,
                 cudaStream_t st) {
  fill_nan_kernel<<<grid_for(span), 256, 0, st>>>(p, dt, span);
  check(cudaGetLastError(), "verification fill kernel launch");
  int64_t numel = 1;
  for (int d = 0; d < rank; ++d) numel *= s.shape[d];
  fill_values_kernel<<<grid_for(numel), 256, 0, st>>>(p, dt, rank, s, key, mode);
  check(cudaGetLastError(), "verification fill kernel launch");
}

void launch_fill_nan(void* p, int32_t dt, int64_t span, cudaStream_t st) {
  if (span <= 0) return;
  fill_nan_kernel<<<grid_for(span), 256, 0, st>>>(p, dt, span);
  check(cudaGetLastError(), "fill kernel launch");
}

void launch_store(const void* v, bool is_float, int64_t n, void* p, int32_t dt, int32_t rank, const TensorShape& s,
                  cudaStream_t st) {
  if (n <= 0) return;
  store_kernel<<<grid_for(n), 256, 0, st>>>(v, is_float, n, p, dt, rank, s);
  check(cudaGetLastError(), "store kernel launch");
}

void launch_compare(const void* cand, int32_t dt, int32_t rank, const TensorShape& s, const void* ref, bool is_float,
                    int64_t n, double* tmp3, double* host3, cudaStream_t st) {
  check(cudaMemsetAsync(tmp3, 0, 3 * sizeof(double), st), "cudaMemsetAsync");
  sumsq_kernel<<<grid_for(n), 256, 0, st>>>(ref, is_float, n, tmp3 + 2);
  check(cudaGetLastError(), "compare kernel launch");
  double h[3];
  check(cudaMemcpyAsync(h, tmp3, 3 * sizeof(double), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
  check(cudaStreamSynchronize(st), "compare synchronize");
  const double scale = n > 0 ? std::sqrt(h[2] / static_cast<double>(n)) : 0.0;
  compare_kernel<<<grid_for(n), 256, 0, st>>>(cand, dt, rank, s, ref, is_float, scale, tmp3);
  check(cudaGetLastError(), "compare kernel launch");
  check(cudaMemcpyAsync(host3, tmp3, 2 * sizeof(double), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
  check(cudaStreamSynchronize(st), "compare synchronize");
  host3[2] = scale;
}

}  // namespace ev
}  // namespace tmb
