// Task mappings lowered to device index arithmetic.
//
// Two forms of the paper's repeat/spatial algebra (Hidet §5.1, reference
// proj/src/mapping.cpp:46-99 for the atoms and :155-188 for assign):
//
//  * compile-time:  Repeat<...>, Spatial<...>, Compose<A, B> types whose
//    task(w, i, coord) is a constexpr closed form, used for the fixed
//    thread/warp mappings inside kernels (e.g. the paper's CUDA-core mapping
//    spatial(4,2)*repeat(2,2)*spatial(4,8)*repeat(4,4) in the SIMT kernel).
//  * run-time:      DevMapping, a flattened chain of up to kMaxAtoms atoms,
//    used for the persistent CTA -> tile scheduler whose shape depends on
//    the problem size.
//
// Both follow the closed form of assign() for chains of atoms:
//   split the worker id mixed-radix over the spatial atoms (leftmost most
//   significant), split the task ordinal mixed-radix over the repeat atoms
//   (leftmost = outermost loop), and combine coordinates as
//   coord[d] = sum_a c_a[d] * prod_{b right of a} dims_b[d].
// (compose(f1,f2): t = t1 (.) d2 + t2, t1 outer — mapping.cpp:169-185.)
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#define TMB_HD
#define TMB_UNROLL
#else
#define TMB_HD __host__ __device__
#define TMB_UNROLL _Pragma("unroll")
#endif

namespace tmb {
namespace tm {

// ------------------------------------------------------------ compile time --
template <int... D>
struct Dims {
  static constexpr int rank = sizeof...(D);
  // extent of dimension i (a function, not a static array: usable in device code)
  TMB_HD static constexpr int get(int i) {
    int k = 0, r = 1;
    ((k++ == i ? (r = D, 0) : 0), ...);
    return r;
  }
  TMB_HD static constexpr int volume() { return (1 * ... * D); }
};

// row-major unlinearisation of `flat` over D
template <class D>
TMB_HD constexpr void unflatten(uint32_t flat, int* out) {
  for (int i = D::rank - 1; i >= 0; --i) {
    out[i] = static_cast<int>(flat % static_cast<uint32_t>(D::get(i)));
    flat /= static_cast<uint32_t>(D::get(i));
  }
}

template <int... D>
struct Repeat {
  using dims_t = Dims<D...>;
  static constexpr int rank = dims_t::rank;
  static constexpr uint32_t workers = 1;
  static constexpr uint32_t tasks = dims_t::volume();
  TMB_HD static constexpr int dim(int i) { return dims_t::get(i); }
  TMB_HD static constexpr void task(uint32_t /*w*/, uint32_t i, int* coord) {
    unflatten<dims_t>(i, coord);
  }
};

template <int... D>
struct Spatial {
  using dims_t = Dims<D...>;
  static constexpr int rank = dims_t::rank;
  static constexpr uint32_t workers = dims_t::volume();
  static constexpr uint32_t tasks = 1;
  TMB_HD static constexpr int dim(int i) { return dims_t::get(i); }
  TMB_HD static constexpr void task(uint32_t w, uint32_t /*i*/, int* coord) {
    unflatten<dims_t>(w, coord);
  }
};

template <class F1, class F2>
struct Compose {
  static_assert(F1::rank == F2::rank, "composed task mappings need equal task dimension");
  static constexpr int rank = F1::rank;
  static constexpr uint32_t workers = F1::workers * F2::workers;
  static constexpr uint32_t tasks = F1::tasks * F2::tasks;
  TMB_HD static constexpr int dim(int i) { return F1::dim(i) * F2::dim(i); }
  TMB_HD static constexpr void task(uint32_t w, uint32_t i, int* coord) {
    int c1[rank] = {}, c2[rank] = {};
    F1::task(w / F2::workers, i / F2::tasks, c1);
    F2::task(w % F2::workers, i % F2::tasks, c2);
    for (int d = 0; d < rank; ++d) coord[d] = c1[d] * F2::dim(d) + c2[d];
  }
};

// Left-associative chain helper: Chain<A, B, C> == Compose<Compose<A, B>, C>.
template <class F, class... Rest>
struct ChainImpl {
  using type = F;
};
template <class F, class G, class... Rest>
struct ChainImpl<F, G, Rest...> {
  using type = typename ChainImpl<Compose<F, G>, Rest...>::type;
};
template <class... F>
using Chain = typename ChainImpl<F...>::type;

// --------------------------------------------------------------- run time --
constexpr int kMaxAtoms = 6;
constexpr int kMaxRank = 3;

struct DevMapping {
  int32_t n_atoms;
  int32_t rank;
  int32_t is_spatial[kMaxAtoms];
  int32_t dims[kMaxAtoms][kMaxRank];
  uint32_t workers;  // product of spatial atom volumes
  uint32_t tasks;    // product of repeat atom volumes
  int32_t shape[kMaxRank];
};

// Task `i` (0 <= i < tasks) of worker `w` (0 <= w < workers).
TMB_HD inline void dev_task(const DevMapping& m, uint32_t w, uint32_t i, int32_t* coord) {
  int32_t scale[kMaxRank];
  for (int d = 0; d < m.rank; ++d) {
    coord[d] = 0;
    scale[d] = 1;
  }
  for (int a = m.n_atoms - 1; a >= 0; --a) {
    uint32_t vol = 1;
    for (int d = 0; d < m.rank; ++d) vol *= static_cast<uint32_t>(m.dims[a][d]);
    uint32_t flat;
    if (m.is_spatial[a]) {
      flat = w % vol;
      w /= vol;
    } else {
      flat = i % vol;
      i /= vol;
    }
    for (int d = m.rank - 1; d >= 0; --d) {
      const uint32_t e = static_cast<uint32_t>(m.dims[a][d]);
      coord[d] += static_cast<int32_t>(flat % e) * scale[d];
      flat /= e;
      scale[d] *= static_cast<int32_t>(e);
    }
  }
}

// dev_task for a chain whose atom count and rank are known at compile time
// (the kernels' CTA -> tile mapping is always 2 atoms over rank 3): fully
// unrolled, ~20 instructions per division instead of the generic loop nest,
// which keeps the per-tile scheduler out of the instruction-cache budget.
template <int NA, int R>
TMB_HD inline void dev_task_fixed(const DevMapping& m, uint32_t w, uint32_t i, int32_t* coord) {
  int32_t scale[R];
TMB_UNROLL
  for (int d = 0; d < R; ++d) {
    coord[d] = 0;
    scale[d] = 1;
  }
TMB_UNROLL
  for (int a = NA - 1; a >= 0; --a) {
    uint32_t vol = 1;
TMB_UNROLL
    for (int d = 0; d < R; ++d) vol *= static_cast<uint32_t>(m.dims[a][d]);
    uint32_t flat;
    if (m.is_spatial[a]) {
      flat = w % vol;
      w /= vol;
    } else {
      flat = i % vol;
      i /= vol;
    }
TMB_UNROLL
    for (int d = R - 1; d >= 0; --d) {
      const uint32_t e = static_cast<uint32_t>(m.dims[a][d]);
      const uint32_t q = flat / e;
      coord[d] += static_cast<int32_t>(flat - q * e) * scale[d];
      flat = q;
      scale[d] *= static_cast<int32_t>(e);
    }
  }
}

}  // namespace tm
}  // namespace tmb
