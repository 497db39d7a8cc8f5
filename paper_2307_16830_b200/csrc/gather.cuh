// Gathered dot products of the sparse KKT / IPM kernels: sum over
// t in [t0, t1) of a[ia(t)] * b[ib(t)], accumulated in ascending t (the
// order of the plain loop, bitwise), with the index and value loads of four
// terms issued before their accumulation -- the gathers' memory latency
// overlaps instead of being paid term by term (rows have ~2-10 terms).
#pragma once

#include <cstdint>

namespace gn {

template <class IA, class IB>
__device__ __forceinline__ void gather4(int64_t t, int64_t t1, const double *__restrict__ a, IA ia,
                                        const double *__restrict__ b, IB ib, double (&va)[4], double (&vb)[4]) {
  int64_t pa[4], pb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const bool ok = t + u < t1;
    pa[u] = ok ? ia(t + u) : 0;
    pb[u] = ok ? ib(t + u) : 0;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const bool ok = t + u < t1;
    va[u] = ok ? a[pa[u]] : 0.0;
    vb[u] = ok ? b[pb[u]] : 0.0;
  }
}

// no contraction: __dadd_rn(acc, __dmul_rn(a, b)) per term
template <class IA, class IB>
__device__ __forceinline__ double gather_dot(int64_t t0, int64_t t1, const double *__restrict__ a, IA ia,
                                             const double *__restrict__ b, IB ib) {
  double acc = 0.0;
  for (int64_t t = t0; t < t1; t += 4) {
    double va[4], vb[4];
    gather4(t, t1, a, ia, b, ib, va, vb);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u < t1) acc = __dadd_rn(acc, __dmul_rn(va[u], vb[u]));
  }
  return acc;
}

// fused: acc = fma(a, b, acc) per term
template <class IA, class IB>
__device__ __forceinline__ double gather_dot_fma(int64_t t0, int64_t t1, const double *__restrict__ a, IA ia,
                                                 const double *__restrict__ b, IB ib) {
  double acc = 0.0;
  for (int64_t t = t0; t < t1; t += 4) {
    double va[4], vb[4];
    gather4(t, t1, a, ia, b, ib, va, vb);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u < t1) acc = fma(va[u], vb[u], acc);
  }
  return acc;
}

}  // namespace gn
