// Deterministic grid-wide reductions: per-CTA partials reduced by the last
// CTA to finish, in CTA-index order (bitwise reproducible sums; max/min
// exact), no floating-point atomics.
#pragma once

#include <cfloat>

#include "device.cuh"

namespace gn {

enum RedOp : int { RED_SUM = 0, RED_MAX = 1, RED_MIN = 2 };

constexpr int kRedThreads = 256;
// 8 CTAs per SM on 148 SMs: the fused IPM kernels gather (Aᵀy, A·dx) per
// element, so memory-level parallelism, not the partials, sets their time
constexpr int kRedMaxBlocks = 1184;
constexpr int kRedMaxSlots = 40;
static_assert(GN_RED_PARTIALS == kRedMaxBlocks * kRedMaxSlots, "gridopf.h GN_RED_PARTIALS out of date");

// Batched launches reduce every instance (blockIdx.y) separately: its CTA
// partials at partials + (y * gridDim.x + blockIdx.x) * kRedMaxSlots, its
// counter at counter[y], its outputs at out + y * out_stride.
struct RedSpec {
  int k;                      // number of reduced quantities (<= kRedMaxSlots)
  int op[kRedMaxSlots];       // RedOp per slot
  double *out;                // k outputs (device)
  double *partials;           // gridDim.y * gridDim.x * kRedMaxSlots scratch
  unsigned int *counter;      // gridDim.y counters, zero-initialised; reset by the last CTA
  int64_t out_stride;         // between instances' outputs
};

__device__ __forceinline__ double red_identity(int op) {
  return op == RED_SUM ? 0.0 : (op == RED_MAX ? -DBL_MAX : DBL_MAX);
}

__device__ __forceinline__ double red_combine(int op, double a, double b) {
  if (op == RED_SUM) return a + b;
  if (a != a) return a;  // NaN propagates like numpy's max/min
  if (b != b) return b;
  if (op == RED_MAX) return b > a ? b : a;
  return b < a ? b : a;
}

inline int red_grid(int64_t n, int per_thread = 1) {
  int64_t g = (n + static_cast<int64_t>(kRedThreads) * per_thread - 1) / (kRedThreads * per_thread);
  if (g < 1) g = 1;
  if (g > kRedMaxBlocks) g = kRedMaxBlocks;
  return static_cast<int>(g);
}

// Reduce vals[0..spec.k) held by every thread of the grid (blockDim ==
// kRedThreads); the last CTA to finish writes spec.out.  Must be reached by
// all threads of every CTA.  Every combine happens in a fixed position (lane
// strides and shuffle trees), so results are bitwise run-to-run identical.
template <int K>
__device__ void grid_reduce(const RedSpec &spec, double (&vals)[K]) {
  __shared__ double sh[K][kRedThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (k >= spec.k) break;
    double v = vals[k];
    for (int o = 16; o > 0; o >>= 1) v = red_combine(spec.op[k], v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) sh[k][warp] = v;
  }
  __syncthreads();
  const int64_t inst = blockIdx.y;
  double *partials = spec.partials + inst * gridDim.x * kRedMaxSlots;
  unsigned int *counter = spec.counter + inst;
  if (threadIdx.x < spec.k) {   // one thread per slot combines the warps
    const int k = threadIdx.x;
    double v = sh[k][0];
    for (int w = 1; w < nw; ++w) v = red_combine(spec.op[k], v, sh[k][w]);
    partials[blockIdx.x * kRedMaxSlots + k] = v;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int done = atomicAdd(counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double *out = spec.out + inst * spec.out_stride;
  for (int k = warp; k < spec.k; k += nw) {   // one warp per slot over the CTA partials
    const int op = spec.op[k];
    double v = red_identity(op);
    for (unsigned b0 = lane; b0 < gridDim.x; b0 += 32 * 8) {   // 8 loads in flight, same order
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned b = b0 + 32u * u;
        t[u] = b < gridDim.x ? __ldcg(partials + b * kRedMaxSlots + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b0 + 32u * u < gridDim.x) v = red_combine(op, v, t[u]);
    }
    for (int o = 16; o > 0; o >>= 1) v = red_combine(op, v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) out[k] = v;
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// ------------------------------------------------------------- batching
// Instance batches (K12): B independent problems of one sparsity pattern,
// vectors stored instance-major ([B][n], [B][m], [B][nnzH], [B][nnzJ]),
// kernels launched with gridDim.y = B.  The per-instance scalar operands
// live in a device array bp[B][GN_BP_STRIDE] (gridopf.h); bp == nullptr is
// the single-instance call (scalars passed by value, blockIdx.y == 0).
struct Bx {
  const double *bp;
  int64_t n, m, nh, nj;
};

__device__ __forceinline__ double bpar(const Bx &x, int k, double dflt) {
  return x.bp ? x.bp[blockIdx.y * GN_BP_STRIDE + k] : dflt;
}
__device__ __forceinline__ bool b_active(const Bx &x) {
  return !x.bp || x.bp[blockIdx.y * GN_BP_STRIDE + GN_BP_ACTIVE] != 0.0;
}
__device__ __forceinline__ void shift(gn_kkt_state &s, const Bx &x) {
  const int64_t b = blockIdx.y;
  if (b == 0 && !x.bp) return;
  s.w += b * x.nh;
  s.a += b * x.nj;
  s.dxl += b * x.n;
  s.dxu += b * x.n;
  s.zxl += b * x.n;
  s.zxu += b * x.n;
  s.sx += b * x.n;
  s.dsl += b * x.m;
  s.dsu += b * x.m;
  s.zsl += b * x.m;
  s.zsu += b * x.m;
  s.ss += b * x.m;
  if (x.bp) {
    s.dw = x.bp[b * GN_BP_STRIDE + GN_BP_DW];
    s.dc = x.bp[b * GN_BP_STRIDE + GN_BP_DC];
  }
}
__device__ __forceinline__ void shift(gn_vec7 &v, const Bx &x) {
  const int64_t b = blockIdx.y;
  if (b == 0) return;
  v.x += b * x.n;
  v.zxl += b * x.n;
  v.zxu += b * x.n;
  v.s += b * x.m;
  v.y += b * x.m;
  v.zsl += b * x.m;
  v.zsu += b * x.m;
}
__device__ __forceinline__ void shift(gn_ipm_vecs &v, const Bx &x) {
  const int64_t b = blockIdx.y;
  if (b == 0) return;
  const int64_t n = b * x.n, m = b * x.m;
  v.x += n; v.zxl += n; v.zxu += n; v.xl += n; v.xu += n; v.dxl += n; v.dxu += n; v.sx += n;
  v.grad += n; v.dual_x += n;
  v.s += m; v.y += m; v.zsl += m; v.zsu += m; v.sl += m; v.su += m; v.dsl += m; v.dsu += m;
  v.ss += m; v.c += m; v.dual_s += m; v.primal += m;
  v.jac += b * x.nj;
}
template <class T>
__device__ __forceinline__ T *shift_ptr(T *p, int64_t len) {
  return p ? p + static_cast<int64_t>(blockIdx.y) * len : p;
}

}  // namespace gn
