// Deterministic grid-wide reductions: per-CTA partials reduced by the last
// CTA to finish, in CTA-index order (bitwise reproducible sums; max/min
// exact), no floating-point atomics.
#pragma once

#include <cfloat>

#include "device.cuh"

namespace gn {

enum RedOp : int { RED_SUM = 0, RED_MAX = 1, RED_MIN = 2 };

constexpr int kRedThreads = 256;
constexpr int kRedMaxBlocks = 296;   // 2 CTAs per SM on 148 SMs
constexpr int kRedMaxSlots = 40;

struct RedSpec {
  int k;                      // number of reduced quantities (<= kRedMaxSlots)
  int op[kRedMaxSlots];       // RedOp per slot
  double *out;                // k outputs (device)
  double *partials;           // kRedMaxBlocks * kRedMaxSlots scratch
  unsigned int *counter;      // zero-initialised; reset by the last CTA
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
  if (threadIdx.x < spec.k) {   // one thread per slot combines the warps
    const int k = threadIdx.x;
    double v = sh[k][0];
    for (int w = 1; w < nw; ++w) v = red_combine(spec.op[k], v, sh[k][w]);
    spec.partials[blockIdx.x * kRedMaxSlots + k] = v;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int done = atomicAdd(spec.counter, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = warp; k < spec.k; k += nw) {   // one warp per slot over the CTA partials
    const int op = spec.op[k];
    double v = red_identity(op);
    for (unsigned b = lane; b < gridDim.x; b += 32)
      v = red_combine(op, v, __ldcg(spec.partials + b * kRedMaxSlots + k));
    for (int o = 16; o > 0; o >>= 1) v = red_combine(op, v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) spec.out[k] = v;
  }
  if (threadIdx.x == 0) *spec.counter = 0u;
}

}  // namespace gn
