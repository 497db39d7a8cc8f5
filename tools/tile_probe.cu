// Microbenchmark of one trailing-update tile (diagnostics): the DMMA strip
// tile of chol.cu's trailing_update (mode 1) on one warp, with the tile's
// values in L2 (written by another kernel) and the panel in shared memory;
// clock64 around the whole call, best of 20 (each rep rewrites the tile).
#include <cstdio>
#include "../paper_2307_16830_b200/csrc/chol.cu"

namespace gn {
__global__ void writer(double *F, int n, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) F[i] = v + i * 1e-9;
}
__global__ void __launch_bounds__(kThreads, 1) tile_kernel(double *F, int ld, int r, int kb, int ntiles_warps, long long *cyc) {
  extern __shared__ double Ps[];
  const int ldp = ((r + 15) & ~15) + 8;
  for (int e = threadIdx.x; e < kb * ldp; e += blockDim.x) Ps[e] = 1e-3 * (e % 97);
  __syncthreads();
  const long long t0 = clock64();
  // warps [0, ntiles_warps) each take one strip tile
  if ((threadIdx.x >> 5) < ntiles_warps) trailing_update(Ps, ldp, F, ld, r, kb, threadIdx.x >> 5, 1 << 20, 1);
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
}  // namespace gn

int main() {
  const int s = 244, ld = 244, kb = 32;
  double *F; long long *cyc;
  cudaMalloc(&F, sizeof(double) * ld * s);
  cudaMalloc(&cyc, 8);
  const int ldp = ((s + 15) & ~15) + 8;
  cudaFuncSetAttribute(gn::tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ldp * kb * 8);
  for (int nw : {1, 7}) {
    long long best = 1ll << 60;
    for (int rep = 0; rep < 20; ++rep) {
      gn::writer<<<148, 256>>>(F, ld * s, rep);
      gn::tile_kernel<<<1, gn::kThreads, ldp * kb * 8>>>(F, ld, s, kb, nw, cyc);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      best = c < best ? c : best;
    }
    printf("%d strip tile(s) on %d warp(s): %lld cycles (%s)\n", nw, nw, best, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
