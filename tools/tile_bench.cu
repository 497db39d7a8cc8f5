// Cycle-level microbenchmark of the PANEL diagonal sweep (csrc/chol.cu
// panel_diag) on one 384-thread CTA, warm (repeated) and in isolation.
// Diagnostics only.  Build + run: tools/tile_bench.sh
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_2307_16830_b200/csrc/chol.cu"

namespace gn {
__global__ void __launch_bounds__(kDagThreads, 1) tile_bench_kernel(Plan P, double *F, int s, int reps,
                                                                    long long *fail, int rows, int bg_iters) {
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long bars[kPanelGroups];
  if (threadIdx.x < kPanelGroups) mbar_init(bars + threadIdx.x, 1);
  __syncthreads();
  FrontMeta fm{};
  fm.f_off = 0;
  fm.first = 0;
  fm.ncols = s;
  fm.nrows = s;
  const int warp = threadIdx.x >> 5;
  if (blockIdx.x > 0) {   // background load on the other SMs: DMMA streams
    double acc[2][2][2] = {};
    double fa[2] = {1e-3 * threadIdx.x, 2e-3}, fb[2] = {3e-3, 1e-3 * warp};
    for (int it = 0; it < bg_iters; ++it)
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma884(acc[a][b], fa[a], fb[b]);
    if (acc[0][0][0] == 12345.0) fail[1] = 1;
    return;
  }
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x < 32) panel_diag(P, fm, 0, 32, F + (r & 1) * s * s, smem, bars, fail, r == reps - 1 ? 0 : -1);
    else if (rows && (warp & 3)) {
      const int lw = warp - (warp >> 2) - 1;
      if (lw < rows) panel_rows(fm, 0, 32, 32 * (1 + (lw % (s / 32 - 1))), 32, F + 2 * s * s, smem, bars, r & 1);
    }
    __syncthreads();
  }
}
}  // namespace gn

int main(int argc, char **argv) {
  using namespace gn;
  const int s = 256;
  std::vector<double> h(static_cast<size_t>(2) * s * s);   // two copies of the front
  const char *mode = argc > 1 ? argv[1] : "dd";
  for (int copy = 0; copy < 2; ++copy)
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < s; ++i) {
        double v = (i == j) ? 2.0 * s : 1.0 / (1 + i + j);
        if (mode[0] == 'w') {   // wide dynamic range (IPM-like): D^1/2 A D^1/2, D in [1e-8, 1e10]
          const double di = std::pow(10.0, -8.0 + 18.0 * ((i * 37) % s) / s);
          const double dj = std::pow(10.0, -8.0 + 18.0 * ((j * 37) % s) / s);
          v *= std::sqrt(di * dj);
        }
        if (mode[0] == 't') v *= 1e-300;   // tiny (subnormal products)
        if (mode[0] == 'r') v = 0.0;        // random SPD below
        h[copy * s * s + j * s + i] = v;
      }
  if (mode[0] == 'r') {   // M M^T / s + I, M uniform in [-1, 1] (tools/chol_trace.py dense)
    std::vector<double> M(static_cast<size_t>(s) * s);
    unsigned long long z = 12345;
    for (auto &m : M) {
      z = z * 6364136223846793005ULL + 1442695040888963407ULL;
      m = ((z >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
    }
    for (int j = 0; j < s; ++j)
      for (int i = 0; i < s; ++i) {
        double acc = (i == j) ? 1.0 : 0.0;
        for (int q = 0; q < s; ++q) acc += M[i * s + q] * M[j * s + q] / s;
        h[j * s + i] = h[s * s + j * s + i] = acc;
      }
  }
  double *F;
  long long *fail, *tr;
  cudaMalloc(&F, sizeof(double) * (8 * h.size()));
  cudaMalloc(&fail, 16);
  cudaMalloc(&tr, 8 * 400);
  Plan P{};
  P.dinv_off = 6LL * s * s;
  P.ptrace = tr;
  cudaFuncSetAttribute(tile_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDagSmem);
  for (int grid : {1})
  for (int rows : {0})
  for (int reps : {1, 2, 3, 20}) {
    cudaMemcpy(F, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(F + 2 * s * s, h.data(), sizeof(double) * h.size() / 2, cudaMemcpyHostToDevice);
    tile_bench_kernel<<<grid, kDagThreads, kDagSmem>>>(P, F, s, reps, fail, rows, 400000);
    if (reps == 20 && argc > 2) break;
    cudaError_t e = cudaDeviceSynchronize();
    long long hc[5];
    cudaMemcpy(hc, tr + 5 * 16, 40, cudaMemcpyDeviceToHost);
    printf("grid %d rows %d reps %d (%s): panel_diag phase1 %lld  phase2 %lld  tail %lld cycles\n", grid, rows, reps, cudaGetErrorString(e),
           hc[1] - hc[0], hc[2] - hc[1], hc[3] - hc[2]);
    (void)rows;
  }
  return 0;
}
