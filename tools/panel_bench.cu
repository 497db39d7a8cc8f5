// Cycle-level microbenchmark of the dense panel factorisation used by the
// multifrontal kernels (factor_panel in csrc/chol.cu): one CTA factors an
// r x kb SPD panel `reps` times; clock64 probes split phase A (warp 0,
// diagonal block), the barrier, and phase B (row triangular solve).
// Build: see tools/panel_bench.sh.  Diagnostics only.
#include <cstdio>
#include <cstdlib>
#include <vector>
__device__ long long g_probe[16];
// per-thread register accumulators: _pa[k] = cycles since the previous probe
#define GN_PANEL_PROBE_DECL long long _pt = clock64(), _pa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define GN_PANEL_PROBE(k)          \
  do {                             \
    const long long _t = clock64(); \
    _pa[k] += _t - _pt;            \
    _pt = _t;                      \
  } while (0)
#define GN_PANEL_PROBE_END                                                          \
  do {                                                                              \
    if (threadIdx.x == 0)                                                           \
      for (int _i = 0; _i < 8; ++_i) g_probe[_i] += _pa[_i];                        \
    if (threadIdx.x == 32) g_probe[8] += _pa[3];                                     \
  } while (0)
#include "../paper_2307_16830_b200/csrc/chol.cu"

namespace gn {
template <int NB, int R>
__global__ void __launch_bounds__(kThreads, 1)
panel_bench_kernel(const double *A, int r, int kb, int reps, long long *fail, double *out, long long *cyc) {
  extern __shared__ double Ps[];
  __shared__ double s_dinv[NB];
  __shared__ __align__(16) double s_col[NB][NB];
  __shared__ unsigned long long s_bar[NB / gn::kPanelGroup];
  const int ldp = ((r + 15) & ~15) + 8;
  long long tot = 0;
  if (threadIdx.x < NB / kPanelGroup) mbar_init(s_bar + threadIdx.x, 1);
  __syncthreads();
  for (int rep = 0; rep < reps; ++rep) {
    load_panel(Ps, ldp, A, r, r, kb);
    __syncthreads();
    const long long t0 = clock64();
    factor_panel<NB, R>(Ps, ldp, r, kb, s_dinv, s_col, s_bar, rep & 1, fail, 0);
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) cyc[0] = tot / reps;
  for (int e = threadIdx.x; e < r * kb; e += blockDim.x) {
    const int c = e / r, i = e % r;
    out[e] = i >= c ? Ps[c * ldp + i] : 0.0;
  }
}
}  // namespace gn

template <int NB, int R>
static void run(int r, int kb, int reps, int threads = gn::kThreads) {
  std::vector<double> M(size_t(r) * r), A(size_t(r) * kb);
  srand(1);
  for (auto &v : M) v = rand() / double(RAND_MAX) - 0.5;
  for (int c = 0; c < kb; ++c)
    for (int i = 0; i < r; ++i) {
      double s = (i == c) ? r : 0.0;
      for (int t = 0; t < r; ++t) s += M[size_t(i) * r + t] * M[size_t(c) * r + t];
      A[size_t(c) * r + i] = s;
    }
  double *dA, *dO;
  long long *dF, *dC;
  cudaMalloc(&dA, A.size() * 8);
  cudaMalloc(&dO, A.size() * 8);
  cudaMalloc(&dF, 8);
  cudaMalloc(&dC, 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  long long big = 1ll << 62, zero[16] = {};
  cudaMemcpy(dF, &big, 8, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(g_probe, zero, sizeof(zero));
  const int ldp = ((r + 15) & ~15) + 8;
  const size_t smem = size_t(ldp) * NB * 8;
  auto k = gn::panel_bench_kernel<NB, R>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k<<<1, threads, smem>>>(dA, r, kb, reps, dF, dO, dC);
  cudaError_t e = cudaDeviceSynchronize();
  long long cyc = 0, pr[16];
  cudaMemcpy(&cyc, dC, 8, cudaMemcpyDeviceToHost);
  cudaMemcpyFromSymbol(pr, g_probe, sizeof(pr));
  // reference: unblocked Cholesky of the panel (same column order)
  std::vector<double> L(A);
  for (int k2 = 0; k2 < kb; ++k2) {
    double d = std::sqrt(L[size_t(k2) * r + k2]);
    for (int i = k2; i < r; ++i) L[size_t(k2) * r + i] /= d;
    for (int j = k2 + 1; j < kb; ++j)
      for (int i = j; i < r; ++i) L[size_t(j) * r + i] -= L[size_t(k2) * r + i] * L[size_t(k2) * r + j];
  }
  std::vector<double> O(A.size());
  cudaMemcpy(O.data(), dO, O.size() * 8, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int c = 0; c < kb; ++c)
    for (int i = c; i < r; ++i) err = std::max(err, std::abs(O[size_t(c) * r + i] - L[size_t(c) * r + i]));
  printf("threads=%d NB=%d R=%d r=%d kb=%d: %s  %lld cycles/panel  max|err| %.2e\n", threads, NB, R, r, kb,
         cudaGetErrorString(e), cyc, err);
  printf("   warp0: setup %.0f  diagonal block %.0f | warp1 rows %.0f\n", double(pr[0]) / reps, double(pr[1]) / reps,
         double(pr[8]) / reps);
}

int main(int argc, char **argv) {
  const int which = argc > 1 ? atoi(argv[1]) : -1;
  if (which < 0 || which == 0) run<32, 1>(244, 32, 50);
  if (which < 0 || which == 1) run<32, 1>(128, 32, 50);
  if (which < 0 || which == 2) run<16, 2>(400, 16, 50);
  if (which < 0 || which == 3) run<16, 4>(1000, 16, 50);
  if (which == 4) run<32, 1>(32, 32, 50, 32);
  if (which == 5) run<32, 1>(64, 32, 50, 64);
  if (which == 6) run<32, 1>(100, 13, 50);
  if (which == 7) run<16, 3>(700, 7, 50);
  return 0;
}
