// Cycle probe of fwd_diag (csrc/chol.cu) alone and next to other CTAs on
// the same SMs (spinning on a flag, or streaming loads).  Diagnostics only.
#include <cstdio>
#include "../paper_2307_16830_b200/csrc/chol.cu"
namespace gn {
__global__ void fwd_bench_kernel(long long *cyc, double *out, int mode, int *flag, const double *big, size_t nbig) {
  __shared__ double sv[64], M[33 * kLdS + 32], dv[32];
  if (blockIdx.x != 0) {   // neighbours
    if (mode == 1) {
      while (ld_relaxed(flag) == 0) __nanosleep(100);
    } else if (mode == 2) {
      while (ld_acquire(flag) == 0) __nanosleep(20);
    } else if (mode == 3) {
      double acc = 0.0;
      while (ld_relaxed(flag) == 0)
        for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nbig; i += gridDim.x * blockDim.x) acc += __ldg(big + i);
      if (acc == 1.2345) out[1] = acc;
    }
    return;
  }
  const double mval = mode == 4 ? 1e-310 : (mode == 5 ? 1e-160 : 1e-3);
  for (int e = threadIdx.x; e < 32 * kLdS; e += blockDim.x) M[e] = (e % kLdS) > (e / kLdS) ? mval : 0.0;
  if (threadIdx.x < 32) { sv[threadIdx.x] = 1.0; dv[threadIdx.x] = 0.5; }
  __syncthreads();
  __nanosleep(100000);
  long long t0 = 0, t1 = 0;
  for (int r = 0; r < 10; ++r) {
    if (threadIdx.x < 32) {
      t0 = clock64();
      fwd_diag(smem_u32(sv), smem_u32(M), smem_u32(dv), 32);
      t1 = clock64();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = sv[5]; atomicExch(flag, 1); }
}
}
int main() {
  long long *c; double *o, *big; int *flag;
  const size_t nbig = 64 << 20;
  cudaMalloc(&c, 8); cudaMalloc(&o, 16); cudaMalloc(&flag, 4); cudaMalloc(&big, nbig * 8);
  cudaMemset(big, 0, nbig * 8);
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int mode : {0, 4, 5}) {
    cudaMemset(flag, 0, 4);
    const int grid = mode == 0 || mode >= 4 ? 1 : nsm * 6;
    gn::fwd_bench_kernel<<<grid, 256>>>(c, o, mode, flag, big, nbig);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (0 alone, 1 relaxed spinners, 2 acquire spinners, 3 streaming): fwd_diag %lld cycles (%s)\n",
           mode, h, cudaGetErrorString(cudaGetLastError()));
  }
}
