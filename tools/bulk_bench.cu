// Panel-load microbenchmark (diagnostics): one CTA of 256 threads copies a
// 32-column x r-row panel of a column-major front (ld s) from global memory
// (L2-resident: written just before by another CTA) into shared memory,
// (a) ld.global.cg, 32 per thread in flight, (b) cp.async.bulk per column
// (16-byte aligned columns), completion on an mbarrier.  Prints cycles.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned su32(const void *p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ double ldcg(const double *p) { double v; asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }

__global__ void writer(double *F, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) F[i] = i * 0.5;
}

__global__ void __launch_bounds__(256, 1) bench(const double *F, int s, int r, int kb, int ldp, long long *cyc, double *sink, int mode) {
  extern __shared__ __align__(16) double Ps[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  __syncthreads();
  long long best = 1ll << 60;
  for (int rep = 0; rep < 20; ++rep) {
    __syncthreads();
    const long long t0 = clock64();
    if (mode == 0) {
      const int tot = kb * r;
      for (int e0 = threadIdx.x; e0 < tot; e0 += 32 * 256) {
        double v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int e = e0 + q * 256;
          const int c = e / r, i = e - c * r;
          v[q] = e < tot ? ldcg(F + (long long)c * s + i) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int e = e0 + q * 256;
          const int c = e / r, i = e - c * r;
          if (e < tot) Ps[c * ldp + i] = v[q];
        }
      }
      __syncthreads();
    } else {
      const unsigned bytes = r * 8u;
      if (threadIdx.x == 0)
        asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(su32(&bar)), "r"(bytes * kb) : "memory");
      __syncthreads();
      if (threadIdx.x < kb) {
        const int c = threadIdx.x;
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(Ps + c * ldp)), "l"(F + (long long)c * s), "r"(bytes), "r"(su32(&bar)) : "memory");
      }
      asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)), "r"(rep & 1) : "memory");
      __syncthreads();
    }
    const long long t1 = clock64();
    best = min(best, t1 - t0);
  }
  if (threadIdx.x == 0) { cyc[0] = best; sink[0] = Ps[5 * ldp + 7]; }
}

int main() {
  const int s = 256, r = 244, kb = 32, ldp = 264;
  double *F, *sink; long long *cyc;
  cudaMalloc(&F, sizeof(double) * s * s * 4);
  cudaMalloc(&sink, 8); cudaMalloc(&cyc, 8);
  for (int mode = 0; mode < 2; ++mode) {
    writer<<<148, 256>>>(F, s * s * 4);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, ldp * 32 * 8);
    bench<<<1, 256, ldp * 32 * 8>>>(F + 16, s, r, kb, ldp, cyc, sink, mode);
    cudaError_t e = cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %s  %lld cycles for %d KB\n", mode, mode ? "bulk" : "ld.cg", cudaGetErrorString(e), c, r * kb * 8 / 1024);
  }
  return 0;
}
