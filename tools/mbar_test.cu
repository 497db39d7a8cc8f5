#include <cstdio>
__device__ __forceinline__ unsigned smem_u32(const void *p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait_phase0(unsigned long long *b) {
  asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], 0;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__global__ void k(int *out) {
  __shared__ unsigned long long bar[32];
  __shared__ int val[32];
  for (int rep = 0; rep < 3; ++rep) {
    if (threadIdx.x < 32) mbar_init(bar + threadIdx.x, 1);
    __syncthreads();
    if (threadIdx.x < 32) {
      for (int kk = 0; kk < 32; ++kk) {
        if (threadIdx.x == 0) { val[kk] = kk + rep; }
        __syncwarp();
        if (threadIdx.x == 0) mbar_arrive(bar + kk);
      }
    } else {
      int s = 0;
      for (int kk = 0; kk < 32; ++kk) { mbar_wait_phase0(bar + kk); s += val[kk]; }
      if (threadIdx.x == 32) out[rep] = s;
    }
    __syncthreads();
  }
}
int main() {
  int *d; cudaMalloc(&d, 16);
  k<<<1, 256>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  int h[3]; cudaMemcpy(h, d, 12, cudaMemcpyDeviceToHost);
  printf("%s %d %d %d\n", cudaGetErrorString(e), h[0], h[1], h[2]);
}
