// FP64 FMA issue throughput per SM (diagnostics): W warps x 16 independent chains.
#include <cstdio>
__global__ void tput(double *out, long long *cyc, double a, double b) {
  double y[16];
  for (int j = 0; j < 16; ++j) y[j] = a + threadIdx.x + j;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) y[j] = fma(y[j], b, a);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  double x = 0;
  for (int j = 0; j < 16; ++j) x += y[j];
  out[threadIdx.x] = x;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
  for (int w : {1, 2, 4, 8, 16, 32}) {
    tput<<<1, 32 * w>>>(o, c, 1e-3, 0.999);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double instr = 256.0 * 16 * w;
    printf("warps %2d: %.2f cycles per warp-DFMA per SM  (%.1f FMA/clk/SM)\n", w, h / instr, 32 * instr / h);
  }
}
