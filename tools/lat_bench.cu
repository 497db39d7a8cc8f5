// Latency probes for the panel-factor building blocks (diagnostics).
#include <cstdio>
__global__ void lat(double *out, long long *cyc, double a, double b) {
  __shared__ double sm[64];
  double x = a + threadIdx.x;
  long long t0, t1;
  // dependent DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, b, a);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // dependent DMUL chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = x * b;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // rsqrt chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = rsqrt(x) + a;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // shfl chain (double)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + a;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // STS -> syncwarp -> LDS chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    sm[threadIdx.x] = x;
    __syncwarp();
    x = sm[(threadIdx.x + 1) & 31] + a;
    __syncwarp();
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  // DFMA throughput: 8 independent chains
  double y[8];
  for (int j = 0; j < 8; ++j) y[j] = x + j;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) y[j] = fma(y[j], b, a);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0);
  for (int j = 0; j < 8; ++j) x += y[j];
  out[threadIdx.x] = x;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
  for (int w : {32, 128, 256}) {
    lat<<<1, w>>>(o, c, 1e-3, 0.999);
    cudaDeviceSynchronize();
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("threads %d: dfma %.1f dmul %.1f rsqrt+add %.1f shfl+add %.1f sts-sync-lds+add %.1f  dfma x8 indep %.1f cycles/iter\n",
           w, h[0] / 1e3, h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3, h[5] / 1e3);
  }
  return 0;
}
