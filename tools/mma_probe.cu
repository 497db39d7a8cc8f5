// FP64 MMA shape microbenchmark (diagnostics): one warp computes a 32x32
// tile update with K = 32 from shared-memory operands using
// (a) mma.m8n8k4.f64 (16 accumulator tiles x 8 k-steps = 128 MMAs) and
// (b) mma.m16n8k16.f64 (8 accumulator tiles x 2 k-steps = 16 MMAs);
// cycles for the whole update, 1 warp and 4 warps (one per SMSP) per CTA.
#include <cstdio>
__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
__global__ void k884(const double *g, double *out, long long *cyc, int reps) {
  __shared__ double Ps[32 * 40];
  for (int e = threadIdx.x; e < 32 * 40; e += blockDim.x) Ps[e] = g[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[4][4][2] = {};
  const long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
    for (int kk = 0; kk < 32; kk += 4) {
      const int c = kk + (lane & 3);
      double fa[4], fb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        fa[u] = -Ps[c * 40 + u * 8 + (lane >> 2)];
        fb[u] = Ps[c * 40 + u * 8 + (lane >> 2) + 1];
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) mma884(acc[a][b], fa[a], fb[b]);
    }
  const long long t1 = clock64();
  double s = 0;
  for (int a = 0; a < 4; ++a) for (int b = 0; b < 4; ++b) s += acc[a][b][0] + acc[a][b][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
__global__ void k16816(const double *g, double *out, long long *cyc, int reps) {
  __shared__ double Ps[32 * 40];
  for (int e = threadIdx.x; e < 32 * 40; e += blockDim.x) Ps[e] = g[e];
  __syncthreads();
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  double acc[2][4][4] = {};
  const long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep)
    for (int k0 = 0; k0 < 32; k0 += 16) {
      double fa[2][8], fb[4][4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          fa[mi][2 * q] = -Ps[(k0 + tig + 4 * q) * 40 + mi * 16 + gid];
          fa[mi][2 * q + 1] = -Ps[(k0 + tig + 4 * q) * 40 + mi * 16 + gid + 8];
        }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int q = 0; q < 4; ++q) fb[ni][q] = Ps[(k0 + tig + 4 * q) * 40 + ni * 8 + gid + 1];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) mma16816(acc[mi][ni], fa[mi], fb[ni]);
    }
  const long long t1 = clock64();
  double s = 0;
  for (int a = 0; a < 2; ++a) for (int b = 0; b < 4; ++b) for (int q = 0; q < 4; ++q) s += acc[a][b][q];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
int main() {
  double *g, *out; long long *cyc;
  cudaMalloc(&g, 8 * 32 * 40); cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8);
  cudaMemset(g, 0, 8 * 32 * 40);
  for (int warps : {1, 4, 8}) {
    long long c1, c2;
    k884<<<1, 32 * warps>>>(g, out, cyc, 50); cudaMemcpy(&c1, cyc, 8, cudaMemcpyDeviceToHost);
    k16816<<<1, 32 * warps>>>(g, out, cyc, 50); cudaMemcpy(&c2, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%d warp(s)/CTA: 32x32x32 update  m8n8k4 %lld cycles   m16n8k16 %lld cycles  (%s)\n", warps, c1, c2,
           cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
