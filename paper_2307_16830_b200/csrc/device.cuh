// Device-side helpers shared by the CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "internal.h"

namespace gn {

#define GN_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      throw ::gn::Error(std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define GN_LAUNCH_CHECK() GN_CUDA(cudaGetLastError())

// kernel launch + error check + launch accounting (gn_stats)
#define GN_LAUNCH(kern, grid, block, smem, st, ...)     \
  do {                                                  \
    kern<<<grid, block, smem, st>>>(__VA_ARGS__);       \
    ::gn::count_launch();                               \
    GN_CUDA(cudaGetLastError());                        \
  } while (0)

void count_launch();
void count_h2d(size_t bytes);
bool timing_on();
double host_now();
void add_upload_time(double malloc_s, double copy_s);

void *dev_malloc(size_t bytes);   // cached device allocation (alloc.cu)
void dev_free(void *p);
void alloc_trim();               // return cached blocks to the driver

template <class T, class A>
T *dev_upload(const std::vector<T, A> &v) {
  T *p = static_cast<T *>(dev_malloc(sizeof(T) * (v.empty() ? 1 : v.size())));
  const bool tm = timing_on();
  const double t0 = tm ? host_now() : 0.0;
  if (!v.empty()) GN_CUDA(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  if (tm) add_upload_time(0.0, host_now() - t0);
  count_h2d(sizeof(T) * v.size());
  return p;
}

template <class T>
T *dev_alloc(size_t count) {
  return static_cast<T *>(dev_malloc(sizeof(T) * (count ? count : 1)));
}

template <class D, class S, class A>
uvec<D> narrow(const std::vector<S, A> &v) {
  uvec<D> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = static_cast<D>(v[i]);
  return out;
}


inline int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 1;
}

// L2-coherent load for data produced by another CTA of the same launch.
template <class T>
__device__ __forceinline__ T ld_cg(const T *p) {
  return __ldcg(p);
}

__device__ __forceinline__ int ld_volatile(const int *p) {
  return *reinterpret_cast<const volatile int *>(p);
}

}  // namespace gn
