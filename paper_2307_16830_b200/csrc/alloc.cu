// Device memory for the resident plans (model, KKT, symbolic factor).
//
// Plans are created per solve and dropped with the model, so a process that
// solves case after case would otherwise pay cudaMalloc's page mapping
// (~0.3 ms per array on B200) on every solve.  Freed blocks are kept in a
// per-device cache keyed by rounded size and handed out again; a block goes
// back to the cache only after the device has finished with it (the same
// device-wide synchronisation cudaFree performs), so reuse needs no stream
// bookkeeping.  GN_ALLOC_CACHE=0 disables the cache.
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>

#include "device.cuh"

namespace gn {
namespace {

constexpr size_t kCacheLimit = size_t(8) << 30;   // bytes kept per device

struct Cache {
  std::mutex mu;
  std::multimap<size_t, void *> free_blocks[64];   // per device: rounded size -> block
  size_t cached[64] = {};
  std::unordered_map<void *, std::pair<int, size_t>> live;   // block -> (device, rounded size)
};

Cache &cache() {
  static Cache *c = new Cache;   // never destroyed (frees can run at interpreter exit)
  return *c;
}

bool cache_on() {
  static const bool on = [] {
    const char *e = std::getenv("GN_ALLOC_CACHE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// 4 size classes per power of two above 4 KiB (waste <= 25 %)
size_t round_size(size_t b) {
  if (b <= 4096) return 4096;
  int k = 63 - __builtin_clzll(b - 1);          // 2^k < b <= 2^(k+1)
  const size_t q = size_t(1) << (k - 2);
  return (b + q - 1) / q * q;
}

}  // namespace

void *dev_malloc(size_t bytes) {
  const bool tm = timing_on();
  const double t0 = tm ? host_now() : 0.0;
  void *p = nullptr;
  if (!cache_on()) {
    GN_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
  } else {
    int dev = 0;
    GN_CUDA(cudaGetDevice(&dev));
    GN_REQUIRE(dev >= 0 && dev < 64, "device ordinal out of range");
    const size_t r = round_size(bytes);
    Cache &c = cache();
    {
      std::lock_guard<std::mutex> g(c.mu);
      auto it = c.free_blocks[dev].find(r);
      if (it != c.free_blocks[dev].end()) {
        p = it->second;
        c.free_blocks[dev].erase(it);
        c.cached[dev] -= r;
        c.live[p] = {dev, r};
      }
    }
    if (!p) {
      GN_CUDA(cudaMalloc(&p, r));
      std::lock_guard<std::mutex> g(c.mu);
      c.live[p] = {dev, r};
    }
  }
  if (tm) add_upload_time(host_now() - t0, 0.0);
  return p;
}

void dev_free(void *p) {
  if (!p) return;
  if (!cache_on()) {
    cudaFree(p);
    return;
  }
  Cache &c = cache();
  int dev;
  size_t r;
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return;
    dev = it->second.first;
    r = it->second.second;
    c.live.erase(it);
  }
  // the device must be done with the block before anyone may reuse it
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  const bool ok = cudaDeviceSynchronize() == cudaSuccess;
  bool keep = false;
  if (ok) {
    std::lock_guard<std::mutex> g(c.mu);
    if (c.cached[dev] + r <= kCacheLimit) {
      c.free_blocks[dev].emplace(r, p);
      c.cached[dev] += r;
      keep = true;
    }
  }
  if (!keep) cudaFree(p);
  if (cur != dev) cudaSetDevice(cur);
}

}  // namespace gn
