// Device memory for the resident plans (model, KKT, symbolic factor).
//
// Plans are created per solve and dropped with the model, so a process that
// solves case after case would otherwise pay cudaMalloc's page mapping
// (~0.3 ms per array on B200) on every solve.  Freed blocks are kept in a
// per-device cache keyed by rounded size and handed out again.
//
// A freed block may still be in use by work queued on any stream, so it is
// first parked on a per-device PENDING list; freeing never synchronises.  An
// allocation that finds no ready block of its size but a pending one waits
// for the device once (one cudaDeviceSynchronize for the whole pending list,
// instead of one per free) and then reuses it.  Concurrent solves on other
// threads are therefore only stalled by an allocation that actually reuses
// memory, never by a teardown.  `gn_alloc_trim` returns every cached block
// to the driver (torch's allocator cannot see this cache; device.py calls it
// on a torch out-of-memory error and from `release_all`).  GN_ALLOC_CACHE=0
// disables the cache.
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "device.cuh"

namespace gn {
namespace {

constexpr size_t kCacheLimit = size_t(8) << 30;   // bytes kept per device (ready + pending)

struct Cache {
  std::mutex mu;
  std::multimap<size_t, void *> ready[64];     // per device: rounded size -> block, device done with it
  std::multimap<size_t, void *> pending[64];   // freed, possibly still referenced by queued work
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

// caller holds c.mu; `dev` is the current device
void *take(Cache &c, int dev, size_t r) {
  auto it = c.ready[dev].find(r);
  if (it == c.ready[dev].end()) return nullptr;
  void *p = it->second;
  c.ready[dev].erase(it);
  c.cached[dev] -= r;
  c.live[p] = {dev, r};
  return p;
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
    bool drain = false;
    {
      std::lock_guard<std::mutex> g(c.mu);
      p = take(c, dev, r);
      drain = !p && c.pending[dev].count(r) > 0;
    }
    if (drain) {
      // a pending block of this size exists: wait for the device once, then
      // every pending block of the device is ready
      GN_CUDA(cudaDeviceSynchronize());
      std::lock_guard<std::mutex> g(c.mu);
      // only blocks parked before the synchronisation are moved (a block
      // freed meanwhile by another thread stays pending)
      for (auto &kv : c.pending[dev]) c.ready[dev].emplace(kv.first, kv.second);
      c.pending[dev].clear();
      p = take(c, dev, r);
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
  bool keep = false;
  {
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return;
    const int dev = it->second.first;
    const size_t r = it->second.second;
    c.live.erase(it);
    if (c.cached[dev] + r <= kCacheLimit) {
      c.pending[dev].emplace(r, p);
      c.cached[dev] += r;
      keep = true;
    }
  }
  if (!keep) cudaFree(p);   // cudaFree itself waits for the device
}

void alloc_trim() {
  if (!cache_on()) return;
  Cache &c = cache();
  std::vector<std::pair<int, void *>> out;
  {
    std::lock_guard<std::mutex> g(c.mu);
    for (int d = 0; d < 64; ++d) {
      for (auto &kv : c.ready[d]) out.emplace_back(d, kv.second);
      for (auto &kv : c.pending[d]) out.emplace_back(d, kv.second);
      c.ready[d].clear();
      c.pending[d].clear();
      c.cached[d] = 0;
    }
  }
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto &dp : out) {
    if (dp.first != cur) cudaSetDevice(dp.first);
    cudaFree(dp.second);
    if (dp.first != cur) cudaSetDevice(cur);
  }
}

}  // namespace gn

extern "C" int gn_alloc_trim(int64_t *cached_bytes_before) {
  return gn::guarded([&] {
    if (cached_bytes_before) {
      gn::Cache &c = gn::cache();
      std::lock_guard<std::mutex> g(c.mu);
      int64_t s = 0;
      for (int d = 0; d < 64; ++d) s += static_cast<int64_t>(c.cached[d]);
      *cached_bytes_before = s;
    }
    gn::alloc_trim();
  });
}
