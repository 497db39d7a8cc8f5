// Error reporting and launch/transfer accounting for the C-ABI (gridopf.h).
#include <malloc.h>
#include <omp.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "internal.h"

namespace gn {
// Host heap policy.  The symbolic analysis of every solve builds and drops
// tens of MB of index arrays; with glibc's defaults those large blocks are
// mmap'd and unmapped per call, so every solve pays a fresh page fault per
// 4 KiB (about half of the C3 condensation's time).  Serving them from the
// heap and never trimming it keeps the pages mapped across solves.
// GN_HOST_HEAP_RETAIN=0 keeps the allocator's defaults.
__attribute__((constructor)) static void host_heap_policy() {
  const char *e = std::getenv("GN_HOST_HEAP_RETAIN");
  if (e && e[0] == '0') return;
  mallopt(M_MMAP_MAX, 0);                 // no per-allocation mmap
  mallopt(M_TRIM_THRESHOLD, 1 << 30);     // keep freed heap pages mapped
  mallopt(M_TOP_PAD, 16 << 20);
}

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};
static std::atomic<int64_t> g_h2d{0};
void set_error(const std::string &msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void count_h2d(size_t bytes) { g_h2d.fetch_add(static_cast<int64_t>(bytes), std::memory_order_relaxed); }

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static std::atomic<int64_t> g_malloc_ns{0}, g_copy_ns{0}, g_nalloc{0};
static void print_upload_totals() {
  std::fprintf(stderr, "[gn host] device allocations %lld: malloc %.2f ms, H2D copies %.2f ms\n",
               static_cast<long long>(g_nalloc.load()), 1e-6 * g_malloc_ns.load(), 1e-6 * g_copy_ns.load());
}
bool timing_on() {
  static const bool on = [] {
    const char *e = std::getenv("GN_HOST_TIMING");
    const bool v = e && e[0] == '1';
    if (v) std::atexit(print_upload_totals);
    return v;
  }();
  return on;
}
double host_now() { return now_s(); }
void add_upload_time(double malloc_s, double copy_s) {
  if (malloc_s > 0) g_nalloc.fetch_add(1);
  g_malloc_ns.fetch_add(static_cast<int64_t>(malloc_s * 1e9));
  g_copy_ns.fetch_add(static_cast<int64_t>(copy_s * 1e9));
}
PhaseTimer::PhaseTimer(const char *n) : name(n), t0(timing_on() ? now_s() : 0.0) {}
PhaseTimer::~PhaseTimer() {
  if (timing_on()) std::fprintf(stderr, "[gn host] %-28s %8.2f ms\n", name, 1e3 * (now_s() - t0));
}
}  // namespace gn

extern "C" const char *gn_last_error(void) { return gn::g_last_error.c_str(); }
extern "C" int gn_version(void) { return 1; }

extern "C" int gn_set_host_threads(int k) {
  omp_set_num_threads(k > 0 ? k : omp_get_num_procs());
  return 0;
}

// plan-upload host time (GN_HOST_TIMING=1 only): device allocations and
// their time, H2D copy time; diagnostics
extern "C" void gn_upload_stats(int64_t *n_alloc, double *malloc_ms, double *copy_ms, int reset) {
  if (n_alloc) *n_alloc = gn::g_nalloc.load();
  if (malloc_ms) *malloc_ms = 1e-6 * static_cast<double>(gn::g_malloc_ns.load());
  if (copy_ms) *copy_ms = 1e-6 * static_cast<double>(gn::g_copy_ns.load());
  if (reset) {
    gn::g_nalloc.store(0);
    gn::g_malloc_ns.store(0);
    gn::g_copy_ns.store(0);
  }
}

extern "C" void gn_stats(int64_t *launches, int64_t *h2d_bytes, int reset) {
  if (launches) *launches = gn::g_launches.load();
  if (h2d_bytes) *h2d_bytes = gn::g_h2d.load();
  if (reset) {
    gn::g_launches.store(0);
    gn::g_h2d.store(0);
  }
}
