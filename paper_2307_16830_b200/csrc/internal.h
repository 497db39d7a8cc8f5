// Internal definitions shared by the host symbolic code and the CUDA kernels.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <mutex>
#include <memory>
#include <utility>
#include <vector>

#include "../../include/gridopf.h"

namespace gn {
// std::allocator that default-initialises: resize() of a uvec leaves
// trivial elements unwritten (the host analysis fills its big index arrays
// itself; zero-filling them first cost a serial memset per solve)
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U> &) noexcept {}
  template <class U, class... A>
  void construct(U *p, A &&...a) {
    if constexpr (sizeof...(A) == 0)
      ::new (static_cast<void *>(p)) U;
    else
      ::new (static_cast<void *>(p)) U(std::forward<A>(a)...);
  }
};
template <class T>
using uvec = std::vector<T, NoInitAlloc<T>>;
}  // namespace gn

namespace gn {

// Sorted unique 64-bit keys (LSD radix sort for large inputs).
inline void sort_unique(std::vector<uint64_t> &k) {
  // LSD radix sort on 64-bit keys (8 passes of 8 bits would be slow for small
  // inputs; use std::sort below 1M keys).
  if (k.size() < (1u << 20)) {
    std::sort(k.begin(), k.end());
  } else {
    std::vector<uint64_t> tmp(k.size());
    for (int shift = 0; shift < 64; shift += 16) {
      std::vector<size_t> cnt(65537, 0);
      for (uint64_t v : k) cnt[((v >> shift) & 0xFFFF) + 1]++;
      for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
      for (uint64_t v : k) tmp[cnt[(v >> shift) & 0xFFFF]++] = v;
      k.swap(tmp);
    }
  }
  k.erase(std::unique(k.begin(), k.end()), k.end());
}


void set_error(const std::string &msg);

// GN_HOST_TIMING=1 prints the duration of instrumented host phases (stderr)
struct PhaseTimer {
  const char *name;
  double t0;
  explicit PhaseTimer(const char *n);
  ~PhaseTimer();
};

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define GN_REQUIRE(cond, msg)                         \
  do {                                                \
    if (!(cond)) throw ::gn::Error(std::string(msg)); \
  } while (0)

// Guard for extern "C" entry points: C++ exceptions never cross the ABI.
template <class F>
int guarded(F &&f) {
  try {
    f();
    return 0;
  } catch (const std::exception &e) {
    set_error(e.what());
    return -1;
  } catch (...) {
    set_error("unknown error");
    return -1;
  }
}

constexpr int kMaxTape = 64;   // device INTERPRETER: tape entries per instruction
constexpr int kMaxSlots = 16;  // device INTERPRETER: variable slots per record
// the generated pattern kernels (ad_codegen.cpp) keep a tape's values in
// registers / local memory and have no structural limit; these bound the
// generated source size only
constexpr int kMaxTapeGen = 4096;
constexpr int kMaxSlotsGen = 256;

// ---------------------------------------------------------------- AD plan
struct DevBlock {                // one pattern block as seen by the device
  int32_t kind;                  // 0 obj, 1 define, 2 increment
  int32_t nv, np, T, out;
  int32_t nfirst, npairs, nsweep, nconst;
  int64_t R;
  int64_t var_off, par_off, tgt_off;   // into SoA record arrays
  int64_t contrib_off;                 // [value | first slots | pairs] x R
  int32_t tape_off, const_off;         // into the tape pools
  int32_t slot_off;                    // into the small per-block int pool
  int32_t spec;                        // specialised kernel id, 0 = interpreter
  int64_t cta_begin;                   // first CTA of this block in the record launch
};

struct Model {
  int64_t n = 0, m = 0;
  // host copies of the blocks (canonical order)
  struct HBlock {
    int32_t kind, nv, np, out;
    int64_t R;
    std::vector<int64_t> var_idx;  // row-major R x nv
    std::vector<double> params;    // row-major R x np
    std::vector<int64_t> targets;
    std::vector<int32_t> ops;      // T x 3
    std::vector<double> consts;
    std::vector<int32_t> first, pairs, grad_order;
  };
  std::vector<HBlock> blocks;
  std::vector<int64_t> jac_rows, jac_cols, hess_rows, hess_cols;
  std::vector<int64_t> jac_slots, hess_slots;  // concatenated (see gridopf.h)
  std::vector<double> hess_factor;
  int64_t n_contrib = 0;
  // gather plans over contribution ids (CSR)
  std::vector<int64_t> c_ptr, grad_ptr, jac_ptr, hess_ptr;
  std::vector<int64_t> c_src, grad_src, jac_src, hess_src;
  std::vector<int64_t> obj_src;  // objective value contributions, block order
  std::vector<int64_t> obj_block_ptr;
  // device
  bool uploaded = false;
  std::vector<DevBlock> dblocks;
  int64_t n_ctas_rec = 0;
  void *pattern_fn = nullptr;        // NVRTC-compiled pattern kernel (nullptr: interpreter)
  void *d_genblk = nullptr;          // its per-block table (device)
  std::string pattern_error;         // why the interpreter is used, if it is
  bool jac_direct = false;           // every J slot has exactly one contribution
  bool needs_patterns = false;       // a tape / slot count beyond the interpreter's limits
  int batch_cap = 0;                 // instances the objective scratch holds
  int64_t n_params = 0;              // device parameter layout size (doubles)
  struct Dev {
    DevBlock *blocks = nullptr;
    int32_t *tape = nullptr;  // int4-packed (op, a, b, 0)
    double *consts = nullptr;
    int32_t *slots = nullptr;  // per block: first[], pair a/b[], sweep[], grad_order[]
    int32_t *var_idx = nullptr;  // SoA int32
    double *params = nullptr;    // SoA
    int32_t *targets = nullptr;
    int64_t *c_ptr = nullptr, *grad_ptr = nullptr, *jac_ptr = nullptr, *hess_ptr = nullptr;
    int32_t *c_src = nullptr, *grad_src = nullptr, *jac_src = nullptr, *hess_src = nullptr;
    int32_t *obj_src = nullptr;
    int32_t *jac_rows = nullptr;
    int64_t *obj_block_ptr = nullptr;
    int32_t n_obj_blocks = 0;
    int32_t *jslots = nullptr;       // Jacobian slot per constraint contribution (direct writes)
    double *obj_partials = nullptr;  // objective reduction scratch
    unsigned *obj_counter = nullptr;
    long long *bstrides = nullptr;   // batched strides (x, y/cs, contrib, params, jac)
    long long *bstrides_shared = nullptr;   // same with shared parameters
  } d;
  ~Model();
};

// --------------------------------------------------------- condensation
struct Condense {
  int64_t n = 0, nnz_h = 0, nnz_j = 0, np = 0;
  std::vector<int64_t> indptr;
  uvec<int64_t> indices;
  // K slot of every coordinate, in input order: the nnz_h W entries
  // (w_map), the n diagonal entries (diag_map), the np A^T A products
  // (ata_map) -- the reference's three maps as slices of one array
  uvec<int64_t> slot;
  // Jacobian row segments: start, product offset (np.tril_indices order),
  // constraint row; one trailing entry
  std::vector<int64_t> seg, seg_poff, seg_row;
  uvec<int32_t> k_ptr, k_row, k_s1, k_s2;   // products grouped by K slot
  // the Jacobian by column (entries ascending): A^T's CSR, reused by the KKT plan
  std::vector<int64_t> a_colptr;
  uvec<int32_t> a_colent;
  bool plan_built = false;
  std::mutex plan_mu;
  void ensure_assembly_plan();
  int64_t w_map(int64_t p) const { return slot[p]; }
  int64_t diag_map(int64_t i) const { return slot[nnz_h + i]; }
  int64_t ata_map(int64_t q) const { return slot[nnz_h + n + q]; }
  // product q -> (Jacobian row, first factor slot, second factor slot)
  void product(int64_t q, int64_t g, int64_t &row, int64_t &s1, int64_t &s2) const;
  int64_t product_segment(int64_t q) const;
};

// ------------------------------------------------------- symbolic factor
// leading dimension of a front's column-major storage: even, so that with
// even front offsets every column starts 16-byte aligned (bulk copies)
inline int64_t front_ld(int64_t s) { return s + (s & 1); }

constexpr int kWarpFrontRows = 32;   // fronts this small are factored by one warp
constexpr int kTopFronts = 96;       // at most this many top fronts go to the cluster kernel
constexpr int kTopMinRows = 96;      // ... and only fronts at least this tall

// device record of one front (loaded with four 16-byte loads)
struct alignas(16) FrontMeta {
  int64_t f_off;      // front storage (doubles), s x s column-major
  int64_t a_begin;    // first entry of the front's A scatter
  int32_t a_count;
  int32_t first, ncols, nrows;
  int32_t parent, child_begin, child_end, v_off;
  int32_t rows_off, relmap_off, pad;
};

struct Symbolic {
  int64_t n = 0, nnz_a = 0, nnz_l = 0;
  std::vector<int64_t> perm, parent, a_rowptr, row_ptr, l_colptr;
  uvec<int64_t> a_rowcol, a_srcslot;
  uvec<int64_t> row_cols;   // row patterns of L, each row in etree-reach order
  // the reference L row indices (CSC) and the L -> front map are only needed
  // for exports: built on first use (ensure_l_csc / ensure_l_export)
  std::vector<int64_t> l_rowidx;
  void ensure_l_csc();
  void ensure_l_export();
  std::mutex lazy_mu;
  // ---- supernodal front plan (internal order = reference elimination order)
  int64_t nf = 0;                              // number of fronts
  std::vector<int32_t> f_first, f_ncols, f_nrows, f_parent;
  std::vector<int64_t> f_rows_off;             // into f_rows
  uvec<int32_t> f_rows;                        // sorted internal row indices per front
  std::vector<int64_t> f_off;                  // F storage offset (doubles)
  std::vector<int64_t> f_voff;                 // solve scratch offset (doubles)
  std::vector<int32_t> f_child_ptr, f_child;   // CSR children
  std::vector<int64_t> f_relmap_off;           // per front: r entries into relmap
  uvec<int32_t> relmap;                        // child update rows -> parent local rows
  std::vector<int64_t> f_a_ptr;                // CSR A scatter per front
  uvec<int64_t> a_kslot, a_fpos;               // (kvals slot, F offset)
  std::vector<int32_t> order;                  // task order: [small by level | large by level]
  int64_t nf_small = 0;                        // warp-task fronts (prefix of order)
  int64_t nf_top = 0;                          // cluster-task fronts (suffix of order)
  std::vector<int32_t> small_lptr;             // level boundaries within order[0, nf_small)
  std::vector<int32_t> level;
  std::vector<int64_t> l_export;               // reference L slot -> F offset
  int64_t dinv_off = 0;   // fronts buffer: [fronts | inverse diagonal (n)]
  int64_t xp_off = 0;     // solve workspace: [front vectors | permuted vector (n)]
  int64_t front_doubles = 0, vec_doubles = 0, max_front = 0, max_cols = 0, n_levels = 0;
  int64_t flops = 0;
  long long *trace = nullptr;   // optional device [3][nf][4] timing stamps
  // the large-front kernels run on `aux`, forked after the counter reset and
  // joined before the caller's next work, so they overlap the small-front
  // kernel of the same sweep (their fronts wait on dependency counters)
  void *aux = nullptr, *ev_fork = nullptr, *ev_join = nullptr;
  void *aux2 = nullptr, *ev_join2 = nullptr;   // the top-front factor kernel
  int64_t counters_cap = 0;     // instances the dependency-counter array holds
  // device
  bool uploaded = false;
  struct Dev {
    FrontMeta *meta = nullptr;        // per-front metadata (one 64-byte record)
    void *cinfo = nullptr;            // per child edge: the child's extend-add fields
    int32_t *f_rows = nullptr;
    int32_t *f_child = nullptr;
    int32_t *relmap = nullptr;
    int32_t *a_kslot = nullptr;
    int32_t *a_loc = nullptr;
    int32_t *order = nullptr;
    int32_t *nchild = nullptr;        // template counters (large children only)
    int32_t *small_lptr = nullptr;
    int32_t *bar = nullptr;           // grid barrier: [count, generation]
    int32_t *counters = nullptr;      // scratch counters
    int64_t *l_export = nullptr;
    int64_t *perm = nullptr;          // internal position -> original index
  } d;
  ~Symbolic();
};

// ---------------------------------------------------------- KKT gathers
struct Kkt {
  int64_t n = 0, m = 0, nh = 0, nj = 0, nk = 0, np = 0;
  bool has_assembly = false;
  int batch_cap = 0;     // instances the reduction / m-vector scratch holds
  struct Dev {
    int64_t *a_rowptr = nullptr;   // A by rows (jac order)
    int32_t *a_col = nullptr;
    int64_t *at_ptr = nullptr;     // A by columns: jac positions + rows
    int32_t *at_p = nullptr, *at_row = nullptr;
    int64_t *w_ptr = nullptr;      // symmetric W per row: hess positions + partner
    int32_t *w_p = nullptr, *w_j = nullptr;
    int32_t *k_ptr = nullptr;      // assembly: per K slot products (row, s1, s2)
    int32_t *k_row = nullptr, *k_s1 = nullptr, *k_s2 = nullptr;
    int32_t *k_w = nullptr, *k_diag = nullptr;
    double *partials = nullptr;
    unsigned int *counter = nullptr;
    double *scratch = nullptr;     // m doubles
    double *dvec = nullptr;        // D per row (assembly)
  } d;
  ~Kkt();
};

}  // namespace gn

struct gn_kkt : gn::Kkt {};
struct gn_model : gn::Model {};
struct gn_condense : gn::Condense {};
struct gn_symbolic : gn::Symbolic {};
