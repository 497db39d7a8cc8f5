// Pattern-block AD evaluator on sm_100a.
//
// One launch evaluates every record of every pattern block: CTA ranges map
// to blocks, one thread per record runs the block's instruction tape
// (forward values, reverse adjoints, forward-over-reverse Hessian columns)
// exactly as the reference interpreter does (expressions.py:222-409,
// including its "absent adjoint" semantics), and writes per-record
// contributions to a fixed contribution array.  A second launch gathers
// the contributions of every output slot (constraint rows, gradient
// entries, Jacobian / Hessian COO slots) in the reference's np.add.at
// order (autodiff.py:57-142): deterministic, no floating-point atomics.
// A single-CTA kernel reduces the objective.
#include <new>
#include <cmath>

#include <cstdio>
#include <cstdlib>

#include "ad_codegen.h"
#include "device.cuh"

namespace gn {
namespace {

constexpr int kRecThreads = 128;
enum { OP_VAR = 0, OP_PAR, OP_CONST, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_POW, OP_NEG, OP_SIN,
       OP_COS, OP_LOG, OP_SQRT, OP_EXP };

// numpy's scalar fast paths for array ** c (square, sqrt, reciprocal, identity)
__device__ __forceinline__ double powc(double v, double c) {
  if (c == 2.0) return v * v;
  if (c == 1.0) return v;
  if (c == 0.0) return 1.0;
  if (c == 0.5) return sqrt(v);
  if (c == -1.0) return 1.0 / v;
  return pow(v, c);
}

struct Partials {
  double fa, fb;
  bool has_b;
};

// (d entry/d a, d entry/d b) -- expressions.py:259-285
__device__ __forceinline__ Partials partials(int op, int a, int b, int i, const double *v,
                                             const double *consts) {
  switch (op) {
    case OP_ADD: return {1.0, 1.0, true};
    case OP_SUB: return {1.0, -1.0, true};
    case OP_MUL: return {v[b], v[a], true};
    case OP_DIV: return {1.0 / v[b], -v[a] / (v[b] * v[b]), true};
    case OP_POW: { double c = consts[b]; return {c * powc(v[a], c - 1.0), 0.0, false}; }
    case OP_NEG: return {-1.0, 0.0, false};
    case OP_SIN: return {cos(v[a]), 0.0, false};
    case OP_COS: return {-sin(v[a]), 0.0, false};
    case OP_LOG: return {1.0 / v[a], 0.0, false};
    case OP_SQRT: return {0.5 / v[i], 0.0, false};
    default: return {v[i], 0.0, false};  // EXP
  }
}

__device__ __forceinline__ bool is_binary(int op) { return op >= OP_ADD && op <= OP_DIV; }

__device__ __forceinline__ void acc(double *arr, uint64_t &mask, int k, double val) {
  if ((mask >> k) & 1ull) arr[k] += val;
  else { arr[k] = val; mask |= 1ull << k; }
}

__global__ void __launch_bounds__(kRecThreads)
ad_records_kernel(const DevBlock *__restrict__ blocks, int nblocks, const int4 *__restrict__ tape,
                  const double *__restrict__ consts_pool, const int32_t *__restrict__ slot_pool,
                  const int32_t *__restrict__ var_idx, const double *__restrict__ params,
                  const int32_t *__restrict__ targets, const double *__restrict__ x,
                  const double *__restrict__ y, const double *__restrict__ con_scale,
                  double obj_w, uint32_t what, double *__restrict__ contrib) {
  __shared__ DevBlock sb;
  __shared__ int4 s_tape[kMaxTape];
  __shared__ double s_const[kMaxTape];
  __shared__ int32_t s_slots[kMaxSlots + 3 * kMaxSlots * (kMaxSlots + 1) / 2 + kMaxSlots];
  if (threadIdx.x == 0) {
    int lo = 0, hi = nblocks - 1;
    while (lo < hi) {  // last block with cta_begin <= blockIdx.x
      int mid = (lo + hi + 1) >> 1;
      if (blocks[mid].cta_begin <= static_cast<int64_t>(blockIdx.x)) lo = mid; else hi = mid - 1;
    }
    sb = blocks[lo];
  }
  __syncthreads();
  const DevBlock &B = sb;
  const bool obj = B.kind == 0;
  const bool need_val = obj ? (what & GN_AD_F) : (what & GN_AD_C);
  const bool need_first = obj ? (what & GN_AD_GRAD) : (what & GN_AD_JAC);
  const bool need_hess = (what & GN_AD_HESS) && B.npairs > 0;
  if (!need_val && !need_first && !need_hess) return;
  for (int t = threadIdx.x; t < B.T; t += blockDim.x) s_tape[t] = tape[B.tape_off + t];
  for (int t = threadIdx.x; t < B.nconst; t += blockDim.x) s_const[t] = consts_pool[B.const_off + t];
  const int nslot = B.nfirst + 2 * B.npairs + B.nsweep;
  for (int t = threadIdx.x; t < nslot; t += blockDim.x) s_slots[t] = slot_pool[B.slot_off + t];
  __syncthreads();
  const int64_t r = (static_cast<int64_t>(blockIdx.x) - B.cta_begin) * blockDim.x + threadIdx.x;
  if (r >= B.R) return;
  const int *first = s_slots;
  const int *pair_a = s_slots + B.nfirst;
  const int *pair_b = pair_a + B.npairs;
  const int *sweep = pair_b + B.npairs;
  const int T = B.T;
  const int64_t R = B.R;

  double X[kMaxSlots];
  for (int s = 0; s < B.nv; ++s) X[s] = x[var_idx[B.var_off + s * R + r]];
  double v[kMaxTape];
  // ---- forward (expressions.py:222-254)
  for (int i = 0; i < T; ++i) {
    int4 e = s_tape[i];
    double o;
    switch (e.x) {
      case OP_VAR: o = X[e.y]; break;
      case OP_PAR: o = params[B.par_off + e.y * R + r]; break;
      case OP_CONST: o = s_const[e.z]; break;
      case OP_ADD: o = v[e.y] + v[e.z]; break;
      case OP_SUB: o = v[e.y] - v[e.z]; break;
      case OP_MUL: o = v[e.y] * v[e.z]; break;
      case OP_DIV: o = v[e.y] / v[e.z]; break;
      case OP_POW: o = powc(v[e.y], s_const[e.z]); break;
      case OP_NEG: o = -v[e.y]; break;
      case OP_SIN: o = sin(v[e.y]); break;
      case OP_COS: o = cos(v[e.y]); break;
      case OP_LOG: o = log(v[e.y]); break;
      case OP_SQRT: o = sqrt(v[e.y]); break;
      default: o = exp(v[e.y]); break;
    }
    v[i] = o;
  }
  double *out = contrib + B.contrib_off;
  if (need_val) out[r] = v[B.out];
  if (!need_first && !need_hess) return;

  // ---- reverse sweep (expressions.py:287-314)
  double adj[kMaxTape];
  uint64_t amask = 1ull << B.out;
  adj[B.out] = 1.0;
  double g[kMaxSlots];
  uint32_t gmask = 0;
  for (int i = T - 1; i >= 0; --i) {
    if (!((amask >> i) & 1ull)) continue;
    int4 e = s_tape[i];
    double ai = adj[i];
    if (e.x == OP_VAR) {
      if ((gmask >> e.y) & 1u) g[e.y] += ai; else { g[e.y] = ai; gmask |= 1u << e.y; }
      continue;
    }
    if (e.x == OP_PAR || e.x == OP_CONST) continue;
    Partials p = partials(e.x, e.y, e.z, i, v, s_const);
    acc(adj, amask, e.y, p.fa * ai);
    if (p.has_b) acc(adj, amask, e.z, p.fb * ai);
  }
  if (need_first)
    for (int k = 0; k < B.nfirst; ++k) {
      int s = first[k];
      out[(1 + k) * R + r] = ((gmask >> s) & 1u) ? g[s] : 0.0;
    }
  if (!need_hess) return;

  // ---- Hessian columns (expressions.py:316-409)
  double w;
  if (obj) w = obj_w;
  else {
    int t = targets[B.tgt_off + r];
    w = y[t] * (con_scale ? con_scale[t] : 1.0);
  }
  const int64_t hbase = (1 + B.nfirst) * R;
  for (int sw = 0; sw < B.nsweep; ++sw) {
    const int ts = sweep[sw];
    double dot[kMaxTape];
    uint64_t dmask = 0;
    for (int i = 0; i < T; ++i) {
      int4 e = s_tape[i];
      if (e.x == OP_VAR) {
        if (e.y == ts) { dot[i] = 1.0; dmask |= 1ull << i; }
        continue;
      }
      if (e.x == OP_PAR || e.x == OP_CONST) continue;
      bool ha = (dmask >> e.y) & 1ull;
      bool hb = is_binary(e.x) && ((dmask >> e.z) & 1ull);
      if (!ha && !hb) continue;
      Partials p = partials(e.x, e.y, e.z, i, v, s_const);
      double t = 0.0;
      bool have = false;
      if (ha) { t = p.fa * dot[e.y]; have = true; }
      if (hb) { t = have ? t + p.fb * dot[e.z] : p.fb * dot[e.z]; }
      dot[i] = t;
      dmask |= 1ull << i;
    }
    double adot[kMaxTape];
    uint64_t admask = 0;
    double hcol[kMaxSlots];
    uint32_t hmask = 0;
    for (int i = T - 1; i >= 0; --i) {
      bool hai = (amask >> i) & 1ull;
      bool hadi = (admask >> i) & 1ull;
      if (!hai && !hadi) continue;
      int4 e = s_tape[i];
      if (e.x == OP_VAR) {
        if (hadi) {
          if ((hmask >> e.y) & 1u) hcol[e.y] += adot[i]; else { hcol[e.y] = adot[i]; hmask |= 1u << e.y; }
        }
        continue;
      }
      if (e.x == OP_PAR || e.x == OP_CONST) continue;
      const int a = e.y, b = e.z;
      Partials p = partials(e.x, a, b, i, v, s_const);
      const bool hda = (dmask >> a) & 1ull;
      const bool hdb = is_binary(e.x) && ((dmask >> b) & 1ull);
      const double da = hda ? dot[a] : 0.0;
      const double db = hdb ? dot[b] : 0.0;
      double dfa = 0.0, dfb = 0.0;
      bool hdfa = false, hdfb = false;
      switch (e.x) {
        case OP_MUL:
          if (hdb) { dfa = db; hdfa = true; }
          if (hda) { dfb = da; hdfb = true; }
          break;
        case OP_DIV: {
          double vb = v[b];
          if (hdb) { dfa = -db / (vb * vb); hdfa = true; }
          if (hda) { dfb = -da / (vb * vb); hdfb = true; }
          if (hdb) {
            double t2 = 2.0 * v[a] * db / (vb * vb * vb);
            dfb = hdfb ? dfb + t2 : t2;
            hdfb = true;
          }
          break;
        }
        case OP_POW: {
          double c = s_const[b];
          if (hda && c != 1.0) { dfa = c * (c - 1.0) * powc(v[a], c - 2.0) * da; hdfa = true; }
          break;
        }
        case OP_SIN: if (hda) { dfa = -sin(v[a]) * da; hdfa = true; } break;
        case OP_COS: if (hda) { dfa = -cos(v[a]) * da; hdfa = true; } break;
        case OP_LOG: if (hda) { dfa = -da / (v[a] * v[a]); hdfa = true; } break;
        case OP_SQRT: if (hda) { dfa = -0.25 * da / (v[a] * v[i]); hdfa = true; } break;
        case OP_EXP: if (hda) { dfa = v[i] * da; hdfa = true; } break;
        default: break;  // ADD, SUB, NEG: constant partials
      }
      if (hai && hdfa) acc(adot, admask, a, dfa * adj[i]);
      if (hadi) acc(adot, admask, a, p.fa * adot[i]);
      if (p.has_b) {
        if (hai && hdfb) acc(adot, admask, b, dfb * adj[i]);
        if (hadi) acc(adot, admask, b, p.fb * adot[i]);
      }
    }
    for (int k = 0; k < B.npairs; ++k) {
      if (pair_b[k] != ts) continue;
      const int a = pair_a[k];
      double c = 0.0;
      if (((hmask >> a) & 1u) && !(obj && obj_w == 0.0)) {
        double fac = 1.0;
        if (a != ts && var_idx[B.var_off + a * R + r] == var_idx[B.var_off + ts * R + r]) fac = 2.0;
        c = (w * fac) * hcol[a];
      }
      out[hbase + k * R + r] = c;
    }
  }
}

struct GatherSeg {
  int64_t n_out;
  const int64_t *ptr;
  const int32_t *src;
  double *out;
  int mode;  // 0 none, 1 scalar, 2 scale[o], 3 scale[rows[o]]
  double scalar;
  const double *scale;
  const int32_t *rows;
  int32_t bit;
};

struct GatherArgs {
  GatherSeg seg[4];
  int nseg;
  int64_t begin[5];
  // instance batches (blockIdx.y): contributions per instance, scale vectors
  // (con_scale) per instance, scalar (obj_scale) from scal_b[instance]
  int64_t contrib_stride, scale_stride;
  const double *scal_b;
};

// Objective: the flattened contribution list (block order) in contiguous
// chunks, one CTA each; fixed-order tree sum per CTA, then the last CTA to
// finish adds the CTA partials in order (deterministic, no FP atomics).
// These CTAs lead the gather launch (one launch for everything after the
// pattern kernels).
constexpr int kGatherThreads = 256;
constexpr int kObjMaxCtas = 128;
struct ObjArgs {
  const int32_t *src;
  int64_t total;
  double scale;
  double *f;
  double *partials;
  unsigned *counter;
  int64_t f_stride;
  const double *scale_b;
  int nctas;   // leading CTAs of the launch that reduce the objective (0: none)
};

__device__ __forceinline__ void objective_cta(const ObjArgs &ob, const double *__restrict__ contrib, int32_t *flags) {
  __shared__ double red[kGatherThreads];
  __shared__ bool last;
  const int64_t bi = blockIdx.y;
  const unsigned cta = blockIdx.x, nct = static_cast<unsigned>(ob.nctas);
  double *partials = ob.partials + bi * kObjMaxCtas;
  unsigned *counter = ob.counter + bi;
  double *f = ob.f + bi * ob.f_stride;
  const double scale = ob.scale_b ? ob.scale_b[bi] : ob.scale;
  const int64_t per = (ob.total + nct - 1) / nct;
  const int64_t lo = per * cta, hi = min(ob.total, lo + per);
  double part = 0.0;
  for (int64_t p = lo + threadIdx.x; p < hi; p += 4 * kGatherThreads) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t q = p + u * kGatherThreads;
      v[u] = q < hi ? contrib[__ldg(ob.src + q)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) part += v[u];
  }
  red[threadIdx.x] = part;
  __syncthreads();
  for (int w = kGatherThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[cta] = red[0];
    __threadfence();
    last = atomicAdd(counter, 1u) == nct - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double total_sum = 0.0;
    for (unsigned b = 0; b < nct; ++b) total_sum += __ldcg(partials + b);
    if (!isfinite(total_sum)) atomicOr(flags, GN_AD_F);
    *f = total_sum * scale;
    *counter = 0u;
  }
}

__global__ void __launch_bounds__(kGatherThreads)
ad_gather_kernel(GatherArgs ga, ObjArgs ob, const double *__restrict__ contrib, int32_t *flags) {
  const int64_t bi = blockIdx.y;
  contrib += bi * ga.contrib_stride;
  flags += bi;
  if (static_cast<int>(blockIdx.x) < ob.nctas) {
    objective_cta(ob, contrib, flags);
    return;
  }
  int64_t t = static_cast<int64_t>(blockIdx.x - ob.nctas) * blockDim.x + threadIdx.x;
  if (t >= ga.begin[ga.nseg]) return;
  int s = 0;
  while (t >= ga.begin[s + 1]) ++s;
  const GatherSeg &G = ga.seg[s];
  int64_t o = t - ga.begin[s];
  double acc = 0.0;
  const int64_t p1 = G.ptr[o + 1];
  for (int64_t p = G.ptr[o]; p < p1; p += 4) {   // four terms' loads in flight, same order
    int64_t src[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) src[u] = p + u < p1 ? G.src[p + u] : 0;
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = p + u < p1 ? contrib[src[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (p + u < p1) acc = __dadd_rn(acc, v[u]);
  }
  if (!isfinite(acc)) atomicOr(flags, G.bit);
  double sc = 1.0;
  const double *scale = G.scale ? G.scale + bi * ga.scale_stride : nullptr;
  if (G.mode == 1) sc = ga.scal_b ? ga.scal_b[bi] : G.scalar;
  else if (G.mode == 2 && scale) sc = scale[o];
  else if (G.mode == 3 && scale) sc = scale[G.rows[o]];
  G.out[bi * G.n_out + o] = G.mode == 0 ? acc : acc * sc;
}

}  // namespace

static void release_model(Model &M) {
  if (!M.uploaded) return;
  dev_free(M.d.jslots);
  M.d.jslots = nullptr;
  dev_free(M.d.bstrides);
  dev_free(M.d.bstrides_shared);
  M.d.bstrides = M.d.bstrides_shared = nullptr;
  M.batch_cap = 0;
  dev_free(M.d.obj_partials);
  dev_free(M.d.obj_counter);
  M.d.obj_partials = nullptr;
  M.d.obj_counter = nullptr;
  void *ps[] = {M.d.blocks, M.d.tape, M.d.consts, M.d.slots, M.d.var_idx, M.d.params, M.d.targets,
                M.d.c_ptr, M.d.grad_ptr, M.d.jac_ptr, M.d.hess_ptr, M.d.c_src, M.d.grad_src,
                M.d.jac_src, M.d.hess_src, M.d.obj_src, M.d.jac_rows, M.d.obj_block_ptr};
  for (void *p : ps) dev_free(p);
  dev_free(M.d_genblk);
  M.d_genblk = nullptr;
  M.pattern_fn = nullptr;
  M.d = Model::Dev{};
  M.uploaded = false;
}

Model::~Model() { release_model(*this); }

static void upload_model(Model &M) {
  PhaseTimer tm("upload_model");
  PhaseTimer tm_b("upload_model.blocks");
  std::vector<DevBlock> db;
  std::vector<int4> tape;
  std::vector<double> consts;
  std::vector<int32_t> slots;
  // the record arrays (SoA, slot-major) are sized first and filled in
  // parallel: they are the bulk of the plan
  int64_t nvid = 0, npar = 0, ntg = 0;
  for (auto &b : M.blocks) {
    nvid += b.R * b.nv;
    npar += b.R * b.np;
    ntg += static_cast<int64_t>(b.targets.size());
  }
  uvec<int32_t> vidx(nvid), tg(ntg);
  uvec<double> par(npar);
  int64_t ovid = 0, opar = 0, otg = 0;
  int64_t cta = 0, coff = 0;
  for (auto &b : M.blocks) {
    DevBlock d{};
    d.kind = b.kind;
    d.nv = b.nv;
    d.np = b.np;
    d.T = static_cast<int32_t>(b.ops.size() / 3);
    d.out = b.out;
    d.nfirst = static_cast<int32_t>(b.first.size());
    d.npairs = static_cast<int32_t>(b.pairs.size() / 2);
    d.R = b.R;
    d.var_off = ovid;
    d.par_off = opar;
    d.tgt_off = otg;
    d.contrib_off = coff;
    coff += b.R * (1 + d.nfirst + d.npairs);
    d.tape_off = static_cast<int32_t>(tape.size());
    d.const_off = static_cast<int32_t>(consts.size());
    d.nconst = static_cast<int32_t>(b.consts.size());
    d.slot_off = static_cast<int32_t>(slots.size());
    d.cta_begin = cta;
    cta += (b.R + kRecThreads - 1) / kRecThreads;
    for (int t = 0; t < d.T; ++t) tape.push_back(make_int4(b.ops[3 * t], b.ops[3 * t + 1], b.ops[3 * t + 2], 0));
    consts.insert(consts.end(), b.consts.begin(), b.consts.end());

    for (int s : b.first) slots.push_back(s);
    std::vector<int> sw;
    for (int p = 0; p < d.npairs; ++p) slots.push_back(b.pairs[2 * p]);
    for (int p = 0; p < d.npairs; ++p) {
      slots.push_back(b.pairs[2 * p + 1]);
      if (std::find(sw.begin(), sw.end(), b.pairs[2 * p + 1]) == sw.end()) sw.push_back(b.pairs[2 * p + 1]);
    }
    std::sort(sw.begin(), sw.end());
    d.nsweep = static_cast<int32_t>(sw.size());
    for (int s : sw) slots.push_back(s);
    const int64_t R = b.R, nv = b.nv, npb = b.np, nt = static_cast<int64_t>(b.targets.size());
    int32_t *vo = vidx.data() + ovid;
    double *po = par.data() + opar;
    int32_t *to = tg.data() + otg;
#pragma omp parallel for schedule(static) if (R > 16384)
    for (int64_t r = 0; r < R; ++r) {
      for (int64_t q = 0; q < nv; ++q) vo[q * R + r] = static_cast<int32_t>(b.var_idx[r * nv + q]);
      for (int64_t q = 0; q < npb; ++q) po[q * R + r] = b.params[r * npb + q];
      if (r < nt) to[r] = static_cast<int32_t>(b.targets[r]);
    }
    for (int64_t r = R; r < nt; ++r) to[r] = static_cast<int32_t>(b.targets[r]);
    ovid += R * nv;
    opar += R * npb;
    otg += nt;
    db.push_back(d);
  }
  tm_b.~PhaseTimer();
  new (&tm_b) PhaseTimer("upload_model.blocks_done");
  GN_REQUIRE(coff == M.n_contrib, "contribution layout mismatch");
  GN_REQUIRE(coff < (int64_t(1) << 31), "contribution array too large for int32 gather lists");
  PhaseTimer tm_up("upload_model.copies");
  M.dblocks = db;
  M.n_ctas_rec = cta;
  M.d.blocks = dev_upload(db);
  M.d.tape = reinterpret_cast<int32_t *>(dev_upload(tape));
  M.d.consts = dev_upload(consts);
  M.d.slots = dev_upload(slots);
  M.d.var_idx = dev_upload(vidx);
  M.d.params = dev_upload(par);
  M.d.targets = dev_upload(tg);
  M.d.c_ptr = dev_upload(M.c_ptr);
  M.d.grad_ptr = dev_upload(M.grad_ptr);
  M.d.jac_ptr = dev_upload(M.jac_ptr);
  M.d.hess_ptr = dev_upload(M.hess_ptr);
  M.d.c_src = dev_upload(narrow<int32_t>(M.c_src));
  M.d.grad_src = dev_upload(narrow<int32_t>(M.grad_src));
  M.d.jac_src = dev_upload(narrow<int32_t>(M.jac_src));
  M.d.hess_src = dev_upload(narrow<int32_t>(M.hess_src));
  M.d.obj_src = dev_upload(narrow<int32_t>(M.obj_src));
  M.d.obj_block_ptr = dev_upload(M.obj_block_ptr);
  M.d.obj_partials = dev_alloc<double>(kObjMaxCtas);
  M.d.obj_counter = dev_upload(std::vector<unsigned>{0u});
  M.batch_cap = 1;
  M.n_params = npar;
  M.d.n_obj_blocks = static_cast<int32_t>(M.obj_block_ptr.size()) - 1;
  M.d.jac_rows = dev_upload(narrow<int32_t>(M.jac_rows));
  tm_up.~PhaseTimer();
  new (&tm_up) PhaseTimer("upload_model.rest");
  // pattern kernels generated from the tapes (NVRTC, cached per source)
  M.pattern_fn = nullptr;
  const char *env = std::getenv("GN_AD_INTERPRETER");
  if (!(env && env[0] == '1') && !db.empty()) {
    std::vector<int> pat;
    PhaseTimer tm_src("upload_model.pattern_source+compile");
    const std::string src = pattern_source(M, pat);
    M.pattern_fn = compile_patterns(src, M.pattern_error);
    tm_src.~PhaseTimer();
    new (&tm_src) PhaseTimer("upload_model.pattern_tail");
    if (M.pattern_fn) {
      struct GenBlk { long long cta_begin, R, var_off, par_off, tgt_off, contrib_off, jslot_off; int pattern, pad; };
      std::vector<GenBlk> gb(db.size());
      long long joff = 0;
      for (size_t b = 0; b < db.size(); ++b) {
        const bool con = M.blocks[b].kind != 0;
        gb[b] = {db[b].cta_begin, db[b].R, db[b].var_off, db[b].par_off, db[b].tgt_off, db[b].contrib_off,
                 con ? joff : -1, pat[b], 0};
        if (con) joff += db[b].R * static_cast<long long>(M.blocks[b].first.size());
      }
      M.d_genblk = dev_upload(gb);
      // Jacobian slots with exactly one contribution each -> direct writes
      M.jac_direct = !M.jac_rows.empty();
      for (size_t o = 0; o + 1 < M.jac_ptr.size() && M.jac_direct; ++o)
        M.jac_direct = M.jac_ptr[o + 1] - M.jac_ptr[o] == 1;
      if (M.jac_direct) M.d.jslots = dev_upload(narrow<int32_t>(M.jac_slots));
    }
  } else {
    M.pattern_error = "disabled by GN_AD_INTERPRETER=1";
  }
  GN_REQUIRE(M.pattern_fn || !M.needs_patterns,
             "a pattern block's tape or slot count exceeds the device interpreter's limits (64 entries, "
             "16 slots); it needs the generated pattern kernels (NVRTC), unavailable: " + M.pattern_error);
  M.uploaded = true;
}

// Batched (B > 1, K12): every instance has its own x / y / con_scale /
// parameters / outputs (instance-major, strides n, m, nnz, params) and its
// own objective weight and scale (device arrays objw_b / objs_b, [B]); the
// plan -- record indices, tapes, gather lists -- is shared.  f has stride
// f_stride, flags one word per instance.
static void ad_eval(Model &M, const double *x, const double *y, double obj_w, const double *con_scale,
                    double obj_scale, double *f, double *c, double *grad, double *jac, double *hess,
                    uint32_t what, double *contrib, int32_t *flags, cudaStream_t st, int B = 1,
                    const double *params_b = nullptr, const double *objw_b = nullptr,
                    const double *objs_b = nullptr, int64_t f_stride = 0) {
  GN_REQUIRE(M.uploaded, "model not uploaded to the device");
  GN_REQUIRE(B >= 1, "batch size must be positive");
  if (what & GN_AD_HESS) GN_REQUIRE(y != nullptr || M.m == 0, "Hessian needs multipliers");
  if (B > 1) GN_REQUIRE(M.pattern_fn != nullptr, "batched AD needs the generated pattern kernels (NVRTC)");
  if (what & GN_AD_RESET_FLAGS) {
    GN_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * B, st));
    what &= ~GN_AD_RESET_FLAGS;
  }
  if (B > M.batch_cap) {   // objective reduction scratch for B instances
    GN_CUDA(cudaStreamSynchronize(st));
    dev_free(M.d.obj_partials);
    dev_free(M.d.obj_counter);
    M.d.obj_partials = dev_alloc<double>(static_cast<int64_t>(kObjMaxCtas) * B);
    M.d.obj_counter = dev_alloc<unsigned>(B);
    GN_CUDA(cudaMemset(M.d.obj_counter, 0, sizeof(unsigned) * B));
    M.batch_cap = B;
  }
  const int64_t par_size = static_cast<int64_t>(M.n_params);
  if (B > 1 && !M.d.bstrides) {
    const std::vector<long long> bs = {static_cast<long long>(M.n), static_cast<long long>(M.m),
                                       static_cast<long long>(M.n_contrib), static_cast<long long>(par_size),
                                       static_cast<long long>(M.jac_rows.size())};
    M.d.bstrides = dev_upload(bs);
  }
  if (M.n_ctas_rec > 0 && M.pattern_fn) {
    int nblk = static_cast<int>(M.dblocks.size());
    const void *blk = M.d_genblk;
    const int32_t *vi = M.d.var_idx, *tg = M.d.targets;
    const double *pa = M.d.params;
    unsigned w = what;
    const int32_t *jsl = M.d.jslots;
    int jdirect = (M.jac_direct && (what & GN_AD_JAC)) ? 1 : 0;
    double *jac_out = jac;
    if (B > 1 && params_b) pa = params_b;   // per-instance parameter values, shared layout
    const long long *bs = B > 1 ? M.d.bstrides : nullptr;
    // shared parameters: stride 0 (bs[3] is the per-instance layout size)
    const long long *bs_use = bs;
    if (B > 1 && !params_b) {
      if (!M.d.bstrides_shared) {
        const std::vector<long long> b2 = {static_cast<long long>(M.n), static_cast<long long>(M.m),
                                           static_cast<long long>(M.n_contrib), 0LL,
                                           static_cast<long long>(M.jac_rows.size())};
        M.d.bstrides_shared = dev_upload(b2);
      }
      bs_use = M.d.bstrides_shared;
    }
    int32_t *fl = flags;
    void *args[] = {&blk, &nblk, &vi, &pa, &tg, &x, &y, &con_scale, &obj_w, &w, &contrib, &jsl, &jac_out, &jdirect,
                    &bs_use, &objw_b, &fl};
    GN_REQUIRE(launch_patterns(M.pattern_fn, static_cast<unsigned>(M.n_ctas_rec), st, args,
                               static_cast<unsigned>(B)),
               "pattern kernel launch failed");
    count_launch();
  } else if (M.n_ctas_rec > 0) {
    GN_LAUNCH(ad_records_kernel, static_cast<unsigned>(M.n_ctas_rec), kRecThreads, 0, st,
        M.d.blocks, static_cast<int>(M.dblocks.size()), reinterpret_cast<const int4 *>(M.d.tape),
        M.d.consts, M.d.slots, M.d.var_idx, M.d.params, M.d.targets, x, y, con_scale, obj_w, what,
        contrib);
  }
  GN_LAUNCH_CHECK();
  GatherArgs ga{};
  int ns = 0;
  auto add = [&](int64_t n_out, const int64_t *ptr, const int32_t *src, double *out, int mode,
                 double scalar, const double *scale, const int32_t *rows, int bit) {
    if (n_out == 0) return;
    ga.seg[ns] = GatherSeg{n_out, ptr, src, out, mode, scalar, scale, rows, bit};
    ga.begin[ns + 1] = ga.begin[ns] + n_out;
    ++ns;
  };
  ga.begin[0] = 0;
  ga.contrib_stride = M.n_contrib;
  ga.scale_stride = M.m;
  ga.scal_b = objs_b;
  if (what & GN_AD_C) add(M.m, M.d.c_ptr, M.d.c_src, c, con_scale ? 2 : 0, 1.0, con_scale, nullptr, GN_AD_C);
  if (what & GN_AD_GRAD)
    add(M.n, M.d.grad_ptr, M.d.grad_src, grad, (obj_scale != 1.0 || objs_b) ? 1 : 0, obj_scale, nullptr, nullptr,
        GN_AD_GRAD);
  if ((what & GN_AD_JAC) && !(M.pattern_fn && M.jac_direct))
    add(static_cast<int64_t>(M.jac_rows.size()), M.d.jac_ptr, M.d.jac_src, jac, con_scale ? 3 : 0, 1.0,
        con_scale, M.d.jac_rows, GN_AD_JAC);
  // directly written J: the pattern kernels flag non-finite values themselves
  if (what & GN_AD_HESS)
    add(static_cast<int64_t>(M.hess_rows.size()), M.d.hess_ptr, M.d.hess_src, hess, 0, 1.0, nullptr, nullptr, GN_AD_HESS);
  ga.nseg = ns;
  ObjArgs ob{};
  if (what & GN_AD_F) {
    const int64_t total = static_cast<int64_t>(M.obj_src.size());
    if (total > 0) {
      ob = ObjArgs{M.d.obj_src, total, obj_scale, f, M.d.obj_partials, M.d.obj_counter, f_stride, objs_b,
                   static_cast<int>(std::min<int64_t>(kObjMaxCtas, (total + 4095) / 4096))};
    } else if (B == 1) {
      GN_CUDA(cudaMemsetAsync(f, 0, sizeof(double), st));
    } else {
      GN_CUDA(cudaMemset2DAsync(f, sizeof(double) * f_stride, 0, sizeof(double), B, st));
    }
  }
  const int64_t tot = ns > 0 ? ga.begin[ns] : 0;
  const int64_t ctas = ob.nctas + (tot + kGatherThreads - 1) / kGatherThreads;
  if (ctas > 0) {
    GN_LAUNCH(ad_gather_kernel, dim3(static_cast<unsigned>(ctas), B), kGatherThreads, 0, st, ga, ob, contrib,
              flags);
    GN_LAUNCH_CHECK();
  }
}

}  // namespace gn

using namespace gn;

extern "C" int gn_ad_eval_batched(gn_model *M, int32_t B, const double *x, const double *y, const double *objw_b,
                                  const double *con_scale, const double *objs_b, const double *params_b, double *f,
                                  int64_t f_stride, double *c, double *grad, double *jac, double *hess,
                                  uint32_t what, double *contrib_ws, int32_t *flags, void *stream) {
  return guarded([&] {
    ad_eval(*M, x, y, 1.0, con_scale, 1.0, f, c, grad, jac, hess, what, contrib_ws, flags,
            static_cast<cudaStream_t>(stream), B, params_b, objw_b, objs_b, f_stride);
  });
}

extern "C" int gn_model_param_count(const gn_model *M, int64_t *count) {
  return guarded([&] { *count = static_cast<int64_t>(M->n_params); });
}

extern "C" int gn_model_upload(gn_model *M) {
  return guarded([&] {
    if (!M->uploaded) upload_model(*M);
  });
}

extern "C" int gn_model_pattern_source(const gn_model *M, char *buf, size_t len, size_t *needed) {
  return guarded([&] {
    std::vector<int> pat;
    const std::string src = pattern_source(*M, pat);
    if (needed) *needed = src.size() + 1;
    if (buf && len) std::snprintf(buf, len, "%s", src.c_str());
  });
}

extern "C" int gn_model_traffic(const gn_model *M, uint32_t what, int64_t *bytes) {
  return guarded([&] {
    const Model &m = *M;
    int64_t b = 8 * m.n;                                    // x
    if (what & GN_AD_HESS) b += 8 * m.m;                    // y
    if (what & (GN_AD_C | GN_AD_JAC | GN_AD_HESS)) b += 8 * m.m;   // con_scale
    for (const auto &blk : m.blocks)                        // record data (SoA)
      b += blk.R * (4 * blk.nv + 8 * blk.np + (blk.kind != 0 ? 4 : 0));
    auto gather = [&](const std::vector<int64_t> &ptr, const std::vector<int64_t> &src, int64_t out) {
      return static_cast<int64_t>(8 * ptr.size() + 4 * src.size() + 8 * out);
    };
    if (what & GN_AD_C) b += gather(m.c_ptr, m.c_src, m.m);
    if (what & GN_AD_GRAD) b += gather(m.grad_ptr, m.grad_src, m.n);
    if (what & GN_AD_JAC) {
      const int64_t nj = static_cast<int64_t>(m.jac_rows.size());
      // direct writes need the slot map only; the gathered path its CSR + rows
      b += (m.pattern_fn && m.jac_direct) ? 12 * nj : gather(m.jac_ptr, m.jac_src, nj) + 4 * nj;
    }
    if (what & GN_AD_HESS) b += gather(m.hess_ptr, m.hess_src, static_cast<int64_t>(m.hess_rows.size()));
    if (what & GN_AD_F) b += 4 * static_cast<int64_t>(m.obj_src.size()) + 8;
    *bytes = b;
  });
}

extern "C" int gn_model_ad_backend(const gn_model *M, char *buf, size_t len) {
  return guarded([&] {
    std::string s = M->pattern_fn ? "patterns" : ("interpreter: " + M->pattern_error);
    if (buf && len) {
      std::snprintf(buf, len, "%s", s.c_str());
    }
  });
}

extern "C" int gn_model_release(gn_model *M) {
  return guarded([&] { release_model(*M); });
}

extern "C" int gn_ad_eval(gn_model *M, const double *x, const double *y, double obj_weight,
                          const double *con_scale, double obj_scale, double *f, double *c,
                          double *grad, double *jac, double *hess, uint32_t what, double *contrib_ws,
                          int32_t *flags, void *stream) {
  return guarded([&] {
    ad_eval(*M, x, y, obj_weight, con_scale, obj_scale, f, c, grad, jac, hess, what, contrib_ws, flags,
            static_cast<cudaStream_t>(stream));
  });
}
