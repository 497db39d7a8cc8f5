// Condensed-KKT device kernels: matvecs, condensed assembly, right-hand
// side, recoveries, the double-double seven-block residual and the matrix
// scale (reference src/gridnlp/kkt.py:96-229, 300-312).
//
// Every kernel is a gather: each output entry is owned by one thread and
// accumulates its inputs in the order the reference's np.add.at scatter
// would, so values are deterministic and -- for the FMA-free assembly --
// bitwise equal to the reference given equal inputs.
#include <cmath>

#include "gather.cuh"
#include "reduce.cuh"

namespace gn {

Kkt::~Kkt() {
  void *ps[] = {d.a_rowptr, d.a_col, d.at_ptr, d.at_p, d.at_row, d.w_ptr, d.w_p, d.w_j,
                d.k_ptr, d.k_row, d.k_s1, d.k_s2, d.k_w, d.k_diag, d.partials, d.counter,
                d.scratch, d.dvec};
  for (void *p : ps) dev_free(p);
}

namespace {

constexpr int kT = 256;

__device__ __forceinline__ double inv_or_zero(double w) { return isfinite(w) ? 1.0 / w : 0.0; }

unsigned blocks_for(int64_t n) { return static_cast<unsigned>((n + kT - 1) / kT > 0 ? (n + kT - 1) / kT : 1); }

// ------------------------------------------------------------ double-double
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick(double s, double e) {
  double h = s + e;
  return {h, e - (h - s)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  dd t = two_sum(x.lo, y.lo);
  double e = s.lo + t.hi;
  dd u = quick(s.hi, e);
  return quick(u.hi, t.lo + u.lo);
}
__device__ __forceinline__ dd dd_prod(double a, double b) {
  double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_from(double a) { return {a, 0.0}; }
// dd * double
__device__ __forceinline__ dd dd_mul_d(dd x, double b) {
  dd p = dd_prod(x.hi, b);
  return quick(p.hi, p.lo + x.lo * b);
}
__device__ __forceinline__ double dd_round(dd x) { return x.hi + x.lo; }

// ------------------------------------------------------------ kernels
__global__ void sigma_kernel(int64_t len, const double *dl, const double *du, const double *zl,
                             const double *zu, double *out) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i < len) out[i] = __dadd_rn(__dmul_rn(zl[i], inv_or_zero(dl[i])), __dmul_rn(zu[i], inv_or_zero(du[i])));
}

// sum_t a[ia[t]] * b[ib[t]] over t in [t0, t1) in double-double, accumulated
// in ascending t (the order of the plain loop) with the index and value
// loads of four terms issued before their sequential accumulation: the
// gathers' L2 latency overlaps instead of being paid per term
template <class IA, class IB>
__device__ __forceinline__ dd dd_gather_dot(int64_t t0, int64_t t1, const double *__restrict__ a, IA ia,
                                            const double *__restrict__ b, IB ib) {
  dd acc = {0.0, 0.0};
  for (int64_t t = t0; t < t1; t += 4) {   // predicated chunks: no serial remainder loop
    double va[4], vb[4];
    gather4(t, t1, a, ia, b, ib, va, vb);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u < t1) acc = dd_add(acc, dd_prod(va[u], vb[u]));
  }
  return acc;
}

// Two gathered double-double dot products with their first four terms each
// in flight together (indices of both, then values of both), then the rest
// in chunks of four; each sum accumulates in ascending t as dd_gather_dot.
template <class IA1, class IB1, class IA2, class IB2>
__device__ __forceinline__ void dd_gather_dot2(int64_t s0, int64_t s1, const double *__restrict__ a1, IA1 ia1,
                                               const double *__restrict__ b1, IB1 ib1, int64_t u0, int64_t u1,
                                               const double *__restrict__ a2, IA2 ia2,
                                               const double *__restrict__ b2, IB2 ib2, dd &r1, dd &r2) {
  int64_t p1[4], q1[4], p2[4], q2[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    p1[u] = s0 + u < s1 ? ia1(s0 + u) : 0;
    q1[u] = s0 + u < s1 ? ib1(s0 + u) : 0;
    p2[u] = u0 + u < u1 ? ia2(u0 + u) : 0;
    q2[u] = u0 + u < u1 ? ib2(u0 + u) : 0;
  }
  double x1[4], y1[4], x2[4], y2[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    x1[u] = s0 + u < s1 ? a1[p1[u]] : 0.0;
    y1[u] = s0 + u < s1 ? b1[q1[u]] : 0.0;
    x2[u] = u0 + u < u1 ? a2[p2[u]] : 0.0;
    y2[u] = u0 + u < u1 ? b2[q2[u]] : 0.0;
  }
  r1 = {0.0, 0.0};
  r2 = {0.0, 0.0};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (s0 + u < s1) r1 = dd_add(r1, dd_prod(x1[u], y1[u]));
    if (u0 + u < u1) r2 = dd_add(r2, dd_prod(x2[u], y2[u]));
  }
  for (int64_t t = s0 + 4; t < s1; t += 4) {
    double va[4], vb[4];
    gather4(t, s1, a1, ia1, b1, ib1, va, vb);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u < s1) r1 = dd_add(r1, dd_prod(va[u], vb[u]));
  }
  for (int64_t t = u0 + 4; t < u1; t += 4) {
    double va[4], vb[4];
    gather4(t, u1, a2, ia2, b2, ib2, va, vb);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u < u1) r2 = dd_add(r2, dd_prod(va[u], vb[u]));
  }
}

// W v from the lower triangle: first every entry's row contribution, then
// the mirrored off-diagonal contributions (kkt.py:132-138)
__global__ void w_matvec_kernel(int64_t n, const int64_t *ptr, const int32_t *wp, const int32_t *wj,
                                const double *w, const double *v, double *out) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i >= n) return;
  out[i] = gather_dot(ptr[i], ptr[i + 1], w, [&](int64_t t) { return wp[t]; }, v,
                      [&](int64_t t) { return wj[t]; });
}

__global__ void a_matvec_kernel(int64_t m, const int64_t *rowptr, const int32_t *col, const double *a,
                                const double *v, double *out) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i >= m) return;
  out[i] = gather_dot(rowptr[i], rowptr[i + 1], a, [](int64_t p) { return p; }, v,
                      [&](int64_t p) { return col[p]; });
}

__global__ void at_matvec_kernel(int64_t n, const int64_t *ptr, const int32_t *pp, const int32_t *row,
                                 const double *a, const double *u, double *out) {
  int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (j >= n) return;
  out[j] = gather_dot(ptr[j], ptr[j + 1], a, [&](int64_t t) { return pp[t]; }, u,
                      [&](int64_t t) { return row[t]; });
}

// D = (Sigma_s + dw) C, C = 1 / (dc Sigma_s + (1 + dc dw)) per row
// (kkt.py:153-157), once per row instead of once per product
__global__ void d_rows_kernel(int64_t m, gn_kkt_state st, double *d, Bx bx) {
  int64_t r = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (r >= m) return;
  shift(st, bx);
  d = shift_ptr(d, m);
  const double ssr = st.ss[r];
  const double cfac = __dadd_rn(1.0, __dmul_rn(st.dc, st.dw));
  const double c = 1.0 / __dadd_rn(__dmul_rn(st.dc, ssr), cfac);
  d[r] = __dmul_rn(__dadd_rn(ssr, st.dw), c);
}

// K[slot] = ((0 + W) + (sigma_x + dw)) + sum (d[row] * a[s1]) * a[s2] in
// product order (kkt.py:300-312); no FMA contraction, so the values are
// bitwise the reference's.  One thread per K slot; the indices of up to four
// products are loaded before their values (memory-level parallelism).
__global__ void __launch_bounds__(kT)
assemble_kernel(int64_t nk, const int32_t *__restrict__ kp, const int32_t *__restrict__ krow,
                const int32_t *__restrict__ ks1, const int32_t *__restrict__ ks2,
                const int32_t *__restrict__ kw, const int32_t *__restrict__ kd, gn_kkt_state st,
                const double *__restrict__ d, double *K, Bx bx) {
  int64_t s = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (s >= nk) return;
  shift(st, bx);
  d = shift_ptr(d, bx.m);
  K = shift_ptr(K, nk);
  const int p0 = __ldg(kp + s), p1 = __ldg(kp + s + 1);
  const int w = __ldg(kw + s), dg = __ldg(kd + s);
  double acc = 0.0;
  if (w >= 0) acc = __dadd_rn(acc, __ldg(st.w + w));
  if (dg >= 0) acc = __dadd_rn(acc, __dadd_rn(__ldg(st.sx + dg), st.dw));
  for (int p = p0; p < p1; p += 4) {
    int r[4], a1[4], a2[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = p + u < p1;
      r[u] = ok ? __ldg(krow + p + u) : 0;
      a1[u] = ok ? __ldg(ks1 + p + u) : 0;
      a2[u] = ok ? __ldg(ks2 + p + u) : 0;
    }
    double dv[4], v1[4], v2[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      dv[u] = __ldg(d + r[u]);
      v1[u] = __ldg(st.a + a1[u]);
      v2[u] = __ldg(st.a + a2[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (p + u < p1) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(dv[u], v1[u]), v2[u]));
  }
  K[s] = acc;
}

__device__ __forceinline__ double c_of(const gn_kkt_state &st, double ssr) {
  return 1.0 / __dadd_rn(__dmul_rn(st.dc, ssr), __dadd_rn(1.0, __dmul_rn(st.dc, st.dw)));
}

// m-side of the condensed rhs: qs, qy and u = C qs + D qy
__global__ void rhs_rows_kernel(int64_t m, gn_kkt_state st, gn_vec7 pv, double *qs, double *qy, double *u,
                                Bx bx) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i >= m) return;
  shift(st, bx);
  shift(pv, bx);
  qs = shift_ptr(qs, m);
  qy = shift_ptr(qy, m);
  u = shift_ptr(u, m);
  const double q_s = __dsub_rn(__dadd_rn(pv.s[i], __dmul_rn(inv_or_zero(st.dsl[i]), pv.zsl[i])),
                               __dmul_rn(inv_or_zero(st.dsu[i]), pv.zsu[i]));
  const double q_y = pv.y[i];
  const double c = c_of(st, st.ss[i]);
  const double d = __dmul_rn(__dadd_rn(st.ss[i], st.dw), c);
  qs[i] = q_s;
  qy[i] = q_y;
  u[i] = __dadd_rn(__dmul_rn(c, q_s), __dmul_rn(d, q_y));
}

// n-side: qx and rhs = qx + A^T u
__global__ void rhs_cols_kernel(int64_t n, const int64_t *ptr, const int32_t *pp, const int32_t *row,
                                gn_kkt_state st, gn_vec7 pv, const double *u, double *qx, double *rhs, Bx bx) {
  int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (j >= n) return;
  shift(st, bx);
  shift(pv, bx);
  u = shift_ptr(u, bx.m);
  qx = shift_ptr(qx, n);
  rhs = shift_ptr(rhs, n);
  const double q_x = __dsub_rn(__dadd_rn(pv.x[j], __dmul_rn(inv_or_zero(st.dxl[j]), pv.zxl[j])),
                               __dmul_rn(inv_or_zero(st.dxu[j]), pv.zxu[j]));
  const double acc = gather_dot(ptr[j], ptr[j + 1], st.a, [&](int64_t t) { return pp[t]; }, u,
                                [&](int64_t t) { return row[t]; });
  qx[j] = q_x;
  rhs[j] = __dadd_rn(q_x, acc);
}

__global__ void recover_sd_kernel(int64_t m, const int64_t *rowptr, const int32_t *col, gn_kkt_state st,
                                  const double *dx, const double *qs, const double *qy, double *ds,
                                  double *dy, Bx bx) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i >= m) return;
  shift(st, bx);
  dx = shift_ptr(dx, bx.n);
  qs = shift_ptr(qs, m);
  qy = shift_ptr(qy, m);
  ds = shift_ptr(ds, m);
  dy = shift_ptr(dy, m);
  const double ax = gather_dot(rowptr[i], rowptr[i + 1], st.a, [](int64_t p) { return p; }, dx,
                               [&](int64_t p) { return col[p]; });
  const double c = c_of(st, st.ss[i]);
  const double dsi = __dmul_rn(c, __dsub_rn(__dadd_rn(ax, __dmul_rn(st.dc, qs[i])), qy[i]));
  ds[i] = dsi;
  dy[i] = __dsub_rn(__dmul_rn(__dadd_rn(st.ss[i], st.dw), dsi), qs[i]);
}

__global__ void recover_bd_kernel(int64_t len, const double *dl, const double *du, const double *zl,
                                  const double *zu, const double *pzl, const double *pzu, const double *dv,
                                  double *dzl, double *dzu, int32_t *flags) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i >= len) return;
  // batched: every array is [B][len], flags [B]
  dl = shift_ptr(dl, len); du = shift_ptr(du, len); zl = shift_ptr(zl, len); zu = shift_ptr(zu, len);
  pzl = shift_ptr(pzl, len); pzu = shift_ptr(pzu, len); dv = shift_ptr(dv, len);
  dzl = shift_ptr(dzl, len); dzu = shift_ptr(dzu, len); flags = shift_ptr(flags, 1);
  const double wl = dl[i], wu = du[i];
  if ((isfinite(wl) && !(wl > 0.0)) || (isfinite(wu) && !(wu > 0.0))) atomicOr(flags, 1);
  dzl[i] = __dmul_rn(inv_or_zero(wl), __dsub_rn(pzl[i], __dmul_rn(zl[i], dv[i])));
  dzu[i] = __dmul_rn(inv_or_zero(wu), __dadd_rn(pzu[i], __dmul_rn(zu[i], dv[i])));
}

// x-side residual blocks in double-double: rx, rzxl, rzxu (kkt.py:199-206)
__global__ void residual_x_kernel(int64_t n, const int64_t *wptr, const int32_t *wp, const int32_t *wj,
                                  const int64_t *atptr, const int32_t *atp, const int32_t *atrow,
                                  gn_kkt_state st, gn_vec7 step, gn_vec7 pv, gn_vec7 res, RedSpec rs, Bx bx) {
  shift(st, bx);
  shift(step, bx);
  shift(pv, bx);
  shift(res, bx);
  double vmax[1] = {0.0};
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; j < n;
       j += static_cast<int64_t>(gridDim.x) * kT) {
    const double dxj = step.x[j];
    dd wv, atv;
    dd_gather_dot2(wptr[j], wptr[j + 1], st.w, [&](int64_t t) { return wp[t]; }, step.x,
                   [&](int64_t t) { return wj[t]; }, atptr[j], atptr[j + 1], st.a,
                   [&](int64_t t) { return atp[t]; }, step.y, [&](int64_t t) { return atrow[t]; }, wv, atv);
    dd rx = dd_from(pv.x[j]);
    rx = dd_add(rx, dd_neg(wv));
    rx = dd_add(rx, dd_neg(dd_prod(st.dw, dxj)));
    rx = dd_add(rx, dd_neg(atv));
    rx = dd_add(rx, dd_from(step.zxl[j]));
    rx = dd_add(rx, dd_from(-step.zxu[j]));
    const double wl = st.dxl[j], wu = st.dxu[j];
    dd rl = dd_add(dd_from(pv.zxl[j]), dd_neg(dd_prod(st.zxl[j], dxj)));
    rl = dd_add(rl, dd_neg(dd_prod(isfinite(wl) ? wl : 1.0, step.zxl[j])));
    dd ru = dd_add(dd_from(pv.zxu[j]), dd_prod(st.zxu[j], dxj));
    ru = dd_add(ru, dd_neg(dd_prod(isfinite(wu) ? wu : 1.0, step.zxu[j])));
    const double a = dd_round(rx), b = dd_round(rl), c = dd_round(ru);
    res.x[j] = a;
    res.zxl[j] = b;
    res.zxu[j] = c;
    double mx = fmax(fmax(fabs(a), fabs(b)), fabs(c));
    if (a != a || b != b || c != c) mx = a + b + c;
    vmax[0] = red_combine(RED_MAX, vmax[0], mx);
  }
  grid_reduce<1>(rs, vmax);
}

// s/y-side residual blocks: rs, ry, rzsl, rzsu (kkt.py:202-208)
__global__ void residual_s_kernel(int64_t m, const int64_t *rowptr, const int32_t *col, gn_kkt_state st,
                                  gn_vec7 step, gn_vec7 pv, gn_vec7 res, RedSpec rs, Bx bx) {
  shift(st, bx);
  shift(step, bx);
  shift(pv, bx);
  shift(res, bx);
  double vmax[1] = {0.0};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * kT) {
    const double dsi = step.s[i], dyi = step.y[i];
    const dd ax = dd_gather_dot(rowptr[i], rowptr[i + 1], st.a, [](int64_t p) { return p; }, step.x,
                                [&](int64_t p) { return col[p]; });
    dd r_s = dd_add(dd_from(pv.s[i]), dd_neg(dd_prod(st.dw, dsi)));
    r_s = dd_add(r_s, dd_from(dyi));
    r_s = dd_add(r_s, dd_from(step.zsl[i]));
    r_s = dd_add(r_s, dd_from(-step.zsu[i]));
    dd r_y = dd_add(dd_from(pv.y[i]), dd_neg(ax));
    r_y = dd_add(r_y, dd_from(dsi));
    r_y = dd_add(r_y, dd_prod(st.dc, dyi));
    const double wl = st.dsl[i], wu = st.dsu[i];
    dd rl = dd_add(dd_from(pv.zsl[i]), dd_neg(dd_prod(st.zsl[i], dsi)));
    rl = dd_add(rl, dd_neg(dd_prod(isfinite(wl) ? wl : 1.0, step.zsl[i])));
    dd ru = dd_add(dd_from(pv.zsu[i]), dd_prod(st.zsu[i], dsi));
    ru = dd_add(ru, dd_neg(dd_prod(isfinite(wu) ? wu : 1.0, step.zsu[i])));
    const double a = dd_round(r_s), b = dd_round(r_y), c = dd_round(rl), e = dd_round(ru);
    res.s[i] = a;
    res.y[i] = b;
    res.zsl[i] = c;
    res.zsu[i] = e;
    double mx = fmax(fmax(fabs(a), fabs(b)), fmax(fabs(c), fabs(e)));
    if (a != a || b != b || c != c || e != e) mx = a + b + c + e;
    vmax[0] = red_combine(RED_MAX, vmax[0], mx);
  }
  grid_reduce<1>(rs, vmax);
}

// out[i * stride] = max(a[i * stride], b[i * stride]) for every instance i
__global__ void max2_kernel(const double *a, const double *b, double *out, int B, int64_t stride) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  double x = a[i * stride], y = b[i * stride];
  out[i * stride] = (x != x) ? x : ((y != y) ? y : fmax(x, y));
}

// max over |w|, |a|, |Sigma|, |z|, finite widths (kkt.py:211-221)
__global__ void matrix_scale_kernel(int64_t n, int64_t m, int64_t nh, int64_t nj, gn_kkt_state st, RedSpec rs,
                                    Bx bx) {
  shift(st, bx);
  double v[1] = {1.0};
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double acc = fmax(1.0, fmax(st.dw, st.dc));
  for (int64_t t = t0; t < nh; t += stride) acc = fmax(acc, fabs(st.w[t]));
  for (int64_t t = t0; t < nj; t += stride) acc = fmax(acc, fabs(st.a[t]));
  for (int64_t t = t0; t < n; t += stride) {
    acc = fmax(acc, fmax(fabs(st.sx[t]), fmax(fabs(st.zxl[t]), fabs(st.zxu[t]))));
    if (isfinite(st.dxl[t])) acc = fmax(acc, st.dxl[t]);
    if (isfinite(st.dxu[t])) acc = fmax(acc, st.dxu[t]);
  }
  for (int64_t t = t0; t < m; t += stride) {
    acc = fmax(acc, fmax(fabs(st.ss[t]), fmax(fabs(st.zsl[t]), fabs(st.zsu[t]))));
    if (isfinite(st.dsl[t])) acc = fmax(acc, st.dsl[t]);
    if (isfinite(st.dsu[t])) acc = fmax(acc, st.dsu[t]);
  }
  v[0] = acc;
  grid_reduce<1>(rs, v);
}

__global__ void axpy7_kernel(int64_t n, int64_t m, gn_vec7 y, gn_vec7 x, double alpha, Bx bx) {
  if (bx.bp) {   // batched: per-instance alpha (0 leaves an instance unchanged)
    alpha = bpar(bx, GN_BP_ALPHA, alpha);
    if (alpha == 0.0) return;
    shift(y, bx);
    shift(x, bx);
  }
  int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i < n) {
    y.x[i] += alpha * x.x[i];
    y.zxl[i] += alpha * x.zxl[i];
    y.zxu[i] += alpha * x.zxu[i];
  }
  if (i < m) {
    y.s[i] += alpha * x.s[i];
    y.y[i] += alpha * x.y[i];
    y.zsl[i] += alpha * x.zsl[i];
    y.zsu[i] += alpha * x.zsu[i];
  }
}

RedSpec max_spec(Kkt &K, double *out, int64_t out_stride = 0) {
  RedSpec r{};
  r.k = 1;
  r.op[0] = RED_MAX;
  r.out = out;
  r.partials = K.d.partials;
  r.counter = K.d.counter;
  r.out_stride = out_stride;
  return r;
}

Bx single(const Kkt &K) { return Bx{nullptr, K.n, K.m, K.nh, K.nj}; }
Bx batched(const Kkt &K, const double *bp) { return Bx{bp, K.n, K.m, K.nh, K.nj}; }

}  // namespace

static void kkt_create(Kkt &K, int64_t n, int64_t m, int64_t nh, const int64_t *hr, const int64_t *hc,
                       int64_t nj, const int64_t *jr, const int64_t *jc, const Condense *cs) {
  PhaseTimer tm("kkt_create");
  K.n = n;
  K.m = m;
  K.nh = nh;
  K.nj = nj;
  // A rows (jac is row-major sorted)
  std::vector<int64_t> rowptr(m + 1, 0);
  const bool have_segs = cs && cs->nnz_j == nj && cs->n == n && !cs->seg.empty();
  if (have_segs) {
    // the condensation checked the order and the columns and split the
    // Jacobian into row segments: the row pointers from the segments
    const int64_t nseg = static_cast<int64_t>(cs->seg.size()) - 1;
    for (int64_t g = 0; g < nseg; ++g) {
      GN_REQUIRE(cs->seg_row[g] >= 0 && cs->seg_row[g] < m, "Jacobian index out of range");
      rowptr[cs->seg_row[g] + 1] = cs->seg[g + 1] - cs->seg[g];
    }
  } else {
    for (int64_t p = 0; p < nj; ++p) {
      GN_REQUIRE(jr[p] >= 0 && jr[p] < m && jc[p] >= 0 && jc[p] < n, "Jacobian index out of range");
      GN_REQUIRE(p == 0 || jr[p] >= jr[p - 1], "Jacobian must be sorted by row");
      rowptr[jr[p] + 1]++;
    }
  }
  for (int64_t i = 0; i < m; ++i) rowptr[i + 1] += rowptr[i];
  uvec<int32_t> col(nj), at_p(nj), at_row(nj);
  for (int64_t p = 0; p < nj; ++p) col[p] = static_cast<int32_t>(jc[p]);
  std::vector<int64_t> atptr;
  if (cs && static_cast<int64_t>(cs->a_colptr.size()) == n + 1 &&
      static_cast<int64_t>(cs->a_colent.size()) == nj) {
    // the condensation already bucketed the Jacobian by column (same order)
    atptr = cs->a_colptr;
    for (int64_t q = 0; q < nj; ++q) {
      at_p[q] = cs->a_colent[q];
      at_row[q] = static_cast<int32_t>(jr[at_p[q]]);
    }
  } else {
    atptr.assign(n + 1, 0);
    for (int64_t p = 0; p < nj; ++p) atptr[jc[p] + 1]++;
    for (int64_t j = 0; j < n; ++j) atptr[j + 1] += atptr[j];
    std::vector<int64_t> fl(atptr.begin(), atptr.end() - 1);
    for (int64_t p = 0; p < nj; ++p) {
      int64_t q = fl[jc[p]]++;
      at_p[q] = static_cast<int32_t>(p);
      at_row[q] = static_cast<int32_t>(jr[p]);
    }
  }
  // W symmetric gather: pass 1 rows (all entries), pass 2 mirrored off-diagonals
  std::vector<int64_t> wptr(n + 1, 0);
  for (int64_t p = 0; p < nh; ++p) {
    GN_REQUIRE(hr[p] >= 0 && hr[p] < n && hc[p] >= 0 && hc[p] <= hr[p], "Hessian index out of range");
    wptr[hr[p] + 1]++;
    if (hr[p] != hc[p]) wptr[hc[p] + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) wptr[i + 1] += wptr[i];
  uvec<int32_t> wp(wptr[n]), wj(wptr[n]);
  {
    std::vector<int64_t> fl(wptr.begin(), wptr.end() - 1);
    for (int64_t p = 0; p < nh; ++p) {
      int64_t q = fl[hr[p]]++;
      wp[q] = static_cast<int32_t>(p);
      wj[q] = static_cast<int32_t>(hc[p]);
    }
    for (int64_t p = 0; p < nh; ++p)
      if (hr[p] != hc[p]) {
        int64_t q = fl[hc[p]]++;
        wp[q] = static_cast<int32_t>(p);
        wj[q] = static_cast<int32_t>(hr[p]);
      }
  }
  PhaseTimer tm_up("kkt_create.copies");
  K.d.a_rowptr = dev_upload(rowptr);
  K.d.a_col = dev_upload(col);
  K.d.at_ptr = dev_upload(atptr);
  K.d.at_p = dev_upload(at_p);
  K.d.at_row = dev_upload(at_row);
  K.d.w_ptr = dev_upload(wptr);
  K.d.w_p = dev_upload(wp);
  K.d.w_j = dev_upload(wj);
  K.d.partials = dev_alloc<double>(kRedMaxBlocks * kRedMaxSlots);
  K.d.counter = dev_alloc<unsigned int>(1);
  GN_CUDA(cudaMemset(K.d.counter, 0, sizeof(unsigned int)));
  K.d.scratch = dev_alloc<double>(m > 0 ? m : 1);
  K.d.dvec = dev_alloc<double>(m > 0 ? m : 1);
  K.batch_cap = 1;
  if (cs) {
    GN_REQUIRE(cs->n == n && cs->nnz_h == nh && cs->nnz_j == nj, "condensed structure mismatch");
    const_cast<Condense *>(cs)->ensure_assembly_plan();
    const int64_t nk = static_cast<int64_t>(cs->indices.size());
    const int64_t np = cs->np;
    K.nk = nk;
    K.np = np;
    std::vector<int32_t> kw(nk, -1), kd(nk, -1);
    for (int64_t p = 0; p < nh; ++p) {
      GN_REQUIRE(kw[cs->w_map(p)] == -1, "duplicate W entry in a K slot");
      kw[cs->w_map(p)] = static_cast<int32_t>(p);
    }
    for (int64_t i = 0; i < n; ++i) kd[cs->diag_map(i)] = static_cast<int32_t>(i);
    K.d.k_ptr = dev_upload(cs->k_ptr);
    K.d.k_row = dev_upload(cs->k_row);
    K.d.k_s1 = dev_upload(cs->k_s1);
    K.d.k_s2 = dev_upload(cs->k_s2);
    K.d.k_w = dev_upload(kw);
    K.d.k_diag = dev_upload(kd);
    K.has_assembly = true;
  }
}

}  // namespace gn

using namespace gn;

#define ST(s) static_cast<cudaStream_t>(s)

extern "C" int gn_kkt_create(int64_t n, int64_t m, int64_t nh, const int64_t *hr, const int64_t *hc,
                             int64_t nj, const int64_t *jr, const int64_t *jc, const gn_condense *cs,
                             gn_kkt **out) {
  return guarded([&] {
    auto *K = new gn_kkt();
    try {
      kkt_create(*K, n, m, nh, hr, hc, nj, jr, jc, cs);
    } catch (...) {
      delete K;
      throw;
    }
    *out = K;
  });
}

extern "C" void gn_kkt_destroy(gn_kkt *K) { delete K; }

namespace gn {
// Scratch of batched launches: reduction partials/counters and the m-vectors
// (condensed-rhs u, assembly D) for B instances; grown on demand.  The
// stream is synchronised before a buffer is replaced (queued work may still
// read the old one).
void kkt_reserve(Kkt &K, int B, cudaStream_t st) {
  const int64_t blocks = static_cast<int64_t>(B) * kRedMaxBlocks;
  if (B <= K.batch_cap) return;
  GN_CUDA(cudaStreamSynchronize(st));
  dev_free(K.d.partials);
  dev_free(K.d.counter);
  dev_free(K.d.scratch);
  dev_free(K.d.dvec);
  K.d.partials = dev_alloc<double>(blocks * kRedMaxSlots);
  K.d.counter = dev_alloc<unsigned int>(B);
  GN_CUDA(cudaMemset(K.d.counter, 0, sizeof(unsigned int) * B));
  K.d.scratch = dev_alloc<double>(K.m > 0 ? K.m * B : 1);
  K.d.dvec = dev_alloc<double>(K.m > 0 ? K.m * B : 1);
  K.batch_cap = B;
}

namespace {
dim3 bgrid(unsigned gx, int B) { return dim3(gx, static_cast<unsigned>(B), 1); }

void assemble(Kkt &K, int B, const gn_kkt_state *st, const double *bp, double *kvals, cudaStream_t s) {
  GN_REQUIRE(K.has_assembly, "KKT plan built without the condensed structure");
  if (K.nk == 0) return;
  kkt_reserve(K, B, s);
  const Bx bx = bp ? batched(K, bp) : single(K);
  if (K.m) GN_LAUNCH(d_rows_kernel, bgrid(blocks_for(K.m), B), kT, 0, s, K.m, *st, K.d.dvec, bx);
  GN_LAUNCH(assemble_kernel, bgrid(blocks_for(K.nk), B), kT, 0, s, K.nk, K.d.k_ptr, K.d.k_row, K.d.k_s1,
            K.d.k_s2, K.d.k_w, K.d.k_diag, *st, K.d.dvec, kvals, bx);
}

void condense_rhs(Kkt &K, int B, const gn_kkt_state *st, const double *bp, const gn_vec7 *pv, double *qx,
                  double *qs, double *qy, double *rhs, cudaStream_t s) {
  kkt_reserve(K, B, s);
  const Bx bx = bp ? batched(K, bp) : single(K);
  if (K.m)
    GN_LAUNCH(rhs_rows_kernel, bgrid(blocks_for(K.m), B), kT, 0, s, K.m, *st, *pv, qs, qy, K.d.scratch, bx);
  if (K.n)
    GN_LAUNCH(rhs_cols_kernel, bgrid(blocks_for(K.n), B), kT, 0, s, K.n, K.d.at_ptr, K.d.at_p, K.d.at_row, *st,
              *pv, K.d.scratch, qx, rhs, bx);
}

void recover_sd(Kkt &K, int B, const gn_kkt_state *st, const double *bp, const double *dx, const double *qs,
                const double *qy, double *ds, double *dy, cudaStream_t s) {
  const Bx bx = bp ? batched(K, bp) : single(K);
  if (K.m)
    GN_LAUNCH(recover_sd_kernel, bgrid(blocks_for(K.m), B), kT, 0, s, K.m, K.d.a_rowptr, K.d.a_col, *st, dx, qs,
              qy, ds, dy, bx);
}

void recover_bd(Kkt &K, int B, const gn_kkt_state *st, const double *dx, const double *ds, const gn_vec7 *pv,
                double *dzxl, double *dzxu, double *dzsl, double *dzsu, int32_t *flags, cudaStream_t s) {
  if (K.n)
    GN_LAUNCH(recover_bd_kernel, bgrid(blocks_for(K.n), B), kT, 0, s, K.n, st->dxl, st->dxu, st->zxl, st->zxu,
              pv->zxl, pv->zxu, dx, dzxl, dzxu, flags);
  if (K.m)
    GN_LAUNCH(recover_bd_kernel, bgrid(blocks_for(K.m), B), kT, 0, s, K.m, st->dsl, st->dsu, st->zsl, st->zsu,
              pv->zsl, pv->zsu, ds, dzsl, dzsu, flags);
}

// norm[b * stride + 0] = residual max of instance b (norm[.. + 1] scratch)
void residual(Kkt &K, int B, const gn_kkt_state *st, const double *bp, const gn_vec7 *steps, const gn_vec7 *pv,
              gn_vec7 *res, double *norm, int64_t stride, cudaStream_t s) {
  kkt_reserve(K, B, s);
  const Bx bx = bp ? batched(K, bp) : single(K);
  RedSpec rx = max_spec(K, norm, stride);
  if (K.n)
    GN_LAUNCH(residual_x_kernel, bgrid(red_grid(K.n), B), kRedThreads, 0, s, K.n, K.d.w_ptr, K.d.w_p, K.d.w_j,
              K.d.at_ptr, K.d.at_p, K.d.at_row, *st, *steps, *pv, *res, rx, bx);
  else
    GN_CUDA(cudaMemsetAsync(norm, 0, sizeof(double), s));   // single instance only
  RedSpec rs = max_spec(K, norm + 1, stride);
  if (K.m)
    GN_LAUNCH(residual_s_kernel, bgrid(red_grid(K.m), B), kRedThreads, 0, s, K.m, K.d.a_rowptr, K.d.a_col, *st,
              *steps, *pv, *res, rs, bx);
  else
    GN_CUDA(cudaMemsetAsync(norm + 1, 0, sizeof(double), s));
  GN_LAUNCH(max2_kernel, (B + 127) / 128, 128, 0, s, norm, norm + 1, norm, B, stride);
}

void matrix_scale(Kkt &K, int B, const gn_kkt_state *st, const double *bp, double *out, int64_t stride,
                  cudaStream_t s) {
  kkt_reserve(K, B, s);
  const Bx bx = bp ? batched(K, bp) : single(K);
  int64_t big = std::max(std::max(K.n, K.m), std::max(K.nh, K.nj));
  RedSpec r = max_spec(K, out, stride);
  GN_LAUNCH(matrix_scale_kernel, bgrid(red_grid(big, 4), B), kRedThreads, 0, s, K.n, K.m, K.nh, K.nj, *st, r, bx);
}

void axpy7(Kkt &K, int B, gn_vec7 *y, const gn_vec7 *x, double alpha, const double *bp, cudaStream_t s) {
  int64_t len = std::max(K.n, K.m);
  if (len == 0) return;
  const Bx bx = bp ? batched(K, bp) : single(K);
  GN_LAUNCH(axpy7_kernel, bgrid(blocks_for(len), B), kT, 0, s, K.n, K.m, *y, *x, alpha, bx);
}
}  // namespace
}  // namespace gn

extern "C" int gn_kkt_sigma(int64_t len, const double *dl, const double *du, const double *zl,
                            const double *zu, double *sigma, void *stream) {
  return guarded([&] {
    if (len == 0) return;
    GN_LAUNCH(sigma_kernel, blocks_for(len), kT, 0, ST(stream), len, dl, du, zl, zu, sigma);
  });
}

extern "C" int gn_kkt_matvec(gn_kkt *K, int kind, const double *vals, const double *v, double *out,
                             void *stream) {
  return guarded([&] {
    if (kind == 0 && K->n)
      GN_LAUNCH(w_matvec_kernel, blocks_for(K->n), kT, 0, ST(stream), K->n, K->d.w_ptr, K->d.w_p, K->d.w_j, vals, v, out);
    else if (kind == 1 && K->m)
      GN_LAUNCH(a_matvec_kernel, blocks_for(K->m), kT, 0, ST(stream), K->m, K->d.a_rowptr, K->d.a_col, vals, v, out);
    else if (kind == 2 && K->n)
      GN_LAUNCH(at_matvec_kernel, blocks_for(K->n), kT, 0, ST(stream), K->n, K->d.at_ptr, K->d.at_p, K->d.at_row, vals, v, out);
  });
}

extern "C" int gn_kkt_assemble(gn_kkt *K, const gn_kkt_state *st, double *kvals, void *stream) {
  return guarded([&] { assemble(*K, 1, st, nullptr, kvals, ST(stream)); });
}

extern "C" int gn_kkt_assembly_traffic(const gn_kkt *K, int64_t *bytes) {
  return guarded([&] {
    GN_REQUIRE(K->has_assembly, "KKT plan built without the condensed structure");
    // index maps (kp, row/s1/s2, W and diagonal sources), inputs (A, W,
    // Sigma_x, Sigma_s; D written and read once), output K
    *bytes = 4 * (K->nk + 1) + 12 * K->np + 8 * K->nk + 8 * (K->nj + K->nh + K->n) + 8 * K->m * 3 + 8 * K->nk;
  });
}

extern "C" int gn_kkt_condense_rhs(gn_kkt *K, const gn_kkt_state *st, const gn_vec7 *pv, double *qx,
                                   double *qs, double *qy, double *rhs, void *stream) {
  return guarded([&] { condense_rhs(*K, 1, st, nullptr, pv, qx, qs, qy, rhs, ST(stream)); });
}

extern "C" int gn_kkt_recover_slack_dual(gn_kkt *K, const gn_kkt_state *st, const double *dx,
                                         const double *qs, const double *qy, double *ds, double *dy,
                                         void *stream) {
  return guarded([&] { recover_sd(*K, 1, st, nullptr, dx, qs, qy, ds, dy, ST(stream)); });
}

extern "C" int gn_kkt_recover_bound_duals(gn_kkt *K, const gn_kkt_state *st, const double *dx,
                                          const double *ds, const gn_vec7 *pv, double *dzxl, double *dzxu,
                                          double *dzsl, double *dzsu, int32_t *flags, void *stream) {
  return guarded([&] { recover_bd(*K, 1, st, dx, ds, pv, dzxl, dzxu, dzsl, dzsu, flags, ST(stream)); });
}

extern "C" int gn_kkt_residual(gn_kkt *K, const gn_kkt_state *st, const gn_vec7 *steps, const gn_vec7 *pv,
                               gn_vec7 *res, double *norm, void *stream) {
  return guarded([&] { residual(*K, 1, st, nullptr, steps, pv, res, norm, 0, ST(stream)); });
}

extern "C" int gn_kkt_matrix_scale(gn_kkt *K, const gn_kkt_state *st, double *out, void *stream) {
  return guarded([&] { matrix_scale(*K, 1, st, nullptr, out, 0, ST(stream)); });
}

extern "C" int gn_vec7_axpy(gn_kkt *K, gn_vec7 *y, const gn_vec7 *x, double alpha, void *stream) {
  return guarded([&] { axpy7(*K, 1, y, x, alpha, nullptr, ST(stream)); });
}

// ----------------------------------------------------------- batched (K12)
extern "C" int gn_kkt_assemble_batched(gn_kkt *K, int32_t B, const gn_kkt_state *st, const double *bp,
                                       double *kvals, void *stream) {
  return guarded([&] { assemble(*K, B, st, bp, kvals, ST(stream)); });
}

extern "C" int gn_kkt_condense_rhs_batched(gn_kkt *K, int32_t B, const gn_kkt_state *st, const double *bp,
                                           const gn_vec7 *pv, double *qx, double *qs, double *qy, double *rhs,
                                           void *stream) {
  return guarded([&] { condense_rhs(*K, B, st, bp, pv, qx, qs, qy, rhs, ST(stream)); });
}

extern "C" int gn_kkt_recover_slack_dual_batched(gn_kkt *K, int32_t B, const gn_kkt_state *st, const double *bp,
                                                 const double *dx, const double *qs, const double *qy, double *ds,
                                                 double *dy, void *stream) {
  return guarded([&] { recover_sd(*K, B, st, bp, dx, qs, qy, ds, dy, ST(stream)); });
}

extern "C" int gn_kkt_recover_bound_duals_batched(gn_kkt *K, int32_t B, const gn_kkt_state *st, const double *dx,
                                                  const double *ds, const gn_vec7 *pv, double *dzxl, double *dzxu,
                                                  double *dzsl, double *dzsu, int32_t *flags, void *stream) {
  return guarded([&] { recover_bd(*K, B, st, dx, ds, pv, dzxl, dzxu, dzsl, dzsu, flags, ST(stream)); });
}

extern "C" int gn_kkt_residual_batched(gn_kkt *K, int32_t B, const gn_kkt_state *st, const double *bp,
                                       const gn_vec7 *steps, const gn_vec7 *pv, gn_vec7 *res, double *norm,
                                       void *stream) {
  return guarded([&] { residual(*K, B, st, bp, steps, pv, res, norm, GN_BATCH_SCAL, ST(stream)); });
}

extern "C" int gn_kkt_matrix_scale_batched(gn_kkt *K, int32_t B, const gn_kkt_state *st, const double *bp,
                                           double *out, void *stream) {
  return guarded([&] { matrix_scale(*K, B, st, bp, out, GN_BATCH_SCAL, ST(stream)); });
}

extern "C" int gn_vec7_axpy_batched(gn_kkt *K, int32_t B, gn_vec7 *y, const gn_vec7 *x, const double *bp,
                                    void *stream) {
  return guarded([&] {
    GN_REQUIRE(bp != nullptr, "batched axpy needs the per-instance alpha array");
    axpy7(*K, B, y, x, 0.0, bp, ST(stream));
  });
}
