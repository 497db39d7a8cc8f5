// Interior-point vector algebra on the device (reference src/gridnlp/ipm.py:
// 150-157 kkt_residual, 340-346 barrier_phi, 393-442 iterate prep and right-
// hand side, 455-476 fraction-to-boundary and dphi, 482-492 trial merit,
// 521-548 step acceptance with the kappa_sigma safeguard).
//
// The prep/direction/merit kernels fuse the elementwise work with every
// reduction the host control flow branches on; each writes a small scalar
// block that the driver reads back in one copy.
#include <cmath>

#include "gather.cuh"
#include "reduce.cuh"

namespace gn {
namespace {

__device__ __forceinline__ double inv0(double w) { return isfinite(w) ? 1.0 / w : 0.0; }
__device__ __forceinline__ double width_lo(double v, double b) { return isfinite(b) ? v - b : INFINITY; }
__device__ __forceinline__ double width_hi(double v, double b) { return isfinite(b) ? b - v : INFINITY; }

struct MuList {
  int n;
  double mu[GN_IPM_MAX_MU];
  const double *dev;   // batched: [B][GN_IPM_MAX_MU] candidates on the device
};

__device__ __forceinline__ double mu_k(const MuList &mus, int k) {
  return mus.dev ? mus.dev[blockIdx.y * GN_IPM_MAX_MU + k] : mus.mu[k];
}

RedSpec spec(Kkt &K, double *out, int k, const int *ops, int64_t out_stride = 0) {
  RedSpec r{};
  r.k = k;
  for (int i = 0; i < k; ++i) r.op[i] = ops[i];
  r.out = out;
  r.partials = K.d.partials;
  r.counter = K.d.counter;
  r.out_stride = out_stride;
  return r;
}

__global__ void __launch_bounds__(kRedThreads)
prep_x_kernel(int64_t n, const int64_t *atptr, const int32_t *atp, const int32_t *atrow, gn_ipm_vecs v,
              MuList mus, RedSpec rs, Bx bx) {
  shift(v, bx);
  double acc[4 + GN_IPM_MAX_MU];
  acc[0] = 0.0;
  acc[1] = 0.0;
  acc[2] = 0.0;
  acc[3] = 0.0;
  for (int k = 0; k < mus.n; ++k) acc[4 + k] = 0.0;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; j < n;
       j += static_cast<int64_t>(gridDim.x) * kRedThreads) {
    const double x = v.x[j];
    const double wl = width_lo(x, v.xl[j]), wu = width_hi(x, v.xu[j]);
    const double zl = v.zxl[j], zu = v.zxu[j];
    v.dxl[j] = wl;
    v.dxu[j] = wu;
    v.sx[j] = __dadd_rn(__dmul_rn(zl, inv0(wl)), __dmul_rn(zu, inv0(wu)));
    const double aty = gather_dot_fma(atptr[j], atptr[j + 1], v.jac, [&](int64_t t) { return atp[t]; }, v.y,
                                      [&](int64_t t) { return atrow[t]; });
    const double dx = ((v.grad[j] + aty) - zl) + zu;
    v.dual_x[j] = dx;
    acc[0] = red_combine(RED_MAX, acc[0], fabs(dx));
    acc[1] += fabs(zl) + fabs(zu);
    const bool fl = isfinite(wl), fu = isfinite(wu);
    if (fl) acc[2] += log(wl);
    if (fu) acc[3] += log(wu);
    for (int k = 0; k < mus.n; ++k) {
      double c = 0.0;
      const double mk = mu_k(mus, k);
      if (fl) c = fabs(zl * wl - mk);
      if (fu) c = red_combine(RED_MAX, c, fabs(zu * wu - mk));
      acc[4 + k] = red_combine(RED_MAX, acc[4 + k], c);
    }
  }
  grid_reduce(rs, acc);
}

__global__ void __launch_bounds__(kRedThreads)
prep_s_kernel(int64_t m, gn_ipm_vecs v, MuList mus, RedSpec rs, Bx bx) {
  shift(v, bx);
  double acc[7 + GN_IPM_MAX_MU];
  for (int k = 0; k < 7 + mus.n; ++k) acc[k] = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * kRedThreads) {
    const double s = v.s[i], y = v.y[i];
    const double wl = width_lo(s, v.sl[i]), wu = width_hi(s, v.su[i]);
    const double zl = v.zsl[i], zu = v.zsu[i];
    v.dsl[i] = wl;
    v.dsu[i] = wu;
    v.ss[i] = __dadd_rn(__dmul_rn(zl, inv0(wl)), __dmul_rn(zu, inv0(wu)));
    const double ds = (-y - zl) + zu;
    const double pr = v.c[i] - s;
    v.dual_s[i] = ds;
    v.primal[i] = pr;
    acc[0] = red_combine(RED_MAX, acc[0], fabs(ds));
    acc[1] = red_combine(RED_MAX, acc[1], fabs(pr));
    acc[2] += fabs(zl) + fabs(zu);
    acc[3] += fabs(y);
    acc[4] += fabs(pr);
    const bool fl = isfinite(wl), fu = isfinite(wu);
    if (fl) acc[5] += log(wl);
    if (fu) acc[6] += log(wu);
    for (int k = 0; k < mus.n; ++k) {
      double c = 0.0;
      const double mk = mu_k(mus, k);
      if (fl) c = fabs(zl * wl - mk);
      if (fu) c = red_combine(RED_MAX, c, fabs(zu * wu - mk));
      acc[7 + k] = red_combine(RED_MAX, acc[7 + k], c);
    }
  }
  grid_reduce(rs, acc);
}

__global__ void pvec_kernel(int64_t n, int64_t m, gn_ipm_vecs v, double mu, gn_vec7 pv, Bx bx) {
  shift(v, bx);
  shift(pv, bx);
  mu = bpar(bx, GN_BP_MU, mu);
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const double wl = v.dxl[i], wu = v.dxu[i];
    pv.x[i] = -v.dual_x[i];
    pv.zxl[i] = (isfinite(wl) ? mu : 0.0) - v.zxl[i] * (isfinite(wl) ? wl : 0.0);
    pv.zxu[i] = (isfinite(wu) ? mu : 0.0) - v.zxu[i] * (isfinite(wu) ? wu : 0.0);
  }
  if (i < m) {
    const double wl = v.dsl[i], wu = v.dsu[i];
    pv.s[i] = -v.dual_s[i];
    pv.y[i] = -v.primal[i];
    pv.zsl[i] = (isfinite(wl) ? mu : 0.0) - v.zsl[i] * (isfinite(wl) ? wl : 0.0);
    pv.zsu[i] = (isfinite(wu) ? mu : 0.0) - v.zsu[i] * (isfinite(wu) ? wu : 0.0);
  }
}

// fraction to the boundary for one primal entry (ipm.py:265-273)
__device__ __forceinline__ double ftb1(double val, double dv, double lo, double hi, double tau) {
  double a = 1.0;
  if (dv < 0 && isfinite(lo)) a = fmin(a, -tau * (val - lo) / dv);
  if (dv > 0 && isfinite(hi)) a = fmin(a, tau * (hi - val) / dv);
  return a;
}
__device__ __forceinline__ double dftb1(double z, double dz, double tau) {
  return dz < 0 ? -tau * z / dz : 1.0;
}

__global__ void __launch_bounds__(kRedThreads)
direction_kernel(int64_t n, int64_t m, gn_ipm_vecs v, gn_vec7 st, double mu, double tau, RedSpec rs, Bx bx) {
  shift(v, bx);
  shift(st, bx);
  mu = bpar(bx, GN_BP_MU, mu);
  tau = bpar(bx, GN_BP_TAU, tau);
  double acc[4] = {1.0, 1.0, 1.0, 0.0};
  const int64_t len = n > m ? n : m;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * kRedThreads) {
    if (i < n) {
      acc[0] = fmin(acc[0], ftb1(v.x[i], st.x[i], v.xl[i], v.xu[i], tau));
      acc[2] = fmin(acc[2], fmin(dftb1(v.zxl[i], st.zxl[i], tau), dftb1(v.zxu[i], st.zxu[i], tau)));
      double g = v.grad[i];
      if (isfinite(v.dxl[i])) g -= mu / v.dxl[i];
      if (isfinite(v.dxu[i])) g += mu / v.dxu[i];
      acc[3] += g * st.x[i];
    }
    if (i < m) {
      acc[1] = fmin(acc[1], ftb1(v.s[i], st.s[i], v.sl[i], v.su[i], tau));
      acc[2] = fmin(acc[2], fmin(dftb1(v.zsl[i], st.zsl[i], tau), dftb1(v.zsu[i], st.zsu[i], tau)));
      double g = 0.0;
      if (isfinite(v.dsl[i])) g -= mu / v.dsl[i];
      if (isfinite(v.dsu[i])) g += mu / v.dsu[i];
      acc[3] += g * st.s[i];
    }
  }
  grid_reduce(rs, acc);
}

__global__ void trial_point_kernel(int64_t n, int64_t m, gn_ipm_vecs v, gn_vec7 st, double alpha,
                                   double *xt, double *s_t, Bx bx) {
  shift(v, bx);
  shift(st, bx);
  alpha = bpar(bx, GN_BP_ALPHA, alpha);
  xt = shift_ptr(xt, n);
  s_t = shift_ptr(s_t, m);
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) xt[i] = v.x[i] + alpha * st.x[i];
  if (i < m) s_t[i] = v.s[i] + alpha * st.s[i];
}

// first trial of the line search at alpha_max = min(alpha_x, alpha_s) read
// from the device (Python's min(a0, a1)), so it needs no host round trip
__global__ void trial_point_at_kernel(int64_t n, int64_t m, gn_ipm_vecs v, gn_vec7 st,
                                      const double *alpha_pair, double *xt, double *s_t, Bx bx) {
  shift(v, bx);
  shift(st, bx);
  alpha_pair = shift_ptr(alpha_pair, GN_BATCH_SCAL);
  xt = shift_ptr(xt, n);
  s_t = shift_ptr(s_t, m);
  const double a0 = alpha_pair[0], a1 = alpha_pair[1];
  const double alpha = a1 < a0 ? a1 : a0;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) xt[i] = v.x[i] + alpha * st.x[i];
  if (i < m) s_t[i] = v.s[i] + alpha * st.s[i];
}

__global__ void __launch_bounds__(kRedThreads)
trial_merit_kernel(int64_t n, int64_t m, gn_ipm_vecs v, const double *ct, const double *xt,
                   const double *s_t, RedSpec rs, Bx bx) {
  shift(v, bx);
  ct = shift_ptr(ct, m);
  xt = shift_ptr(xt, n);
  s_t = shift_ptr(s_t, m);
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const int64_t len = n > m ? n : m;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * kRedThreads) {
    if (i < n) {
      const double x = xt[i];
      if (isfinite(v.xl[i])) acc[1] += log(x - v.xl[i]);
      if (isfinite(v.xu[i])) acc[2] += log(v.xu[i] - x);
    }
    if (i < m) {
      const double s = s_t[i];
      acc[0] += fabs(ct[i] - s);
      if (isfinite(v.sl[i])) acc[3] += log(s - v.sl[i]);
      if (isfinite(v.su[i])) acc[4] += log(v.su[i] - s);
    }
  }
  grid_reduce(rs, acc);
}

__device__ __forceinline__ double safeguard(double z, double w, double mu, double ks) {
  if (!isfinite(w)) return z;
  return fmin(fmax(z, mu / (ks * w)), ks * mu / w);
}

__global__ void accept_kernel(int64_t n, int64_t m, gn_ipm_vecs v, gn_vec7 st, double alpha, double az,
                              double mu, double ks, int32_t *flags, Bx bx) {
  if (!b_active(bx)) return;
  shift(v, bx);
  shift(st, bx);
  alpha = bpar(bx, GN_BP_ALPHA, alpha);
  az = bpar(bx, GN_BP_ALPHA_Z, az);
  mu = bpar(bx, GN_BP_MU, mu);
  flags = shift_ptr(flags, 1);
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const double x = v.x[i] + alpha * st.x[i];
    v.x[i] = x;
    const double wl = width_lo(x, v.xl[i]), wu = width_hi(x, v.xu[i]);
    v.zxl[i] = safeguard(v.zxl[i] + az * st.zxl[i], wl, mu, ks);
    v.zxu[i] = safeguard(v.zxu[i] + az * st.zxu[i], wu, mu, ks);
    if ((isfinite(wl) && !(wl > 0.0)) || (isfinite(wu) && !(wu > 0.0))) atomicOr(flags, 2);
  }
  if (i < m) {
    const double s = v.s[i] + alpha * st.s[i];
    v.s[i] = s;
    v.y[i] = v.y[i] + alpha * st.y[i];
    const double wl = width_lo(s, v.sl[i]), wu = width_hi(s, v.su[i]);
    v.zsl[i] = safeguard(v.zsl[i] + az * st.zsl[i], wl, mu, ks);
    v.zsu[i] = safeguard(v.zsu[i] + az * st.zsu[i], wu, mu, ks);
    if ((isfinite(wl) && !(wl > 0.0)) || (isfinite(wu) && !(wu > 0.0))) atomicOr(flags, 4);
  }
}

unsigned ew_blocks(int64_t len) { return static_cast<unsigned>(len > 0 ? (len + 255) / 256 : 1); }

// ---- problem setup: frozen gradient scaling at x0 (ipm.py:179-193),
// relax_equalities on the scaled ranges (ipm.py:112-123), the start point,
// the unit bound duals (ipm.py:360-369) and the initial slacks from g(x0)
// (ipm.py:371-380) -- one elementwise pass each instead of a chain of
// tensor ops.  The maxima go through atomicMax on the IEEE bits of |v|
// (non-negative doubles order like their bit patterns, and a NaN bit
// pattern wins like numpy's max), so they are exact and order-free.
__device__ __forceinline__ unsigned long long abs_bits(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(fabs(v)));
}
__device__ __forceinline__ double nan_max(double a, double b) {   // torch.maximum
  return (a != a || b != b) ? NAN : (a > b ? a : b);
}
__device__ __forceinline__ double nan_min(double a, double b) {   // torch.minimum
  return (a != a || b != b) ? NAN : (a < b ? a : b);
}
__device__ __forceinline__ double unit_scale(double mx) {   // where(mx > 0, min(100 / mx, 1), 1)
  return mx > 0.0 ? fmin(__ddiv_rn(100.0, mx), 1.0) : 1.0;
}

__global__ void setup_max_kernel(int64_t n, const double *__restrict__ g0, int64_t nj,
                                 const double *__restrict__ j0, const int64_t *__restrict__ jrow,
                                 unsigned long long *bits /* [0] max |g0|, [1 + i] row i max |j0| */) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long gm = 0;
  for (int64_t i = t0; i < n; i += stride) gm = max(gm, abs_bits(g0[i]));
  for (int o = 16; o; o >>= 1) gm = max(gm, __shfl_xor_sync(0xffffffffu, gm, o));
  if ((threadIdx.x & 31) == 0 && gm) atomicMax(bits, gm);
  for (int64_t t = t0; t < nj; t += stride) {
    const unsigned long long v = abs_bits(j0[t]);
    if (v) atomicMax(bits + 1 + jrow[t], v);
  }
}

__global__ void setup_vec_kernel(int64_t n, int64_t m, int scaling, double tol,
                                 const unsigned long long *__restrict__ bits, const double *__restrict__ x0,
                                 const double *__restrict__ xl, const double *__restrict__ xu,
                                 const double *__restrict__ rlo, const double *__restrict__ rhi, double *x,
                                 double *s, double *y, double *zxl, double *zxu, double *zsl, double *zsu,
                                 double *con_scale, double *sl, double *su, double *obj_scale) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) *obj_scale = scaling ? unit_scale(__longlong_as_double(static_cast<long long>(bits[0]))) : 1.0;
  if (i < n) {
    x[i] = x0[i];
    zxl[i] = isfinite(xl[i]) ? 1.0 : 0.0;
    zxu[i] = isfinite(xu[i]) ? 1.0 : 0.0;
  }
  if (i < m) {
    const double cs = scaling ? unit_scale(__longlong_as_double(static_cast<long long>(bits[1 + i]))) : 1.0;
    con_scale[i] = cs;
    const double lo = __dmul_rn(rlo[i], cs), hi = __dmul_rn(rhi[i], cs);
    const double l = isfinite(lo) ? __dsub_rn(lo, __dmul_rn(tol, nan_max(1.0, fabs(lo)))) : -INFINITY;
    const double u = isfinite(hi) ? __dadd_rn(hi, __dmul_rn(tol, nan_max(1.0, fabs(hi)))) : INFINITY;
    sl[i] = l;
    su[i] = u;
    zsl[i] = isfinite(l) ? 1.0 : 0.0;
    zsu[i] = isfinite(u) ? 1.0 : 0.0;
    s[i] = 0.0;
    y[i] = 0.0;
  }
}

__global__ void __launch_bounds__(kRedThreads)
init_slacks_kernel(int64_t m, const double *__restrict__ g, const double *__restrict__ sl,
                   const double *__restrict__ su, double push_tol, double *s, RedSpec rs) {
  double acc[1] = {0.0};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * kRedThreads) {
    const double l = sl[i], u = su[i];
    const double lo = isfinite(l) ? __dadd_rn(l, push_tol) : -INFINITY;
    const double hi = isfinite(u) ? __dsub_rn(u, push_tol) : INFINITY;
    double s0 = nan_min(nan_max(g[i], lo), hi);
    if (lo > hi) s0 = __dmul_rn(0.5, __dadd_rn(l, u));
    s[i] = s0;
    acc[0] += fabs(__dsub_rn(g[i], s0));
  }
  grid_reduce(rs, acc);
}

}  // namespace
}  // namespace gn

using namespace gn;
#define ST(s) static_cast<cudaStream_t>(s)

namespace gn {
void kkt_reserve(Kkt &K, int B, cudaStream_t st);   // kkt.cu
namespace {
dim3 bgrid(unsigned gx, int B) { return dim3(gx, static_cast<unsigned>(B), 1); }
Bx bx_of(const Kkt &K, const double *bp) { return Bx{bp, K.n, K.m, K.nh, K.nj}; }

void prep(Kkt &K, int B, const gn_ipm_vecs *v, int n_mu, const double *mus_host, const double *mus_dev,
          const double *bp, double *scal, int64_t sstride, cudaStream_t s) {
  GN_REQUIRE(n_mu >= 0 && n_mu <= GN_IPM_MAX_MU, "too many barrier candidates");
  kkt_reserve(K, B, s);
  MuList mus{};
  mus.n = n_mu;
  mus.dev = mus_dev;
  if (mus_host)
    for (int k = 0; k < n_mu; ++k) mus.mu[k] = mus_host[k];
  int ops_x[4 + GN_IPM_MAX_MU] = {RED_MAX, RED_SUM, RED_SUM, RED_SUM};
  for (int k = 0; k < n_mu; ++k) ops_x[4 + k] = RED_MAX;
  int ops_s[7 + GN_IPM_MAX_MU] = {RED_MAX, RED_MAX, RED_SUM, RED_SUM, RED_SUM, RED_SUM, RED_SUM};
  for (int k = 0; k < n_mu; ++k) ops_s[7 + k] = RED_MAX;
  if (B == 1) {
    GN_CUDA(cudaMemsetAsync(scal, 0, sizeof(double) * GN_PREP_DOUBLES, s));
  } else {
    GN_CUDA(cudaMemset2DAsync(scal, sizeof(double) * sstride, 0, sizeof(double) * GN_PREP_DOUBLES, B, s));
  }
  const Bx bx = bx_of(K, bp);
  if (K.n)
    GN_LAUNCH(prep_x_kernel, bgrid(red_grid(K.n), B), kRedThreads, 0, s, K.n, K.d.at_ptr, K.d.at_p, K.d.at_row,
              *v, mus, spec(K, scal, 4 + n_mu, ops_x, sstride), bx);
  if (K.m)
    GN_LAUNCH(prep_s_kernel, bgrid(red_grid(K.m), B), kRedThreads, 0, s, K.m, *v, mus,
              spec(K, scal + GN_PREP_S, 7 + n_mu, ops_s, sstride), bx);
}
}  // namespace
}  // namespace gn

extern "C" int gn_ipm_prep(gn_kkt *K, const gn_ipm_vecs *v, int32_t n_mu, const double *mus_host,
                           double *scal, void *stream) {
  return guarded([&] { prep(*K, 1, v, n_mu, mus_host, nullptr, nullptr, scal, 0, ST(stream)); });
}

extern "C" int gn_ipm_pvec(gn_kkt *K, const gn_ipm_vecs *v, double mu, gn_vec7 *pv, void *stream) {
  return guarded([&] {
    GN_LAUNCH(pvec_kernel, ew_blocks(std::max(K->n, K->m)), 256, 0, ST(stream), K->n, K->m, *v, mu, *pv,
              bx_of(*K, nullptr));
  });
}

extern "C" int gn_ipm_direction(gn_kkt *K, const gn_ipm_vecs *v, const gn_vec7 *steps, double mu, double tau,
                                double *scal, void *stream) {
  return guarded([&] {
    int ops[4] = {RED_MIN, RED_MIN, RED_MIN, RED_SUM};
    GN_LAUNCH(direction_kernel, red_grid(std::max(K->n, K->m)), kRedThreads, 0, ST(stream), K->n, K->m, *v,
              *steps, mu, tau, spec(*K, scal, 4, ops), bx_of(*K, nullptr));
  });
}

extern "C" int gn_ipm_trial_point(gn_kkt *K, const gn_ipm_vecs *v, const gn_vec7 *steps, double alpha,
                                  double *xt, double *st, void *stream) {
  return guarded([&] {
    GN_LAUNCH(trial_point_kernel, ew_blocks(std::max(K->n, K->m)), 256, 0, ST(stream), K->n, K->m, *v, *steps,
              alpha, xt, st, bx_of(*K, nullptr));
  });
}

extern "C" int gn_ipm_trial_point_at(gn_kkt *K, const gn_ipm_vecs *v, const gn_vec7 *steps,
                                     const double *alpha_pair, double *xt, double *st, void *stream) {
  return guarded([&] {
    GN_LAUNCH(trial_point_at_kernel, ew_blocks(std::max(K->n, K->m)), 256, 0, ST(stream), K->n, K->m, *v,
              *steps, alpha_pair, xt, st, bx_of(*K, nullptr));
  });
}

extern "C" int gn_ipm_trial_merit(gn_kkt *K, const gn_ipm_vecs *v, const double *ct, const double *xt,
                                  const double *st, double *scal, void *stream) {
  return guarded([&] {
    int ops[5] = {RED_SUM, RED_SUM, RED_SUM, RED_SUM, RED_SUM};
    GN_LAUNCH(trial_merit_kernel, red_grid(std::max(K->n, K->m)), kRedThreads, 0, ST(stream), K->n, K->m, *v,
              ct, xt, st, spec(*K, scal, 5, ops), bx_of(*K, nullptr));
  });
}

extern "C" int gn_ipm_accept(gn_kkt *K, const gn_ipm_vecs *v, const gn_vec7 *steps, double alpha,
                             double alpha_z, double mu, double kappa_sigma, int32_t *flags, void *stream) {
  return guarded([&] {
    GN_LAUNCH(accept_kernel, ew_blocks(std::max(K->n, K->m)), 256, 0, ST(stream), K->n, K->m, *v, *steps, alpha,
              alpha_z, mu, kappa_sigma, flags, bx_of(*K, nullptr));
  });
}

// ----------------------------------------------------------- batched (K12)
// bp: [B][GN_BP_STRIDE] per-instance operands; scal: [B][GN_BATCH_SCAL]
extern "C" int gn_ipm_prep_batched(gn_kkt *K, int32_t B, const gn_ipm_vecs *v, int32_t n_mu, const double *mus_dev,
                                   double *scal, void *stream) {
  return guarded([&] { prep(*K, B, v, n_mu, nullptr, mus_dev, nullptr, scal, GN_BATCH_SCAL, ST(stream)); });
}

extern "C" int gn_ipm_pvec_batched(gn_kkt *K, int32_t B, const gn_ipm_vecs *v, const double *bp, gn_vec7 *pv,
                                   void *stream) {
  return guarded([&] {
    GN_LAUNCH(pvec_kernel, bgrid(ew_blocks(std::max(K->n, K->m)), B), 256, 0, ST(stream), K->n, K->m, *v, 0.0,
              *pv, bx_of(*K, bp));
  });
}

extern "C" int gn_ipm_direction_batched(gn_kkt *K, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps,
                                        const double *bp, double *scal, void *stream) {
  return guarded([&] {
    kkt_reserve(*K, B, ST(stream));
    int ops[4] = {RED_MIN, RED_MIN, RED_MIN, RED_SUM};
    GN_LAUNCH(direction_kernel, bgrid(red_grid(std::max(K->n, K->m)), B), kRedThreads, 0, ST(stream), K->n, K->m,
              *v, *steps, 0.0, 0.0, spec(*K, scal, 4, ops, GN_BATCH_SCAL), bx_of(*K, bp));
  });
}

extern "C" int gn_ipm_trial_point_batched(gn_kkt *K, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps,
                                          const double *bp, double *xt, double *st, void *stream) {
  return guarded([&] {
    GN_LAUNCH(trial_point_kernel, bgrid(ew_blocks(std::max(K->n, K->m)), B), 256, 0, ST(stream), K->n, K->m, *v,
              *steps, 0.0, xt, st, bx_of(*K, bp));
  });
}

extern "C" int gn_ipm_trial_point_at_batched(gn_kkt *K, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps,
                                             const double *alpha_pairs, double *xt, double *st, void *stream) {
  return guarded([&] {
    GN_LAUNCH(trial_point_at_kernel, bgrid(ew_blocks(std::max(K->n, K->m)), B), 256, 0, ST(stream), K->n, K->m,
              *v, *steps, alpha_pairs, xt, st, bx_of(*K, nullptr));
  });
}

extern "C" int gn_ipm_trial_merit_batched(gn_kkt *K, int32_t B, const gn_ipm_vecs *v, const double *ct,
                                          const double *xt, const double *st, double *scal, void *stream) {
  return guarded([&] {
    kkt_reserve(*K, B, ST(stream));
    int ops[5] = {RED_SUM, RED_SUM, RED_SUM, RED_SUM, RED_SUM};
    GN_LAUNCH(trial_merit_kernel, bgrid(red_grid(std::max(K->n, K->m)), B), kRedThreads, 0, ST(stream), K->n,
              K->m, *v, ct, xt, st, spec(*K, scal, 5, ops, GN_BATCH_SCAL), bx_of(*K, nullptr));
  });
}

extern "C" int gn_ipm_accept_batched(gn_kkt *K, int32_t B, const gn_ipm_vecs *v, const gn_vec7 *steps,
                                     const double *bp, double kappa_sigma, int32_t *flags, void *stream) {
  return guarded([&] {
    GN_LAUNCH(accept_kernel, bgrid(ew_blocks(std::max(K->n, K->m)), B), 256, 0, ST(stream), K->n, K->m, *v,
              *steps, 0.0, 0.0, 0.0, kappa_sigma, flags, bx_of(*K, bp));
  });
}

extern "C" int gn_ipm_setup(int64_t n, int64_t m, int64_t nj, const double *g0, const double *j0,
                            const int64_t *jac_rows, const double *x0, const double *xl, const double *xu,
                            const double *rlo, const double *rhi, int32_t scaling, double tol_r,
                            uint64_t *scratch, double *x, double *s, double *y, double *zxl, double *zxu,
                            double *zsl, double *zsu, double *con_scale, double *sl, double *su,
                            double *obj_scale, void *stream) {
  return guarded([&] {
    GN_REQUIRE(n >= 0 && m >= 0 && nj >= 0, "negative size");
    auto *bits = reinterpret_cast<unsigned long long *>(scratch);
    GN_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long) * (m + 1), ST(stream)));
    if (scaling && (n || nj))
      GN_LAUNCH(setup_max_kernel, ew_blocks(std::max(n, nj)), 256, 0, ST(stream), n, g0, nj, j0, jac_rows, bits);
    GN_LAUNCH(setup_vec_kernel, ew_blocks(std::max<int64_t>(1, std::max(n, m))), 256, 0, ST(stream), n, m,
              static_cast<int>(scaling), tol_r, bits, x0, xl, xu, rlo, rhi, x, s, y, zxl, zxu, zsl, zsu,
              con_scale, sl, su, obj_scale);
  });
}

extern "C" int gn_ipm_init_slacks(int64_t m, const double *g, const double *sl, const double *su,
                                  double push_tol, double *s, double *theta, double *red_partials,
                                  uint32_t *red_counter, void *stream) {
  return guarded([&] {
    if (m <= 0) return;
    RedSpec r{};
    r.k = 1;
    r.op[0] = RED_SUM;
    r.out = theta;
    r.partials = red_partials;
    r.counter = red_counter;
    GN_LAUNCH(init_slacks_kernel, red_grid(m), kRedThreads, 0, ST(stream), m, g, sl, su, push_tol, s, r);
  });
}
