"""Condensed-space interior-point loop with every iterate resident in HBM.

Same algorithm, options, statuses and report as reference
src/gridnlp/ipm.py (Algorithm 1): equality relaxation, frozen
gradient scaling, the kappa_eps barrier update, the condensed Newton step
with double-double refinement, fraction-to-boundary, the filter / Armijo
line search and the kappa_sigma dual safeguard.

The driver stays in Python and only sequences device work: AD kernels
(csrc/ad.cu), fused iterate/merit reductions (csrc/ipm.cu), condensed
assembly and recoveries (csrc/kkt.cu) and the multifrontal factor/solve
(csrc/chol.cu).  Host <-> device traffic per iteration is a handful of
scalar blocks at the points where the reference's control flow branches
(residual norms, PD flag, refinement norms, step lengths, trial merits).
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .autodiff import C, F, GRAD, HESS, JAC, RESET, NonFiniteResult, evaluator
from .kkt import (CondensedBackend, DegenerateInterior, FactorizationFailed, HostAnalysis,
                  KKTWorkspace, PVec, RegState, RegularizationExhausted, Steps, assemble_steps,
                  iterative_refinement, solve_with_regularization)
from .profiling import span

OPTIMAL = "optimal"
MAX_ITER = "max_iter"
REGULARIZATION_EXHAUSTED = "regularization_exhausted"
LINE_SEARCH_FAILURE = "line_search_failure"
EVAL_ERROR = "eval_error"


@dataclass
class SolverOptions:
    """Options and defaults of the reference (ipm.py:43-74)."""
    tol: float = 1e-4
    max_iter: int = 3000
    mu_init: float = 0.1
    bound_push: float = 0.01
    bound_relax: float | None = None
    mu_min: float | None = None
    kappa_eps: float = 10.0
    kappa_mu: float = 0.2
    theta_mu: float = 1.5
    tau_min: float = 0.99
    eta_phi: float = 1e-8
    gamma_theta: float = 1e-5
    gamma_phi: float = 1e-5
    s_theta: float = 1.1
    s_phi: float = 2.3
    delta: float = 1.0
    kappa_sigma: float = 1e10
    alpha_min: float = 1e-12
    s_max: float = 100.0
    fixed_var_eps: float = 1e-8
    scaling: bool = True
    backend: str = "condensed"
    log_level: int = 0
    record_trace: bool = True
    keep_workspace: bool = False
    ordering: object = None   # optional injected fill-reducing permutation

    def __post_init__(self):
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")
        if self.backend != "condensed":
            raise ValueError("only the condensed GPU backend is provided "
                             "(the dense augmented LDL^T is the CPU oracle's)")


@dataclass
class SolveReport:
    status: str
    objective: float = np.nan
    constraint_violation: float = np.nan
    residual_scaled: float = np.nan
    iterations: int = 0
    seconds: dict = field(default_factory=dict)
    final_mu: float = np.nan
    n_var: int = 0
    n_con: int = 0
    refinement_relative_residual: float = np.nan
    message: str = ""
    x: np.ndarray | None = None
    trace: list = field(default_factory=list)
    debug: dict = field(default_factory=dict)

    @property
    def success(self) -> bool:
        return self.status == OPTIMAL


# -- host helpers (once per solve; identical to the reference) -------------
def relax_equalities(m, ranges, tol):
    """Slack intervals (ipm.py:112-123)."""
    if ranges is None:
        lo, hi = np.zeros(m), np.zeros(m)
    else:
        r = np.asarray(ranges, dtype=float)
        lo, hi = r[:, 0].copy(), r[:, 1].copy()
    with np.errstate(invalid="ignore"):
        sl = np.where(np.isfinite(lo), lo - tol * np.maximum(1.0, np.abs(lo)), -np.inf)
        su = np.where(np.isfinite(hi), hi + tol * np.maximum(1.0, np.abs(hi)), np.inf)
    return sl, su


def initial_slacks(g0, sl, su, tol, push):
    """Clamp g(x0) into the strict interior (ipm.py:126-134)."""
    lo = np.where(np.isfinite(sl), sl + push * tol, -np.inf)
    hi = np.where(np.isfinite(su), su - push * tol, np.inf)
    s = np.minimum(np.maximum(g0, lo), hi)
    crossed = lo > hi
    return np.where(crossed, 0.5 * (sl + su), s) if np.any(crossed) else s


def kkt_residual(dual_x, dual_s, primal, comps, z_l1, y_l1, m, n_bounds, s_max=100.0):
    """Scaled optimality residual (ipm.py:150-157) from arrays."""
    amax = lambda *arrs: max([0.0] + [float(np.abs(a).max()) for a in arrs if np.size(a)])
    return kkt_residual_scalars(max(amax(dual_x), amax(dual_s)), amax(primal), amax(*comps),
                                z_l1, y_l1, m, n_bounds, s_max)


def kkt_residual_scalars(dual_max, primal_max, comp_max, z_l1, y_l1, m, n_bounds, s_max=100.0):
    """Same residual from the device reductions."""
    s_d = max(s_max, (y_l1 + z_l1) / max(1, m + n_bounds)) / s_max
    s_c = max(s_max, z_l1 / max(1, n_bounds)) / s_max
    comp = comp_max / s_c if n_bounds else 0.0
    return max(dual_max / s_d, primal_max, comp)


class _Filter:
    def __init__(self):
        self.entries: list[tuple[float, float]] = []

    def acceptable(self, theta, phi):
        return all(theta < th or phi < ph for th, ph in self.entries)

    def add(self, theta, phi):
        self.entries = [(th, ph) for th, ph in self.entries if not (th >= theta and ph >= phi)]
        self.entries.append((theta, phi))

    def clear(self):
        self.entries.clear()


def _mu_candidates(mu, mu_min, opts, k):
    """[0, mu, update(mu), ...] -- the values the barrier loop may visit."""
    out = [0.0, mu]
    cur = mu
    while len(out) < k and cur > mu_min * (1 + 1e-12):
        cur = max(mu_min, min(opts.kappa_mu * cur, cur ** opts.theta_mu))
        out.append(cur)
    return out


class _Timer:
    """Host perf_counter phase splits, as the reference keeps them
    (ipm.py:381-391, 431-453).  CUDA events here cost ~5-10 us of Python per
    record on the solver's critical path (the GPU waits on the host there);
    device-side kernel times come from profiling.span / bench.py instead."""

    def __init__(self):
        self.spans = {"ad": 0.0, "linear": 0.0}

    @staticmethod
    def start():
        return time.perf_counter()

    def stop(self, name, t0):
        self.spans[name] += time.perf_counter() - t0

    def totals(self):
        return dict(self.spans)


def _prepared_inputs(model, opts, ranges) -> dict:
    """Bounds with fixed variables widened, the pushed-in start point, the
    constraint ranges and the bound count (host and device), prepared once
    and kept on the model while the raw inputs are unchanged (compared by
    value; dropped by ``release_device``)."""
    m = model.n_con
    rr = None if ranges is None else np.asarray(ranges, dtype=float)
    raw = (model.lower, model.upper, model.start, rr)
    c = model.__dict__.get("_prepared_inputs")
    if c is not None and c["eps"] == opts.fixed_var_eps and all(
            (a is None and b is None) or (a is not None and b is not None and a.shape == b.shape
                                          and np.array_equal(a, b))
            for a, b in zip(c["raw"], raw)):
        return c
    xl, xu = model.lower.copy(), model.upper.copy()
    fixed = xl == xu
    if np.any(fixed):
        eps = opts.fixed_var_eps * np.maximum(1.0, np.abs(xl))
        xl, xu = np.where(fixed, xl - eps, xl), np.where(fixed, xu + eps, xu)
    x0 = np.minimum(np.maximum(model.start, xl), xu)
    if rr is None:
        rlo, rhi = np.zeros(m), np.zeros(m)
    else:
        rlo, rhi = rr[:, 0].copy(), rr[:, 1].copy()
    c = {"eps": opts.fixed_var_eps, "raw": tuple(None if a is None else a.copy() for a in raw),
         "xl": xl, "xu": xu, "x0": x0, "rlo": rlo, "rhi": rhi,
         # scaling keeps finiteness, so the bound count needs no device data
         "n_bounds": int(np.isfinite(xl).sum() + np.isfinite(xu).sum()
                         + np.isfinite(rlo).sum() + np.isfinite(rhi).sum()),
         "xl_d": D.to_dev(xl), "xu_d": D.to_dev(xu), "x0_d": D.to_dev(x0),
         "rlo_d": D.to_dev(rlo) if m else None, "rhi_d": D.to_dev(rhi) if m else None}
    model.__dict__["_prepared_inputs"] = c
    return c


class _DeviceSolve:
    """Device buffers and scalar mailboxes of one solve."""

    def __init__(self, model, opts, ranges):
        self.model = model
        self.opts = opts
        n, m = model.n_var, model.n_con
        self.n, self.m = n, m
        self.tol_r = opts.bound_relax if opts.bound_relax is not None else opts.tol
        pin = _prepared_inputs(model, opts, ranges)
        xl, xu = pin["xl"], pin["xu"]
        self.xl_h, self.xu_h = xl, xu
        self.x0 = pin["x0"]
        self.ev = evaluator(model)
        dev = D.require_cuda()
        self.dev = dev
        self.obj_scale = 1.0
        # scalar mailbox: [0:48) prep | 48 f | 49 f_trial | 50.. misc, then the
        # two int32 flag words [AD flags, IPM flags] in the last double, so one
        # copy brings scalars and flags back; the AD kernels write their flags
        # into it directly
        self.mail = D.zeros(97)
        self.scal = self.mail[:96]
        self.flags = self.mail[96:].view(torch.int32)
        self.flag_ad = self.flags[0:1]
        self.host_mail = torch.zeros(97, dtype=torch.float64, pin_memory=True)
        self.host = self.host_mail[:96]
        self.host_flags = self.host_mail[96:].view(torch.int32)
        self.stream = torch.cuda.current_stream()
        # the Newton right-hand side (independent of the factorisation) is
        # built on a second stream while the speculative factorisation runs
        self.aux = torch.cuda.Stream(device=dev)
        self.ev_prep, self.ev_rhs = torch.cuda.Event(), torch.cuda.Event()
        # frozen gradient scaling at x0 (ipm.py:179-193), relax_equalities on
        # the scaled ranges (ipm.py:112-123), the start point and the unit
        # bound duals, all on the device (gn_ipm_setup); the flags of the
        # scaling evaluation land in the mailbox's second word and obj_scale
        # in scal[61], so one read later brings obj_scale, theta0 and both
        # evaluations' flags back
        x0d = pin["x0_d"]
        g0 = D.empty(n)
        j0 = D.empty(max(1, model.nnz_jac))
        self.ev.launch(x0d, GRAD | JAC, grad=g0, jac=j0, flags=self.flags[1:2])
        self.rlo, self.rhi = pin["rlo"], pin["rhi"]
        self.rlo_d, self.rhi_d = pin["rlo_d"], pin["rhi_d"]
        self.n_bounds = pin["n_bounds"]
        self.xl, self.xu = pin["xl_d"], pin["xu_d"]
        mm = max(1, m)
        self.x = D.empty(n)
        self.s, self.y = D.empty(m), D.empty(m)
        self.zxl, self.zxu = D.empty(n), D.empty(n)
        self.zsl, self.zsu = D.empty(m), D.empty(m)
        self.con_scale, self.sl, self.su = D.empty(mm), D.empty(mm), D.empty(mm)
        if not m:   # placeholders the kernels never read
            self.con_scale.fill_(0.0 if opts.scaling else 1.0)
            self.sl.zero_()
            self.su.zero_()
        bits = torch.empty(m + 1, dtype=torch.int64, device=dev)
        L.check(L.lib().gn_ipm_setup(
            n, m, model.nnz_jac, L.ptr(g0), L.ptr(j0),
            L.ptr(model.jac_rows_device()) if model.nnz_jac else None, L.ptr(x0d), L.ptr(self.xl),
            L.ptr(self.xu), L.ptr(self.rlo_d), L.ptr(self.rhi_d), 1 if opts.scaling else 0,
            float(self.tol_r), L.ptr(bits), L.ptr(self.x), L.ptr(self.s), L.ptr(self.y), L.ptr(self.zxl),
            L.ptr(self.zxu), L.ptr(self.zsl), L.ptr(self.zsu), L.ptr(self.con_scale), L.ptr(self.sl),
            L.ptr(self.su), L.ptr(self.scal[61:62]), D.stream_ptr()))
        self.grad, self.c = D.empty(n), D.empty(mm)
        self.dual_x, self.dual_s, self.primal = D.empty(n), D.empty(mm), D.empty(mm)
        self.xt, self.st, self.ct = D.empty(n), D.empty(mm), D.empty(mm)
        # reduction scratch of the initial-slack sum (counter left zeroed)
        red = model.__dict__.get("_setup_red")
        if red is None or red[0].device != dev:
            red = (torch.empty(L.GN_RED_PARTIALS, dtype=torch.float64, device=dev),
                   torch.zeros(1, dtype=torch.int32, device=dev))
            model.__dict__["_setup_red"] = red
        self.red = red

    def vecs(self, ws) -> L.IpmVecs:
        return L.IpmVecs(*(t.data_ptr() for t in (
            self.x, self.s, self.y, self.zxl, self.zxu, self.zsl, self.zsu, self.xl, self.xu,
            self.sl, self.su, ws.dxl, ws.dxu, ws.dsl, ws.dsu, ws.sigma_x, ws.sigma_s, self.grad,
            self.c, ws.a_vals, self.dual_x, self.dual_s, self.primal)))

    def read_async(self, lo, hi):
        """Start copying scal[lo:hi] and the flag words (one copy); returns
        the event to wait on."""
        D.TRANSFER["d2h"] += 8 * (97 - lo)
        self.host_mail[lo:].copy_(self.mail[lo:], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(self.stream)
        return ev

    def read_wait(self, ev, lo, hi):
        ev.synchronize()
        f = self.host_flags.tolist()
        return self.host[lo:hi].numpy(), f[0], f[1]

    def read(self, lo, hi):
        """Copy scal[lo:hi] and both flag words to the host (one copy, one
        stream sync)."""
        D.TRANSFER["d2h"] += 8 * (97 - lo)
        self.host_mail[lo:].copy_(self.mail[lo:], non_blocking=True)
        self.stream.synchronize()
        f = self.host_flags.tolist()
        return self.host[lo:hi].numpy(), f[0], f[1]


def _plan_lookup(model, ordering):
    """The cached symbolic plans of `model` for `ordering`, or a started host
    analysis.  Keyed on the ordering's CONTENT (a copy is kept): a new array
    that reuses a freed one's id, or one mutated in place, is a different
    key.  Returns (key, analysis or None on a hit)."""
    key = None if ordering is None else np.array(ordering, dtype=np.int64, copy=True)
    cache = getattr(model, "_kkt_cache", None)
    hit = cache is not None and ((cache[0] is None and key is None) or (
        cache[0] is not None and key is not None and cache[0].shape == key.shape
        and np.array_equal(cache[0], key)))
    return key, (None if hit else HostAnalysis(model, ordering))


def _plan_finish(model, key, analysis, setup):
    """KKT workspace + condensed backend (device plans) of the analysis, or
    the cached ones; cached on the model."""
    if analysis is None:
        _, ws, backend = model._kkt_cache
        return ws, backend
    n, m = model.n_var, model.n_con
    t0 = time.perf_counter()
    cs = analysis.condensed()
    setup["wait_condense"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ws = KKTWorkspace(n, m, model.hess_rows, model.hess_cols, model.jac_rows, model.jac_cols,
                      condensed=cs)
    setup["kkt_workspace"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    sym = analysis.symbolic()
    setup["wait_symbolic"] = time.perf_counter() - t0
    backend = CondensedBackend(ws, timings=setup, structure=cs, symbolic=sym)
    setup.update({"worker_" + k: v for k, v in analysis.timings.items()})
    model._kkt_cache = (key, ws, backend)
    return ws, backend


def plans(model, ordering=None):
    """(KKTWorkspace, CondensedBackend) of a model: the symbolic analysis and
    device plans, computed once per sparsity pattern and ordering."""
    key, analysis = _plan_lookup(model, ordering)
    return _plan_finish(model, key, analysis, {})


def solve(model, options: SolverOptions | None = None, constraint_ranges=None) -> SolveReport:
    """Solve min f s.t. g in ranges, bounds -- on the GPU (ipm.py:301-563)."""
    opts = options if options is not None else SolverOptions()
    t_start = time.perf_counter()
    report = SolveReport(status=MAX_ITER, n_var=model.n_var, n_con=model.n_con)
    setup = {}
    # symbolic analysis (condensed pattern, ordering, symbolic factor, device
    # plans) is a function of the sparsity only: cached on the model.  On a
    # miss its host part starts on a worker thread right away.
    key, analysis = _plan_lookup(model, opts.ordering)
    try:
        P = _DeviceSolve(model, opts, constraint_ranges)
        setup["problem"] = time.perf_counter() - t_start
    except NonFiniteResult as exc:
        report.status = EVAL_ERROR
        report.message = str(exc)
        report.seconds = {"total": time.perf_counter() - t_start, "ad": 0.0, "linear": 0.0,
                          "internal": 0.0}
        return report
    n, m = P.n, P.m
    mu_min = opts.mu_min if opts.mu_min is not None else opts.tol / 10.0
    lib = L.lib()
    stream = D.stream_ptr()
    timer = _Timer()

    ws, backend = _plan_finish(model, key, analysis, setup)
    backend.n_factorizations = 0
    # the workspace reads the solver's duals in place (no copies per iteration)
    ws.zxl, ws.zxu, ws.zsl, ws.zsu = P.zxl, P.zxu, P.zsl, P.zsu
    ws.__dict__["_stream"] = P.stream
    ws.delta_w = ws.delta_c = 0.0
    reg = RegState()
    V = P.vecs(ws)
    ev = P.ev
    fil = _Filter()
    state = {"mu": opts.mu_init, "it": 0}
    flagp = L.ptr(P.flags)

    def finish(status, message=""):
        P.stream.synchronize()
        total = time.perf_counter() - t_start
        report.status = status
        report.message = message
        report.iterations = state["it"]
        report.final_mu = state["mu"]
        report.x = D.to_host(P.x)
        try:
            # unscaled objective and bound violation of g(x) (ipm.py:350-357)
            P.flag_ad.zero_()
            ev.launch(P.x, F | C, f=P.scal[62:63], c=P.ct, flags=P.flag_ad)
            if m:
                g = P.ct[:m]
                zero = torch.zeros_like(g)
                viol = torch.maximum(torch.maximum(P.rlo_d - g, zero),
                                     torch.maximum(g - P.rhi_d, zero))
                P.scal[63] = viol.max()
            fin, adf, _ = P.read(62, 64)
            # ipm.py:352-355: a non-finite objective leaves both NaN; a
            # non-finite g(x) keeps the objective and leaves the violation NaN
            if not adf & F:
                report.objective = float(fin[0])
                if not adf & C:
                    report.constraint_violation = float(fin[1]) if m else 0.0
        except NonFiniteResult:
            pass
        if state.get("reg") is not None:   # the last Newton step's regularisation
            ws.delta_w, ws.delta_c = state["reg"]
        sec = timer.totals()
        internal = max(0.0, total - sec["ad"] - sec["linear"])
        report.seconds = {"total": total, "ad": sec["ad"], "linear": sec["linear"],
                          "internal": internal}
        if opts.record_trace:
            report.debug["filter"] = list(fil.entries)
        report.debug["n_factorizations"] = backend.n_factorizations
        report.debug["setup_seconds"] = setup
        report.debug["symbolic"] = dict(backend.symbolic.info)
        if opts.keep_workspace:
            report.debug["workspace"] = ws
            report.debug["backend"] = backend
            report.debug["problem"] = P
        return report

    def check_ipm_flags(ipm_flags):
        if ipm_flags & 2:
            raise DegenerateInterior("x slack lost strict interiority")
        if ipm_flags & 4:
            raise DegenerateInterior("s slack lost strict interiority")

    # initial slacks from g(x0) (ipm.py:371-380), on the device; one read
    # returns obj_scale, theta0 and the flags of both evaluations at x0 (the
    # mailbox is fresh: both flag words start at zero)
    t0 = timer.start()
    ev.launch(P.x, C, con_scale=P.con_scale, c=P.c, flags=P.flag_ad)
    timer.stop("ad", t0)
    if m:
        L.check(lib.gn_ipm_init_slacks(m, L.ptr(P.c), L.ptr(P.sl), L.ptr(P.su),
                                       opts.bound_push * P.tol_r, L.ptr(P.s), L.ptr(P.scal[60:61]),
                                       L.ptr(P.red[0]), L.ptr(P.red[1]), stream))
    sc0, adf0, adf_x0 = P.read(60, 62)
    if adf_x0:
        # the scaling evaluations at x0 failed: _Problem's constructor raised
        # in the reference (ipm.py:305-312), so the report carries no x
        try:
            ev.raise_on_flags(adf_x0, order=(GRAD, JAC))
        except NonFiniteResult as exc:
            report.status = EVAL_ERROR
            report.message = str(exc)
            report.seconds = {"total": time.perf_counter() - t_start, "ad": 0.0, "linear": 0.0,
                              "internal": 0.0}
            return report
    P.flags.zero_()
    if adf0:
        return finish(EVAL_ERROR, "constraint evaluation produced a non-finite value")
    P.obj_scale = float(sc0[1])
    theta0 = float(sc0[0]) if m else 0.0
    theta_min = 1e-4 * max(1.0, theta0)
    theta_max = 1e4 * max(1.0, theta0)
    f_ptr = L.ptr(P.scal[48:49])
    ft_ptr = L.ptr(P.scal[49:50])

    pv_buf = PVec.empty(n, m)

    def launch_eval_prep(mu):
        """Derivatives at x (ipm.py:384-391), then widths, Sigma, residual
        blocks and reductions (ipm.py:393-429) and the async read of their
        scalars.  Issued right after the previous iteration's accept, ahead
        of its host bookkeeping."""
        t0 = timer.start()
        with span("ad_full"):
            ev.launch(P.x, F | C | GRAD | JAC | HESS | RESET, y=P.y, obj_weight=P.obj_scale,
                      con_scale=P.con_scale, obj_scale=P.obj_scale, f=P.scal[48:49], c=P.c,
                      grad=P.grad, jac=ws.a_vals, hess=ws.w_vals, flags=P.flag_ad)
        timer.stop("ad", t0)
        cands = _mu_candidates(mu, mu_min, opts, L.IPM_MAX_MU)
        mus = (ctypes.c_double * len(cands))(*cands)
        with span("prep"):
            L.check(lib.gn_ipm_prep(ws.handle, ctypes.byref(V), len(cands), mus, L.ptr(P.scal),
                                    stream))
        P.ev_prep.record(P.stream)
        return P.read_async(0, 49), cands

    pending = launch_eval_prep(state["mu"]) if opts.max_iter > 0 else None
    for _ in range(opts.max_iter):
        mu = state["mu"]
        ev_prep, cands = pending
        # the condensed matrix does not depend on mu: assemble and factor it
        # (delta_w = delta_c = 0, the first try of kkt.py:424-447) while the
        # host reads the residuals and runs the barrier update; the PD flag is
        # checked with the first refinement read
        t_lin = timer.start()
        ws.delta_w = ws.delta_c = 0.0
        backend.factorize_async()
        sc, adf, ipf = P.read_wait(ev_prep, 0, 49)
        check_ipm_flags(ipf)
        if adf:
            try:
                ev.raise_on_flags(adf)
            except NonFiniteResult as exc:
                backend.n_factorizations -= 1
                return finish(EVAL_ERROR, str(exc))
        fval = float(sc[48])
        S0 = L.PREP_S
        dual_max = max(sc[0], sc[S0 + 0])
        primal_max = sc[S0 + 1]
        z_l1 = sc[1] + sc[S0 + 2]
        y_l1 = sc[S0 + 3]
        comp = lambda k: max(sc[4 + k] if n else 0.0, sc[S0 + 7 + k] if m else 0.0)
        resid = lambda k: kkt_residual_scalars(dual_max, primal_max, comp(k), z_l1, y_l1, m,
                                               P.n_bounds, opts.s_max)
        e_0 = resid(0)
        if e_0 < opts.tol:
            report.residual_scaled = e_0
            backend.n_factorizations -= 1   # the speculative factorisation is not used
            return finish(OPTIMAL)
        k = 1
        e_mu = resid(k)
        while e_mu <= opts.kappa_eps * mu and mu > mu_min * (1 + 1e-12):
            mu = max(mu_min, min(opts.kappa_mu * mu, mu ** opts.theta_mu))
            fil.clear()
            k += 1
            if k < len(cands) and cands[k] == mu:
                e_mu = resid(k)
            else:   # beyond the precomputed candidates: one more reduction pass
                more = (ctypes.c_double * 2)(0.0, mu)
                L.check(lib.gn_ipm_prep(ws.handle, ctypes.byref(V), 2, more, L.ptr(P.scal), stream))
                sc2, _, _ = P.read(0, 48)
                sc = np.concatenate([sc2, sc[48:]])
                cands = [0.0, mu]
                k = 1
                e_mu = resid(1)
        state["mu"] = mu
        theta_cur = float(sc[S0 + 4]) if m else 0.0
        phi_cur = fval
        for lsum in (sc[2], sc[3], sc[S0 + 5], sc[S0 + 6]):
            phi_cur -= mu * float(lsum)
        # ---- Newton step (ipm.py:434-453)
        pv = pv_buf          # overwritten in full by gn_ipm_pvec
        pvc = pv.c_struct()
        # right-hand side and its condensation on the second stream, after
        # the prep (which precedes the factorisation on the solver's stream):
        # they run beside the factorisation; the solve waits for them
        with torch.cuda.stream(P.aux):
            P.aux.wait_event(P.ev_prep)
            L.check(lib.gn_ipm_pvec(ws.handle, ctypes.byref(V), mu, ctypes.byref(pvc), P.aux.cuda_stream))
            cond = ws._condense(pv, "main")
            ws.matrix_scale_device(ws._scal[2:3])   # the refinement's scale (delta_w = delta_c = 0)
            P.ev_rhs.record(P.aux)
        P.stream.wait_event(P.ev_rhs)
        t0 = t_lin
        try:
            # the speculative factorisation above is used without reading the
            # pivot flag; it comes back with the first refinement read, and
            # only a failure falls back to the regularisation schedule of
            # solve_with_regularization (kkt.py:424-447)
            dx, ds, dy = backend.solve_condensed(cond, "main")
            delta_w = 0.0
            steps = assemble_steps(ws, pv, dx, ds, dy, check=False, slot="main")
            try:
                ir = iterative_refinement(ws, backend, steps, pv, check_factor=backend.fws.fail,
                                          scale_ready=True)
            except FactorizationFailed:
                (dx, ds, dy), delta_w = solve_with_regularization(ws, backend, pv, reg, "main")
                steps = assemble_steps(ws, pv, dx, ds, dy, check=False, slot="main")
                ir = iterative_refinement(ws, backend, steps, pv)
        except RegularizationExhausted as exc:
            timer.stop("linear", t0)
            return finish(REGULARIZATION_EXHAUSTED, str(exc))
        timer.stop("linear", t0)
        state["reg"] = (ws.delta_w, ws.delta_c)
        if opts.log_level >= 3:
            print(f"  newton: delta_w {delta_w:.3e} ir rounds {ir.rounds} "
                  f"residual {ir.initial_residual:.3e} -> {ir.final_residual:.3e} scale {ir.scale:.3e}")
        report.refinement_relative_residual = ir.relative_residual
        # ---- fraction to the boundary and dphi (ipm.py:455-476)
        tau = max(opts.tau_min, 1.0 - mu)
        stc = steps.c_struct()
        L.check(lib.gn_ipm_direction(ws.handle, ctypes.byref(V), ctypes.byref(stc), mu, tau,
                                     L.ptr(P.scal[50:54]), stream))
        # ---- filter line search (ipm.py:478-519); the first trial runs at
        # alpha_max read on the device and returns with the direction scalars
        alpha = alpha_z = dphi = 0.0
        accepted = f_type = False
        theta_t = phi_t = np.nan
        first = True
        while True:
            if first:
                L.check(lib.gn_ipm_trial_point_at(ws.handle, ctypes.byref(V), ctypes.byref(stc),
                                                  L.ptr(P.scal[50:52]), L.ptr(P.xt), L.ptr(P.st),
                                                  stream))
            else:
                if alpha < opts.alpha_min:
                    break
                L.check(lib.gn_ipm_trial_point(ws.handle, ctypes.byref(V), ctypes.byref(stc), alpha,
                                               L.ptr(P.xt), L.ptr(P.st), stream))
            t0 = timer.start()
            with span("ad_trial"):
                ev.launch(P.xt, F | C | RESET, con_scale=P.con_scale, obj_scale=P.obj_scale,
                          f=P.scal[49:50], c=P.ct, flags=P.flag_ad)
            timer.stop("ad", t0)
            L.check(lib.gn_ipm_trial_merit(ws.handle, ctypes.byref(V), L.ptr(P.ct), L.ptr(P.xt),
                                           L.ptr(P.st), L.ptr(P.scal[54:59]), stream))
            tv, adf, _ = P.read(49, 59)
            if opts.log_level >= 3:
                print(f"  trial alpha {alpha:.3e} adf {adf} merit {list(map(float, tv))}")
            if first:
                first = False
                alpha = min(float(tv[1]), float(tv[2]))
                alpha_z, dphi = float(tv[3]), float(tv[4])
                if alpha < opts.alpha_min:
                    break
            if adf:
                alpha *= 0.5
                continue
            ft = float(tv[0])
            theta_t = float(tv[5]) if m else 0.0
            phi_t = ft
            for lsum in tv[6:10]:
                phi_t -= mu * float(lsum)
            if not np.isfinite(phi_t) or theta_t > theta_max:
                alpha *= 0.5
                continue
            if not fil.acceptable(theta_t, phi_t):
                alpha *= 0.5
                continue
            switching = (dphi < 0.0 and alpha * (-dphi) ** opts.s_phi
                         > opts.delta * theta_cur ** opts.s_theta)
            if theta_cur <= theta_min and switching:
                if phi_t <= phi_cur + opts.eta_phi * alpha * dphi:
                    accepted = f_type = True
                    break
            elif (theta_t <= (1.0 - opts.gamma_theta) * theta_cur
                  or phi_t <= phi_cur - opts.gamma_phi * theta_cur):
                accepted = True
                break
            alpha *= 0.5
        if not accepted:
            return finish(LINE_SEARCH_FAILURE, f"step size below {opts.alpha_min:g}")
        if not f_type:
            fil.add((1.0 - opts.gamma_theta) * theta_cur, phi_cur - opts.gamma_phi * theta_cur)
        # ---- accept + dual safeguard + interiority (ipm.py:521-548)
        L.check(lib.gn_ipm_accept(ws.handle, ctypes.byref(V), ctypes.byref(stc), alpha, alpha_z,
                                  mu, opts.kappa_sigma, L.ptr(P.flags[1:2]), stream))
        state["it"] += 1
        if state["it"] < opts.max_iter:   # the next iteration's device work first
            pending = launch_eval_prep(state["mu"])
        if opts.record_trace:
            report.trace.append((state["it"], fval / P.obj_scale, float(primal_max),
                                 float(dual_max), mu, alpha, delta_w))
            report.debug.setdefault("accepted", []).append((theta_t, phi_t, list(fil.entries)))
            report.debug.setdefault("ir_rounds", []).append(ir.rounds)
        if opts.log_level >= 2:
            print(f"iter {state['it']:4d} obj {fval / P.obj_scale: .8e} inf_pr {primal_max:.2e} "
                  f"inf_du {dual_max:.2e} mu {mu:.1e} alpha {alpha:.2e} dw {delta_w:.1e}")
        report.residual_scaled = e_0
    P.stream.synchronize()
    check_ipm_flags(int(P.flags[1].item()))
    return finish(MAX_ITER)
