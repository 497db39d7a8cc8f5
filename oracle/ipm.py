"""Filter line-search interior-point loop (oracle).

Restates reference src/gridnlp/ipm.py:112-563: equality relaxation
(112-123), initial slacks (126-134), frozen gradient scaling (179-203),
the scaled KKT residual (150-157), the barrier update (422-429), the
condensed Newton step with refinement (434-453), fraction-to-boundary
(265-281, 455-462), the filter / Armijo line search (284-298, 464-519),
the step update with the kappa_sigma dual safeguard (521-548).

``solve`` takes an oracle model (oracle/model.py ``OModel``), the
reference option values and an optional injected ordering (the
"loop-fair" CPU baseline).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import kkt as K
from . import model as M

OPTIMAL, MAX_ITER = "optimal", "max_iter"
REGULARIZATION_EXHAUSTED, LINE_SEARCH_FAILURE, EVAL_ERROR = (
    "regularization_exhausted", "line_search_failure", "eval_error")


@dataclass
class Options:
    """SolverOptions defaults (ipm.py:43-74)."""
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
    verbose: bool = False


@dataclass
class Report:
    status: str
    objective: float = np.nan
    constraint_violation: float = np.nan
    residual_scaled: float = np.nan
    iterations: int = 0
    final_mu: float = np.nan
    x: np.ndarray | None = None
    trace: list = field(default_factory=list)
    seconds: dict = field(default_factory=dict)
    n_factorizations: int = 0
    ir_rounds: list = field(default_factory=list)


def relax_equalities(m, ranges, tol):
    lo, hi = (np.zeros(m), np.zeros(m)) if ranges is None else (
        np.asarray(ranges, float)[:, 0].copy(), np.asarray(ranges, float)[:, 1].copy())
    sl = np.where(np.isfinite(lo), lo - tol * np.maximum(1.0, np.abs(lo)), -np.inf)
    su = np.where(np.isfinite(hi), hi + tol * np.maximum(1.0, np.abs(hi)), np.inf)
    return sl, su


def initial_slacks(g0, sl, su, tol, push):
    lo = np.where(np.isfinite(sl), sl + push * tol, -np.inf)
    hi = np.where(np.isfinite(su), su - push * tol, np.inf)
    s = np.minimum(np.maximum(g0, lo), hi)
    crossed = lo > hi
    return np.where(crossed, 0.5 * (sl + su), s) if np.any(crossed) else s


def width(v, bound, upper=False):
    return np.where(np.isfinite(bound), (bound - v) if upper else (v - bound), np.inf)


def amax(*arrs):
    out = 0.0
    for a in arrs:
        if a.size:
            out = max(out, float(np.abs(a).max()))
    return out


def kkt_residual(dual_x, dual_s, primal, comps, z_l1, y_l1, m, n_bounds, s_max=100.0):
    s_d = max(s_max, (y_l1 + z_l1) / max(1, m + n_bounds)) / s_max
    s_c = max(s_max, z_l1 / max(1, n_bounds)) / s_max
    comp = amax(*comps) / s_c if n_bounds else 0.0
    return max(max(amax(dual_x), amax(dual_s)) / s_d, amax(primal), comp)


def ftb(v, dv, lo, hi, tau):
    a = 1.0
    neg = (dv < 0) & np.isfinite(lo)
    if np.any(neg):
        a = min(a, float(np.min(-tau * (v[neg] - lo[neg]) / dv[neg])))
    pos = (dv > 0) & np.isfinite(hi)
    if np.any(pos):
        a = min(a, float(np.min(tau * (hi[pos] - v[pos]) / dv[pos])))
    return a


def dual_ftb(z, dz, tau):
    neg = dz < 0
    return min(1.0, float(np.min(-tau * z[neg] / dz[neg]))) if np.any(neg) else 1.0


def solve(om: M.OModel, lower, upper, start, opts: Options | None = None,
          ranges=None, ordering=None) -> Report:
    opts = opts or Options()
    t0 = time.perf_counter()
    ad_t = [0.0]
    lin_t = 0.0
    n, m = om.n, om.m
    tol_r = opts.bound_relax if opts.bound_relax is not None else opts.tol
    rep = Report(status=MAX_ITER)

    xl, xu = np.array(lower, float), np.array(upper, float)
    fixed = xl == xu
    if np.any(fixed):
        e = opts.fixed_var_eps * np.maximum(1.0, np.abs(xl))
        xl, xu = np.where(fixed, xl - e, xl), np.where(fixed, xu + e, xu)
    x0 = np.minimum(np.maximum(np.asarray(start, float), xl), xu)

    def timed(fn, *a):
        t = time.perf_counter()
        try:
            return fn(*a)
        finally:
            ad_t[0] += time.perf_counter() - t

    try:
        g0x = M.gradient(om, x0)
        j0 = M.jacobian(om, x0)
    except M.NonFinite:
        rep.status = EVAL_ERROR
        return rep
    if opts.scaling:
        gm = amax(g0x)
        osc = min(1.0, 100.0 / gm) if gm > 0 else 1.0
        rmax = np.zeros(m)
        if j0.size:
            np.maximum.at(rmax, om.jac_rows, np.abs(j0))
        csc = np.ones(m)
        pos = rmax > 0
        csc[pos] = np.minimum(1.0, 100.0 / rmax[pos])
    else:
        osc, csc = 1.0, np.ones(m)
    rlo, rhi = (np.zeros(m), np.zeros(m)) if ranges is None else (
        np.asarray(ranges, float)[:, 0].copy(), np.asarray(ranges, float)[:, 1].copy())
    sl, su = relax_equalities(m, np.column_stack([rlo * csc, rhi * csc]) if m else None, tol_r)

    f_obj = lambda x: osc * timed(M.objective, om, x)
    f_con = lambda x: csc * timed(M.constraints, om, x)
    f_grad = lambda x: osc * timed(M.gradient, om, x)
    f_jac = lambda x: timed(M.jacobian, om, x) * csc[om.jac_rows] if om.jac_rows.size else np.zeros(0)
    f_hess = lambda x, y: timed(M.hessian, om, x, y * csc if m else y, osc)

    mu_min = opts.mu_min if opts.mu_min is not None else opts.tol / 10.0
    ws = K.OWorkspace(n, m, om.hess_rows, om.hess_cols, om.jac_rows, om.jac_cols)
    backend = K.OCondensedBackend(ws, ordering)
    reg = K.RegState()
    st = dict(x=x0.copy(), s=np.zeros(m), y=np.zeros(m),
              zxl=np.where(np.isfinite(xl), 1.0, 0.0), zxu=np.where(np.isfinite(xu), 1.0, 0.0),
              zsl=np.where(np.isfinite(sl), 1.0, 0.0), zsu=np.where(np.isfinite(su), 1.0, 0.0))
    mu = opts.mu_init
    filt: list = []
    nb = int(np.isfinite(xl).sum() + np.isfinite(xu).sum() + np.isfinite(sl).sum()
             + np.isfinite(su).sum())
    it = 0

    def phi(fv, ws4):
        out = fv
        for w in ws4:
            f = np.isfinite(w)
            if np.any(f):
                out -= mu * float(np.log(w[f]).sum())
        return out

    def finish(status):
        rep.status = status
        rep.iterations = it
        rep.final_mu = mu
        rep.x = st["x"].copy()
        try:
            rep.objective = M.objective(om, st["x"])
            g = M.constraints(om, st["x"])
            rep.constraint_violation = float(np.maximum(np.maximum(rlo - g, 0.0),
                                                        np.maximum(g - rhi, 0.0)).max()) if m else 0.0
        except M.NonFinite:
            pass
        total = time.perf_counter() - t0
        rep.seconds = {"total": total, "ad": ad_t[0], "linear": lin_t,
                       "internal": max(0.0, total - ad_t[0] - lin_t)}
        rep.n_factorizations = backend.n_factorizations
        return rep

    try:
        g0 = f_con(st["x"])
    except M.NonFinite:
        return finish(EVAL_ERROR)
    st["s"] = initial_slacks(g0, sl, su, tol_r, opts.bound_push)
    theta_fn = lambda g, s: float(np.abs(g - s).sum()) if m else 0.0
    th0 = theta_fn(g0, st["s"])
    th_min, th_max = 1e-4 * max(1.0, th0), 1e4 * max(1.0, th0)

    for _ in range(opts.max_iter):
        x, s = st["x"], st["s"]
        try:
            fval, g, grad = f_obj(x), f_con(x), f_grad(x)
            jv, wv = f_jac(x), f_hess(x, st["y"])
        except M.NonFinite:
            return finish(EVAL_ERROR)
        dxl, dxu = width(x, xl), width(x, xu, True)
        dsl, dsu = width(s, sl), width(s, su, True)
        ws.set_iterate(wv, jv, dxl, dxu, st["zxl"], st["zxu"], dsl, dsu, st["zsl"], st["zsu"])
        dual_x = grad + ws.at_mv(st["y"]) - st["zxl"] + st["zxu"]
        dual_s = -st["y"] - st["zsl"] + st["zsu"]
        primal = g - s
        pairs = ((st["zxl"], dxl), (st["zxu"], dxu), (st["zsl"], dsl), (st["zsu"], dsu))
        comps = lambda mu_: [z[np.isfinite(w)] * w[np.isfinite(w)] - mu_ for z, w in pairs]
        z_l1 = float(sum(np.abs(st[k]).sum() for k in ("zxl", "zxu", "zsl", "zsu")))
        y_l1 = float(np.abs(st["y"]).sum())
        kw = dict(z_l1=z_l1, y_l1=y_l1, m=m, n_bounds=nb, s_max=opts.s_max)
        e0 = kkt_residual(dual_x, dual_s, primal, comps(0.0), **kw)
        if e0 < opts.tol:
            rep.residual_scaled = e0
            return finish(OPTIMAL)
        emu = kkt_residual(dual_x, dual_s, primal, comps(mu), **kw)
        while emu <= opts.kappa_eps * mu and mu > mu_min * (1 + 1e-12):
            mu = max(mu_min, min(opts.kappa_mu * mu, mu ** opts.theta_mu))
            filt.clear()
            emu = kkt_residual(dual_x, dual_s, primal, comps(mu), **kw)
        muv = lambda w: np.where(np.isfinite(w), mu, 0.0)
        fin0 = lambda w: np.where(np.isfinite(w), w, 0.0)
        pv = K.Vec7(-dual_x, -dual_s, -primal,
                    muv(dxl) - st["zxl"] * fin0(dxl), muv(dxu) - st["zxu"] * fin0(dxu),
                    muv(dsl) - st["zsl"] * fin0(dsl), muv(dsu) - st["zsu"] * fin0(dsu))
        tl = time.perf_counter()
        try:
            (dx, ds, dy), dw = K.solve_with_regularization(ws, backend, pv, reg)
            steps = K.assemble_steps(ws, pv, dx, ds, dy)
            rounds = K.iterative_refinement(ws, backend, steps, pv)[0]
            rep.ir_rounds.append(rounds)
        except K.RegExhausted:
            lin_t += time.perf_counter() - tl
            return finish(REGULARIZATION_EXHAUSTED)
        lin_t += time.perf_counter() - tl

        tau = max(opts.tau_min, 1.0 - mu)
        a_max = min(ftb(x, steps.x, xl, xu, tau), ftb(s, steps.s, sl, su, tau))
        a_z = 1.0
        for k in ("zxl", "zxu", "zsl", "zsu"):
            a_z = min(a_z, dual_ftb(st[k], getattr(steps, k), tau))
        th_cur = theta_fn(g, s)
        ph_cur = phi(fval, (dxl, dxu, dsl, dsu))
        gpx = grad.copy()
        f = np.isfinite(dxl)
        gpx[f] -= mu / dxl[f]
        f = np.isfinite(dxu)
        gpx[f] += mu / dxu[f]
        gps = np.zeros(m)
        f = np.isfinite(dsl)
        gps[f] -= mu / dsl[f]
        f = np.isfinite(dsu)
        gps[f] += mu / dsu[f]
        dphi = float(gpx @ steps.x + (gps @ steps.s if m else 0.0))

        alpha, ok, ftype = a_max, False, False
        if getattr(opts, "verbose", False):
            print(f"  oracle newton: dw {dw:.3e} ir {rounds} a_max {a_max:.3e} a_z {a_z:.3e} dphi {dphi:.6e}"
                  f" th_cur {th_cur:.6e} ph_cur {ph_cur:.10e}")
        while alpha >= opts.alpha_min:
            xt, stt = x + alpha * steps.x, s + alpha * steps.s
            try:
                ft, gt = f_obj(xt), f_con(xt)
            except M.NonFinite:
                alpha *= 0.5
                continue
            th_t = theta_fn(gt, stt)
            ph_t = phi(ft, (width(xt, xl), width(xt, xu, True), width(stt, sl),
                            width(stt, su, True)))
            if not np.isfinite(ph_t) or th_t > th_max:
                alpha *= 0.5
                continue
            if not all(th_t < a or ph_t < b for a, b in filt):
                alpha *= 0.5
                continue
            switching = dphi < 0.0 and alpha * (-dphi) ** opts.s_phi > opts.delta * th_cur ** opts.s_theta
            if th_cur <= th_min and switching:
                if ph_t <= ph_cur + opts.eta_phi * alpha * dphi:
                    ok = ftype = True
                    break
            elif th_t <= (1.0 - opts.gamma_theta) * th_cur or ph_t <= ph_cur - opts.gamma_phi * th_cur:
                ok = True
                break
            alpha *= 0.5
        if not ok:
            return finish(LINE_SEARCH_FAILURE)
        if not ftype:
            ent = ((1.0 - opts.gamma_theta) * th_cur, ph_cur - opts.gamma_phi * th_cur)
            filt[:] = [e for e in filt if not (e[0] >= ent[0] and e[1] >= ent[1])]
            filt.append(ent)

        st["x"] = x + alpha * steps.x
        st["s"] = s + alpha * steps.s
        st["y"] = st["y"] + alpha * steps.y
        for k in ("zxl", "zxu", "zsl", "zsu"):
            st[k] = st[k] + a_z * getattr(steps, k)
        for k, v, bd, up in (("zxl", "x", xl, False), ("zxu", "x", xu, True),
                             ("zsl", "s", sl, False), ("zsu", "s", su, True)):
            w = width(st[v], bd, up)
            f = np.isfinite(w)
            if np.any(f):
                z = st[k]
                z[f] = np.minimum(np.maximum(z[f], mu / (opts.kappa_sigma * w[f])),
                                  opts.kappa_sigma * mu / w[f])
        for v, bd, up in (("x", xl, False), ("x", xu, True), ("s", sl, False), ("s", su, True)):
            w = width(st[v], bd, up)
            if np.any(w[np.isfinite(w)] <= 0.0):
                raise K.Degenerate(f"{v} lost strict interiority")
        it += 1
        rep.trace.append((it, fval / osc, amax(primal), amax(dual_x, dual_s), mu, alpha, dw))
        rep.residual_scaled = e0
    return finish(MAX_ITER)
