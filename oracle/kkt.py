"""Condensed KKT algebra, regularisation and refinement (oracle).

Restates reference src/gridnlp/kkt.py: the seven-block Newton system, its
condensation to W + dw I + Sigma_x + A^T D A (kkt.py:1-28), diagonal
recoveries (159-187), the extended-precision residual (190-209,
``np.longdouble``), the inertia-correction schedule (424-447) and
iterative refinement (467-491).  The condensed backend uses the oracle's
sparse restatement (oracle/sparse.py) with an injected ordering.
"""
from __future__ import annotations

import numpy as np

from . import sparse as S
from .ordering import min_degree_order

DELTA_W_INIT, DELTA_W_MIN, DELTA_W_MAX = 1e-4, 1e-20, 1e40   # kkt.py:39-41
DELTA_C_VALUE, KAPPA_IR, MAX_IR_ROUNDS = 1e-8, 10.0, 10      # kkt.py:42-44
FIELDS = ("x", "s", "y", "zxl", "zxu", "zsl", "zsu")


class RegExhausted(RuntimeError):
    pass


class Degenerate(RuntimeError):
    pass


class Vec7:
    """Seven-block vector (PVec / Steps, kkt.py:60-85)."""

    def __init__(self, *arrs):
        for f, a in zip(FIELDS, arrs):
            setattr(self, f, a)

    def parts(self):
        return [getattr(self, f) for f in FIELDS]

    def axpy(self, other, alpha=1.0):
        for f in FIELDS:
            getattr(self, f)[...] += alpha * getattr(other, f)


def inv_or_zero(w):
    out = np.zeros_like(w)
    fin = np.isfinite(w)
    out[fin] = 1.0 / w[fin]
    return out


class OWorkspace:
    """kkt.py:96-221"""

    def __init__(self, n, m, hr, hc, jr, jc):
        self.n, self.m = n, m
        self.hr, self.hc, self.jr, self.jc = hr, hc, jr, jc
        self.w = np.zeros(hr.size)
        self.a = np.zeros(jr.size)
        self.dw = self.dc = 0.0
        for f in ("dxl", "dxu", "zxl", "zxu"):
            setattr(self, f, np.zeros(n))
        for f in ("dsl", "dsu", "zsl", "zsu"):
            setattr(self, f, np.zeros(m))
        self.sx, self.ss = np.zeros(n), np.zeros(m)

    def set_iterate(self, w, a, dxl, dxu, zxl, zxu, dsl, dsu, zsl, zsu):
        self.w[:], self.a[:] = w, a
        self.dxl, self.dxu, self.zxl, self.zxu = (np.array(v, float) for v in (dxl, dxu, zxl, zxu))
        self.dsl, self.dsu, self.zsl, self.zsu = (np.array(v, float) for v in (dsl, dsu, zsl, zsu))
        self.sx = self.zxl * inv_or_zero(self.dxl) + self.zxu * inv_or_zero(self.dxu)
        self.ss = self.zsl * inv_or_zero(self.dsl) + self.zsu * inv_or_zero(self.dsu)

    def w_mv(self, v, dt=float):
        out = np.zeros(self.n, dtype=dt)
        wv = self.w.astype(dt, copy=False)
        np.add.at(out, self.hr, wv * v[self.hc])
        off = self.hr != self.hc
        np.add.at(out, self.hc[off], wv[off] * v[self.hr[off]])
        return out

    def a_mv(self, v, dt=float):
        out = np.zeros(self.m, dtype=dt)
        np.add.at(out, self.jr, self.a.astype(dt, copy=False) * v[self.jc])
        return out

    def at_mv(self, u, dt=float):
        out = np.zeros(self.n, dtype=dt)
        np.add.at(out, self.jc, self.a.astype(dt, copy=False) * u[self.jr])
        return out

    def c_diag(self):
        return 1.0 / (self.dc * self.ss + (1.0 + self.dc * self.dw))

    def d_diag(self):
        return (self.ss + self.dw) * self.c_diag()

    def condense_pvec(self, pv):
        qx = pv.x + inv_or_zero(self.dxl) * pv.zxl - inv_or_zero(self.dxu) * pv.zxu
        qs = pv.s + inv_or_zero(self.dsl) * pv.zsl - inv_or_zero(self.dsu) * pv.zsu
        return qx, qs, pv.y.copy()

    def condensed_rhs(self, qx, qs, qy):
        return qx + self.at_mv(self.c_diag() * qs + self.d_diag() * qy)

    def recover_slack_dual(self, dx, qx, qs, qy):
        ds = self.c_diag() * (self.a_mv(dx) + self.dc * qs - qy)
        return ds, (self.ss + self.dw) * ds - qs

    def recover_bound_duals(self, dx, ds, pv):
        for w in (self.dxl, self.dxu, self.dsl, self.dsu):
            if np.any(w[np.isfinite(w)] <= 0.0):
                raise Degenerate("non-positive bound slack")
        return (inv_or_zero(self.dxl) * (pv.zxl - self.zxl * dx),
                inv_or_zero(self.dxu) * (pv.zxu + self.zxu * dx),
                inv_or_zero(self.dsl) * (pv.zsl - self.zsl * ds),
                inv_or_zero(self.dsu) * (pv.zsu + self.zsu * ds))

    def residual_full(self, st, pv, dt=np.longdouble):
        """pv - M_full * st in extended precision (kkt.py:190-209)."""
        L = lambda a: a.astype(dt)
        one = lambda w: np.where(np.isfinite(w), w, 1.0).astype(dt)
        dx, ds, dy = L(st.x), L(st.s), L(st.y)
        rx = (L(pv.x) - self.w_mv(dx, dt) - self.dw * dx - self.at_mv(dy, dt)
              + L(st.zxl) - L(st.zxu))
        rs = L(pv.s) - self.dw * ds + dy + L(st.zsl) - L(st.zsu)
        ry = L(pv.y) - self.a_mv(dx, dt) + ds + self.dc * dy
        return Vec7(rx, rs, ry,
                    L(pv.zxl) - self.zxl * dx - one(self.dxl) * L(st.zxl),
                    L(pv.zxu) + self.zxu * dx - one(self.dxu) * L(st.zxu),
                    L(pv.zsl) - self.zsl * ds - one(self.dsl) * L(st.zsl),
                    L(pv.zsu) + self.zsu * ds - one(self.dsu) * L(st.zsu))

    def matrix_scale(self):
        out = [1.0, self.dw, self.dc]
        for arr in (self.w, self.a, self.sx, self.ss, self.zxl, self.zxu, self.zsl, self.zsu):
            if arr.size:
                out.append(float(np.abs(arr).max()))
        for w in (self.dxl, self.dxu, self.dsl, self.dsu):
            f = w[np.isfinite(w)]
            if f.size:
                out.append(float(f.max()))
        return max(out)


def residual_norm(v):
    out = 0.0
    for a in v.parts():
        if a.size:
            out = max(out, float(np.abs(a).max()))
    return out


class OCondensedBackend:
    """kkt.py:286-325 with an injectable ordering (kkt.py:289-295)."""

    def __init__(self, ws, ordering=None):
        self.ws = ws
        self.cs = S.condense(ws.hr, ws.hc, ws.jr, ws.jc, ws.n)
        if ordering is None:
            r, c = self.cs.matrix.coords()
            ordering = min_degree_order(ws.n, r, c)
        self.sym = S.symbolic(self.cs.matrix, ordering)
        self.l_vals = None
        self.n_factorizations = 0

    def assemble(self):
        ws = self.ws
        self.cs.matrix.values = S.assemble(self.cs, ws.w, ws.a, ws.sx, ws.dw, ws.d_diag())

    def try_factorize(self):
        self.assemble()
        self.n_factorizations += 1
        self.l_vals, ok, self.failing_column = S.factorize(self.sym, self.cs.matrix.values)
        return ok

    def solve3(self, qx, qs, qy):
        ws = self.ws
        dx = S.solve(self.sym, self.l_vals, ws.condensed_rhs(qx, qs, qy))
        ds, dy = ws.recover_slack_dual(dx, qx, qs, qy)
        return dx, ds, dy


class RegState:
    def __init__(self):
        self.delta_w_last = 0.0


def solve_with_regularization(ws, backend, pv, reg):
    """kkt.py:424-447"""
    ws.dw = ws.dc = 0.0
    if not backend.try_factorize():
        hist = reg.delta_w_last > 0.0
        ws.dc = DELTA_C_VALUE
        ws.dw = max(DELTA_W_MIN, reg.delta_w_last / 3.0) if hist else DELTA_W_INIT
        while not backend.try_factorize():
            ws.dw *= 8.0 if hist else 100.0
            if ws.dw > DELTA_W_MAX:
                raise RegExhausted("delta_w ceiling")
        reg.delta_w_last = ws.dw
    qx, qs, qy = ws.condense_pvec(pv)
    return backend.solve3(qx, qs, qy), ws.dw


def assemble_steps(ws, pv, dx, ds, dy):
    return Vec7(dx, ds, dy, *ws.recover_bound_duals(dx, ds, pv))


def iterative_refinement(ws, backend, steps, pv):
    """-> (rounds, initial, final, scale) (kkt.py:467-491)."""
    scale = ws.matrix_scale()
    target = KAPPA_IR * np.finfo(float).eps * scale
    res = ws.residual_full(steps, pv)
    r0 = residual_norm(res)
    final, rounds = r0, 0
    while final > target and rounds < MAX_IR_ROUNDS:
        rv = Vec7(*(a.astype(float) for a in res.parts()))
        qx, qs, qy = ws.condense_pvec(rv)
        corr = assemble_steps(ws, rv, *backend.solve3(qx, qs, qy))
        steps.axpy(corr)
        res = ws.residual_full(steps, pv)
        new = residual_norm(res)
        rounds += 1
        if new >= final:
            steps.axpy(corr, alpha=-1.0)
            break
        enough = new <= final / 2.0
        final = new
        if not enough:
            break
    return rounds, r0, final, scale
