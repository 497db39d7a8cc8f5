"""Polar ACOPF model construction for the oracle (TEST INFRASTRUCTURE).

Restates reference src/gridnlp/acopf.py:68-246 (variables, the fifteen
pattern blocks, constraint ranges) and the ModelBuilder record handling of
src/gridnlp/model.py:143-226 (push-inside start 75-89, canonical record
order 128-140) directly into oracle blocks (``oracle.model.OBlock``), with
no call into the product library.  Only the instruction front end
(``paper_2307_16830_b200.expressions``: pure-Python expression trees and
their tapes, interchangeable with the reference's) and the MATPOWER parser
(pure-Python input format) are shared.

Used by bench.py's reference arm and ``cpu_baseline`` leg and by tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2307_16830_b200.expressions import Tape, cos, param, sin, var

from . import model as M

BOUND_PUSH = 0.01   # model.py:28


def push_inside(lower, upper, start):
    """model.py:75-89"""
    x = np.array(start, dtype=float)
    fl, fu = np.isfinite(lower), np.isfinite(upper)
    lo = np.where(fl, lower + BOUND_PUSH * np.maximum(1.0, np.abs(np.where(fl, lower, 0.0))), -np.inf)
    hi = np.where(fu, upper - BOUND_PUSH * np.maximum(1.0, np.abs(np.where(fu, upper, 0.0))), np.inf)
    crossed = lo > hi
    x = np.minimum(np.maximum(x, lo), hi)
    mid = fl & fu & crossed
    x[mid] = 0.5 * (lower[mid] + upper[mid])
    return x


class _Builder:
    """ModelBuilder semantics (model.py:143-226) producing oracle blocks."""

    def __init__(self):
        self.n_var = 0
        self.n_con = 0
        self.lower, self.upper, self.start = [], [], []
        self.blocks: list[M.OBlock] = []

    def add_variables(self, count, lower, upper, start):
        lo, hi = np.asarray(lower, float), np.asarray(upper, float)
        self.lower.append(lo)
        self.upper.append(hi)
        self.start.append(push_inside(lo, hi, np.asarray(start, float)))
        idx = np.arange(self.n_var, self.n_var + count, dtype=np.int64)
        self.n_var += count
        return idx

    def _block(self, kind, instr, var_idx, params, targets):
        t = Tape(instr)
        vi = np.asarray(var_idx, np.int64).reshape(-1, t.n_var_slots)
        pa = np.asarray(params, float).reshape(vi.shape[0], t.n_param_slots)
        tg = None if targets is None else np.asarray(targets, np.int64)
        o = M.canonical_order(vi, pa, tg)
        self.blocks.append(M.OBlock(kind, list(t.ops), list(t.consts), t.out, list(t.first_slots),
                                    [tuple(p) for p in t.second_pairs], vi[o], pa[o],
                                    None if tg is None else tg[o]))

    def add_objective(self, instr, var_idx, params):
        self._block(M.OBJ, instr, var_idx, params, None)

    def add_constraints(self, instr, var_idx, params):
        n = np.asarray(var_idx).shape[0]
        rows = np.arange(self.n_con, self.n_con + n, dtype=np.int64)
        self.n_con += n
        self._block(M.DEF, instr, var_idx, params, rows)
        return rows

    def add_constraint_increments(self, instr, var_idx, params, targets):
        self._block(M.INC, instr, var_idx, params, targets)


@dataclass
class OAcopf:
    model: M.OModel
    lower: np.ndarray
    upper: np.ndarray
    start: np.ndarray
    ranges: np.ndarray


def _admittance(br):
    """acopf.py:53-65"""
    y = 1.0 / complex(br.r, br.x)
    g, b = y.real, y.imag
    tt = br.tap * br.tap
    bc2 = br.b_charge / 2.0
    return dict(gff=g / tt, bff=(b + bc2) / tt, gtt=g, btt=b + bc2, gft=g / br.tap, bft=b / br.tap,
                shift=br.shift)


def build(net) -> OAcopf:
    """acopf.py:68-246 -> expanded oracle model + bounds, start, ranges."""
    nb, ng, nl = len(net.buses), len(net.generators), len(net.branches)
    pos = {b.id: k for k, b in enumerate(net.buses)}
    base = net.base_mva
    mb = _Builder()
    va = mb.add_variables(nb, np.full(nb, -np.inf), np.full(nb, np.inf), np.zeros(nb))
    vm = mb.add_variables(nb, [b.vmin for b in net.buses], [b.vmax for b in net.buses], np.ones(nb))
    pg = mb.add_variables(ng, [g.pmin for g in net.generators], [g.pmax for g in net.generators],
                          np.zeros(ng))
    qg = mb.add_variables(ng, [g.qmin for g in net.generators], [g.qmax for g in net.generators],
                          np.zeros(ng))
    rate = np.array([br.rate_a for br in net.branches], float)
    lo = np.where(rate > 0, -rate, -np.inf)
    hi = np.where(rate > 0, rate, np.inf)
    pflow = mb.add_variables(2 * nl, np.tile(lo, 2), np.tile(hi, 2), np.zeros(2 * nl))
    qflow = mb.add_variables(2 * nl, np.tile(lo, 2), np.tile(hi, 2), np.zeros(2 * nl))
    p_from, p_to, q_from, q_to = pflow[:nl], pflow[nl:], qflow[:nl], qflow[nl:]
    ranges: list = []

    def ranged(instr, vi, pa, rlo, rhi):
        rows = mb.add_constraints(instr, vi, pa)
        ranges.extend(zip(np.broadcast_to(np.asarray(rlo, float), rows.shape).tolist(),
                          np.broadcast_to(np.asarray(rhi, float), rows.shape).tolist()))
        return rows

    adm = [_admittance(br) for br in net.branches]
    fb = np.array([pos[br.from_bus] for br in net.branches], dtype=np.int64)
    tb = np.array([pos[br.to_bus] for br in net.branches], dtype=np.int64)
    # (1) generation cost, per-unit coefficients (acopf.py:127-134)
    cost = np.array([[g.cost[0] * base * base, g.cost[1] * base, g.cost[2]]
                     for g in net.generators]).reshape(ng, 3)
    mb.add_objective(param(0) * var(0) ** 2 + param(1) * var(0) + param(2), pg.reshape(-1, 1), cost)
    # (2) reference angle (136-138)
    ranged(var(0), np.array([[va[pos[net.ref_bus]]]]), np.zeros((1, 0)), 0.0, 0.0)
    # (3)-(6) branch flows, slots (flow, vm_f, vm_t, va_f, va_t) (141-176)
    quad = np.column_stack([vm[fb], vm[tb], va[fb], va[tb]]).reshape(nl, 4)
    dlt_f = var(3) - var(4) - param(3)
    dlt_t = var(4) - var(3) + param(3)
    vv = lambda: var(1) * var(2)
    flows = (
        (var(0) - (param(0) * var(1) ** 2 - vv() * (param(1) * cos(dlt_f) + param(2) * sin(dlt_f))),
         p_from, "gff"),
        (var(0) - (-param(0) * var(1) ** 2 - vv() * (param(1) * sin(dlt_f) - param(2) * cos(dlt_f))),
         q_from, "bff"),
        (var(0) - (param(0) * var(2) ** 2 - vv() * (param(1) * cos(dlt_t) + param(2) * sin(dlt_t))),
         p_to, "gtt"),
        (var(0) - (-param(0) * var(2) ** 2 - vv() * (param(1) * sin(dlt_t) - param(2) * cos(dlt_t))),
         q_to, "btt"))
    for instr, flow, key in flows:
        prm = np.array([[a[k] for k in (key, "gft", "bft", "shift")] for a in adm]).reshape(nl, 4)
        ranged(instr, np.column_stack([flow, quad]).reshape(nl, 5), prm, 0.0, 0.0)
    # (7) angle-difference limits (178-199)
    sel, alo, ahi = [], [], []
    for k, br in enumerate(net.branches):
        a0 = br.angmin if br.angmin > -np.pi else -np.inf
        a1 = br.angmax if br.angmax < np.pi else np.inf
        if (br.angmin == 0.0 and br.angmax == 0.0) or not (np.isfinite(a0) or np.isfinite(a1)):
            continue
        sel.append(k)
        alo.append(a0)
        ahi.append(a1)
    sel = np.array(sel, dtype=np.int64)
    ranged(var(0) - var(1), np.column_stack([va[fb[sel]], va[tb[sel]]]).reshape(-1, 2),
           np.zeros((sel.size, 0)), np.array(alo, float), np.array(ahi, float))
    # (8)-(9) apparent-power limits (201-212)
    lim = np.flatnonzero(rate > 0)
    rsq = (rate[lim] ** 2).reshape(-1, 1)
    for pside, qside in ((p_from, q_from), (p_to, q_to)):
        ranged(var(0) ** 2 + var(1) ** 2 - param(0),
               np.column_stack([pside[lim], qside[lim]]).reshape(-1, 2), rsq, -np.inf, 0.0)
    # (10)-(11) bus balances (214-220)
    p_rows = ranged(-param(0) - param(1) * var(0) ** 2, vm.reshape(-1, 1),
                    np.array([[b.pd, b.gs] for b in net.buses]).reshape(nb, 2), 0.0, 0.0)
    q_rows = ranged(-param(0) + param(1) * var(0) ** 2, vm.reshape(-1, 1),
                    np.array([[b.qd, b.bs] for b in net.buses]).reshape(nb, 2), 0.0, 0.0)
    # (12)-(15) increments (222-236)
    gbus = np.array([pos[g.bus] for g in net.generators], dtype=np.int64)
    mb.add_constraint_increments(var(0), pg.reshape(-1, 1), np.zeros((ng, 0)), p_rows[gbus])
    mb.add_constraint_increments(var(0), qg.reshape(-1, 1), np.zeros((ng, 0)), q_rows[gbus])
    for fp, fq, end in ((p_from, q_from, fb), (p_to, q_to, tb)):
        vi = np.concatenate([fp, fq]).reshape(-1, 1)
        mb.add_constraint_increments(-var(0), vi, np.zeros((vi.shape[0], 0)),
                                     np.concatenate([p_rows[end], q_rows[end]]))
    om = M.expand(mb.n_var, mb.n_con, mb.blocks)
    return OAcopf(om, np.concatenate(mb.lower), np.concatenate(mb.upper), np.concatenate(mb.start),
                  np.array(ranges, float).reshape(mb.n_con, 2))


def ordering(oa: OAcopf) -> np.ndarray:
    """The reference's ordering of the condensed pattern (amd.py:18-54 via the
    oracle's heap minimum degree; bit-identical to the shipped scan)."""
    from . import ordering as O
    from . import sparse as S

    om = oa.model
    cs = S.condense(om.hess_rows, om.hess_cols, om.jac_rows, om.jac_cols, om.n)
    r, c = cs.matrix.coords()
    return O.min_degree_order(om.n, r, c)
