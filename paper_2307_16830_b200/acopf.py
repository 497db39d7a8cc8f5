"""Polar ACOPF as fifteen pattern blocks (host model construction).

Same model as reference src/gridnlp/acopf.py:68-246 -- the same variables
in the same order, the same fifteen instructions in the same order, so the
compiled sparsity, row numbering and slot maps are identical (SURVEY.md
Appendix E).  The instructions built here are the patterns the device AD
evaluates: generator cost, reference angle, the four branch flows, angle
and thermal limits, bus balances and the linear increments.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .expressions import cos, param, sin, var
from .matpower import NetworkData
from .model import CompiledModel, ModelBuilder


@dataclass
class AcopfVariables:
    va: np.ndarray
    vm: np.ndarray
    pg: np.ndarray
    qg: np.ndarray
    p_from: np.ndarray
    p_to: np.ndarray
    q_from: np.ndarray
    q_to: np.ndarray


@dataclass
class AcopfModel:
    model: CompiledModel
    variables: AcopfVariables
    ranges: np.ndarray
    network: NetworkData
    p_balance_rows: np.ndarray
    q_balance_rows: np.ndarray


def branch_admittance(br) -> dict:
    """Tap-model admittances (acopf.py:53-65)."""
    y = 1.0 / complex(br.r, br.x)
    g, b = y.real, y.imag
    tt = br.tap * br.tap
    bc2 = br.b_charge / 2.0
    return dict(gff=g / tt, bff=(b + bc2) / tt, gtt=g, btt=b + bc2,
                gft=g / br.tap, bft=b / br.tap, shift=br.shift)


def _flow_instructions():
    """p/q from/to instructions; slots (flow, vm_f, vm_t, va_f, va_t) (acopf.py:141-158)."""
    dlt_f = var(3) - var(4) - param(3)
    dlt_t = var(4) - var(3) + param(3)
    vv = lambda: var(1) * var(2)
    pf = var(0) - (param(0) * var(1) ** 2 - vv() * (param(1) * cos(dlt_f) + param(2) * sin(dlt_f)))
    qf = var(0) - (-param(0) * var(1) ** 2 - vv() * (param(1) * sin(dlt_f) - param(2) * cos(dlt_f)))
    pt = var(0) - (param(0) * var(2) ** 2 - vv() * (param(1) * cos(dlt_t) + param(2) * sin(dlt_t)))
    qt = var(0) - (-param(0) * var(2) ** 2 - vv() * (param(1) * sin(dlt_t) - param(2) * cos(dlt_t)))
    return pf, qf, pt, qt


def build_acopf(net: NetworkData) -> AcopfModel:
    nb, ng, nl = len(net.buses), len(net.generators), len(net.branches)
    pos = net.bus_index()
    base = net.base_mva
    mb = ModelBuilder()
    va = mb.add_variables(nb, np.full(nb, -np.inf), np.full(nb, np.inf), np.zeros(nb))
    vm = mb.add_variables(nb, np.array([b.vmin for b in net.buses]),
                          np.array([b.vmax for b in net.buses]), np.ones(nb))
    pg = mb.add_variables(ng, np.array([g.pmin for g in net.generators]),
                          np.array([g.pmax for g in net.generators]), np.zeros(ng))
    qg = mb.add_variables(ng, np.array([g.qmin for g in net.generators]),
                          np.array([g.qmax for g in net.generators]), np.zeros(ng))
    rate = np.array([br.rate_a for br in net.branches])
    lo = np.where(rate > 0, -rate, -np.inf)
    hi = np.where(rate > 0, rate, np.inf)
    empty = np.zeros(0, dtype=np.int64)
    if nl:
        pflow = mb.add_variables(2 * nl, np.tile(lo, 2), np.tile(hi, 2), np.zeros(2 * nl)).indices
        qflow = mb.add_variables(2 * nl, np.tile(lo, 2), np.tile(hi, 2), np.zeros(2 * nl)).indices
    else:
        pflow = qflow = np.zeros(0, dtype=np.int64)
    V = AcopfVariables(va.indices, vm.indices, pg.indices, qg.indices,
                       pflow[:nl], pflow[nl:], qflow[:nl], qflow[nl:])
    ranges: list = []

    def ranged(instr, vi, pa, rlo, rhi):
        rows = mb.add_constraints(instr, vi, pa)
        ranges.extend(zip(np.broadcast_to(np.asarray(rlo, float), rows.shape).tolist(),
                          np.broadcast_to(np.asarray(rhi, float), rows.shape).tolist()))
        return rows

    adm = [branch_admittance(br) for br in net.branches]
    fb = np.array([pos[br.from_bus] for br in net.branches], dtype=np.int64)
    tb = np.array([pos[br.to_bus] for br in net.branches], dtype=np.int64)

    # (1) generation cost in per-unit coefficients
    cost = np.array([[g.cost[0] * base * base, g.cost[1] * base, g.cost[2]]
                     for g in net.generators]).reshape(ng, 3)
    mb.add_objective(param(0) * var(0) ** 2 + param(1) * var(0) + param(2),
                     V.pg.reshape(-1, 1), cost)
    # (2) reference angle
    ranged(var(0), np.array([[V.va[pos[net.ref_bus]]]]), np.zeros((1, 0)), 0.0, 0.0)
    # (3)-(6) branch flows
    quad = (np.column_stack([V.vm[fb], V.vm[tb], V.va[fb], V.va[tb]])
            if nl else np.zeros((0, 4), dtype=np.int64))

    def prm(keys):
        return np.array([[a[k] for k in keys] for a in adm]).reshape(nl, len(keys))

    pf, qf, pt, qt = _flow_instructions()
    for instr, flow, self_key in ((pf, V.p_from, "gff"), (qf, V.q_from, "bff"),
                                  (pt, V.p_to, "gtt"), (qt, V.q_to, "btt")):
        vi = np.column_stack([flow, quad]) if nl else np.zeros((0, 5), dtype=np.int64)
        ranged(instr, vi, prm((self_key, "gft", "bft", "shift")), 0.0, 0.0)
    # (7) angle-difference limits (+-360 deg or (0, 0) means unconstrained)
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
    ranged(var(0) - var(1),
           np.column_stack([V.va[fb[sel]], V.va[tb[sel]]]) if sel.size else np.zeros((0, 2), np.int64),
           np.zeros((sel.size, 0)),
           np.array(alo) if sel.size else np.zeros(0), np.array(ahi) if sel.size else np.zeros(0))
    # (8)-(9) apparent-power limits on rated branches
    lim = np.flatnonzero(rate > 0)
    rsq = (rate[lim] ** 2).reshape(-1, 1)
    thermal = var(0) ** 2 + var(1) ** 2 - param(0)
    for pside, qside in ((V.p_from, V.q_from), (V.p_to, V.q_to)):
        ranged(thermal,
               np.column_stack([pside[lim], qside[lim]]) if lim.size else np.zeros((0, 2), np.int64),
               rsq, -np.inf, 0.0)
    # (10)-(11) bus balances seeded with load and shunt
    p_rows = ranged(-param(0) - param(1) * var(0) ** 2, V.vm.reshape(-1, 1),
                    np.array([[b.pd, b.gs] for b in net.buses]).reshape(nb, 2), 0.0, 0.0)
    q_rows = ranged(-param(0) + param(1) * var(0) ** 2, V.vm.reshape(-1, 1),
                    np.array([[b.qd, b.bs] for b in net.buses]).reshape(nb, 2), 0.0, 0.0)
    # (12)-(13) generator injections
    gbus = np.array([pos[g.bus] for g in net.generators], dtype=np.int64)
    mb.add_constraint_increments(var(0), V.pg.reshape(-1, 1), np.zeros((ng, 0)), p_rows[gbus])
    mb.add_constraint_increments(var(0), V.qg.reshape(-1, 1), np.zeros((ng, 0)), q_rows[gbus])
    # (14)-(15) flows leaving each branch end
    for fp, fq, end in ((V.p_from, V.q_from, fb), (V.p_to, V.q_to, tb)):
        vi = np.concatenate([fp, fq]).reshape(-1, 1)
        mb.add_constraint_increments(-var(0), vi, np.zeros((vi.shape[0], 0)),
                                     np.concatenate([p_rows[end], q_rows[end]]))
    model = mb.finalize()
    return AcopfModel(model, V, np.array(ranges).reshape(model.n_con, 2), net, p_rows, q_rows)
