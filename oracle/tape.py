"""Vectorised tape interpreter (oracle).

Restates the reference's per-pattern evaluator
(src/gridnlp/expressions.py:222-409): a tape is a list of ``(op, a, b)``
triples (opcodes expressions.py:23-37) evaluated column-wise over all
records of a block.  ``None`` marks structurally absent adjoints/tangents,
exactly as the reference does, so that e.g. an infinite partial that is
never reached does not poison a result with ``0*inf``.
"""
from __future__ import annotations

import numpy as np

VAR, PAR, CONST, ADD, SUB, MUL, DIV, POW, NEG, SIN, COS, LOG, SQRT, EXP = range(14)
_BIN = (ADD, SUB, MUL, DIV)


def forward(ops, consts, X, P):
    """Values of every tape entry (expressions.py:222-254)."""
    v = [None] * len(ops)
    for i, (op, a, b) in enumerate(ops):
        if op == VAR:
            v[i] = X[:, a]
        elif op == PAR:
            v[i] = P[:, a]
        elif op == CONST:
            v[i] = consts[b]
        elif op == ADD:
            v[i] = v[a] + v[b]
        elif op == SUB:
            v[i] = v[a] - v[b]
        elif op == MUL:
            v[i] = v[a] * v[b]
        elif op == DIV:
            v[i] = v[a] / v[b]
        elif op == POW:
            v[i] = v[a] ** consts[b]
        elif op == NEG:
            v[i] = -v[a]
        elif op == SIN:
            v[i] = np.sin(v[a])
        elif op == COS:
            v[i] = np.cos(v[a])
        elif op == LOG:
            v[i] = np.log(v[a])
        elif op == SQRT:
            v[i] = np.sqrt(v[a])
        else:
            v[i] = np.exp(v[a])
    return v


def local_partials(ops, consts, v, i):
    """(d entry / d a, d entry / d b), None where absent (expressions.py:259-285)."""
    op, a, b = ops[i]
    if op == ADD:
        return 1.0, 1.0
    if op == SUB:
        return 1.0, -1.0
    if op == MUL:
        return v[b], v[a]
    if op == DIV:
        return 1.0 / v[b], -v[a] / (v[b] * v[b])
    if op == POW:
        c = consts[b]
        return c * v[a] ** (c - 1.0), None
    if op == NEG:
        return -1.0, None
    if op == SIN:
        return np.cos(v[a]), None
    if op == COS:
        return -np.sin(v[a]), None
    if op == LOG:
        return 1.0 / v[a], None
    if op == SQRT:
        return 0.5 / v[i], None
    if op == EXP:
        return v[i], None
    return None, None


def _acc(lst, k, val):
    lst[k] = val if lst[k] is None else lst[k] + val


def reverse(ops, consts, out, v, n_rec):
    """Adjoint sweep -> ({slot: d out/d slot}, adjoints) (expressions.py:287-314)."""
    adj = [None] * len(ops)
    adj[out] = np.ones(n_rec)
    grad = {}
    for i in range(len(ops) - 1, -1, -1):
        ai = adj[i]
        if ai is None:
            continue
        op, a, b = ops[i]
        if op == VAR:
            grad[a] = grad[a] + ai if a in grad else +ai
            continue
        if op in (PAR, CONST):
            continue
        fa, fb = local_partials(ops, consts, v, i)
        _acc(adj, a, fa * ai)
        if fb is not None:
            _acc(adj, b, fb * ai)
    return grad, adj


def hessian_column(ops, consts, v, adj, tslot):
    """Forward-over-reverse sweep for one tangent slot (expressions.py:316-409).

    Returns {slot: d2 out / (d slot d tslot)}.
    """
    n = len(ops)
    dot = [None] * n
    for i, (op, a, b) in enumerate(ops):
        if op == VAR:
            dot[i] = 1.0 if a == tslot else None
            continue
        if op in (PAR, CONST):
            continue
        da = dot[a]
        db = dot[b] if op in _BIN else None
        if da is None and db is None:
            continue
        fa, fb = local_partials(ops, consts, v, i)
        t = fa * da if da is not None else None
        if db is not None:
            t = fb * db if t is None else t + fb * db
        dot[i] = t
    adot = [None] * n
    hcol = {}
    for i in range(n - 1, -1, -1):
        ai, adi = adj[i], adot[i]
        if ai is None and adi is None:
            continue
        op, a, b = ops[i]
        if op == VAR:
            if adi is not None:
                hcol[a] = adi if a not in hcol else hcol[a] + adi
            continue
        if op in (PAR, CONST):
            continue
        fa, fb = local_partials(ops, consts, v, i)
        da = dot[a]
        db = dot[b] if op in _BIN else None
        dfa = dfb = None
        if op == MUL:
            dfa, dfb = db, da
        elif op == DIV:
            vb = v[b]
            if db is not None:
                dfa = -db / (vb * vb)
            if da is not None:
                dfb = -da / (vb * vb)
            if db is not None:
                t2 = 2.0 * v[a] * db / (vb * vb * vb)
                dfb = t2 if dfb is None else dfb + t2
        elif op == POW:
            c = consts[b]
            if da is not None and c != 1.0:
                dfa = c * (c - 1.0) * v[a] ** (c - 2.0) * da
        elif op in (SIN, COS, LOG, SQRT, EXP) and da is not None:
            if op == SIN:
                dfa = -np.sin(v[a]) * da
            elif op == COS:
                dfa = -np.cos(v[a]) * da
            elif op == LOG:
                dfa = -da / (v[a] * v[a])
            elif op == SQRT:
                dfa = -0.25 * da / (v[a] * v[i])
            else:
                dfa = v[i] * da
        if ai is not None and dfa is not None:
            _acc(adot, a, dfa * ai)
        if adi is not None:
            _acc(adot, a, fa * adi)
        if fb is not None:
            if ai is not None and dfb is not None:
                _acc(adot, b, dfb * ai)
            if adi is not None:
                _acc(adot, b, fb * adi)
    return hcol


def template(ops, consts, out):
    """Structural first slots / second pairs (expressions.py:173-219)."""
    deps, pairs = [], set()

    def cross(u, w):
        for i in u:
            for j in w:
                pairs.add((max(i, j), min(i, j)))

    for op, a, b in ops:
        if op == VAR:
            deps.append(frozenset((a,)))
        elif op in (PAR, CONST):
            deps.append(frozenset())
        elif op in (ADD, SUB):
            deps.append(deps[a] | deps[b])
        elif op == NEG:
            deps.append(deps[a])
        elif op == MUL:
            cross(deps[a], deps[b])
            deps.append(deps[a] | deps[b])
        elif op == DIV:
            cross(deps[a], deps[b])
            cross(deps[b], deps[b])
            deps.append(deps[a] | deps[b])
        elif op == POW:
            c = consts[b]
            if c == 0.0:
                deps.append(frozenset())
                continue
            if c != 1.0:
                cross(deps[a], deps[a])
            deps.append(deps[a])
        else:
            cross(deps[a], deps[a])
            deps.append(deps[a])
    live = deps[out]
    return sorted(live), sorted(p for p in pairs if p[0] in live and p[1] in live)
