"""Pattern-block expansion and AD evaluation (oracle).

Restates reference src/gridnlp/model.py (record order 128-140, COO
expansion and slot maps 229-303) and src/gridnlp/autodiff.py (eval_*
36-142).  Input is a neutral block description so the oracle can consume
models built by either the reference or the product:

    OBlock(kind, ops, consts, out, first_slots, second_pairs,
           var_idx[R, v], params[R, p], targets[R] | None)

``kind`` is one of "objective_sum", "constraint_define",
"constraint_increment" (model.py:24-26).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import tape as T

OBJ, DEF, INC = "objective_sum", "constraint_define", "constraint_increment"


@dataclass
class OBlock:
    kind: str
    ops: list
    consts: list
    out: int
    first_slots: list
    second_pairs: list
    var_idx: np.ndarray
    params: np.ndarray
    targets: np.ndarray | None = None
    jac_slots: list = field(default_factory=list)
    hess_slots: list = field(default_factory=list)
    hess_factor: list = field(default_factory=list)

    @property
    def n(self):
        return self.var_idx.shape[0]


def canonical_order(var_idx, params, targets=None):
    """Record permutation: targets, then var_idx columns, then params (model.py:128-140)."""
    keys = [params[:, c] for c in range(params.shape[1] - 1, -1, -1)]
    keys += [var_idx[:, c] for c in range(var_idx.shape[1] - 1, -1, -1)]
    if targets is not None:
        keys.append(targets)
    if not keys:
        return np.arange(var_idx.shape[0])
    return np.lexsort(keys)


def from_model(model) -> list[OBlock]:
    """Neutral copies of a finalized model's blocks (reference or product)."""
    out = []
    for b in model.pattern_blocks:
        tp = b.tape
        fs, sp = T.template(tp.ops, tp.consts, tp.out)
        out.append(OBlock(b.kind, list(tp.ops), list(tp.consts), tp.out, fs, sp,
                          np.asarray(b.var_idx, np.int64), np.asarray(b.params, float),
                          None if b.targets is None else np.asarray(b.targets, np.int64)))
    return out


@dataclass
class OModel:
    n: int
    m: int
    blocks: list
    jac_rows: np.ndarray
    jac_cols: np.ndarray
    hess_rows: np.ndarray
    hess_cols: np.ndarray


def _dedup(i, j):
    key = np.unique(i.astype(np.int64) << 32 | j.astype(np.int64))
    return key >> 32, key & 0xFFFFFFFF, key


def expand(n, m, blocks) -> OModel:
    """Template expansion + dedup + per-block slot maps (model.py:250-303)."""
    ji, jj, hi, hj = [], [], [], []
    for b in blocks:
        for (a, c) in b.second_pairs:
            ga, gc = b.var_idx[:, a], b.var_idx[:, c]
            hi.append(np.maximum(ga, gc))
            hj.append(np.minimum(ga, gc))
        if b.kind != OBJ:
            for s in b.first_slots:
                ji.append(b.targets)
                jj.append(b.var_idx[:, s])
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)
    jr, jc, jkey = _dedup(cat(ji), cat(jj))
    hr, hc, hkey = _dedup(cat(hi), cat(hj))
    for b in blocks:
        b.jac_slots, b.hess_slots, b.hess_factor = [], [], []
        if b.kind != OBJ:
            for s in b.first_slots:
                b.jac_slots.append(np.searchsorted(jkey, b.targets << 32 | b.var_idx[:, s]))
        for (a, c) in b.second_pairs:
            ga, gc = b.var_idx[:, a], b.var_idx[:, c]
            b.hess_slots.append(np.searchsorted(hkey, np.maximum(ga, gc) << 32 | np.minimum(ga, gc)))
            b.hess_factor.append(np.where(ga == gc, 2.0, 1.0) if a != c else np.ones(b.n))
    return OModel(n, m, blocks, jr, jc, hr, hc)


class NonFinite(ArithmeticError):
    pass


def _gather(b, x):
    return x[b.var_idx] if b.var_idx.shape[1] else np.zeros((b.n, 0))


def _finite(arr, what):
    if not np.all(np.isfinite(arr)):
        raise NonFinite(what)


def _value(b, x):
    v = T.forward(b.ops, b.consts, _gather(b, x), b.params)
    return np.broadcast_to(v[b.out], (b.n,))


def objective(om, x):
    """autodiff.py:45-54"""
    tot = 0.0
    with np.errstate(all="ignore"):
        for b in om.blocks:
            if b.kind == OBJ and b.n:
                tot += float(np.sum(_value(b, x)))
    _finite(tot, "objective")
    return tot


def constraints(om, x):
    """autodiff.py:57-70: defines assign, then increments add in block order."""
    c = np.zeros(om.m)
    with np.errstate(all="ignore"):
        for b in om.blocks:
            if b.kind == DEF and b.n:
                c[b.targets] = _value(b, x)
        for b in om.blocks:
            if b.kind == INC and b.n:
                np.add.at(c, b.targets, _value(b, x))
    _finite(c, "constraint")
    return c


def gradient(om, x):
    """autodiff.py:73-85"""
    g = np.zeros(om.n)
    with np.errstate(all="ignore"):
        for b in om.blocks:
            if b.kind != OBJ or not b.n:
                continue
            v = T.forward(b.ops, b.consts, _gather(b, x), b.params)
            sg, _ = T.reverse(b.ops, b.consts, b.out, v, b.n)
            for s, gv in sg.items():
                np.add.at(g, b.var_idx[:, s], gv)
    _finite(g, "gradient")
    return g


def jacobian(om, x):
    """autodiff.py:88-103"""
    jv = np.zeros(om.jac_rows.size)
    with np.errstate(all="ignore"):
        for b in om.blocks:
            if b.kind == OBJ or not b.n:
                continue
            v = T.forward(b.ops, b.consts, _gather(b, x), b.params)
            sg, _ = T.reverse(b.ops, b.consts, b.out, v, b.n)
            for k, s in enumerate(b.first_slots):
                if s in sg:
                    np.add.at(jv, b.jac_slots[k], np.broadcast_to(sg[s], (b.n,)))
    _finite(jv, "jacobian")
    return jv


def hessian(om, x, y, obj_weight=1.0):
    """Lower triangle of obj_weight*H(f) + sum y_i H(g_i) (autodiff.py:106-142)."""
    hv = np.zeros(om.hess_rows.size)
    with np.errstate(all="ignore"):
        for b in om.blocks:
            if not b.second_pairs or not b.n:
                continue
            if b.kind == OBJ:
                if obj_weight == 0.0:
                    continue
                w = obj_weight
            else:
                w = y[b.targets]
            v = T.forward(b.ops, b.consts, _gather(b, x), b.params)
            _, adj = T.reverse(b.ops, b.consts, b.out, v, b.n)
            cols = {s: T.hessian_column(b.ops, b.consts, v, adj, s)
                    for s in sorted({c for _, c in b.second_pairs})}
            for k, (a, c) in enumerate(b.second_pairs):
                h = cols[c].get(a)
                if h is None:
                    continue
                np.add.at(hv, b.hess_slots[k],
                          np.broadcast_to(w * b.hess_factor[k] * h, (b.n,)))
    _finite(hv, "hessian")
    return hv
