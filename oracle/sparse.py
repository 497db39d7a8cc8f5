"""Symbolic condensation, symbolic/numeric Cholesky and solves (oracle).

Restates reference src/gridnlp/sparse/csc.py:52-76 (``coo_to_csc``),
src/gridnlp/kkt.py:243-283 (``symbolic_condense``) and
src/gridnlp/sparse/cholesky.py:56-217 (etree, row patterns, L pattern,
factorize, solve).  The numeric kernels are the C restatement in
oracle/csrc/chol.c, loaded with ctypes.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .build import build as _build_lib

PIVOT_FLOOR = 1e-30   # cholesky.py:24


@dataclass
class OCsc:
    n: int
    indptr: np.ndarray
    indices: np.ndarray
    values: np.ndarray

    def coords(self):
        cols = np.repeat(np.arange(self.n), np.diff(self.indptr))
        return self.indices.copy(), cols

    def to_dense(self):
        r, c = self.coords()
        a = np.zeros((self.n, self.n))
        a[r, c] = self.values
        a[c, r] = self.values
        return a


def coo_to_csc(n, rows, cols, values):
    """Lower CSC + slot map, column-major unique keys (csc.py:52-76)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    if rows.size and np.any(cols > rows):
        raise ValueError("entry above the diagonal")
    keys = cols << 32 | rows
    uniq, slot = np.unique(keys, return_inverse=True)
    vals = np.zeros(uniq.size)
    np.add.at(vals, slot, np.asarray(values, float))
    indptr = np.zeros(n + 1, np.int64)
    np.add.at(indptr, (uniq >> 32) + 1, 1)
    np.cumsum(indptr, out=indptr)
    return OCsc(n, indptr, uniq & 0xFFFFFFFF, vals), slot


@dataclass
class OCondensed:
    matrix: OCsc
    w_map: np.ndarray
    diag_map: np.ndarray
    ata_map: np.ndarray
    ata_row: np.ndarray
    ata_s1: np.ndarray
    ata_s2: np.ndarray


def condense(hess_rows, hess_cols, jac_rows, jac_cols, n) -> OCondensed:
    """Pattern of W + I + tril(A^T A) and its scatter maps (kkt.py:243-283)."""
    starts = np.flatnonzero(np.diff(jac_rows, prepend=-1))
    ends = np.append(starts[1:], jac_rows.size)
    pi, pj, s1, s2, rw = [], [], [], [], []
    for st, en in zip(starts, ends):
        la, lb = np.tril_indices(en - st)
        cc = jac_cols[st:en]
        pi.append(cc[la])
        pj.append(cc[lb])
        s1.append(st + la)
        s2.append(st + lb)
        rw.append(np.full(la.size, jac_rows[st]))
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)
    pi, pj, s1, s2, rw = map(cat, (pi, pj, s1, s2, rw))
    rows = np.concatenate([hess_rows, np.arange(n), pi])
    cols = np.concatenate([hess_cols, np.arange(n), pj])
    mat, slot = coo_to_csc(n, rows, cols, np.zeros(rows.size))
    nw = hess_rows.size
    return OCondensed(mat, slot[:nw], slot[nw:nw + n], slot[nw + n:], rw, s1, s2)


def assemble(cs: OCondensed, w_vals, a_vals, sigma_x, delta_w, d):
    """K values in the reference's scatter order (kkt.py:300-312)."""
    v = np.zeros(cs.matrix.indices.size)
    np.add.at(v, cs.w_map, w_vals)
    np.add.at(v, cs.diag_map, sigma_x + delta_w)
    if cs.ata_map.size:
        np.add.at(v, cs.ata_map, d[cs.ata_row] * a_vals[cs.ata_s1] * a_vals[cs.ata_s2])
    return v


@dataclass
class OSymbolic:
    n: int
    perm: np.ndarray
    parent: np.ndarray
    a_rowptr: np.ndarray
    a_rowcol: np.ndarray
    a_srcslot: np.ndarray
    row_ptr: np.ndarray
    row_cols: np.ndarray
    l_colptr: np.ndarray
    l_rowidx: np.ndarray


def etree(n, rowptr, rowcol):
    """Liu's elimination tree with path compression (cholesky.py:56-70)."""
    parent = np.full(n, -1, np.int64)
    anc = np.full(n, -1, np.int64)
    rp, rc = rowptr.tolist(), rowcol.tolist()
    par, an = parent.tolist(), anc.tolist()
    for k in range(n):
        for t in range(rp[k], rp[k + 1]):
            i = rc[t]
            while an[i] != -1 and an[i] != k:
                nxt = an[i]
                an[i] = k
                i = nxt
            if an[i] == -1 and i != k:
                an[i] = k
                par[i] = k
    return np.array(par, np.int64)


def row_patterns(n, rowptr, rowcol, parent):
    """Reach of each permuted row in the etree, sorted (cholesky.py:73-91)."""
    mark = [-1] * n
    par = parent.tolist()
    rp, rc = rowptr.tolist(), rowcol.tolist()
    ptr = [0] * (n + 1)
    out = []
    for k in range(n):
        pat = []
        mark[k] = k
        for t in range(rp[k], rp[k + 1]):
            i = rc[t]
            while i != -1 and mark[i] != k:
                mark[i] = k
                pat.append(i)
                i = par[i]
        pat.sort()
        out.extend(pat)
        ptr[k + 1] = ptr[k] + len(pat)
    return np.array(ptr, np.int64), np.array(out, np.int64)


def symbolic(mat: OCsc, perm) -> OSymbolic:
    """cholesky.py:94-144"""
    n = mat.n
    perm = np.asarray(perm, np.int64)
    pinv = np.empty(n, np.int64)
    pinv[perm] = np.arange(n)
    r, c = mat.coords()
    pr = np.maximum(pinv[r], pinv[c])
    pc = np.minimum(pinv[r], pinv[c])
    order = np.lexsort((pc, pr))
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, pr + 1, 1)
    np.cumsum(rowptr, out=rowptr)
    rowcol = pc[order]
    src = np.arange(r.size, dtype=np.int64)[order]
    parent = etree(n, rowptr, rowcol)
    rptr, rcols = row_patterns(n, rowptr, rowcol, parent)
    counts = np.ones(n, np.int64)
    np.add.at(counts, rcols, 1)
    colptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=colptr[1:])
    rowidx = np.empty(int(colptr[-1]), np.int64)
    fill = colptr[:-1].copy()
    rowidx[fill] = np.arange(n)
    fill += 1
    # rows of each factor column in increasing order (diagonal first)
    owner = np.repeat(np.arange(n), np.diff(rptr))
    o = np.argsort(rcols, kind="stable")
    cj, ck = rcols[o], owner[o]
    pos = fill[cj] + (np.arange(cj.size) - np.searchsorted(cj, cj))
    rowidx[pos] = ck
    return OSymbolic(n, perm, parent, rowptr, rowcol, src, rptr, rcols, colptr, rowidx)


_lib = None


def _clib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(_build_lib())
        p = ctypes.c_void_p
        _lib.oracle_chol.restype = ctypes.c_int64
        _lib.oracle_chol.argtypes = [ctypes.c_int64] + [p] * 10 + [ctypes.c_double]
        _lib.oracle_solve.restype = None
        _lib.oracle_solve.argtypes = [ctypes.c_int64, p, p, p, p]
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def factorize(sym: OSymbolic, values):
    """-> (l_vals, ok, failing_column) (cholesky.py:189-205)."""
    n = sym.n
    a = np.ascontiguousarray(np.asarray(values, float)[sym.a_srcslot])
    l_vals = np.zeros(sym.l_rowidx.size)
    cpos = np.zeros(n, np.int64)
    x = np.zeros(n)
    bad = _clib().oracle_chol(n, _ptr(sym.a_rowptr), _ptr(sym.a_rowcol), _ptr(a),
                              _ptr(sym.row_ptr), _ptr(sym.row_cols), _ptr(sym.l_colptr),
                              _ptr(sym.l_rowidx), _ptr(l_vals), _ptr(cpos), _ptr(x),
                              PIVOT_FLOOR)
    if bad >= 0:
        return l_vals, False, int(sym.perm[bad])
    return l_vals, True, -1


def solve(sym: OSymbolic, l_vals, b):
    """P^T L^-T L^-1 P b (cholesky.py:208-217)."""
    xp = np.ascontiguousarray(np.asarray(b, float)[sym.perm])
    _clib().oracle_solve(sym.n, _ptr(sym.l_colptr), _ptr(sym.l_rowidx), _ptr(l_vals), _ptr(xp))
    out = np.empty_like(xp)
    out[sym.perm] = xp
    return out
