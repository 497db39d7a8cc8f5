"""Sparse symmetric storage, ordering, symbolic and numeric Cholesky.

API of reference src/gridnlp/sparse/ (csc.py, amd.py, cholesky.py):
``SparseSymmetric``, ``coo_to_csc``, ``amd_order``, ``symbolic_cholesky``,
``factorize``, ``solve``, ``solve_in_place``, ``NumericFactor``.

Host symbolic work (CSC construction, minimum degree, elimination tree,
row patterns, L pattern and the supernodal front plan) runs in the native
C++ library; the numeric refactorisation and the triangular solves run on
the GPU (``csrc/chol.cu``).  ``values``/right-hand sides may be numpy
arrays (copied to HBM and back, like the reference's arrays) or CUDA
tensors (stay resident).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import device as D

PIVOT_FLOOR = 1e-30


class UpperTriangleEntry(ValueError):
    pass


@dataclass
class SparseSymmetric:
    """Symmetric matrix, lower triangle in CSC (csc.py:13-49)."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return self.indices.size

    def coords(self):
        cols = np.repeat(np.arange(self.n), np.diff(self.indptr))
        return self.indices.copy(), cols

    def to_dense(self) -> np.ndarray:
        r, c = self.coords()
        v = D.to_host(self.values) if D.is_tensor(self.values) else self.values
        a = np.zeros((self.n, self.n))
        a[r, c] = v
        a[c, r] = v
        return a


def coo_to_csc(n, rows, cols, values, accumulate=True):
    """Lower CSC from coordinates + slot map (csc.py:52-76), natively."""
    rows, cols = L.i64(rows), L.i64(cols)
    values = np.asarray(values, dtype=float)
    if rows.size and np.any(cols > rows):
        k = int(np.argmax(cols > rows))
        raise UpperTriangleEntry(f"entry ({rows[k]}, {cols[k]}) lies above the diagonal")
    nnz = ctypes.c_int64()
    lib = L.lib()
    L.check(lib.gn_coo_to_csc(n, rows.size, L.ptr(rows), L.ptr(cols), ctypes.byref(nnz),
                              None, None, None))
    indptr = np.empty(n + 1, np.int64)
    indices = np.empty(nnz.value, np.int64)
    slot = np.empty(rows.size, np.int64)
    L.check(lib.gn_coo_to_csc(n, rows.size, L.ptr(rows), L.ptr(cols), ctypes.byref(nnz),
                              L.ptr(indptr), L.ptr(indices), L.ptr(slot)))
    if not accumulate and nnz.value != rows.size:
        raise ValueError("duplicate coordinates without accumulate")
    vals = np.zeros(nnz.value)
    np.add.at(vals, slot, values)   # host-side construction of a user matrix
    return SparseSymmetric(n, indptr, indices, vals), slot


def amd_order(matrix: SparseSymmetric) -> np.ndarray:
    """Exact greedy minimum degree (amd.py:18-54), bit-identical permutation."""
    perm = np.empty(matrix.n, np.int64)
    ip, ix = L.i64(matrix.indptr), L.i64(matrix.indices)
    L.check(L.lib().gn_min_degree(matrix.n, L.ptr(ip), L.ptr(ix), L.ptr(perm)))
    return perm


class SymbolicFactorization:
    """Fixed-pattern factor structure (cholesky.py:27-45) + native front plan."""

    def __init__(self, matrix: SparseSymmetric, perm):
        self.n = matrix.n
        self.perm = L.i64(perm if perm is not None else np.arange(self.n))
        ip, ix = L.i64(matrix.indptr), L.i64(matrix.indices)
        h = ctypes.c_void_p()
        L.check(L.lib().gn_symbolic_create(self.n, L.ptr(ip), L.ptr(ix), L.ptr(self.perm),
                                           ctypes.byref(h)))
        self._h = h
        info = L.SymbolicInfo()
        L.check(L.lib().gn_symbolic_info(h, ctypes.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in L.SymbolicInfo._fields_}
        self._arrays = None
        self._uploaded = False

    def _export(self):
        if self._arrays is None:
            n, nnz, nl = self.n, self.info["nnz_a"], self.info["nnz_l"]
            a = dict(parent=np.empty(n, np.int64), a_rowptr=np.empty(n + 1, np.int64),
                     a_rowcol=np.empty(nnz, np.int64), a_srcslot=np.empty(nnz, np.int64),
                     row_ptr=np.empty(n + 1, np.int64), row_cols=np.empty(nl - n, np.int64),
                     l_colptr=np.empty(n + 1, np.int64), l_rowidx=np.empty(nl, np.int64))
            L.check(L.lib().gn_symbolic_export(self._h, *(L.ptr(a[k]) for k in (
                "parent", "a_rowptr", "a_rowcol", "a_srcslot", "row_ptr", "row_cols",
                "l_colptr", "l_rowidx"))))
            self._arrays = a
        return self._arrays

    def __getattr__(self, name):
        if name in ("parent", "a_rowptr", "a_rowcol", "a_srcslot", "row_ptr", "row_cols",
                    "l_colptr", "l_rowidx"):
            return self._export()[name]
        raise AttributeError(name)

    @property
    def factor_nnz(self) -> int:
        return self.info["nnz_l"]

    def handle(self):
        """Device plan (uploaded once)."""
        if not self._uploaded:
            D.require_cuda()
            L.check(L.lib().gn_symbolic_upload(self._h))
            self._uploaded = True
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and L._lib is not None:
                L.lib().gn_symbolic_destroy(h)
        except Exception:
            pass
        self._h = None


def symbolic_cholesky(matrix: SparseSymmetric, perm=None) -> SymbolicFactorization:
    return SymbolicFactorization(matrix, perm)


class NumericFactor:
    """Device-resident factor (front storage) of one refactorisation."""

    def __init__(self, symbolic: SymbolicFactorization, fronts: torch.Tensor, fail: torch.Tensor):
        self.symbolic = symbolic
        self.fronts = fronts
        self._fail = fail
        self._ok = None
        self._failing = -1

    def _sync(self):
        if self._ok is None:
            k = int(self._fail.item())
            self._ok = k >= self.symbolic.n
            self._failing = -1 if self._ok else int(self.symbolic.perm[k])
        return self._ok

    @property
    def ok(self) -> bool:
        return self._sync()

    @property
    def failing_column(self) -> int:
        self._sync()
        return self._failing

    @property
    def values(self) -> np.ndarray:
        """Factor values in the reference CSC layout (l_colptr / l_rowidx)."""
        return D.to_host(self.values_device())

    def values_device(self) -> torch.Tensor:
        out = D.empty(self.symbolic.factor_nnz)
        L.check(L.lib().gn_chol_export_l(self.symbolic.handle(), L.ptr(self.fronts), L.ptr(out),
                                         D.stream_ptr()))
        return out


class FactorWorkspace:
    """Reusable device buffers for repeated refactorisations of one pattern."""

    def __init__(self, symbolic: SymbolicFactorization):
        self.fronts = D.empty(max(1, symbolic.info["front_doubles"]))
        self.vec = D.empty(max(1, symbolic.info["vec_doubles"]))
        self.fail = torch.empty(1, dtype=torch.int64, device=self.fronts.device)


def factorize_device(symbolic: SymbolicFactorization, kvals: torch.Tensor,
                     ws: FactorWorkspace | None = None) -> NumericFactor:
    """Refactorise on the GPU; kvals is a CUDA tensor in the matrix's CSC order."""
    h = symbolic.handle()
    ws = ws or FactorWorkspace(symbolic)
    L.check(L.lib().gn_chol_factor(h, L.ptr(kvals), L.ptr(ws.fronts), L.ptr(ws.fail),
                                   D.stream_ptr()))
    f = NumericFactor(symbolic, ws.fronts, ws.fail)
    f._ws = ws
    return f


def factorize(symbolic: SymbolicFactorization, values, out=None) -> NumericFactor:
    """Numeric refactorisation with fresh values (cholesky.py:189-205)."""
    kv = D.to_dev(values)
    return factorize_device(symbolic, kv, getattr(out, "_ws", None))


def solve_device(factor: NumericFactor, b: torch.Tensor, x: torch.Tensor | None = None) -> torch.Tensor:
    sym = factor.symbolic
    x = b if x is None else x
    ws = getattr(factor, "_ws", None) or FactorWorkspace(sym)
    L.check(L.lib().gn_chol_solve(sym.handle(), L.ptr(factor.fronts), L.ptr(b), L.ptr(x),
                                  L.ptr(ws.vec), D.stream_ptr()))
    return x


def solve_in_place(factor: NumericFactor, rhs):
    """rhs <- P^T L^-T L^-1 P rhs (cholesky.py:208-213)."""
    if D.is_tensor(rhs):
        return solve_device(factor, rhs)
    t = D.to_dev(rhs)
    solve_device(factor, t)
    rhs[...] = D.to_host(t)
    return rhs


def solve(factor: NumericFactor, b):
    """cholesky.py:216-217"""
    if D.is_tensor(b):
        return solve_device(factor, b.clone())
    return D.to_host(solve_device(factor, D.to_dev(b)))


def estimate_condition(factor: NumericFactor, matrix: SparseSymmetric) -> float:
    """Hager 1-norm condition estimate (cholesky.py:220-241) using device solves."""
    n = matrix.n
    if n == 0:
        return 1.0
    r, c = matrix.coords()
    v = np.abs(D.to_host(matrix.values) if D.is_tensor(matrix.values) else matrix.values)
    s = np.zeros(n)
    np.add.at(s, r, v)
    off = r != c
    np.add.at(s, c[off], v[off])
    norm_a = float(s.max())
    x = np.full(n, 1.0 / n)
    est = 0.0
    for _ in range(5):
        y = solve(factor, x)
        est_new = float(np.abs(y).sum())
        xi = np.sign(y)
        xi[xi == 0.0] = 1.0
        z = solve(factor, xi)
        j = int(np.argmax(np.abs(z)))
        if np.abs(z[j]) <= z @ x or est_new <= est:
            est = max(est, est_new)
            break
        est = est_new
        x = np.zeros(n)
        x[j] = 1.0
    return norm_a * est


def front_plan(symbolic: SymbolicFactorization) -> dict:
    """The supernodal front plan of a symbolic factorisation (diagnostics)."""
    nf = symbolic.info["n_fronts"]
    out = {k: np.empty(nf, np.int32) for k in ("first", "ncols", "nrows", "parent", "order")}
    nsm = ctypes.c_int64()
    L.check(L.lib().gn_symbolic_fronts(symbolic._h, *(L.ptr(out[k]) for k in
                                                      ("first", "ncols", "nrows", "parent", "order")),
                                       ctypes.byref(nsm)))
    out["nf_small"] = nsm.value
    return out


def trace_factor_solve(symbolic: SymbolicFactorization, kvals: torch.Tensor, b: torch.Tensor):
    """Run one refactorisation and one solve with per-front %globaltimer
    stamps; returns int64 [3][n_fronts][4] (factor, forward, backward) of
    (start, dependencies met, assembled, done) in ns (0 = not stamped), and
    [64][5] panel stamps of the last front (start, loaded, diagonal block,
    TRSM, trailing update)."""
    nf = symbolic.info["n_fronts"]
    tr = torch.zeros(3 * nf * 4 + 64 * 5 + 256, dtype=torch.int64, device=kvals.device)
    h = symbolic.handle()
    L.check(L.lib().gn_chol_set_trace(h, L.ptr(tr)))
    try:
        f = factorize_device(symbolic, kvals)
        solve_device(f, b.clone())
        torch.cuda.synchronize()
    finally:
        L.check(L.lib().gn_chol_set_trace(h, None))
    t = tr.cpu().numpy()
    trace_factor_solve.last_probes = t[12 * nf + 320:]   # kernel-specific probe stamps (diagnostics)
    return t[:12 * nf].reshape(3, nf, 4), t[12 * nf:12 * nf + 320].reshape(64, 5)
