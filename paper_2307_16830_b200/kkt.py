"""Condensed KKT machinery on the GPU.

Same structure and API as reference src/gridnlp/kkt.py: the seven-block
Newton system, its condensation to

    (W + dw I + Sigma_x + A^T D A) dx = qx + A^T (C qs + D qy),
    C = (dc Sigma_s + (1 + dc dw) I)^-1,  D = (Sigma_s + dw I) C,

diagonal recoveries, the inertia-correction schedule and iterative
refinement against the full system.  Every vector lives in HBM; the
arithmetic runs in the native kernels of ``csrc/kkt.cu`` (assembly, rhs,
recoveries, double-double residual) and ``csrc/chol.cu`` (factor/solve).
Host code only sequences kernels and reads back the scalars the control
flow branches on (PD flag, residual norms).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from . import device as D
from . import sparse as S
from .profiling import span

DELTA_W_INIT = 1e-4
DELTA_W_MIN = 1e-20
DELTA_W_MAX = 1e40
DELTA_C_VALUE = 1e-8
KAPPA_IR = 10.0
MAX_IR_ROUNDS = 10

FIELDS = ("x", "s", "y", "zxl", "zxu", "zsl", "zsu")


class DegenerateInterior(RuntimeError):
    """A finite-bound slack is not strictly positive."""


class RegularizationExhausted(RuntimeError):
    """No positive-definite condensed system below the delta_w ceiling."""


@dataclass
class RegState:
    delta_w_last: float = 0.0


class _Vec7:
    """Seven device vectors (x, s, y, zxl, zxu, zsl, zsu)."""

    def __setattr__(self, name, value):
        object.__setattr__(self, name, value)
        if name in FIELDS:
            object.__setattr__(self, "_cs", None)   # pointer struct is rebuilt on demand

    def __init__(self, x, s, y, zxl, zxu, zsl, zsu):
        self.x, self.s, self.y = D.to_dev(x), D.to_dev(s), D.to_dev(y)
        self.zxl, self.zxu = D.to_dev(zxl), D.to_dev(zxu)
        self.zsl, self.zsu = D.to_dev(zsl), D.to_dev(zsu)

    @classmethod
    def empty(cls, n, m):
        obj = cls.__new__(cls)
        for f, k in zip(FIELDS, (n, m, m, n, n, m, m)):
            setattr(obj, f, D.empty(k))
        return obj

    def parts(self):
        return [getattr(self, f) for f in FIELDS]

    def c_struct(self) -> L.Vec7:
        cs = getattr(self, "_cs", None)
        if cs is None:
            cs = L.Vec7(*(t.data_ptr() for t in self.parts()))
            object.__setattr__(self, "_cs", cs)
        return cs

    def numpy(self):
        return [D.to_host(t) for t in self.parts()]


class PVec(_Vec7):
    """Right-hand side of the seven-block Newton system (kkt.py:60-70)."""


class Steps(_Vec7):
    """Newton steps (kkt.py:73-85)."""

    def axpy(self, other: "Steps", alpha=1.0) -> None:
        for f in FIELDS:
            getattr(self, f).add_(getattr(other, f), alpha=alpha)


def _bind(kkt, y: _Vec7, x: _Vec7, alpha):
    yc, xc = y.c_struct(), x.c_struct()
    L.check(L.lib().gn_vec7_axpy(kkt, ctypes.byref(yc), ctypes.byref(xc), alpha, D.stream_ptr()))


@dataclass
class CondensedStructure:
    """Pattern of W + I + tril(A^T A) and its scatter maps (kkt.py:232-240).

    The native plan (``handle``) is what the device path uses; the numpy
    views of the maps are exported from it on first access."""

    _MAPS = ("w_map", "diag_map", "ata_map", "ata_row", "ata_s1", "ata_s2")

    def __init__(self, matrix: S.SparseSymmetric, handle, nnz_w, n_products):
        self.matrix = matrix
        self.handle = handle
        self._nw, self._np = int(nnz_w), int(n_products)
        self._maps = None

    def _export(self):
        if self._maps is None:
            n = self.matrix.n
            m = {"w_map": np.empty(self._nw, np.int64), "diag_map": np.empty(n, np.int64)}
            for k in ("ata_map", "ata_row", "ata_s1", "ata_s2"):
                m[k] = np.empty(self._np, np.int64)
            L.check(L.lib().gn_condense_export(self.handle, None, None,
                                               *(L.ptr(m[k]) for k in self._MAPS)))
            self._maps = m
        return self._maps

    def __getattr__(self, name):
        if name in CondensedStructure._MAPS:
            return self._export()[name]
        raise AttributeError(name)

    def __del__(self):
        try:
            if self.__dict__.get("handle") is not None and L._lib is not None:
                L.lib().gn_condense_destroy(self.handle)
        except Exception:
            pass
        self.handle = None


def symbolic_condense(hess_rows, hess_cols, jac_rows, jac_cols, n) -> CondensedStructure:
    """Pattern of W + diag + tril(A^T A) plus scatter maps (kkt.py:243-283), natively."""
    hr, hc, jr, jc = (L.i64(a) for a in (hess_rows, hess_cols, jac_rows, jac_cols))
    h = ctypes.c_void_p()
    L.check(L.lib().gn_condense_create(n, hr.size, L.ptr(hr), L.ptr(hc), jr.size, L.ptr(jr),
                                       L.ptr(jc), ctypes.byref(h)))
    nk, npr = ctypes.c_int64(), ctypes.c_int64()
    L.check(L.lib().gn_condense_info(h, ctypes.byref(nk), ctypes.byref(npr)))
    indptr, indices = np.empty(n + 1, np.int64), np.empty(nk.value, np.int64)
    L.check(L.lib().gn_condense_export(h, L.ptr(indptr), L.ptr(indices), None, None, None, None,
                                       None, None))
    mat = S.SparseSymmetric(n, indptr, indices, np.zeros(nk.value))
    return CondensedStructure(mat, h, hr.size, npr.value)


class HostAnalysis:
    """The host half of the symbolic analysis -- condensed pattern, ordering,
    symbolic factor and front plan -- on a worker thread (the native calls
    release the GIL), so it overlaps the device-side problem setup and the
    KKT plan upload of the calling thread.  Pure host work: no CUDA calls."""

    _pool = None
    # While an analysis runs, the interpreter's thread switch interval is cut
    # to 0.1 ms: the worker needs the GIL for a moment between its native
    # calls, and the launching thread is busy in Python (device setup), so
    # the default 5 ms interval would stall the worker at every hand-over.
    _active = 0
    _saved_interval = None
    _lock = None

    def __init__(self, model, ordering=None):
        import concurrent.futures as cf
        import sys
        import threading

        if HostAnalysis._pool is None:
            HostAnalysis._pool = cf.ThreadPoolExecutor(max_workers=4,
                                                       thread_name_prefix="gn-analysis")
            HostAnalysis._lock = threading.Lock()
        with HostAnalysis._lock:
            if HostAnalysis._active == 0:
                HostAnalysis._saved_interval = sys.getswitchinterval()
                sys.setswitchinterval(min(1e-4, HostAnalysis._saved_interval))
            HostAnalysis._active += 1
        self._released = False
        self.timings = {}
        self._cs_ready = threading.Event()
        self._cs = None
        self._fut = HostAnalysis._pool.submit(self._run, model, ordering)

    def _release(self):
        import sys

        if self._released:
            return
        self._released = True
        with HostAnalysis._lock:
            HostAnalysis._active -= 1
            if HostAnalysis._active == 0 and HostAnalysis._saved_interval is not None:
                sys.setswitchinterval(HostAnalysis._saved_interval)

    def _run(self, model, ordering):
        import os
        import time

        # this process's share of the host cores (one process per GPU under
        # torchrun), minus one for the launching thread (device setup)
        share = len(os.sched_getaffinity(0)) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        L.lib().gn_set_host_threads(max(1, share - 1))
        try:
            t = time.perf_counter()
            self._cs = symbolic_condense(model.hess_rows, model.hess_cols, model.jac_rows,
                                         model.jac_cols, model.n_var)
            self.timings["condense"] = time.perf_counter() - t
        finally:
            self._cs_ready.set()
        t = time.perf_counter()
        if ordering is None:
            ordering = S.amd_order(self._cs.matrix)
        self.timings["ordering"] = time.perf_counter() - t
        t = time.perf_counter()
        sym = S.symbolic_cholesky(self._cs.matrix, ordering)
        self.timings["symbolic"] = time.perf_counter() - t
        return sym

    def condensed(self) -> CondensedStructure:
        self._cs_ready.wait()
        if self._cs is None:       # condensation failed: raise its error
            self._fut.result()
        return self._cs

    def symbolic(self):
        try:
            return self._fut.result()
        finally:
            self._release()

    def __del__(self):
        try:
            if not self._released:
                self._fut.result()
                self._release()
        except Exception:
            pass


class KKTWorkspace:
    """Device values of the full KKT system at the current iterate (kkt.py:96-221)."""

    def __init__(self, n, m, hess_rows, hess_cols, jac_rows, jac_cols, condensed=None):
        self.n, self.m = int(n), int(m)
        self.hess_rows, self.hess_cols = L.i64(hess_rows), L.i64(hess_cols)
        self.jac_rows, self.jac_cols = L.i64(jac_rows), L.i64(jac_cols)
        D.require_cuda()
        h = ctypes.c_void_p()
        L.check(L.lib().gn_kkt_create(self.n, self.m, self.hess_rows.size, L.ptr(self.hess_rows),
                                      L.ptr(self.hess_cols), self.jac_rows.size, L.ptr(self.jac_rows),
                                      L.ptr(self.jac_cols),
                                      None if condensed is None else condensed.handle,
                                      ctypes.byref(h)))
        self.handle = h
        self._has_assembly = condensed is not None
        self.w_vals = D.zeros(self.hess_rows.size)
        self.a_vals = D.zeros(self.jac_rows.size)
        self.delta_w = 0.0
        self.delta_c = 0.0
        for f in ("dxl", "dxu", "zxl", "zxu", "sigma_x"):
            setattr(self, f, D.zeros(self.n))
        for f in ("dsl", "dsu", "zsl", "zsu", "sigma_s"):
            setattr(self, f, D.zeros(self.m))
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.w_vals.device)
        self._scal = D.zeros(4)

    def attach_condensed(self, condensed: CondensedStructure):
        """Rebuild the plan with the assembly maps of ``condensed``."""
        if self._has_assembly:
            return
        L.lib().gn_kkt_destroy(self.handle)
        h = ctypes.c_void_p()
        L.check(L.lib().gn_kkt_create(self.n, self.m, self.hess_rows.size, L.ptr(self.hess_rows),
                                      L.ptr(self.hess_cols), self.jac_rows.size, L.ptr(self.jac_rows),
                                      L.ptr(self.jac_cols), condensed.handle, ctypes.byref(h)))
        self.handle = h
        self._has_assembly = True

    def __del__(self):
        h = getattr(self, "handle", None)
        try:
            if h is not None and L._lib is not None:
                L.lib().gn_kkt_destroy(h)
        except Exception:
            pass
        self.handle = None

    # -- state -------------------------------------------------------------
    def set_iterate(self, w_vals, a_vals, dxl, dxu, zxl, zxu, dsl, dsu, zsl, zsu):
        for name, v in (("w_vals", w_vals), ("a_vals", a_vals), ("dxl", dxl), ("dxu", dxu),
                        ("zxl", zxl), ("zxu", zxu), ("dsl", dsl), ("dsu", dsu), ("zsl", zsl),
                        ("zsu", zsu)):
            dst = getattr(self, name)
            if D.is_tensor(v) and v.data_ptr() == dst.data_ptr():
                continue
            dst.copy_(D.to_dev(v))
        st = D.stream_ptr()
        lib = L.lib()
        L.check(lib.gn_kkt_sigma(self.n, *(L.ptr(t) for t in (self.dxl, self.dxu, self.zxl,
                                                                self.zxu, self.sigma_x)), st))
        L.check(lib.gn_kkt_sigma(self.m, *(L.ptr(t) for t in (self.dsl, self.dsu, self.zsl,
                                                                self.zsu, self.sigma_s)), st))

    _STATE_FIELDS = ("w_vals", "a_vals", "dxl", "dxu", "dsl", "dsu", "zxl", "zxu", "zsl", "zsu",
                     "sigma_x", "sigma_s")

    def __setattr__(self, name, value):
        object.__setattr__(self, name, value)
        if name in KKTWorkspace._STATE_FIELDS:
            object.__setattr__(self, "_state", None)

    def state(self) -> L.KktState:
        """The C struct of device pointers + (delta_w, delta_c); rebuilt only
        when a buffer is rebound or a regularisation changes."""
        key = (float(self.delta_w), float(self.delta_c))
        st = getattr(self, "_state", None)
        if st is None or getattr(self, "_state_key", None) != key:
            st = L.KktState(*(getattr(self, f).data_ptr() for f in KKTWorkspace._STATE_FIELDS), *key)
            object.__setattr__(self, "_state", st)
            object.__setattr__(self, "_state_key", key)
        return st

    # -- matrix-vector products ----------------------------------------------
    def _mv(self, kind, vals, v, n_out):
        out = D.empty(n_out)
        v = D.to_dev(v)
        L.check(L.lib().gn_kkt_matvec(self.handle, kind, L.ptr(vals), L.ptr(v), L.ptr(out),
                                      D.stream_ptr()))
        return out

    def w_matvec(self, v):
        return self._mv(0, self.w_vals, v, self.n)

    def a_matvec(self, v):
        return self._mv(1, self.a_vals, v, self.m)

    def at_matvec(self, u):
        return self._mv(2, self.a_vals, u, self.n)

    # -- condensation formulas (convenience; the solver uses fused kernels) ---
    def c_diag(self):
        return 1.0 / (self.delta_c * self.sigma_s + (1.0 + self.delta_c * self.delta_w))

    def d_diag(self):
        return (self.sigma_s + self.delta_w) * self.c_diag()

    def condense_pvec(self, pv: PVec):
        qx, qs, qy, _ = self._condense(pv)
        return qx, qs, qy

    def _buf(self, key, n):
        """A persistent device buffer per (role, slot): the solver's hot path
        allocates nothing per call.  The IPM's Newton step ("main") and a
        refinement correction ("corr") use different slots, so a correction
        never overwrites the step it refines."""
        bufs = self.__dict__.setdefault("_bufs", {})
        t = bufs.get(key)
        if t is None or t.numel() != n:
            t = D.empty(n)
            bufs[key] = t
        return t

    def _condense(self, pv, slot=None):
        if slot is None:
            qx, rhs = D.empty(self.n), D.empty(self.n)
            qs, qy = D.empty(self.m), D.empty(self.m)
        else:
            qx, rhs = self._buf(("qx", slot), self.n), self._buf(("rhs", slot), self.n)
            qs, qy = self._buf(("qs", slot), self.m), self._buf(("qy", slot), self.m)
        st, pc = self.state(), pv.c_struct()
        L.check(L.lib().gn_kkt_condense_rhs(self.handle, ctypes.byref(st), ctypes.byref(pc),
                                            L.ptr(qx), L.ptr(qs), L.ptr(qy), L.ptr(rhs),
                                            D.stream_ptr()))
        return qx, qs, qy, rhs

    def condensed_rhs(self, qx, qs, qy):
        z_n, z_m = D.zeros(self.n), D.zeros(self.m)
        return self._condense(PVec(qx, qs, qy, z_n, z_n, z_m, z_m))[3]

    def recover_slack_dual(self, dx, qx, qs, qy, slot=None):
        if slot is None:
            ds, dy = D.empty(self.m), D.empty(self.m)
        else:
            ds, dy = self._buf(("ds", slot), self.m), self._buf(("dy", slot), self.m)
        st = self.state()
        L.check(L.lib().gn_kkt_recover_slack_dual(self.handle, ctypes.byref(st), L.ptr(D.to_dev(dx)),
                                                  L.ptr(D.to_dev(qs)), L.ptr(D.to_dev(qy)), L.ptr(ds),
                                                  L.ptr(dy), D.stream_ptr()))
        return ds, dy

    def recover_bound_duals(self, dx, ds, pv: PVec, check=True, slot=None):
        if slot is None:
            out = [D.empty(k) for k in (self.n, self.n, self.m, self.m)]
        else:
            out = [self._buf((f, slot), k) for f, k in zip(("zxl", "zxu", "zsl", "zsu"),
                                                          (self.n, self.n, self.m, self.m))]
        st, pc = self.state(), pv.c_struct()
        if check:
            self.flags.zero_()
        L.check(L.lib().gn_kkt_recover_bound_duals(
            self.handle, ctypes.byref(st), L.ptr(D.to_dev(dx)), L.ptr(D.to_dev(ds)), ctypes.byref(pc),
            *(L.ptr(t) for t in out), L.ptr(self.flags), D.stream_ptr()))
        if check and int(self.flags.item()) & 1:
            raise DegenerateInterior("non-positive bound slack at an interior iterate")
        return tuple(out)

    # -- full seven-block system ----------------------------------------------
    def residual_full(self, st_: Steps, pv: PVec, norm_out=None, reuse=False):
        """pv - M_full * steps, accumulated in double-double (kkt.py:190-209).
        reuse: into the workspace's persistent residual (the refinement loop,
        which consumes each residual before the next one is formed)."""
        if reuse:
            res = self.__dict__.get("_res")
            if res is None:
                res = PVec.empty(self.n, self.m)
                self.__dict__["_res"] = res
        else:
            res = PVec.empty(self.n, self.m)
        st, sc, pc, rc = self.state(), st_.c_struct(), pv.c_struct(), res.c_struct()
        norm = norm_out if norm_out is not None else self._scal[0:2]
        L.check(L.lib().gn_kkt_residual(self.handle, ctypes.byref(st), ctypes.byref(sc),
                                        ctypes.byref(pc), ctypes.byref(rc), L.ptr(norm),
                                        D.stream_ptr()))
        res._norm = norm
        return res

    def matrix_scale_device(self, out):
        st = self.state()
        L.check(L.lib().gn_kkt_matrix_scale(self.handle, ctypes.byref(st), L.ptr(out), D.stream_ptr()))
        return out

    def matrix_scale(self) -> float:
        return float(self.matrix_scale_device(self._scal[2:3]).item())


def residual_norm(pv) -> float:
    """max |block| over the seven blocks (kkt.py:224-229)."""
    nrm = getattr(pv, "_norm", None)
    if nrm is not None:
        return float(nrm[0].item())
    out = 0.0
    for t in pv.parts():
        if t.numel():
            out = max(out, float(t.abs().max().item()))
    return out


class CondensedBackend:
    """Sparse Cholesky of the condensed primal system on the GPU (kkt.py:286-325)."""

    def __init__(self, ws: KKTWorkspace, ordering=None, timings=None, structure=None,
                 symbolic=None):
        import time

        tm = timings if timings is not None else {}
        self.ws = ws
        if structure is None:
            t = time.perf_counter()
            structure = symbolic_condense(ws.hess_rows, ws.hess_cols, ws.jac_rows, ws.jac_cols,
                                          ws.n)
            tm["condense"] = time.perf_counter() - t
        self.structure = structure
        ws.attach_condensed(self.structure)
        if symbolic is None:
            t = time.perf_counter()
            if ordering is None:
                ordering = S.amd_order(self.structure.matrix)
            tm["ordering"] = time.perf_counter() - t
            t = time.perf_counter()
            symbolic = S.symbolic_cholesky(self.structure.matrix, ordering)
            tm["symbolic"] = time.perf_counter() - t
        self.symbolic = symbolic
        t = time.perf_counter()
        self.symbolic.handle()
        self.kvals = D.zeros(self.structure.matrix.nnz)
        self.structure.matrix.values = self.kvals
        self.fws = S.FactorWorkspace(self.symbolic)
        self.factor = None
        self.n_factorizations = 0
        self._dx = D.empty(ws.n)
        tm["factor_upload"] = time.perf_counter() - t

    def assemble(self) -> None:
        st = self.ws.state()
        with span("assemble"):
            L.check(L.lib().gn_kkt_assemble(self.ws.handle, ctypes.byref(st), L.ptr(self.kvals),
                                            D.stream_ptr()))

    def factorize_async(self):
        self.assemble()
        self.n_factorizations += 1
        with span("refactor"):
            self.factor = S.factorize_device(self.symbolic, self.kvals, self.fws)
        return self.factor

    def try_factorize(self) -> bool:
        return self.factorize_async().ok

    def solve3(self, qx, qs, qy):
        ws = self.ws
        rhs = ws.condensed_rhs(qx, qs, qy)
        dx = S.solve_device(self.factor, rhs, D.empty(ws.n))
        ds, dy = ws.recover_slack_dual(dx, qx, qs, qy)
        return dx, ds, dy

    def solve_pvec(self, pv: PVec, slot=None):
        """Fused condense_pvec + solve3 for the solver's hot path (outputs in
        the workspace's persistent buffers of `slot` when given)."""
        ws = self.ws
        with span("rhs"):
            qx, qs, qy, rhs = ws._condense(pv, slot)
        with span("solve"):
            dx = S.solve_device(self.factor, rhs, D.empty(ws.n) if slot is None else ws._buf(("dx", slot), ws.n))
        with span("recover"):
            ds, dy = ws.recover_slack_dual(dx, qx, qs, qy, slot)
        return dx, ds, dy

    def solve_condensed(self, cond, slot=None):
        """solve_pvec's solve and recovery for a right-hand side condensed
        beforehand (`cond` = ws._condense(pv, slot), e.g. on another stream)."""
        ws = self.ws
        qx, qs, qy, rhs = cond
        with span("solve"):
            dx = S.solve_device(self.factor, rhs, D.empty(ws.n) if slot is None else ws._buf(("dx", slot), ws.n))
        with span("recover"):
            ds, dy = ws.recover_slack_dual(dx, qx, qs, qy, slot)
        return dx, ds, dy


def solve_with_regularization(ws, backend, pv: PVec, reg: RegState, slot=None):
    """Factorize with the inertia-correction schedule, then solve (kkt.py:424-447)."""
    ws.delta_w = 0.0
    ws.delta_c = 0.0
    if not backend.try_factorize():
        had = reg.delta_w_last > 0.0
        ws.delta_c = DELTA_C_VALUE
        ws.delta_w = max(DELTA_W_MIN, reg.delta_w_last / 3.0) if had else DELTA_W_INIT
        while not backend.try_factorize():
            ws.delta_w *= 8.0 if had else 100.0
            if ws.delta_w > DELTA_W_MAX:
                raise RegularizationExhausted(
                    f"delta_w exceeded {DELTA_W_MAX:g} without positive definiteness")
        reg.delta_w_last = ws.delta_w
    if hasattr(backend, "solve_pvec"):
        dx, ds, dy = backend.solve_pvec(pv, slot)
    else:
        qx, qs, qy = ws.condense_pvec(pv)
        dx, ds, dy = backend.solve3(qx, qs, qy)
    return (dx, ds, dy), ws.delta_w


def assemble_steps(ws, pv: PVec, dx, ds, dy, check=True, slot=None) -> Steps:
    dz = ws.recover_bound_duals(dx, ds, pv, check=check, slot=slot)
    if slot is not None:   # the slot's Steps object: same buffers, pointer struct kept
        cache = ws.__dict__.setdefault("_steps", {})
        st = cache.get(slot)
        if st is not None and st.x is dx and st.s is ds and st.y is dy and st.zxl is dz[0]:
            return st
    st = Steps.__new__(Steps)
    st.x, st.s, st.y = D.to_dev(dx), D.to_dev(ds), D.to_dev(dy)
    st.zxl, st.zxu, st.zsl, st.zsu = dz
    if slot is not None:
        ws.__dict__["_steps"][slot] = st
    return st


@dataclass
class RefinementStats:
    rounds: int = 0
    initial_residual: float = 0.0
    final_residual: float = 0.0
    scale: float = 1.0

    @property
    def relative_residual(self) -> float:
        return self.final_residual / self.scale


def _read4(ws, scal):
    """scal[0:4] -> host through a pinned buffer (one stream sync)."""
    pin = getattr(ws, "_pin4", None)
    if pin is None:
        pin = torch.zeros(4, dtype=torch.float64, pin_memory=True)
        object.__setattr__(ws, "_pin4", pin)
    pin.copy_(scal[0:4], non_blocking=True)
    st = ws.__dict__.get("_stream")
    (st if st is not None else torch.cuda.current_stream()).synchronize()
    return pin.numpy()


class FactorizationFailed(RuntimeError):
    """Raised by iterative_refinement(check_factor=...) when the speculative
    factorisation behind ``steps`` was not positive definite."""


def iterative_refinement(ws, backend, steps: Steps, pv: PVec, check_factor=None,
                         scale_ready=False) -> RefinementStats:
    """Refine against the full seven-block system in place (kkt.py:467-491).

    The matrix scale and the first residual norm come back in one read;
    ``check_factor`` (the device failing-pivot word of a factorisation whose
    success was not checked yet) rides along in the same read.
    """
    scal = ws._scal
    if not scale_ready:   # (the caller may have queued it already, for the same delta_w / delta_c)
        ws.matrix_scale_device(scal[2:3])
    res = ws.residual_full(steps, pv, norm_out=scal[0:2], reuse=True)
    if check_factor is not None:
        scal[3:4].copy_(check_factor)
    host = _read4(ws, scal)
    if check_factor is not None and host[3] < ws.n:
        raise FactorizationFailed("condensed matrix not positive definite")
    scale, rnorm = float(host[2]), float(host[0])
    target = KAPPA_IR * np.finfo(float).eps * scale
    stats = RefinementStats(initial_residual=rnorm, final_residual=rnorm, scale=scale)
    while stats.final_residual > target and stats.rounds < MAX_IR_ROUNDS:
        dx, ds, dy = backend.solve_pvec(res, "corr")
        corr = assemble_steps(ws, res, dx, ds, dy, check=False, slot="corr")
        _bind(ws.handle, steps, corr, 1.0)
        res = ws.residual_full(steps, pv, norm_out=scal[0:2], reuse=True)
        new = float(_read4(ws, scal)[0])
        stats.rounds += 1
        if new >= stats.final_residual:
            _bind(ws.handle, steps, corr, -1.0)
            break
        enough = new <= stats.final_residual / 2.0
        stats.final_residual = new
        if not enough:
            break
    return stats
