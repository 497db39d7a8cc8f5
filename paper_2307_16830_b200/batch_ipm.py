"""Instance-batched interior-point solve.

B ACOPF instances that share one sparsity pattern -- the load-perturbed C5
batch -- are solved TOGETHER: one launch per kernel for all B instances
(the ``*_batched`` C-ABI entry points), every plan (AD records and gather
lists, KKT gathers, assembly products, symbolic factor) shared, and every
iterate stored instance-major in HBM ([B][n], [B][m], ...).  The host reads
ONE [B]-block of scalars per sync point -- the same sync points as the
single-instance driver (ipm.py) -- and runs each instance's control flow
(barrier update, inertia correction, refinement stop test, filter line
search, termination) on its own scalars.  Instances that finish are masked
out of every state-changing kernel.

The arithmetic of every instance is that of ``ipm.solve`` on that instance
alone (same kernels, same reduction shapes), so each instance's iterates
are bitwise those of a single solve (tested).  The reference has no batch
solver; its multi-instance path is ``run_suite(paths, parallel=P)``
(src/bench.py:166-186), a process pool of independent solves.
"""
from __future__ import annotations

import ctypes
import threading
import time

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .autodiff import C, F, GRAD, HESS, JAC, RESET, NonFiniteResult
from .ipm import (EVAL_ERROR, LINE_SEARCH_FAILURE, MAX_ITER, OPTIMAL, REGULARIZATION_EXHAUSTED,
                  SolveReport, SolverOptions, _Filter, _mu_candidates, kkt_residual_scalars, plans)
from .kkt import (DELTA_C_VALUE, DELTA_W_INIT, DELTA_W_MAX, DELTA_W_MIN, KAPPA_IR, MAX_IR_ROUNDS)

SC = 64          # GN_BATCH_SCAL: doubles per instance in a scalar block
BP = 8           # GN_BP_STRIDE
BP_MU, BP_TAU, BP_ALPHA, BP_ALPHA_Z, BP_DW, BP_DC, BP_ACTIVE, BP_OBJW = range(8)
# scal block layout per instance (same offsets as the single driver's mailbox)
S_F, S_FT, S_DIR, S_MERIT, S_NORM, S_SCALE = 48, 49, 50, 54, 60, 62


class _Inst:
    """Host control state of one instance."""

    def __init__(self, opts, mu_min):
        self.mu = opts.mu_init
        self.mu_min = mu_min
        self.filter = _Filter()
        self.it = 0
        self.status = None
        self.message = ""
        self.delta_w_last = 0.0
        self.residual = np.nan
        self.ir_rel = np.nan
        self.trace = []
        self.obj_scale = 1.0
        self.theta_min = self.theta_max = 0.0
        self.cands = [0.0, self.mu]

    @property
    def active(self):
        return self.status is None


def _check_same_plan(models):
    ref = models[0]
    for m in models[1:]:
        if (m.n_var, m.n_con) != (ref.n_var, ref.n_con):
            raise ValueError("instances differ in size")
        for f in ("jac_rows", "jac_cols", "hess_rows", "hess_cols"):
            if not np.array_equal(getattr(m, f), getattr(ref, f)):
                raise ValueError(f"instances differ in sparsity ({f})")
        for a, b in zip(m.pattern_blocks, ref.pattern_blocks):
            if not np.array_equal(a.var_idx, b.var_idx) or (
                    a.targets is not None and not np.array_equal(a.targets, b.targets)):
                raise ValueError("instances differ in record structure")


def _param_layout(model) -> np.ndarray:
    """Parameter values in the device plan's layout (per block, slot-major;
    ad.cu upload_model)."""
    parts = [np.ascontiguousarray(b.params, dtype=float).T.ravel() for b in model.pattern_blocks]
    return np.concatenate(parts) if parts else np.zeros(0)


def _param_layout_batch(models) -> np.ndarray:
    """[B, P] stack of _param_layout, one transposing copy per block for the
    whole batch (not one per instance)."""
    cols = []
    for j in range(len(models[0].pattern_blocks)):
        blk = np.stack([np.asarray(mdl.pattern_blocks[j].params, dtype=float) for mdl in models])   # [B, R, np]
        cols.append(blk.transpose(0, 2, 1).reshape(len(models), -1))
    return np.concatenate(cols, axis=1) if cols else np.zeros((len(models), 0))


_PINNED: dict = {}


def _pinned(shape, dtype, tag):
    """Page-locked host buffers cached across batched solves (cudaHostAlloc
    costs milliseconds per call)."""
    key = (tuple(shape), dtype, tag, threading.get_ident())   # per thread: concurrent batches never share
    t = _PINNED.get(key)
    if t is None:
        t = torch.zeros(*shape, dtype=dtype, pin_memory=True)
        _PINNED[key] = t
    return t


class _Batch:
    """Device buffers of a batch (instance-major)."""

    def __init__(self, models, opts, ranges, ws, backend):
        B = len(models)
        base = models[0]
        n, m = base.n_var, base.n_con
        self.B, self.n, self.m = B, n, m
        self.nj, self.nh = base.nnz_jac, base.nnz_hess
        self.ws, self.backend = ws, backend
        dev = D.require_cuda()
        f64 = dict(dtype=torch.float64, device=dev)
        z = lambda *sh: torch.zeros(*sh, **f64)
        mm = max(1, m)
        # prepared inputs (ipm.py _prepared_inputs), per instance
        xl = np.stack([b.lower for b in models])
        xu = np.stack([b.upper for b in models])
        fixed = xl == xu
        if np.any(fixed):
            eps = opts.fixed_var_eps * np.maximum(1.0, np.abs(xl))
            xl, xu = np.where(fixed, xl - eps, xl), np.where(fixed, xu + eps, xu)
        x0 = np.minimum(np.maximum(np.stack([b.start for b in models]), xl), xu)
        if ranges is None:
            rlo, rhi = np.zeros((B, m)), np.zeros((B, m))
        else:
            rr = np.stack([np.asarray(r, dtype=float).reshape(m, 2) for r in ranges])
            rlo, rhi = rr[:, :, 0].copy(), rr[:, :, 1].copy()
        self.n_bounds = (np.isfinite(xl).sum(1) + np.isfinite(xu).sum(1) + np.isfinite(rlo).sum(1)
                         + np.isfinite(rhi).sum(1)).astype(int)
        self.xl, self.xu = D.to_dev(xl), D.to_dev(xu)
        self.rlo, self.rhi = D.to_dev(rlo), D.to_dev(rhi)
        self.x0 = D.to_dev(x0)
        self.x = self.x0.clone()
        self.s, self.y = z(B, mm), z(B, mm)
        self.zxl, self.zxu = torch.isfinite(self.xl).double(), torch.isfinite(self.xu).double()
        self.sl, self.su = z(B, mm), z(B, mm)
        self.zsl, self.zsu = z(B, mm), z(B, mm)
        self.dxl, self.dxu, self.sx = z(B, n), z(B, n), z(B, n)
        self.dsl, self.dsu, self.ss = z(B, mm), z(B, mm), z(B, mm)
        self.grad, self.c = z(B, n), z(B, mm)
        self.a_vals, self.w_vals = z(B, max(1, self.nj)), z(B, max(1, self.nh))
        self.dual_x, self.dual_s, self.primal = z(B, n), z(B, mm), z(B, mm)
        self.xt, self.st, self.ct = z(B, n), z(B, mm), z(B, mm)
        self.con_scale = torch.ones(B, mm, **f64)
        self.objs = torch.ones(B, **f64)
        # AD plan inputs
        self.params = D.to_dev(_param_layout_batch(models)) if any(b.pattern_blocks for b in models) else None
        self.contrib = z(B, max(1, base.n_contrib))
        self.ad_flags = torch.zeros(B, dtype=torch.int32, device=dev)
        self.ipm_flags = torch.zeros(B, dtype=torch.int32, device=dev)
        self.bd_flags = torch.zeros(B, dtype=torch.int32, device=dev)
        # KKT / factor
        info = backend.symbolic.info
        self.kvals = z(B, max(1, backend.structure.matrix.nnz))
        self.fronts = z(B, max(1, info["front_doubles"]))
        self.fvec = z(B, max(1, info["vec_doubles"]))
        self.fail = torch.zeros(B, dtype=torch.int64, device=dev)
        vec7 = lambda: [z(B, k) for k in (n, mm, mm, n, n, mm, mm)]
        self.pv, self.steps, self.corr, self.res = vec7(), vec7(), vec7(), vec7()
        self.qx, self.rhs, self.dx = z(B, n), z(B, n), z(B, n)
        self.qs, self.qy = z(B, mm), z(B, mm)
        # scalar blocks
        self.scal = z(B, SC)
        self.host = _pinned((B, SC), torch.float64, "host")
        self.host_i = _pinned((4, B), torch.int64, "host_i")
        # per-instance operands: edited on the host (bp_h, numpy), uploaded
        # through a ring of pinned staging slots -- an asynchronous copy reads
        # its slot when the stream reaches it, so a slot is reused only after
        # a stream synchronisation (every read is one)
        self.bp_h = np.zeros((B, BP))
        self.bp = z(B, BP)
        self.mus = z(B, L.IPM_MAX_MU)
        self._ring = [(_pinned((B, BP), torch.float64, ("bp", k)),
                       _pinned((B, L.IPM_MAX_MU), torch.float64, ("mu", k))) for k in range(8)]
        self._ring_next = 0
        self._ring_used = 0
        self.stream = torch.cuda.current_stream()
        self.words = torch.zeros(4, B, dtype=torch.int64, device=dev)
        # C structs (base pointers; the kernels offset by instance)
        p = lambda t: t.data_ptr()
        self.V = L.IpmVecs(*(p(t) for t in (
            self.x, self.s, self.y, self.zxl, self.zxu, self.zsl, self.zsu, self.xl, self.xu,
            self.sl, self.su, self.dxl, self.dxu, self.dsl, self.dsu, self.sx, self.ss, self.grad,
            self.c, self.a_vals, self.dual_x, self.dual_s, self.primal)))
        self.KS = L.KktState(*(p(t) for t in (self.w_vals, self.a_vals, self.dxl, self.dxu,
                                               self.dsl, self.dsu, self.zxl, self.zxu, self.zsl,
                                               self.zsu, self.sx, self.ss)), 0.0, 0.0)
        v7 = lambda ts: L.Vec7(*(p(t) for t in ts))
        self.PV, self.ST, self.CR, self.RS = v7(self.pv), v7(self.steps), v7(self.corr), v7(self.res)
        self.DIRV = v7([self.dx] + self.corr[1:])   # solve output: dx + (ds, dy) into corr

    def reset(self):
        """Back to the start point for another solve of the same (resident)
        batch: the iterate buffers the setup does not rewrite."""
        self.x.copy_(self.x0)
        self.s.zero_()
        self.y.zero_()
        self.zxl.copy_(torch.isfinite(self.xl).double())
        self.zxu.copy_(torch.isfinite(self.xu).double())
        self.con_scale.fill_(1.0)
        self.objs.fill_(1.0)
        for t in (self.ad_flags, self.ipm_flags, self.bd_flags):
            t.zero_()
        self.bp_h[...] = 0.0

    # -- scalar plumbing ---------------------------------------------------
    def _slot(self):
        if self._ring_used == len(self._ring):   # every slot may still be pending
            self.stream.synchronize()
            self._ring_used = 0
        slot = self._ring[self._ring_next]
        self._ring_next = (self._ring_next + 1) % len(self._ring)
        self._ring_used += 1
        return slot

    def push_bp(self):
        slot = self._slot()[0]
        slot.numpy()[...] = self.bp_h
        self.bp.copy_(slot, non_blocking=True)
        D.TRANSFER["h2d"] += self.B * BP * 8

    def push_mus(self, mus):
        slot = self._slot()[1]
        slot.numpy()[...] = mus
        self.mus.copy_(slot, non_blocking=True)
        D.TRANSFER["h2d"] += self.B * L.IPM_MAX_MU * 8

    def read(self, lo, hi, words=()):
        """scal[:, lo:hi] (+ the named int words) -> host, one stream sync."""
        self.host[:, lo:hi].copy_(self.scal[:, lo:hi], non_blocking=True)
        D.TRANSFER["d2h"] += self.B * (hi - lo) * 8
        for k, w in enumerate(words):
            self.words[k].copy_(w)
        if words:
            self.host_i[:len(words)].copy_(self.words[:len(words)], non_blocking=True)
            D.TRANSFER["d2h"] += len(words) * self.B * 8
        self.stream.synchronize()
        self._ring_used = 0
        return self.host[:, lo:hi].numpy(), self.host_i[:len(words)].numpy()


def release_batch(instances) -> None:
    """Drop the resident device buffers of a batch (see solve_batched)."""
    for am in instances[:1]:
        mdl = am.model if hasattr(am, "model") else am[0]
        mdl.__dict__.pop("_batch_cache", None)


def solve_batched(instances, options: SolverOptions | None = None, ordering=None) -> list[SolveReport]:
    """Solve AcopfModels (or (model, ranges) pairs) sharing one sparsity
    pattern as ONE batch on the current GPU; returns one SolveReport per
    instance (the same reports ``ipm.solve`` gives, without timings)."""
    opts = options if options is not None else SolverOptions()
    pairs = [(am.model, am.ranges) if hasattr(am, "model") else am for am in instances]
    models = [p[0] for p in pairs]
    ranges = [p[1] for p in pairs]
    if not models:
        return []
    t_start = time.perf_counter()
    base = models[0]
    ws, backend = plans(base, ordering)
    # The batch's device buffers and uploaded instance data stay resident on
    # the first model between solves of the SAME instances (the same model
    # and ranges objects, the same bound / start arrays, the same fixed-
    # variable widening); any change rebuilds them (release_batch drops them).
    key = (tuple(id(x) for x in models), tuple(id(r) for r in ranges),
           tuple(id(a) for mdl in models for a in (mdl.lower, mdl.upper, mdl.start)), opts.fixed_var_eps,
           ordering is None)
    cached = base.__dict__.get("_batch_cache")
    if (cached is not None and cached[0] == key and all(a is b for a, b in zip(cached[1], models))
            and all(a is b for a, b in zip(cached[2], ranges)) and cached[3].backend is backend):
        Bt = cached[3]
        Bt.reset()
    else:
        _check_same_plan(models)
        Bt = _Batch(models, opts, None if all(r is None for r in ranges) else
                    [np.zeros((base.n_con, 2)) if r is None else r for r in ranges], ws, backend)
        base.__dict__["_batch_cache"] = (key, list(models), list(ranges), Bt)
    B, n, m = Bt.B, Bt.n, Bt.m
    lib = L.lib()
    stream = D.stream_ptr()
    mu_min = opts.mu_min if opts.mu_min is not None else opts.tol / 10.0
    tol_r = opts.bound_relax if opts.bound_relax is not None else opts.tol
    insts = [_Inst(opts, mu_min) for _ in range(B)]
    M = base.device_plan()
    KH, SH = ws.handle, backend.symbolic.handle()
    ptr = L.ptr
    bp = ptr(Bt.bp)

    def ad(x, what, *, y=None, objw=None, cs=None, objs=None, f=None, c=None, grad=None, jac=None,
           hess=None):
        L.check(lib.gn_ad_eval_batched(M, B, ptr(x), ptr(y), ptr(objw), ptr(cs), ptr(objs),
                                       ptr(Bt.params), ptr(f), SC, ptr(c), ptr(grad), ptr(jac),
                                       ptr(hess), what, ptr(Bt.contrib), ptr(Bt.ad_flags), stream))

    def set_active():
        Bt.bp_h[:, BP_ACTIVE] = [1.0 if it.status is None else 0.0 for it in insts]

    # ---- setup: frozen scaling at x0 (ipm.py:179-203), relaxed slack bounds,
    # initial slacks (ipm.py:371-380); one read
    Bt.ad_flags.zero_()
    ad(Bt.x, GRAD | JAC, grad=Bt.grad, jac=Bt.a_vals)
    flags0 = Bt.ad_flags.clone()
    if opts.scaling:
        gm = Bt.grad.abs().amax(dim=1) if n else torch.zeros(B, dtype=torch.float64, device=Bt.x.device)
        Bt.objs = torch.where(gm > 0, torch.clamp(100.0 / gm, max=1.0), torch.ones_like(gm))
        if m and base.nnz_jac:
            rmax = torch.zeros(B, m, dtype=torch.float64, device=Bt.x.device)
            idx = base.jac_rows_device().unsqueeze(0).expand(B, -1)
            rmax.scatter_reduce_(1, idx, Bt.a_vals[:, :base.nnz_jac].abs(), "amax")
            Bt.con_scale[:, :m] = torch.where(rmax > 0, torch.clamp(100.0 / rmax, max=1.0),
                                              torch.ones_like(rmax))
    if m:
        lo, hi = Bt.rlo * Bt.con_scale[:, :m], Bt.rhi * Bt.con_scale[:, :m]
        one = torch.ones_like(lo)
        inf = torch.full_like(lo, np.inf)
        Bt.sl[:, :m] = torch.where(torch.isfinite(lo), lo - tol_r * torch.maximum(one, lo.abs()), -inf)
        Bt.su[:, :m] = torch.where(torch.isfinite(hi), hi + tol_r * torch.maximum(one, hi.abs()), inf)
        Bt.zsl[:, :m] = torch.isfinite(Bt.sl[:, :m]).double()
        Bt.zsu[:, :m] = torch.isfinite(Bt.su[:, :m]).double()
    Bt.ad_flags.zero_()
    ad(Bt.x, C, cs=Bt.con_scale, c=Bt.c)
    if m:
        g0 = Bt.c[:, :m]
        push = opts.bound_push
        inf = torch.full_like(g0, np.inf)
        lo = torch.where(torch.isfinite(Bt.sl[:, :m]), Bt.sl[:, :m] + push * tol_r, -inf)
        hi = torch.where(torch.isfinite(Bt.su[:, :m]), Bt.su[:, :m] - push * tol_r, inf)
        s0 = torch.minimum(torch.maximum(g0, lo), hi)
        s0 = torch.where(lo > hi, 0.5 * (Bt.sl[:, :m] + Bt.su[:, :m]), s0)
        Bt.s[:, :m] = s0
        Bt.scal[:, 60] = (g0 - s0).abs().sum(dim=1)
    Bt.scal[:, 61] = Bt.objs
    sc0, w0 = Bt.read(60, 62, (Bt.ad_flags, flags0))
    for b, it in enumerate(insts):
        if w0[1][b]:
            it.status, it.message = EVAL_ERROR, "scaling evaluation produced a non-finite value"
            it.no_x = True
        elif w0[0][b]:
            it.status, it.message = EVAL_ERROR, "constraint evaluation produced a non-finite value"
        it.obj_scale = float(sc0[b, 1])
        theta0 = float(sc0[b, 0]) if m else 0.0
        it.theta_min, it.theta_max = 1e-4 * max(1.0, theta0), 1e4 * max(1.0, theta0)
        Bt.bp_h[b, BP_OBJW] = it.obj_scale
    Bt.push_bp()
    objw = Bt.bp[:, BP_OBJW].contiguous()

    def solve_pvec(pv_struct, pv_tensors):
        """condensed rhs + batched solve + slack/dual recovery -> (dx, corr.s, corr.y)."""
        L.check(lib.gn_kkt_condense_rhs_batched(KH, B, ctypes.byref(Bt.KS), bp, ctypes.byref(pv_struct),
                                                ptr(Bt.qx), ptr(Bt.qs), ptr(Bt.qy), ptr(Bt.rhs), stream))
        L.check(lib.gn_chol_solve_batched(SH, B, ptr(Bt.fronts), ptr(Bt.rhs), ptr(Bt.dx), ptr(Bt.fvec),
                                          stream))
        L.check(lib.gn_kkt_recover_slack_dual_batched(KH, B, ctypes.byref(Bt.KS), bp, ptr(Bt.dx),
                                                      ptr(Bt.qs), ptr(Bt.qy), ptr(Bt.corr[1]),
                                                      ptr(Bt.corr[2]), stream))

    def steps_from(pv_struct, out_tensors):
        """assemble_steps: bound-dual recovery of (dx, ds, dy) into out_tensors."""
        out_tensors[0].copy_(Bt.dx)
        if out_tensors is not Bt.corr:
            out_tensors[1].copy_(Bt.corr[1])
            out_tensors[2].copy_(Bt.corr[2])
        L.check(lib.gn_kkt_recover_bound_duals_batched(
            KH, B, ctypes.byref(Bt.KS), ptr(out_tensors[0]), ptr(out_tensors[1]), ctypes.byref(pv_struct),
            *(ptr(t) for t in out_tensors[3:]), ptr(Bt.bd_flags), stream))

    def refactor():
        L.check(lib.gn_kkt_assemble_batched(KH, B, ctypes.byref(Bt.KS), bp, ptr(Bt.kvals), stream))
        L.check(lib.gn_chol_factor_batched(SH, B, ptr(Bt.kvals), ptr(Bt.fronts), ptr(Bt.fail), stream))

    def residual_norms():
        L.check(lib.gn_kkt_residual_batched(KH, B, ctypes.byref(Bt.KS), bp, ctypes.byref(Bt.ST),
                                            ctypes.byref(Bt.PV), ctypes.byref(Bt.RS),
                                            ptr(Bt.scal[:, S_NORM]), stream))

    def newton_and_refine(check_fail):
        """pv -> steps with iterative refinement (kkt.py:467-491), every active
        instance on its own stop test.  Returns the per-instance failed
        speculative-factorisation mask when check_fail (nothing refined)."""
        solve_pvec(Bt.PV, Bt.pv)
        steps_from(Bt.PV, Bt.steps)
        L.check(lib.gn_kkt_matrix_scale_batched(KH, B, ctypes.byref(Bt.KS), bp,
                                                ptr(Bt.scal[:, S_SCALE]), stream))
        residual_norms()
        h, w = Bt.read(S_NORM, S_SCALE + 1, (Bt.fail,))
        if check_fail:
            failed = np.array([it.active and w[0][b] < n for b, it in enumerate(insts)])
            if failed.any():
                return failed
        final = h[:, 0].copy()
        scale = h[:, 2].copy()
        target = KAPPA_IR * np.finfo(float).eps * scale
        running = np.array([it.active for it in insts]) & (final > target)
        rounds = np.zeros(B, dtype=int)
        while running.any():
            solve_pvec(Bt.RS, Bt.res)
            steps_from(Bt.RS, Bt.corr)
            Bt.bp_h[:, BP_ALPHA] = np.where(running, 1.0, 0.0)
            Bt.push_bp()
            L.check(lib.gn_vec7_axpy_batched(KH, B, ctypes.byref(Bt.ST), ctypes.byref(Bt.CR), bp, stream))
            residual_norms()
            h, _ = Bt.read(S_NORM, S_NORM + 1)
            new = h[:, 0]
            rounds += running
            back = running & (new >= final)
            if back.any():
                Bt.bp_h[:, BP_ALPHA] = np.where(back, -1.0, 0.0)
                Bt.push_bp()
                L.check(lib.gn_vec7_axpy_batched(KH, B, ctypes.byref(Bt.ST), ctypes.byref(Bt.CR), bp,
                                                 stream))
            ok = running & ~back
            enough = new <= final / 2.0
            final = np.where(ok, new, final)
            running = ok & enough & (final > target) & (rounds < MAX_IR_ROUNDS)
        for b, it in enumerate(insts):
            if it.active:
                it.ir_rel = final[b] / scale[b]
        return None

    def regularize(failed):
        """The delta_w schedule of kkt.py:424-447 for the failed instances
        (the others keep their delta = 0 factor: refactoring them with the
        same values reproduces it bitwise)."""
        had = {b: insts[b].delta_w_last > 0.0 for b in np.flatnonzero(failed)}
        for b in had:
            Bt.bp_h[b, BP_DC] = DELTA_C_VALUE
            Bt.bp_h[b, BP_DW] = max(DELTA_W_MIN, insts[b].delta_w_last / 3.0) if had[b] else DELTA_W_INIT
        pending = set(had)
        while pending:
            Bt.push_bp()
            refactor()
            _, w = Bt.read(0, 0, (Bt.fail,))
            for b in list(pending):
                if w[0][b] >= n:
                    pending.discard(b)
                    insts[b].delta_w_last = float(Bt.bp_h[b, BP_DW])
                else:
                    Bt.bp_h[b, BP_DW] *= 8.0 if had[b] else 100.0
                    if Bt.bp_h[b, BP_DW] > DELTA_W_MAX:
                        pending.discard(b)
                        insts[b].status = REGULARIZATION_EXHAUSTED
                        insts[b].message = f"delta_w exceeded {DELTA_W_MAX:g} without positive definiteness"
                        Bt.bp_h[b, BP_DW] = Bt.bp_h[b, BP_DC] = 0.0
        Bt.push_bp()

    # ---- main loop.  The per-instance control flow of ipm.solve, vectorised
    # over the batch with numpy (the host work per iteration was a Python
    # loop over B instances: ~7 ms of GPU idle per iteration at B = 256).
    # Elementwise float64 numpy arithmetic rounds exactly like the scalar
    # Python expressions it replaces; Python's max(a, b) / min(a, b) are
    # written as where(b > a, b, a) / where(b < a, b, a) (same NaN behaviour)
    # and the powers stay scalar Python ** (libm pow), so every instance's
    # decisions and pushed operands are bitwise those of a single solve.
    S0 = L.PREP_S
    KMU = L.IPM_MAX_MU
    mu = np.full(B, float(opts.mu_init))
    nbd = np.asarray(Bt.n_bounds, dtype=float)
    th_min = np.array([it.theta_min for it in insts])
    th_max = np.array([it.theta_max for it in insts])
    fcap = 64
    filt = np.zeros((B, fcap, 2))
    fcnt = np.zeros(B, dtype=np.int64)
    mu_floor = mu_min * (1 + 1e-12)

    def pmax(a, b):   # Python max(a, b), elementwise
        return np.where(b > a, b, a)

    def pmin(a, b):
        return np.where(b < a, b, a)

    def powv(a, e):   # scalar libm pow per element
        return np.array([float(v) ** e for v in a], dtype=float)

    def mu_next(cur):
        return pmax(np.full_like(cur, mu_min), pmin(opts.kappa_mu * cur, powv(cur, opts.theta_mu)))

    def residual(s, comp_k, nb):
        """kkt_residual_scalars over rows of scalar blocks s."""
        dual_max = pmax(s[:, 0], s[:, S0])
        primal_max = s[:, S0 + 1]
        z_l1 = s[:, 1] + s[:, S0 + 2]
        y_l1 = s[:, S0 + 3]
        comp_max = pmax(s[:, 4 + comp_k] if n else np.zeros(len(s)), s[:, S0 + 7 + comp_k] if m else np.zeros(len(s)))
        s_max = opts.s_max
        s_d = pmax(np.full(len(s), s_max), (y_l1 + z_l1) / np.maximum(1.0, m + nb)) / s_max
        s_c = pmax(np.full(len(s), s_max), z_l1 / np.maximum(1.0, nb)) / s_max
        comp = np.where(nb > 0, comp_max / s_c, 0.0)
        return pmax(pmax(dual_max / s_d, primal_max), comp), dual_max, primal_max

    def filter_acceptable(rows, theta, phi):
        if fcnt[rows].max(initial=0) == 0:
            return np.ones(len(rows), dtype=bool)
        F_ = filt[rows]
        valid = np.arange(fcap)[None, :] < fcnt[rows][:, None]
        ok = (theta[:, None] < F_[:, :, 0]) | (phi[:, None] < F_[:, :, 1]) | ~valid
        return ok.all(axis=1)

    def filter_add(rows, theta, phi):
        nonlocal filt, fcap
        if len(rows) == 0:
            return
        if fcnt[rows].max() + 1 > fcap:
            filt = np.concatenate([filt, np.zeros((B, fcap, 2))], axis=1)
            fcap *= 2
        F_ = filt[rows]
        valid = np.arange(fcap)[None, :] < fcnt[rows][:, None]
        keep = valid & ~((F_[:, :, 0] >= theta[:, None]) & (F_[:, :, 1] >= phi[:, None]))
        order = np.argsort(~keep, axis=1, kind="stable")
        F_ = np.take_along_axis(F_, order[:, :, None], axis=1)
        cnt = keep.sum(axis=1)
        F_[np.arange(len(rows)), cnt, 0] = theta
        F_[np.arange(len(rows)), cnt, 1] = phi
        filt[rows] = F_
        fcnt[rows] = cnt + 1

    def active_mask():
        return np.array([it.status is None for it in insts])

    for _ in range(opts.max_iter):
        amask = active_mask()
        if not amask.any():
            break
        act = np.flatnonzero(amask)
        # derivatives at x and the residual blocks (ipm.py:384-429)
        ad(Bt.x, F | C | GRAD | JAC | HESS | RESET, y=Bt.y, objw=objw, cs=Bt.con_scale, objs=objw,
           f=Bt.scal[:, S_F], c=Bt.c, grad=Bt.grad, jac=Bt.a_vals, hess=Bt.w_vals)
        # barrier candidates [0, mu, update(mu), ...] (_mu_candidates)
        cands = np.zeros((B, KMU))
        cands[:, 1] = mu
        ncand = np.full(B, 2, dtype=np.int64)
        cur = mu.copy()
        grow = amask.copy()
        for k in range(2, KMU):
            grow &= cur > mu_floor
            if not grow.any():
                break
            rows = np.flatnonzero(grow)
            cur[rows] = mu_next(cur[rows])
            cands[rows, k] = cur[rows]
            ncand[rows] = k + 1
        nmu = int(ncand.max())
        mus = cands.copy()
        for k in range(2, KMU):
            pad = k >= ncand
            mus[pad, k] = cands[pad, np.maximum(ncand[pad] - 1, 0)] if k < nmu else 0.0
        mus[:, nmu:] = 0.0
        Bt.push_mus(mus)
        L.check(lib.gn_ipm_prep_batched(KH, B, ctypes.byref(Bt.V), nmu, ptr(Bt.mus), ptr(Bt.scal), stream))
        # speculative delta = 0 factorisation (kkt.py:424-447, first try)
        Bt.bp_h[act, BP_DW] = 0.0
        Bt.bp_h[act, BP_DC] = 0.0
        set_active()
        Bt.push_bp()
        refactor()
        sc, w = Bt.read(0, 49, (Bt.ad_flags, Bt.ipm_flags))
        for b in act[(w[1][act] != 0) | (w[0][act] != 0)]:   # rare: flagged instances
            it = insts[b]
            if w[1][b]:
                it.status, it.message = EVAL_ERROR, "lost strict interiority"
                continue
            it.status = EVAL_ERROR
            for bit, name in ((F, "objective"), (C, "constraint"), (GRAD, "gradient"),
                              (JAC, "jacobian"), (HESS, "hessian")):
                if w[0][b] & bit:
                    it.message = f"{name} evaluation produced a non-finite value"
                    break
        act = act[(w[1][act] == 0) & (w[0][act] == 0)]
        s_act = sc[act]
        e_0, dual_max, primal_max = residual(s_act, 0, nbd[act])
        fval = s_act[:, S_F].copy()
        done = e_0 < opts.tol
        for j in np.flatnonzero(done):
            insts[act[j]].residual = float(e_0[j])
            insts[act[j]].status = OPTIMAL
        keep = ~done
        act, s_act, e_0, dual_max, primal_max, fval = (a[keep] for a in (act, s_act, e_0, dual_max, primal_max, fval))
        # barrier update (ipm.py:423-428) along the candidates
        mu_a = mu[act].copy()
        e_mu = residual(s_act, 1, nbd[act])[0]
        looping = np.ones(len(act), dtype=bool)
        extra = np.zeros(len(act), dtype=bool)
        kk = np.ones(len(act), dtype=np.int64)
        while looping.any():
            cond = looping & (e_mu <= opts.kappa_eps * mu_a) & (mu_a > mu_floor)
            looping &= cond
            if not cond.any():
                break
            rows = np.flatnonzero(cond)
            mu_a[rows] = mu_next(mu_a[rows])
            fcnt[act[rows]] = 0   # filter.clear()
            kk[rows] += 1
            hit = (kk[rows] < ncand[act[rows]]) & (cands[act[rows], np.minimum(kk[rows], KMU - 1)] == mu_a[rows])
            for kval in np.unique(kk[rows[hit]]):
                r2 = rows[hit][kk[rows[hit]] == kval]
                e_mu[r2] = residual(s_act[r2], int(kval), nbd[act[r2]])[0]
            miss = rows[~hit]
            extra[miss] = True
            looping[miss] = False
        mu[act] = mu_a
        # rare: instances past their candidate list get more reduction passes
        while extra.any():
            mus = np.zeros((B, KMU))
            mus[:, 1] = mu
            Bt.push_mus(mus)
            L.check(lib.gn_ipm_prep_batched(KH, B, ctypes.byref(Bt.V), 2, ptr(Bt.mus), ptr(Bt.scal), stream))
            sc2, _ = Bt.read(0, 48)
            for j in np.flatnonzero(extra):
                b = act[j]
                s = sc2[b]
                comp = max(s[4 + 1] if n else 0.0, s[S0 + 7 + 1] if m else 0.0)
                e_mu_b = kkt_residual_scalars(max(s[0], s[S0]), s[S0 + 1], comp, s[1] + s[S0 + 2],
                                              s[S0 + 3], m, int(Bt.n_bounds[b]), opts.s_max)
                extra[j] = False
                mub = mu[b]
                while e_mu_b <= opts.kappa_eps * mub and mub > mu_min * (1 + 1e-12):
                    mub = max(mu_min, min(opts.kappa_mu * mub, mub ** opts.theta_mu))
                    fcnt[b] = 0
                    extra[j] = True
                    break
                mu[b] = mub
        if len(act) == 0:
            continue
        mu_a = mu[act]
        theta_cur = s_act[:, S0 + 4] if m else np.zeros(len(act))
        phi_cur = fval - mu_a * s_act[:, 2] - mu_a * s_act[:, 3] - mu_a * s_act[:, S0 + 5] - mu_a * s_act[:, S0 + 6]
        Bt.bp_h[act, BP_MU] = mu_a
        Bt.bp_h[act, BP_TAU] = pmax(np.full(len(act), opts.tau_min), 1.0 - mu_a)
        set_active()
        Bt.push_bp()
        # ---- Newton step with refinement (ipm.py:434-453)
        L.check(lib.gn_ipm_pvec_batched(KH, B, ctypes.byref(Bt.V), bp, ctypes.byref(Bt.PV), stream))
        delta_w = np.zeros(B)
        failed = newton_and_refine(check_fail=True)
        if failed is not None:
            regularize(failed)
            fb = np.flatnonzero(failed)
            delta_w[fb] = Bt.bp_h[fb, BP_DW]
            set_active()
            Bt.push_bp()
            newton_and_refine(check_fail=False)
        still = np.array([insts[b].status is None for b in act], dtype=bool)
        act, theta_cur, phi_cur, e_0, dual_max, primal_max, fval = (
            a[still] for a in (act, theta_cur, phi_cur, e_0, dual_max, primal_max, fval))
        if len(act) == 0:
            continue
        mu_a = mu[act]
        # ---- fraction to the boundary, dphi, first trial at alpha_max
        L.check(lib.gn_ipm_direction_batched(KH, B, ctypes.byref(Bt.V), ctypes.byref(Bt.ST), bp,
                                             ptr(Bt.scal[:, S_DIR]), stream))
        L.check(lib.gn_ipm_trial_point_at_batched(KH, B, ctypes.byref(Bt.V), ctypes.byref(Bt.ST),
                                                  ptr(Bt.scal[:, S_DIR]), ptr(Bt.xt), ptr(Bt.st), stream))
        na = len(act)
        searching = np.ones(na, dtype=bool)
        verdict = np.zeros(na, dtype=np.int8)   # 0 none, 1 h-type, 2 f-type
        alpha = np.zeros(na)
        alpha_z = np.zeros(na)
        dphi = np.zeros(na)
        # the switching condition's right side, per instance (libm pow)
        rhs_switch = opts.delta * powv(theta_cur, opts.s_theta)
        first = True
        while searching.any():
            if not first:
                Bt.bp_h[:, BP_ALPHA] = 0.0
                Bt.bp_h[act[searching], BP_ALPHA] = alpha[searching]
                Bt.push_bp()
                L.check(lib.gn_ipm_trial_point_batched(KH, B, ctypes.byref(Bt.V), ctypes.byref(Bt.ST), bp,
                                                       ptr(Bt.xt), ptr(Bt.st), stream))
            ad(Bt.xt, F | C | RESET, cs=Bt.con_scale, objs=objw, f=Bt.scal[:, S_FT], c=Bt.ct)
            L.check(lib.gn_ipm_trial_merit_batched(KH, B, ctypes.byref(Bt.V), ptr(Bt.ct), ptr(Bt.xt),
                                                   ptr(Bt.st), ptr(Bt.scal[:, S_MERIT]), stream))
            tv, w = Bt.read(S_FT, S_MERIT + 5, (Bt.ad_flags,))
            t = tv[act]
            if first:
                alpha = pmin(t[:, 1], t[:, 2])
                alpha_z, dphi = t[:, 3].copy(), t[:, 4].copy()
                searching &= ~(alpha < opts.alpha_min)
            rows = np.flatnonzero(searching)
            bad = w[0][act[rows]] != 0
            theta_t = t[rows, 5] if m else np.zeros(len(rows))
            phi_t = (t[rows, 0] - mu_a[rows] * t[rows, 6] - mu_a[rows] * t[rows, 7] - mu_a[rows] * t[rows, 8]
                     - mu_a[rows] * t[rows, 9])
            cand = ~bad & np.isfinite(phi_t) & ~(theta_t > th_max[act[rows]])
            cand &= filter_acceptable(act[rows], theta_t, phi_t)
            al, dp = alpha[rows], dphi[rows]
            lhs_switch = al * powv(np.where(dp < 0.0, -dp, 0.0), opts.s_phi)
            switching = (dp < 0.0) & (lhs_switch > rhs_switch[rows])
            ftype_branch = (theta_cur[rows] <= th_min[act[rows]]) & switching
            acc_f = cand & ftype_branch & (phi_t <= phi_cur[rows] + opts.eta_phi * al * dp)
            acc_h = cand & ~ftype_branch & ((theta_t <= (1.0 - opts.gamma_theta) * theta_cur[rows])
                                           | (phi_t <= phi_cur[rows] - opts.gamma_phi * theta_cur[rows]))
            verdict[rows[acc_f]] = 2
            verdict[rows[acc_h]] = 1
            accepted_now = acc_f | acc_h
            searching[rows[accepted_now]] = False
            rej = rows[~accepted_now]
            alpha[rej] *= 0.5
            searching[rej[alpha[rej] < opts.alpha_min]] = False
            first = False
        # ---- accept (ipm.py:521-548)
        for j in np.flatnonzero(verdict == 0):
            insts[act[j]].status = LINE_SEARCH_FAILURE
            insts[act[j]].message = f"step size below {opts.alpha_min:g}"
        hrows = np.flatnonzero(verdict == 1)
        filter_add(act[hrows], (1.0 - opts.gamma_theta) * theta_cur[hrows],
                   phi_cur[hrows] - opts.gamma_phi * theta_cur[hrows])
        acc = np.flatnonzero(verdict != 0)
        Bt.bp_h[act[acc], BP_ALPHA] = alpha[acc]
        Bt.bp_h[act[acc], BP_ALPHA_Z] = alpha_z[acc]
        set_active()
        Bt.push_bp()
        L.check(lib.gn_ipm_accept_batched(KH, B, ctypes.byref(Bt.V), ctypes.byref(Bt.ST), bp,
                                          opts.kappa_sigma, ptr(Bt.ipm_flags), stream))
        for j in acc:
            b = act[j]
            it = insts[b]
            it.it += 1
            it.residual = float(e_0[j])
            if opts.record_trace:
                it.trace.append((it.it, float(fval[j]) / it.obj_scale, float(primal_max[j]), float(dual_max[j]),
                                 float(mu[b]), float(alpha[j]), float(delta_w[b])))
            if it.it >= opts.max_iter:
                it.status = MAX_ITER
    for b, it in enumerate(insts):
        it.mu = float(mu[b])
        if it.status is None:
            it.status = MAX_ITER
    # ---- unscaled objective and violation at x (ipm.py:350-357), one read
    Bt.ad_flags.zero_()
    ad(Bt.x, F | C, f=Bt.scal[:, 62], c=Bt.ct)
    if m:
        g = Bt.ct[:, :m]
        zero = torch.zeros_like(g)
        Bt.scal[:, 63] = torch.maximum(torch.maximum(Bt.rlo - g, zero), torch.maximum(g - Bt.rhi, zero)).amax(1)
    fin, w = Bt.read(62, 64, (Bt.ad_flags,))
    xh = D.to_host(Bt.x)
    total = time.perf_counter() - t_start
    reports = []
    for b, it in enumerate(insts):
        rep = SolveReport(status=it.status, n_var=n, n_con=m, iterations=it.it, message=it.message,
                          final_mu=it.mu, residual_scaled=it.residual, trace=it.trace,
                          refinement_relative_residual=it.ir_rel,
                          x=None if getattr(it, "no_x", False) else xh[b].copy(),
                          seconds={"total": total, "ad": np.nan, "linear": np.nan, "internal": np.nan})
        if not getattr(it, "no_x", False) and not w[0][b] & F:
            rep.objective = float(fin[b, 0])
            if not w[0][b] & C:
                rep.constraint_violation = float(fin[b, 1]) if m else 0.0
        rep.debug["batch"] = B
        reports.append(rep)
    return reports
