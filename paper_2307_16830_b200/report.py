"""Case runner and benchmark records (the reporting front end).

Mirrors the reference's `gridnlp.bench` API (src/bench.py:28-218):
`BenchRecord` (same fields, JSON/CSV), `solve_case`, `run_suite`,
`render_csv`, `render_text`. Two things differ on the GPU path:
* `run_suite(parallel=P)` runs P cases at once on one GPU. It uses host
  threads, each with its own CUDA stream and persistent-grid budget
  (gn_set_concurrency), instead of a process pool.
* The condition estimates (condensed and augmented, src/bench.py:68-135)
  run on the device factor: the augmented system's inverse is the condensed
  solve plus the recoveries.
"""
from __future__ import annotations

import csv
import io
import json
import os
from dataclasses import asdict, dataclass, field

import numpy as np

from .acopf import build_acopf
from .ipm import OPTIMAL, SolverOptions, solve
from .matpower import parse_matpower_file

CSV_COLUMNS = [
    "case", "n_var", "n_con", "iterations", "status", "objective",
    "violation", "total_s", "ad_s", "linear_s", "internal_s",
    "condensed_condition", "augmented_condition", "augmented_condition_dense",
]


@dataclass
class BenchRecord:
    case: str
    n_var: int = 0
    n_con: int = 0
    iterations: int = 0
    status: str = ""
    objective: float | None = None
    violation: float | None = None
    seconds: dict = field(default_factory=dict)
    condensed_condition: float | None = None
    augmented_condition: float | None = None
    augmented_condition_dense: float | str | None = None
    error: str = ""

    def to_json(self) -> str:
        return json.dumps(asdict(self))

    @classmethod
    def from_json(cls, text: str) -> "BenchRecord":
        return cls(**json.loads(text))

    def csv_row(self):
        sec = self.seconds or {}
        return [self.case, self.n_var, self.n_con, self.iterations, self.status, self.objective,
                self.violation, sec.get("total"), sec.get("ad"), sec.get("linear"),
                sec.get("internal"), self.condensed_condition, self.augmented_condition,
                self.augmented_condition_dense]


def _finite_or_none(v):
    return None if v is None or not np.isfinite(v) else float(v)


DENSE_CONDITION_LIMIT = 2000          # src/bench.py:25
SKIPPED_TOO_LARGE = "skipped_too_large"


def _augmented_norm1(ws):
    """1-norm (max column |sum|) of the augmented three-block matrix
    [[W + Sigma_x + dw, 0, A^T], [0, Sigma_s + dw, -I], [A, -I, -dc]] of
    src/bench.py:68-90, from the device workspace (duplicates summed before
    the absolute value, as the reference's COO -> CSC does)."""
    import torch

    n, m = ws.n, ws.m
    dev = ws.w_vals.device
    hr = torch.as_tensor(ws.hess_rows, device=dev)
    hc = torch.as_tensor(ws.hess_cols, device=dev)
    jr = torch.as_tensor(ws.jac_rows, device=dev)
    jc = torch.as_tensor(ws.jac_cols, device=dev)
    diag = ws.sigma_x + ws.delta_w
    dmask = hr == hc
    diag = diag.index_add(0, hc[dmask], ws.w_vals[dmask])
    colx = diag.abs()
    off = ~dmask
    wa = ws.w_vals[off].abs()
    colx = colx.index_add(0, hc[off], wa).index_add(0, hr[off], wa)
    aa = ws.a_vals.abs()
    colx = colx.index_add(0, jc, aa)
    cols = (ws.sigma_s + ws.delta_w).abs() + 1.0
    coly = torch.zeros(m, dtype=torch.float64, device=dev).index_add(0, jr, aa) + 1.0 + abs(ws.delta_c)
    return float(torch.cat([colx, cols, coly]).max().item()) if n + m else 0.0


def _augmented_dense(ws):
    """Dense augmented matrix on the device (small systems only)."""
    import torch

    n, m = ws.n, ws.m
    dev = ws.w_vals.device
    a = torch.zeros(n + 2 * m, n + 2 * m, dtype=torch.float64, device=dev)
    hr = torch.as_tensor(ws.hess_rows, device=dev)
    hc = torch.as_tensor(ws.hess_cols, device=dev)
    a.index_put_((hr, hc), ws.w_vals, accumulate=True)
    off = hr != hc
    a.index_put_((hc[off], hr[off]), ws.w_vals[off], accumulate=True)
    ix = torch.arange(n, device=dev)
    a.index_put_((ix, ix), ws.sigma_x + ws.delta_w, accumulate=True)
    jr = torch.as_tensor(ws.jac_rows, device=dev) + n + m
    jc = torch.as_tensor(ws.jac_cols, device=dev)
    a.index_put_((jr, jc), ws.a_vals, accumulate=True)
    a.index_put_((jc, jr), ws.a_vals, accumulate=True)
    iy = torch.arange(m, device=dev)
    a[n + iy, n + iy] += ws.sigma_s + ws.delta_w
    a[n + iy, n + m + iy] -= 1.0
    a[n + m + iy, n + iy] -= 1.0
    a[n + m + iy, n + m + iy] -= ws.delta_c
    return a


def _hager_estimate(solve_fn, dim, iters=6):
    """Hager's 1-norm estimate of ||M^-1|| (src/bench.py:93-110)."""
    x = np.full(dim, 1.0 / dim)
    est = 0.0
    for _ in range(iters):
        y = solve_fn(x)
        est_new = float(np.abs(y).sum())
        xi = np.sign(y)
        xi[xi == 0.0] = 1.0
        z = solve_fn(xi)   # symmetric
        j = int(np.argmax(np.abs(z)))
        if np.abs(z[j]) <= z @ x or est_new <= est:
            est = max(est, est_new)
            break
        est = est_new
        x = np.zeros(dim)
        x[j] = 1.0
    return est


def diagnose_conditioning(report, dense_limit=DENSE_CONDITION_LIMIT) -> dict:
    """Condition estimates of the condensed and augmented systems at the final
    iterate of a solve run with ``keep_workspace=True`` (src/bench.py:113-135).

    * condensed: refactorise with the workspace's current regularisation
      (device), then Hager's estimate over device solves -- only when the
      factorisation is positive definite;
    * augmented: Hager's estimate of the three-block matrix, whose inverse
      is exactly the condensed solve + recoveries (``backend.solve3``), so it
      runs on the device factor too (the reference uses a CPU sparse LU);
    * dense: numpy-equivalent ``cond(M, 1)`` of the dense augmented matrix
      (torch.linalg on the device) up to ``dense_limit`` rows.
    """
    import torch

    from . import device as D
    from . import sparse as S

    ws = report.debug.get("workspace")
    backend = report.debug.get("backend")
    if ws is None or backend is None:
        return {}
    out = {}
    backend.try_factorize()
    if not backend.factor.ok:
        return out
    out["condensed_condition"] = float(S.estimate_condition(backend.factor, backend.structure.matrix))
    n, m = ws.n, ws.m
    dim = n + 2 * m

    def solve_aug(v):
        dx, ds, dy = backend.solve3(D.to_dev(v[:n]), D.to_dev(v[n:n + m]), D.to_dev(v[n + m:]))
        return D.to_host(torch.cat([dx, ds, dy]))

    out["augmented_condition"] = _augmented_norm1(ws) * _hager_estimate(solve_aug, dim)
    if dim <= dense_limit:
        out["augmented_condition_dense"] = float(torch.linalg.cond(_augmented_dense(ws), 1).item())
    else:
        out["augmented_condition_dense"] = SKIPPED_TOO_LARGE
    return out


def solve_case(path, tol=1e-4, max_iter=3000, log_level=0, diagnose=False, backend="condensed"):
    """Parse, build and solve one MATPOWER case file -> (record, report)."""
    net = parse_matpower_file(path)
    am = build_acopf(net)
    opts = SolverOptions(tol=tol, max_iter=max_iter, log_level=log_level, backend=backend,
                         keep_workspace=diagnose)
    rep = solve(am.model, opts, constraint_ranges=am.ranges)
    rec = BenchRecord(case=net.name or str(path), n_var=rep.n_var, n_con=rep.n_con,
                      iterations=rep.iterations, status=rep.status,
                      objective=_finite_or_none(rep.objective),
                      violation=_finite_or_none(rep.constraint_violation),
                      seconds={k: float(v) for k, v in rep.seconds.items()})
    if diagnose and rep.status == OPTIMAL:
        d = diagnose_conditioning(rep)
        rec.condensed_condition = d.get("condensed_condition")
        rec.augmented_condition = d.get("augmented_condition")
        rec.augmented_condition_dense = d.get("augmented_condition_dense")
    return rec, rep


def _suite_worker(path, tol, max_iter, log_level=0):
    try:
        return solve_case(path, tol=tol, max_iter=max_iter, log_level=log_level)[0]
    except Exception as exc:   # a bad case becomes a failure record, never kills the suite
        return BenchRecord(case=os.path.basename(str(path)), status="failed", error=str(exc))


def run_suite(case_paths, tol=1e-4, max_iter=3000, log_level=0, parallel=0):
    """Solve every case; `parallel` > 1 overlaps that many solves on the GPU."""
    paths = [str(p) for p in case_paths]
    if not parallel or parallel <= 1 or len(paths) <= 1:
        return [_suite_worker(p, tol, max_iter, log_level) for p in paths]
    import threading

    import torch

    from . import _lib as L

    workers = min(int(parallel), len(paths))
    out: list = [None] * len(paths)
    dev = torch.cuda.current_device()

    def run(idxs):
        torch.cuda.set_device(dev)
        L.lib().gn_set_concurrency(workers)
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for i in idxs:
                    out[i] = _suite_worker(paths[i], tol, max_iter, log_level)
        finally:
            L.lib().gn_set_concurrency(1)

    threads = [threading.Thread(target=run, args=(list(range(w, len(paths), workers)),))
               for w in range(workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    return out


def render_csv(records) -> str:
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(CSV_COLUMNS)
    for r in records:
        w.writerow(r.csv_row())
    return buf.getvalue()


def render_text(records) -> str:
    head = ["case", "vars", "cons", "iter", "status", "objective", "violation", "ad_s", "lin_s",
            "total_s"]

    def fmt(v, spec):
        return "" if v is None else format(v, spec)

    rows = []
    for r in records:
        sec = r.seconds or {}
        rows.append([r.case, str(r.n_var), str(r.n_con), str(r.iterations), r.status or "failed",
                     fmt(r.objective, ".4f"), fmt(r.violation, ".3e"), fmt(sec.get("ad"), ".3f"),
                     fmt(sec.get("linear"), ".3f"), fmt(sec.get("total"), ".3f")])
    width = [max([len(h)] + [len(row[i]) for row in rows]) for i, h in enumerate(head)]
    lines = ["  ".join(h.ljust(n) for h, n in zip(head, width))]
    lines += ["  ".join(c.ljust(n) for c, n in zip(row, width)) for row in rows]
    return "\n".join(lines) + "\n"
