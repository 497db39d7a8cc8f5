"""Case runner and benchmark records (the reporting front end).

Mirrors the reference's `gridnlp.bench` API (src/bench.py:28-218):
`BenchRecord` (same fields, JSON/CSV), `solve_case`, `run_suite`,
`render_csv`, `render_text`. Two things differ on the GPU path:
* `run_suite(parallel=P)` runs P cases at once on one GPU. It uses host
  threads, each with its own CUDA stream and persistent-grid budget
  (gn_set_concurrency), instead of a process pool.
* The condensed condition estimate uses the device factor and solves
  (`sparse.estimate_condition`, cholesky.py:220-241). The augmented
  estimates belong to the dense CPU oracle and are reported as not computed.
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


def diagnose_conditioning(report) -> dict:
    """Condensed 1-norm condition estimate at the final iterate (device)."""
    from . import sparse as S

    backend = report.debug.get("backend")
    if backend is None or backend.factor is None:
        return {}
    return {"condensed_condition": float(S.estimate_condition(backend.factor,
                                                             backend.structure.matrix)),
            "augmented_condition": None,
            "augmented_condition_dense": "not computed (dense CPU oracle only)"}


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
