"""Per-front timeline of one refactorisation + solve on the GPU (diagnostics).

    python tools/chol_trace.py C3 gpurun_out/trace_C3.npz

Runs one C3 solve to a mid-run iterate (keep_workspace), then traces one
factor + solve of that K and saves the stamps and the front plan.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve, sparse  # noqa: E402


def dense(n, out):
    """One dense SPD front of n rows (single-front timing)."""
    n = int(n)
    g = torch.Generator().manual_seed(0)
    M = torch.randn(n, n, generator=g, dtype=torch.float64)
    A = (M @ M.T / n + torch.eye(n, dtype=torch.float64)).numpy()
    ri, ci = np.tril_indices(n)
    m = sparse.coo_to_csc(n, ri, ci, A[ri, ci])[0]
    sym = sparse.symbolic_cholesky(m, np.arange(n))
    kv = torch.as_tensor(m.values, device="cuda")
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        tr, pt = sparse.trace_factor_solve(sym, kv, b)
    np.savez_compressed(out, trace=tr, panels=pt, probes=getattr(sparse.trace_factor_solve, "last_probes", None),
                        **sparse.front_plan(sym))
    print("saved", out)


def main(wl="C3", out="gpurun_out/trace.npz"):
    if wl.startswith("dense"):
        return dense(wl[5:], out)
    am = build_model(wl)
    rep = solve(am.model, SolverOptions(tol=1e-6, max_iter=6, keep_workspace=True),
                constraint_ranges=am.ranges)
    be = rep.debug["backend"]
    b = torch.ones(am.model.n_var, dtype=torch.float64, device="cuda")
    for _ in range(2):
        tr, pt = sparse.trace_factor_solve(be.symbolic, be.kvals, b)
    fp = sparse.front_plan(be.symbolic)
    np.savez_compressed(out, trace=tr, panels=pt, probes=getattr(sparse.trace_factor_solve, "last_probes", None),
                        **fp)
    print("saved", out, tr.shape)


if __name__ == "__main__":
    main(*sys.argv[1:])
