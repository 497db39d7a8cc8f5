"""Dump refactorisation values (C3 condensed K after 3 IPM iterations, and
dense fronts exercising every panel variant) with a given libgridopf.so, to
check that a kernel change is bitwise neutral:
    python tools/factor_dump.py <lib.so> <out.npz>   (diagnostics)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(libpath, out):
    from paper_2307_16830_b200 import _lib as L

    L.LIB_PATH = os.path.abspath(libpath)
    from bench import build_model
    from paper_2307_16830_b200 import SolverOptions, solve
    from paper_2307_16830_b200 import sparse as S

    res = {}
    am = build_model("C3")
    rep = solve(am.model, SolverOptions(tol=1e-6, max_iter=3, keep_workspace=True), constraint_ranges=am.ranges)
    be = rep.debug["backend"]
    be.assemble()
    res["C3"] = S.factorize_device(be.symbolic, be.kvals).values
    rng = np.random.default_rng(0)
    for n in (200, 330, 700, 900):
        M = rng.normal(size=(n, n))
        A = M @ M.T / n + np.eye(n)
        ri, ci = np.tril_indices(n)
        m = S.coo_to_csc(n, ri, ci, A[ri, ci])[0]
        sym = S.symbolic_cholesky(m, np.arange(n))
        res[f"dense{n}"] = S.factorize(sym, m.values).values
    np.savez(out, **res)
    print("ok", {k: v.shape for k, v in res.items()})


if __name__ == "__main__":
    main(*sys.argv[1:])
