"""Refactorise + solve the C3 condensed matrix a few times (profiling target).

    ncu --set full --import-source on -k regex:mf_factor_large -c 1 -s 2 \
        -o gpurun_out/factor python tools/chol_once.py C3
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve, sparse  # noqa: E402


def main(wl="C3", reps=4):
    am = build_model(wl)
    rep = solve(am.model, SolverOptions(tol=1e-6, max_iter=6, keep_workspace=True),
                constraint_ranges=am.ranges)
    be = rep.debug["backend"]
    b = torch.ones(am.model.n_var, dtype=torch.float64, device="cuda")
    for _ in range(int(reps)):
        f = sparse.factorize_device(be.symbolic, be.kvals, be.fws)
        sparse.solve_device(f, b.clone())
    torch.cuda.synchronize()
    print("ok", be.symbolic.info)


if __name__ == "__main__":
    main(*sys.argv[1:])
