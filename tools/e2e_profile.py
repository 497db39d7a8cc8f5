"""cProfile of from-scratch (e2e) solves with the ordering injected: where
the host time of setup + IPM goes (diagnostics)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, kkt, solve, sparse  # noqa: E402


def main(wl="C3", n=3):
    am = build_model(wl)
    m = am.model
    cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    opts = SolverOptions(tol=1e-6, ordering=sparse.amd_order(cs.matrix))
    del cs
    for _ in range(2):
        m.release_device()
        solve(m, opts, constraint_ranges=am.ranges)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    for _ in range(int(n)):
        m.release_device()
        torch.cuda.synchronize()
        t = time.perf_counter()
        pr.enable()
        solve(m, opts, constraint_ranges=am.ranges)
        torch.cuda.synchronize()
        pr.disable()
        print("wall", time.perf_counter() - t)
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(30)
    st.sort_stats("cumtime").print_stats(40)


if __name__ == "__main__":
    main(*sys.argv[1:])
