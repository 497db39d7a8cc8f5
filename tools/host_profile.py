"""cProfile of resident-plan solves (host overhead diagnostics)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402


def main(wl="C3"):
    am = build_model(wl)
    opts = SolverOptions(tol=1e-6)
    for _ in range(2):
        solve(am.model, opts, constraint_ranges=am.ranges)
    torch.cuda.synchronize()
    t = time.perf_counter()
    solve(am.model, opts, constraint_ranges=am.ranges)
    torch.cuda.synchronize()
    print("wall", time.perf_counter() - t)
    pr = cProfile.Profile()
    pr.enable()
    solve(am.model, opts, constraint_ranges=am.ranges)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main(*sys.argv[1:])
