"""Host-side setup breakdown of one from-scratch solve (diagnostics)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, kkt, solve, sparse  # noqa: E402


def main(wl="C3"):
    am = build_model(wl)
    m = am.model
    cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    perm = sparse.amd_order(cs.matrix)
    for _ in range(3):
        m.release_device()
        torch.cuda.synchronize()
        t = time.perf_counter()
        rep = solve(m, SolverOptions(tol=1e-6, ordering=perm), constraint_ranges=am.ranges)
        torch.cuda.synchronize()
        tot = time.perf_counter() - t
        print(f"total {tot:.3f} s  ipm-seconds {rep.seconds}  setup "
              + " ".join(f"{k}={v:.3f}" for k, v in rep.debug["setup_seconds"].items()))


if __name__ == "__main__":
    main(*sys.argv[1:])
