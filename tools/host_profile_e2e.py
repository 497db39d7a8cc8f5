"""cProfile of one end-to-end solve (release_device + solve with an injected
ordering), the bench's e2e leg (diagnostics)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402
from paper_2307_16830_b200 import kkt as KK, sparse as SP  # noqa: E402

am = build_model(sys.argv[1] if len(sys.argv) > 1 else "C3")
model = am.model
cs0 = KK.symbolic_condense(model.hess_rows, model.hess_cols, model.jac_rows, model.jac_cols, model.n_var)
perm = SP.amd_order(cs0.matrix)
opts = SolverOptions(tol=1e-6, ordering=perm)
for _ in range(3):
    model.release_device()
    rep = solve(model, opts, constraint_ranges=am.ranges)
torch.cuda.synchronize()
for _ in range(3):
    model.release_device()
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = solve(model, opts, constraint_ranges=am.ranges)
    torch.cuda.synchronize()
    print("wall", round(time.perf_counter() - t, 4), "setup", {k: round(v, 4) for k, v in rep.debug["setup_seconds"].items()})
model.release_device()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
rep = solve(model, opts, constraint_ranges=am.ranges)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(30)
