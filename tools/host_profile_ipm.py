"""cProfile of the Python side of one resident C3 solve (diagnostics)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402

am = build_model(sys.argv[1] if len(sys.argv) > 1 else "C3")
opts = SolverOptions(tol=1e-6)
for _ in range(3):
    rep = solve(am.model, opts, constraint_ranges=am.ranges)
torch.cuda.synchronize()
import time  # noqa: E402

t = time.perf_counter()
rep = solve(am.model, opts, constraint_ranges=am.ranges)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t, "iters", rep.iterations, "ir", rep.debug.get("ir_rounds"))
pr = cProfile.Profile()
pr.enable()
rep = solve(am.model, opts, constraint_ranges=am.ranges)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
