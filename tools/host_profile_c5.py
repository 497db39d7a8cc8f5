"""cProfile of the host side of one instance-batched C5 solve (diagnostics)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2307_16830_b200 import SolverOptions, batch as B  # noqa: E402
from paper_2307_16830_b200.batch_ipm import solve_batched  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
inst = B.perturbed_instances(97, list(range(nb)))
opts = SolverOptions(tol=1e-6)
for _ in range(2):
    solve_batched(inst, opts)
torch.cuda.synchronize()
t = time.perf_counter()
solve_batched(inst, opts)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t)
pr = cProfile.Profile()
pr.enable()
solve_batched(inst, opts)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
