"""Kernel sequence with gaps of one resident solve (diagnostics):
prints the first N and last M kernels and every gap > 10 us."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402

am = build_model(sys.argv[1] if len(sys.argv) > 1 else "C3")
opts = SolverOptions(tol=1e-6)
for _ in range(2):
    solve(am.model, opts, constraint_ranges=am.ranges)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    solve(am.model, opts, constraint_ranges=am.ranges)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = t0
for k, e in enumerate(ev):
    g = e.time_range.start - prev
    if k < 120 or k > len(ev) - 40 or g > 10:
        print(f"{k:5d} {(e.time_range.start - t0):9.1f} gap {g:7.1f} dur {e.time_range.end - e.time_range.start:8.1f}  {e.name[:70]}")
    prev = e.time_range.end
