"""GPU timeline of one resident C3 solve via torch.profiler (CUPTI): kernel
durations, GPU idle gaps and what precedes/follows the largest gaps."""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402


def main(wl="C3"):
    am = build_model(wl)
    opts = SolverOptions(tol=1e-6)
    for _ in range(2):
        solve(am.model, opts, constraint_ranges=am.ranges)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        solve(am.model, opts, constraint_ranges=am.ranges)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    gaps = []
    for a, b in zip(ev, ev[1:]):
        g = b.time_range.start - a.time_range.end
        if g > 0:
            gaps.append((g, a.name[:40], b.name[:40]))
    print(f"kernels {len(ev)}  span {span / 1e3:.2f} ms  busy {busy / 1e3:.2f} ms  idle {(span - busy) / 1e3:.2f} ms")
    byk = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        byk[e.name[:50]][0] += 1
        byk[e.name[:50]][1] += e.time_range.end - e.time_range.start
    for k, (c, t) in sorted(byk.items(), key=lambda x: -x[1][1])[:20]:
        print(f"  {k:50s} {c:5d} {t / 1e3:8.3f} ms")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for g, a, b in gaps:
        if g > 3:
            agg[(a, b)][0] += 1
            agg[(a, b)][1] += g
    print("idle gaps > 3us by (before -> after):")
    for (a, b), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"  {t / 1e3:7.3f} ms {c:4d}x  {a} -> {b}")


if __name__ == "__main__":
    main(*sys.argv[1:])
