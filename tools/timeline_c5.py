"""GPU timeline of one instance-batched C5 solve (torch.profiler/CUPTI):
kernel time by name and idle gaps (diagnostics)."""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16830_b200 import SolverOptions, batch as B  # noqa: E402
from paper_2307_16830_b200.batch_ipm import solve_batched  # noqa: E402


def main(nb=256):
    inst = B.perturbed_instances(97, list(range(int(nb))))
    opts = SolverOptions(tol=1e-6)
    for _ in range(2):
        solve_batched(inst, opts)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        reps = solve_batched(inst, opts)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    print(f"instances {nb} iterations max {max(r.iterations for r in reps)} kernels {len(ev)} "
          f"span {span / 1e3:.2f} ms busy {busy / 1e3:.2f} ms idle {(span - busy) / 1e3:.2f} ms")
    byk = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        byk[e.name[:60]][0] += 1
        byk[e.name[:60]][1] += e.time_range.end - e.time_range.start
    for k, (c, t) in sorted(byk.items(), key=lambda x: -x[1][1])[:22]:
        print(f"  {k:60s} {c:5d} {t / 1e3:8.3f} ms")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for a, b in zip(ev, ev[1:]):
        g = b.time_range.start - a.time_range.end
        if g > 3:
            agg[(a.name[:40], b.name[:40])][0] += 1
            agg[(a.name[:40], b.name[:40])][1] += g
    print("idle gaps > 3us by (before -> after):")
    for (a, b), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
        print(f"  {t / 1e3:8.3f} ms {c:4d}x  {a} -> {b}")


if __name__ == "__main__":
    main(*sys.argv[1:])
