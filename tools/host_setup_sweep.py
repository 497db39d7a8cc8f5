"""Host setup phases of the e2e leg vs OpenMP threads (diagnostics):
release_device + plans(model, ordering) + evaluator upload, timed per phase."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve, _lib  # noqa: E402
from paper_2307_16830_b200 import kkt as KK, sparse as SP  # noqa: E402

am = build_model("C3")
model = am.model
cs0 = KK.symbolic_condense(model.hess_rows, model.hess_cols, model.jac_rows, model.jac_cols, model.n_var)
perm = SP.amd_order(cs0.matrix)
print("n_cond", cs0.matrix.n, "nnzK", cs0.matrix.nnz, flush=True)
for nt in [int(a) for a in sys.argv[1:]] or [16]:
    _lib.lib().gn_set_host_threads(nt)
    opts = SolverOptions(tol=1e-6, ordering=perm)
    walls = []
    import ctypes
    for r in range(6):
        model.release_device()
        torch.cuda.synchronize()
        _lib.lib().gn_upload_stats(None, None, None, 1)
        t = time.perf_counter()
        rep = solve(model, opts, constraint_ranges=am.ranges)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t)
        na, mm, cm = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        _lib.lib().gn_upload_stats(ctypes.byref(na), ctypes.byref(mm), ctypes.byref(cm), 0)
        print(f"  solve {r}: {walls[-1]*1e3:.1f} ms, allocs {na.value} malloc {mm.value:.2f} ms copies {cm.value:.2f} ms",
              flush=True)
    s = rep.debug["setup_seconds"]
    print(f"threads {nt}: wall {min(walls)*1e3:.1f} ms  ipm_total {rep.seconds['total']*1e3:.1f}  setup",
          {k: round(v * 1e3, 2) for k, v in s.items()}, flush=True)
