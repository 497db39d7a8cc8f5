"""Per-phase host symbolic timings on the calling thread vs OpenMP threads
(diagnostics; run with GN_HOST_TIMING=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import _lib  # noqa: E402
from paper_2307_16830_b200 import kkt as KK, sparse as SP  # noqa: E402

am = build_model(os.environ.get("WL", "C3"))
model = am.model
cs0 = KK.symbolic_condense(model.hess_rows, model.hess_cols, model.jac_rows, model.jac_cols, model.n_var)
perm = SP.amd_order(cs0.matrix)
for nt in [int(a) for a in sys.argv[1:]] or [16]:
    _lib.lib().gn_set_host_threads(nt)
    for r in range(3):
        print(f"== threads {nt} rep {r}", file=sys.stderr, flush=True)
        t = time.perf_counter()
        cs = KK.symbolic_condense(model.hess_rows, model.hess_cols, model.jac_rows, model.jac_cols, model.n_var)
        t1 = time.perf_counter()
        sym = SP.symbolic_cholesky(cs.matrix, perm)
        t2 = time.perf_counter()
        print(f"threads {nt}: condense {1e3*(t1-t):.2f} symbolic {1e3*(t2-t1):.2f}", file=sys.stderr, flush=True)
