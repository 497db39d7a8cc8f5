"""Minor page faults and wall time of the host symbolic phases (diagnostics)."""
import os
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import kkt as KK, sparse as SP  # noqa: E402

am = build_model(os.environ.get("WL", "C3"))
model = am.model
cs0 = KK.symbolic_condense(model.hess_rows, model.hess_cols, model.jac_rows, model.jac_cols, model.n_var)
perm = SP.amd_order(cs0.matrix)
flt = lambda: resource.getrusage(resource.RUSAGE_SELF).ru_minflt
for r in range(4):
    f0, t0 = flt(), time.perf_counter()
    cs = KK.symbolic_condense(model.hess_rows, model.hess_cols, model.jac_rows, model.jac_cols, model.n_var)
    f1, t1 = flt(), time.perf_counter()
    sym = SP.symbolic_cholesky(cs.matrix, perm)
    f2, t2 = flt(), time.perf_counter()
    print(f"rep {r}: condense {1e3*(t1-t0):.2f} ms {f1-f0} faults | symbolic {1e3*(t2-t1):.2f} ms {f2-f1} faults", flush=True)
    del cs, sym
