"""Trace comparison of the nonconvex regularisation case (GPU vs oracle)."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402

from oracle import ipm as OI  # noqa: E402
from oracle import model as OM  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402
from test_gpu_ipm import nonconvex_model  # noqa: E402

m = nonconvex_model()
om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
for tol in [float(t) for t in (sys.argv[1:] or ["1e-4", "1e-8"])]:
    r = solve(m, SolverOptions(tol=tol, log_level=3))
    o = OI.solve(om, m.lower, m.upper, m.start, OI.Options(tol=tol, verbose=True))
    print("tol", tol, r.status, r.iterations, r.message, o.status, o.iterations)
    for a, b in zip(r.trace, o.trace):
        print(" ours", ["%.10g" % v for v in a])
        print(" orac", ["%.10g" % v for v in b])
    print(" ir_rounds", r.debug.get("ir_rounds"))
    print(" x", r.x, o.x)
