"""Median host-analysis phase times over repeated calls (diagnostics):
    GN_HOST_TIMING=1 python tools/host_ab.py 2> timings.txt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import kkt, sparse  # noqa: E402

am = build_model("C3")
m = am.model
cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
perm = sparse.amd_order(cs.matrix)
for _ in range(12):
    cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    sym = sparse.symbolic_cholesky(cs.matrix, perm)
