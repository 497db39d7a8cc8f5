"""Print GPU vs oracle IPM traces side by side (development aid)."""
import faulthandler
import sys

import numpy as np

faulthandler.dump_traceback_later(100, exit=True)

sys.path.insert(0, ".")
sys.path.insert(0, "tests")

from oracle import ipm as OI
from oracle import model as OM

import paper_2307_16830_b200 as gp
from paper_2307_16830_b200.acopf import build_acopf
from paper_2307_16830_b200.grids import tiled_case
from paper_2307_16830_b200.matpower import parse_matpower

tiles = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
am = build_acopf(parse_matpower(tiled_case(tiles)))
m = am.model
rep = gp.solve(m, gp.SolverOptions(tol=tol, max_iter=40), constraint_ranges=am.ranges)
om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
orep = OI.solve(om, m.lower, m.upper, m.start, OI.Options(tol=tol, max_iter=40), am.ranges)
print("gpu", rep.status, rep.iterations, rep.objective, "oracle", orep.status, orep.iterations, orep.objective)
print("ir gpu", rep.debug.get("ir_rounds"))
print("ir ora", orep.ir_rounds)
for a, b in zip(rep.trace, orep.trace):
    print("G", " ".join(f"{v:.6e}" for v in a))
    print("O", " ".join(f"{v:.6e}" for v in b))
