"""Run each hot kernel group of one IPM iterate a few times (profiling
target for ncu): full AD evaluation, condensed assembly, refactorisation,
solve.  The model is taken to a mid-run iterate first (keep_workspace).

    ncu --set full -k regex:"mf_|gn_ad|assemble" -o prof python tools/kernels_once.py C4
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve, sparse  # noqa: E402
from paper_2307_16830_b200.autodiff import C, F, GRAD, HESS, JAC, RESET  # noqa: E402


def main(wl="C3", reps=3):
    am = build_model(wl)
    rep = solve(am.model, SolverOptions(tol=1e-6, max_iter=6, keep_workspace=True),
                constraint_ranges=am.ranges)
    be, ws, P = rep.debug["backend"], rep.debug["workspace"], rep.debug["problem"]
    b = torch.ones(am.model.n_var, dtype=torch.float64, device="cuda")
    for _ in range(int(reps)):
        P.ev.launch(P.x, F | C | GRAD | JAC | HESS | RESET, y=P.y, obj_weight=P.obj_scale,
                    con_scale=P.con_scale, obj_scale=P.obj_scale, f=P.scal[48:49], c=P.c,
                    grad=P.grad, jac=ws.a_vals, hess=ws.w_vals)
        be.assemble()
        f = sparse.factorize_device(be.symbolic, be.kvals, be.fws)
        sparse.solve_device(f, b.clone())
    torch.cuda.synchronize()
    print("ok", wl, be.symbolic.info)


if __name__ == "__main__":
    main(*sys.argv[1:])
