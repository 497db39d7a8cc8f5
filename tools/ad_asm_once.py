"""AD full evaluation + K assembly at a mid-run iterate (profiling target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_model  # noqa: E402
from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402
from paper_2307_16830_b200.autodiff import C, F, GRAD, HESS, JAC  # noqa: E402


def main(wl="C4", reps=3):
    am = build_model(wl)
    rep = solve(am.model, SolverOptions(tol=1e-6, max_iter=3, keep_workspace=True),
                constraint_ranges=am.ranges)
    P, ws, be = rep.debug["problem"], rep.debug["workspace"], rep.debug["backend"]
    for _ in range(int(reps)):
        P.ev.launch(P.x, F | C | GRAD | JAC | HESS, y=P.y, obj_weight=P.obj_scale, con_scale=P.con_scale,
                    obj_scale=P.obj_scale, f=P.scal[48:49], c=P.c, grad=P.grad, jac=ws.a_vals,
                    hess=ws.w_vals)
        be.assemble()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(*sys.argv[1:])
