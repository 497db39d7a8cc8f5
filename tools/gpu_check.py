"""Stage-by-stage GPU diagnostics (development aid; prints, never asserts)."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")


def stage(name, fn):
    t = time.perf_counter()
    try:
        out = fn()
        print(f"[ok] {name} ({time.perf_counter() - t:.3f}s) {out if out is not None else ''}", flush=True)
    except Exception:
        print(f"[FAIL] {name}", flush=True)
        traceback.print_exc()


def main():
    import faulthandler

    import torch

    faulthandler.dump_traceback_later(240, exit=True)

    print("device", torch.cuda.get_device_name(0), flush=True)
    from paper_2307_16830_b200 import autodiff as ad, kkt as K, sparse as S
    from paper_2307_16830_b200.acopf import build_acopf
    from paper_2307_16830_b200.grids import tiled_case
    from paper_2307_16830_b200.matpower import parse_matpower
    import paper_2307_16830_b200 as gp

    g = dict(np.load("tests/golden/T4.npz"))
    am = build_acopf(parse_matpower(tiled_case(4)))
    m = am.model

    def ad_check():
        x, y = g["ad1_x"], g["ad1_y"]
        out = {}
        for nm, got, ref in (("c", ad.eval_constraints(m, x), g["ad1_c"]),
                             ("grad", ad.eval_gradient(m, x), g["ad1_grad"]),
                             ("jac", ad.eval_jacobian(m, x), g["ad1_jac"]),
                             ("hess", ad.eval_lagrangian_hessian(m, x, y, 0.7), g["ad1_hess"])):
            out[nm] = float(np.abs(got - ref).max() / max(1e-300, np.abs(ref).max()))
        out["f"] = ad.eval_objective(m, x) - float(g["ad1_f"])
        return out

    stage("AD T4", ad_check)

    def kkt_check():
        n, mm = int(g["n"]), int(g["m"])
        ws = K.KKTWorkspace(n, mm, g["hess_rows"], g["hess_cols"], g["jac_rows"], g["jac_cols"])
        ws.set_iterate(*(g["ws_" + f] for f in ("w_vals", "a_vals", "dxl", "dxu", "zxl", "zxu",
                                                 "dsl", "dsu", "zsl", "zsu")))
        ws.delta_w, ws.delta_c = float(g["ws_delta_w"]), float(g["ws_delta_c"])
        back = K.CondensedBackend(ws, ordering=g["sym_perm"])
        ok = back.try_factorize()
        kv = back.kvals.cpu().numpy()
        lv = back.factor.values
        x = S.solve(back.factor, g["solve_b"])
        return dict(ok=ok, K=float(np.abs(kv - g["K_vals"]).max()),
                    L=float(np.abs(lv - g["L_vals"]).max() / np.abs(g["L_vals"]).max()),
                    solve=float(np.abs(x - g["solve_x"]).max() / np.abs(g["solve_x"]).max()),
                    info=back.symbolic.info)

    stage("KKT T4", kkt_check)

    def solve_case(tiles, tol=1e-6):
        a = build_acopf(parse_matpower(tiled_case(tiles)))
        t = time.perf_counter()
        rep = gp.solve(a.model, gp.SolverOptions(tol=tol), constraint_ranges=a.ranges)
        return dict(status=rep.status, it=rep.iterations, obj=rep.objective,
                    wall=time.perf_counter() - t, sec=rep.seconds, msg=rep.message)

    stage("solve C1", lambda: solve_case(1))
    stage("solve T16", lambda: solve_case(16))
    stage("solve C2", lambda: solve_case(143))
    if "--big" in sys.argv:
        stage("solve C3", lambda: solve_case(714))


if __name__ == "__main__":
    main()
