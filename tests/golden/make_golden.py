"""Generate golden vectors by running the REFERENCE package (gridnlp 0.1.0).

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a writable temp dir (numba's cache=True
writes beside the source), imports ``gridnlp`` from there, and writes

* ``networks.json``        parsed case14/30/57/118 tables (NetworkData)
* ``<model>.npz``          structure arrays, AD values, condensed K pattern
                            and maps, ordering, symbolic factor, K/L values,
                            solves and KKT vector kernels at a real iterate
* ``end_to_end.json``      status / iterations / objective of full solves
* ``<cfg>_x.npz``          converged x for the synthetic configurations

The ordering for the synthetic grids >= 2k buses is injected through
``gridnlp.kkt.amd_order`` with the heap minimum degree (bit-identical to
the shipped O(n^2) scan, checked here on every model where both run).
"""
from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from paper_2307_16830_b200.grids import tiled_case  # noqa: E402
from oracle.ordering import min_degree_order  # noqa: E402


def _import_reference():
    tmp = tempfile.mkdtemp(prefix="gridnlp_ref_")
    shutil.copytree("/root/reference/pkg", os.path.join(tmp, "pkg"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba"))
    sys.path.insert(0, os.path.join(tmp, "pkg", "src"))
    import gridnlp  # noqa: F401
    return os.path.join(tmp, "pkg", "src", "gridnlp", "cases")


CASES = _import_reference()
import gridnlp.kkt as RK  # noqa: E402
from gridnlp import autodiff as RA  # noqa: E402
from gridnlp.acopf import build_acopf  # noqa: E402
from gridnlp.ipm import SolverOptions, solve  # noqa: E402
from gridnlp.matpower import parse_matpower, parse_matpower_file  # noqa: E402
from gridnlp.sparse import amd_order, factorize, symbolic_cholesky, solve as rsolve  # noqa: E402

_SHIPPED_AMD = RK.amd_order


def _heap_amd(mat):
    r, c = mat.coords()
    return min_degree_order(mat.n, r, c)


def net_to_dict(net):
    return dict(
        base_mva=net.base_mva, name=net.name,
        buses=[[b.id, b.type, b.pd, b.qd, b.gs, b.bs, b.vm, b.va, b.vmax, b.vmin]
               for b in net.buses],
        generators=[[g.bus, g.pg, g.qg, g.qmax, g.qmin, g.vg, g.pmax, g.pmin, *g.cost]
                    for g in net.generators],
        branches=[[br.from_bus, br.to_bus, br.r, br.x, br.b_charge, br.rate_a, br.tap,
                   br.shift, br.angmin, br.angmax] for br in net.branches])


def dump_model(tag, am, rng, check_shipped_amd=True):
    m = am.model
    out = {"n": m.n_var, "m": m.n_con, "lower": m.lower, "upper": m.upper,
           "start": m.start, "ranges": am.ranges,
           "jac_rows": m.jac_rows, "jac_cols": m.jac_cols,
           "hess_rows": m.hess_rows, "hess_cols": m.hess_cols}
    for bi, blk in enumerate(m.pattern_blocks):
        p = f"b{bi}_"
        out[p + "kind"] = np.array(("objective_sum", "constraint_define",
                                    "constraint_increment").index(blk.kind))
        out[p + "out"] = np.array(blk.tape.out)
        out[p + "var_idx"] = blk.var_idx
        out[p + "params"] = blk.params
        if blk.targets is not None:
            out[p + "targets"] = blk.targets
        out[p + "ops"] = np.asarray(blk.tape.ops, np.int64).reshape(-1, 3)
        out[p + "consts"] = np.asarray(blk.tape.consts, float)
        out[p + "first_slots"] = np.asarray(blk.tape.first_slots, np.int64)
        out[p + "second_pairs"] = np.asarray(blk.tape.second_pairs, np.int64).reshape(-1, 2)
        for k, a in enumerate(blk.jac_slots):
            out[p + f"jac_slots{k}"] = a
        for k, a in enumerate(blk.hess_slots):
            out[p + f"hess_slots{k}"] = a
            out[p + f"hess_factor{k}"] = blk.hess_factor[k]
    out["n_blocks"] = len(m.pattern_blocks)
    # AD at the start point and at a random interior point
    x0 = m.start
    x1 = m.start + rng.uniform(-0.05, 0.05, m.n_var)
    x1 = np.clip(x1, np.where(np.isfinite(m.lower), m.lower + 1e-3, -np.inf),
                 np.where(np.isfinite(m.upper), m.upper - 1e-3, np.inf))
    y1 = rng.normal(size=m.n_con)
    for k, (x, y, w) in enumerate(((x0, np.ones(m.n_con), 1.0), (x1, y1, 0.7))):
        out[f"ad{k}_x"], out[f"ad{k}_y"], out[f"ad{k}_w"] = x, y, w
        out[f"ad{k}_f"] = RA.eval_objective(m, x)
        out[f"ad{k}_c"] = RA.eval_constraints(m, x)
        out[f"ad{k}_grad"] = RA.eval_gradient(m, x)
        out[f"ad{k}_jac"] = RA.eval_jacobian(m, x)
        out[f"ad{k}_hess"] = RA.eval_lagrangian_hessian(m, x, y, w)
    # solve to tol 1e-4 keeping the workspace: a realistic iterate for K/L
    RK.amd_order = _heap_amd
    rep = solve(m, SolverOptions(tol=1e-4, keep_workspace=True), constraint_ranges=am.ranges)
    RK.amd_order = _SHIPPED_AMD
    ws, back = rep.debug["workspace"], rep.debug["backend"]
    st = back.structure
    for f in ("w_map", "diag_map", "ata_map", "ata_row", "ata_s1", "ata_s2"):
        out["cond_" + f] = getattr(st, f)
    out["cond_indptr"], out["cond_indices"] = st.matrix.indptr, st.matrix.indices
    perm = back.symbolic.perm
    if check_shipped_amd:
        assert np.array_equal(perm, _SHIPPED_AMD(st.matrix)), tag
    sym = back.symbolic
    for f in ("perm", "parent", "a_rowptr", "a_rowcol", "a_srcslot", "row_ptr",
              "row_cols", "l_colptr", "l_rowidx"):
        out["sym_" + f] = getattr(sym, f)
    for f in ("w_vals", "a_vals", "dxl", "dxu", "zxl", "zxu", "dsl", "dsu", "zsl", "zsu",
              "sigma_x", "sigma_s"):
        out["ws_" + f] = getattr(ws, f)
    ws.delta_w, ws.delta_c = 1e-6, 1e-8
    out["ws_delta_w"], out["ws_delta_c"] = ws.delta_w, ws.delta_c
    back.assemble()
    out["K_vals"] = st.matrix.values.copy()
    fac = factorize(sym, st.matrix.values)
    assert fac.ok
    out["L_vals"] = fac.values
    b = rng.normal(size=m.n_var)
    out["solve_b"], out["solve_x"] = b, rsolve(fac, b)
    pv = RK.PVec(*(rng.normal(size=k) for k in (m.n_var, m.n_con, m.n_con, m.n_var,
                                                  m.n_var, m.n_con, m.n_con)))
    for f, a in zip(("x", "s", "y", "zxl", "zxu", "zsl", "zsu"),
                    (pv.x, pv.s, pv.y, pv.zxl, pv.zxu, pv.zsl, pv.zsu)):
        out["pv_" + f] = a
    qx, qs, qy = ws.condense_pvec(pv)
    out["q_x"], out["q_s"], out["q_y"] = qx, qs, qy
    out["rhs"] = ws.condensed_rhs(qx, qs, qy)
    back.factor = fac
    dx, ds, dy = back.solve3(qx, qs, qy)
    out["s3_dx"], out["s3_ds"], out["s3_dy"] = dx, ds, dy
    steps = RK.assemble_steps(ws, pv, dx, ds, dy)
    for f in ("zxl", "zxu", "zsl", "zsu"):
        out["st_" + f] = getattr(steps, f)
    res = ws.residual_full(steps, pv)
    for f in ("x", "s", "y", "zxl", "zxu", "zsl", "zsu"):
        out["res_" + f] = getattr(res, f).astype(float)
    out["matrix_scale"] = ws.matrix_scale()
    np.savez_compressed(os.path.join(HERE, f"{tag}.npz"), **out)
    print(tag, m.n_var, m.n_con, "nnzL", sym.l_rowidx.size, flush=True)


def main():
    rng = np.random.default_rng(20230731)
    nets = {c: parse_matpower_file(os.path.join(CASES, f"{c}.m"))
            for c in ("case14", "case30", "case57", "case118")}
    with open(os.path.join(HERE, "networks.json"), "w") as fh:
        json.dump({k: net_to_dict(v) for k, v in nets.items()}, fh)
    dump_model("case14", build_acopf(nets["case14"]), rng)
    dump_model("case118", build_acopf(nets["case118"]), rng)
    dump_model("C1", build_acopf(parse_matpower(tiled_case(1))), rng)
    dump_model("T4", build_acopf(parse_matpower(tiled_case(4))), rng)

    e2e = {}

    def run(tag, am, tol, inject, keep_x=False):
        if inject:
            RK.amd_order = _heap_amd
        t = time.perf_counter()
        rep = solve(am.model, SolverOptions(tol=tol), constraint_ranges=am.ranges)
        dt = time.perf_counter() - t
        RK.amd_order = _SHIPPED_AMD
        e2e[f"{tag}@{tol:g}"] = dict(status=rep.status, iterations=rep.iterations,
                                    objective=rep.objective,
                                    violation=rep.constraint_violation,
                                    residual_scaled=rep.residual_scaled,
                                    trace=[list(map(float, t)) for t in rep.trace],
                                    seconds=rep.seconds, wall=dt,
                                    n_var=rep.n_var, n_con=rep.n_con)
        if keep_x:
            np.savez_compressed(os.path.join(HERE, f"{tag}_{tol:g}_x.npz"), x=rep.x)
        print(tag, tol, rep.status, rep.iterations, rep.objective, f"{dt:.2f}s", flush=True)

    for c, net in nets.items():
        for tol in (1e-4, 1e-6):
            run(c, build_acopf(net), tol, inject=False, keep_x=True)
    run("C1", build_acopf(parse_matpower(tiled_case(1))), 1e-6, False, keep_x=True)
    run("C1", build_acopf(parse_matpower(tiled_case(1))), 1e-4, False, keep_x=True)
    run("T16", build_acopf(parse_matpower(tiled_case(16))), 1e-6, True, keep_x=True)
    for seed in (0, 1, 2):
        run(f"C5s{seed}", build_acopf(parse_matpower(tiled_case(97, seed=seed))), 1e-6, True,
            keep_x=(seed == 0))
    run("C2", build_acopf(parse_matpower(tiled_case(143))), 1e-6, True, keep_x=True)
    if os.environ.get("GOLDEN_C3", "1") == "1":
        run("C3", build_acopf(parse_matpower(tiled_case(714))), 1e-6, True, keep_x=True)
    with open(os.path.join(HERE, "end_to_end.json"), "w") as fh:
        json.dump(e2e, fh, indent=1)


if __name__ == "__main__":
    main()
