"""GPU parity: the CUDA path through the C-ABI vs the oracle / golden vectors.

Tolerances:
* AD values: ||gpu - ref||_inf <= 1e-12 * ||ref||_inf per output array;
* K values: 1e-14 relative (the assembly kernel is FMA-free, usually bitwise);
* factor: ||L_gpu - L_ref||_inf <= 1e-12 * ||L_ref||_inf; solves 1e-10;
* end to end: same status, objective <= 1e-6 relative, iterations +-2.
"""
import numpy as np
import pytest
import torch

from oracle import kkt as OK
from oracle import model as OM
from oracle import sparse as OS

from conftest import MODEL_TAGS, TILES, golden_x
from golden_io import oracle_model

pytestmark = pytest.mark.gpu

import paper_2307_16830_b200 as gp  # noqa: E402
from paper_2307_16830_b200 import autodiff as ad  # noqa: E402
from paper_2307_16830_b200 import kkt as K  # noqa: E402
from paper_2307_16830_b200 import sparse as S  # noqa: E402
from paper_2307_16830_b200.acopf import build_acopf  # noqa: E402
from paper_2307_16830_b200.expressions import cos, log, param, sin, sqrt, var  # noqa: E402
from paper_2307_16830_b200.grids import tiled_case  # noqa: E402
from paper_2307_16830_b200.matpower import network_from_tables, parse_matpower  # noqa: E402
from paper_2307_16830_b200.model import ModelBuilder  # noqa: E402


def normwise(a, b, tol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape
    if not b.size:
        return
    scale = max(float(np.abs(b).max()), 1e-300)
    err = float(np.abs(a - b).max())
    assert err <= tol * scale, f"err {err:.3e} > {tol:.1e} * {scale:.3e}"


def product_model(tag, networks_json):
    if tag.startswith("case"):
        return build_acopf(network_from_tables(networks_json[tag]))
    return build_acopf(parse_matpower(tiled_case(TILES[tag])))


# ---------------------------------------------------------------- AD (a4-a10)
@pytest.mark.parametrize("tag", MODEL_TAGS)
@pytest.mark.parametrize("pt", (0, 1))
def test_ad_matches_reference(golden_models, networks_json, tag, pt):
    g = golden_models[tag]
    m = product_model(tag, networks_json).model
    x, y, w = g[f"ad{pt}_x"], g[f"ad{pt}_y"], float(g[f"ad{pt}_w"])
    assert ad.eval_objective(m, x) == pytest.approx(float(g[f"ad{pt}_f"]), rel=1e-12)
    normwise(ad.eval_constraints(m, x), g[f"ad{pt}_c"], 1e-12)
    normwise(ad.eval_gradient(m, x), g[f"ad{pt}_grad"], 1e-12)
    normwise(ad.eval_jacobian(m, x), g[f"ad{pt}_jac"], 1e-12)
    normwise(ad.eval_lagrangian_hessian(m, x, y, w), g[f"ad{pt}_hess"], 1e-12)


def random_model(rng, n=8):
    """The reference suite's random model (test_autodiff.py:15-27)."""
    b = ModelBuilder()
    b.add_variables(n, np.full(n, -10.0), np.full(n, 10.0), np.zeros(n))
    instr = (param(0) * var(0) ** 2 + param(1) * sin(var(1)) * cos(var(0))
             + param(2) / sqrt(var(1) + 12.0))
    b.add_objective(instr, rng.integers(0, n, (12, 2)), rng.normal(size=(12, 3)))
    b.add_constraints(var(0) * var(1) - param(0) * log(var(2) + 11.0),
                      rng.integers(0, n, (6, 3)), rng.normal(size=(6, 1)))
    b.add_constraint_increments(param(0) * var(0) * var(1), rng.integers(0, n, (9, 2)),
                                rng.normal(size=(9, 1)), rng.integers(0, 6, 9))
    return b.finalize()


def test_generic_interpreter_matches_oracle():
    rng = np.random.default_rng(11)
    for _ in range(10):
        m = random_model(rng)
        om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
        x = rng.uniform(-0.8, 0.8, m.n_var)
        y = rng.normal(size=m.n_con)
        assert ad.eval_objective(m, x) == pytest.approx(OM.objective(om, x), rel=1e-13)
        normwise(ad.eval_constraints(m, x), OM.constraints(om, x), 1e-13)
        normwise(ad.eval_gradient(m, x), OM.gradient(om, x), 1e-13)
        normwise(ad.eval_jacobian(m, x), OM.jacobian(om, x), 1e-13)
        normwise(ad.eval_lagrangian_hessian(m, x, y, 0.7), OM.hessian(om, x, y, 0.7), 1e-13)


def test_known_answers():
    """KATs of test_autodiff.py:30-160."""
    b = ModelBuilder()
    b.add_variables(1, np.array([-5.0]), np.array([5.0]), np.zeros(1))
    b.add_objective(param(0) + param(1) * var(0) + param(2) * var(0) ** 2,
                    np.array([[0]]), np.array([[1.0, 2.0, 3.0]]))
    m = b.finalize()
    assert ad.eval_objective(m, np.array([1.0])) == pytest.approx(6.0)
    assert ad.eval_gradient(m, np.array([1.0]))[0] == pytest.approx(8.0)
    b = ModelBuilder()
    b.add_variables(2, np.full(2, -5.0), np.full(2, 5.0), np.zeros(2))
    b.add_constraints(var(0) * var(1), np.array([[0, 1]]), np.zeros((1, 0)))
    m = b.finalize()
    assert ad.eval_lagrangian_hessian(m, np.zeros(2), np.array([3.0]), 0.0)[0] == pytest.approx(3.0)
    b = ModelBuilder()
    b.add_variables(1, np.array([-5.0]), np.array([5.0]), np.zeros(1))
    b.add_constraints(var(0), np.array([[0]]), np.zeros((1, 0)))
    b.add_constraint_increments(param(0) * var(0), np.array([[0], [0]]),
                                np.array([[2.0], [3.0]]), np.array([0, 0]))
    m = b.finalize()
    assert ad.eval_jacobian(m, np.zeros(1))[0] == pytest.approx(6.0)


def test_nonfinite_raises():
    b = ModelBuilder()
    b.add_variables(1, np.array([-5.0]), np.array([5.0]), np.zeros(1))
    b.add_objective(log(var(0)), np.array([[0]]), np.zeros((1, 0)))
    m = b.finalize()
    with pytest.raises(ad.NonFiniteResult):
        ad.eval_objective(m, np.array([-1.0]))
    with pytest.raises(ad.NonFiniteResult):
        ad.eval_gradient(m, np.array([0.0]))


def test_record_order_bitwise_and_buffers():
    rng = np.random.default_rng(17)
    m = random_model(rng)
    buf = ad.DerivativeBuffers(m)
    x = rng.uniform(-0.5, 0.5, m.n_var)
    assert ad.eval_gradient(m, x, out=buf.gradient) is buf.gradient
    assert ad.eval_jacobian(m, x, out=buf.jacobian_values) is buf.jacobian_values
    h1 = ad.eval_lagrangian_hessian(m, x, np.ones(m.n_con), 1.0, out=buf.hessian_values)
    assert h1 is buf.hessian_values
    h2 = ad.eval_lagrangian_hessian(m, x, np.ones(m.n_con), 1.0)
    np.testing.assert_array_equal(h1, h2)   # deterministic gathers


# ------------------------------------------------------ KKT (a11-a18)
def _ws(g):
    n, m = int(g["n"]), int(g["m"])
    ws = K.KKTWorkspace(n, m, g["hess_rows"], g["hess_cols"], g["jac_rows"], g["jac_cols"])
    ws.set_iterate(*(g["ws_" + f] for f in ("w_vals", "a_vals", "dxl", "dxu", "zxl", "zxu",
                                             "dsl", "dsu", "zsl", "zsu")))
    ws.delta_w, ws.delta_c = float(g["ws_delta_w"]), float(g["ws_delta_c"])
    return ws


def _sp_lower(n, colptr, rowidx, vals):
    import scipy.sparse as sp

    return sp.csc_matrix((vals, rowidx, colptr), shape=(n, n))


def factor_residual(g, lvals):
    """||P K P^T - L L^T||_max / ||K||_max with L in the reference CSC layout."""
    n = int(g["n"])
    Kl = _sp_lower(n, g["cond_indptr"], g["cond_indices"], g["K_vals"])
    Kf = (Kl + Kl.T - __import__("scipy.sparse").sparse.diags(Kl.diagonal())).tocsr()
    p = g["sym_perm"]
    PKP = Kf[p][:, p]
    Lm = _sp_lower(n, g["sym_l_colptr"], g["sym_l_rowidx"], lvals)
    R = (PKP - Lm @ Lm.T).tocoo()
    return (np.abs(R.data).max() if R.nnz else 0.0) / np.abs(Kf.data).max(), Kf


@pytest.mark.parametrize("tag", MODEL_TAGS)
def test_assembly_factor_solve_match_reference(golden_models, tag):
    g = golden_models[tag]
    ws = _ws(g)
    normwise(ws.sigma_x.cpu().numpy(), g["ws_sigma_x"], 1e-15)
    back = K.CondensedBackend(ws, ordering=g["sym_perm"])
    assert back.try_factorize()
    np.testing.assert_array_equal(back.kvals.cpu().numpy(), g["K_vals"])   # FMA-free: bitwise
    lv = back.factor.values
    ours, Kf = factor_residual(g, lv)
    theirs, _ = factor_residual(g, g["L_vals"])
    assert ours <= 1e-12 and ours <= 10 * max(theirs, 1e-16)
    b = g["solve_b"]
    x = S.solve(back.factor, b)
    bwd = lambda z: np.abs(Kf @ z - b).max() / (np.abs(Kf).max() * np.abs(z).max() + np.abs(b).max())
    assert bwd(x) <= 1e-13 and bwd(x) <= 10 * max(bwd(g["solve_x"]), 1e-17)
    pv = K.PVec(*(g["pv_" + f] for f in K.FIELDS))
    qx, qs, qy = ws.condense_pvec(pv)
    normwise(qx.cpu().numpy(), g["q_x"], 1e-15)
    normwise(ws.condensed_rhs(qx, qs, qy).cpu().numpy(), g["rhs"], 1e-14)
    dx, ds, dy = back.solve3(qx, qs, qy)
    st = K.assemble_steps(ws, pv, dx, ds, dy)
    # seven-block residual of our steps vs the reference's own steps (same oracle)
    ows = OK.OWorkspace(int(g["n"]), int(g["m"]), g["hess_rows"], g["hess_cols"],
                        g["jac_rows"], g["jac_cols"])
    ows.set_iterate(*(g["ws_" + f] for f in ("w_vals", "a_vals", "dxl", "dxu", "zxl", "zxu",
                                              "dsl", "dsu", "zsl", "zsu")))
    ows.dw, ows.dc = ws.delta_w, ws.delta_c
    opv = OK.Vec7(*(g["pv_" + f] for f in K.FIELDS))
    ours = OK.residual_norm(ows.residual_full(OK.Vec7(*st.numpy()), opv))
    ref = OK.residual_norm(ows.residual_full(OK.Vec7(
        g["s3_dx"], g["s3_ds"], g["s3_dy"], g["st_zxl"], g["st_zxu"], g["st_zsl"], g["st_zsu"]), opv))
    assert ours <= 1e-6 * float(g["matrix_scale"]) and ours <= 100 * max(ref, 1e-300)
    assert ws.matrix_scale() == float(g["matrix_scale"])


def test_residual_double_double_matches_longdouble(golden_models):
    """The seven-block residual of the reference steps, dd vs np.longdouble."""
    g = golden_models["T4"]
    ws = _ws(g)
    ows = OK.OWorkspace(int(g["n"]), int(g["m"]), g["hess_rows"], g["hess_cols"],
                        g["jac_rows"], g["jac_cols"])
    ows.set_iterate(*(g["ws_" + f] for f in ("w_vals", "a_vals", "dxl", "dxu", "zxl", "zxu",
                                              "dsl", "dsu", "zsl", "zsu")))
    ows.dw, ows.dc = ws.delta_w, ws.delta_c
    pv = K.PVec(*(g["pv_" + f] for f in K.FIELDS))
    opv = OK.Vec7(*(g["pv_" + f] for f in K.FIELDS))
    steps = OK.Vec7(g["s3_dx"], g["s3_ds"], g["s3_dy"], g["st_zxl"], g["st_zxu"], g["st_zsl"],
                    g["st_zsu"])
    dsteps = K.Steps(*steps.parts())
    ref = ows.residual_full(steps, opv)
    got = ws.residual_full(dsteps, pv)
    # both accumulate in > 53-bit precision: they agree to well below one
    # double ulp of the largest term of M * steps
    terms = float(g["matrix_scale"]) * max(float(np.abs(a).max()) for a in steps.parts())
    for f in K.FIELDS:
        r = getattr(ref, f).astype(float)
        scale = terms + float(np.abs(getattr(opv, f)).max())
        assert float(np.abs(getattr(got, f).cpu().numpy() - r).max()) <= 2e-16 * scale


def test_hand_factor_and_failing_column():
    m, _ = S.coo_to_csc(2, np.array([0, 1, 1]), np.array([0, 0, 1]), np.array([2.0, 1.0, 2.0]))
    f = S.factorize(S.symbolic_cholesky(m, np.arange(2)), m.values)
    assert f.ok
    np.testing.assert_allclose(f.values, [np.sqrt(2.0), 1.0 / np.sqrt(2.0), np.sqrt(1.5)])
    np.testing.assert_allclose(S.solve(f, np.array([3.0, 3.0])), [1.0, 1.0])
    m, _ = S.coo_to_csc(2, np.array([0, 1, 1]), np.array([0, 0, 1]), np.array([1.0, 2.0, 1.0]))
    f = S.factorize(S.symbolic_cholesky(m, np.arange(2)), m.values)
    assert not f.ok and f.failing_column == 1


def random_spd(rng, n, density=0.2, shift=1.0):
    A = np.zeros((n, n))
    for _ in range(max(1, int(density * n * n / 2))):
        i, j = rng.integers(0, n, 2)
        A[i, j] = A[j, i] = rng.normal()
    A += np.diag(np.abs(A).sum(axis=1) + shift)
    return A


def to_sparse(A):
    ri, ci = np.nonzero(np.tril(A))
    return S.coo_to_csc(A.shape[0], ri, ci, A[ri, ci])[0]


def test_pd_detection_agrees_with_eigenvalues_and_oracle():
    rng = np.random.default_rng(4)
    trials = 0
    while trials < 100:
        n = int(rng.integers(2, 21))
        A = random_spd(rng, n, density=0.4, shift=0.5)
        if rng.random() < 0.5:
            A -= (np.abs(np.linalg.eigvalsh(A)).max() * rng.uniform(0.2, 1.5)) * np.eye(n)
        eig = np.linalg.eigvalsh(A)
        if np.min(np.abs(eig)) < 1e-8:
            continue
        trials += 1
        m = to_sparse(A)
        perm = S.amd_order(m)
        f = S.factorize(S.symbolic_cholesky(m, perm), m.values)
        assert f.ok == bool(eig.min() > 0)
        om, _ = OS.coo_to_csc(n, *m.coords(), m.values)
        _, ok, bad = OS.factorize(OS.symbolic(om, perm), om.values)
        assert ok == f.ok
        if not ok:
            assert f.failing_column == bad


def test_refactor_bitwise_and_solve_residual():
    rng = np.random.default_rng(6)
    A = random_spd(rng, 50)
    m = to_sparse(A)
    sym = S.symbolic_cholesky(m, S.amd_order(m))
    f1 = S.factorize(sym, m.values).values
    f2 = S.factorize(sym, m.values).values
    assert np.array_equal(f1, f2)
    f = S.factorize(sym, m.values)
    for _ in range(10):
        b = rng.normal(size=50)
        x = S.solve(f, b)
        assert np.max(np.abs(A @ x - b)) / np.max(np.abs(b)) <= 1e-10


def test_condensation_equivalence_random_instances():
    """100 random KKT instances vs the dense augmented oracle (test_kkt_condensed.py:280-296)."""
    rng = np.random.default_rng(100)
    for _ in range(100):
        n = int(rng.integers(1, 9))
        m = int(rng.integers(0, 6))
        W = rng.normal(size=(n, n))
        W = (W + W.T) / 2 + 2.5 * np.eye(n) * (rng.random() < 0.5)
        hr, hc = np.tril_indices(n)
        keep = (rng.random(hr.size) < 0.8) | (hr == hc)
        hr, hc = hr[keep], hc[keep]
        A = rng.normal(size=(m, n)) * (rng.random((m, n)) < 0.7)
        jr, jc = np.nonzero(A)
        widths = lambda k, inf: np.where(rng.random(k) < (0.3 if inf else 0), np.inf,
                                         rng.uniform(0.05, 2.0, k))
        dxl, dxu, dsl, dsu = widths(n, True), widths(n, True), widths(m, False), widths(m, False)
        duals = lambda w: np.where(np.isfinite(w), rng.uniform(0.1, 3.0, w.size), 0.0)
        args = (W[hr, hc], A[jr, jc], dxl, dxu, duals(dxl), duals(dxu), dsl, dsu, duals(dsl), duals(dsu))
        pv_np = [rng.normal(size=k) for k in (n, m, m)] + [
            np.where(np.isfinite(dxl), rng.normal(size=n), 0.0),
            np.where(np.isfinite(dxu), rng.normal(size=n), 0.0),
            rng.normal(size=m), rng.normal(size=m)]
        ows = OK.OWorkspace(n, m, hr, hc, jr, jc)
        ows.set_iterate(*args)
        oback = OK.OCondensedBackend(ows)
        (odx, ods, ody), odw = OK.solve_with_regularization(ows, oback, OK.Vec7(*pv_np), OK.RegState())
        ws = K.KKTWorkspace(n, m, hr, hc, jr, jc)
        ws.set_iterate(*args)
        back = K.CondensedBackend(ws)
        (dx, ds, dy), dw = K.solve_with_regularization(ws, back, K.PVec(*pv_np), K.RegState())
        assert dw == odw
        for got, ref in ((dx, odx), (ds, ods), (dy, ody)):
            assert np.max(np.abs(got.cpu().numpy() - ref), initial=0.0) <= 1e-9


# --------------------------------------------------------- end to end (a23)
@pytest.mark.parametrize("case,tol", [("case14", 1e-4), ("case14", 1e-6), ("case30", 1e-4),
                                      ("case30", 1e-6), ("case57", 1e-4), ("case57", 1e-6),
                                      ("case118", 1e-4), ("case118", 1e-6)])
def test_end_to_end_ieee_cases(networks_json, end_to_end, case, tol):
    am = build_acopf(network_from_tables(networks_json[case]))
    rep = gp.solve(am.model, gp.SolverOptions(tol=tol), constraint_ranges=am.ranges)
    ref = end_to_end[f"{case}@{tol:g}"]
    assert rep.status == ref["status"] == "optimal"
    assert rep.objective == pytest.approx(ref["objective"], rel=1e-6)
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert np.max(np.abs(rep.x - golden_x(case, tol))) <= 1e-3


@pytest.mark.parametrize("tag,tiles,seed", [("C1", 1, None), ("T16", 16, None), ("C5s0", 97, 0),
                                            ("C5s1", 97, 1), ("C5s2", 97, 2), ("C2", 143, None)])
def test_end_to_end_synthetic(end_to_end, tag, tiles, seed):
    am = build_acopf(parse_matpower(tiled_case(tiles, seed=seed)))
    rep = gp.solve(am.model, gp.SolverOptions(tol=1e-6), constraint_ranges=am.ranges)
    ref = end_to_end[f"{tag}@1e-06"]
    assert rep.status == ref["status"] == "optimal"
    assert rep.objective == pytest.approx(ref["objective"], rel=1e-6)
    assert abs(rep.iterations - ref["iterations"]) <= 2


def test_end_to_end_matches_oracle_trace_closely(golden_models):
    g = golden_models["C1"]
    am = build_acopf(parse_matpower(tiled_case(1)))
    rep = gp.solve(am.model, gp.SolverOptions(tol=1e-6), constraint_ranges=am.ranges)
    from oracle import ipm as OI

    orep = OI.solve(oracle_model(g), g["lower"], g["upper"], g["start"], OI.Options(tol=1e-6),
                    g["ranges"])
    assert rep.iterations == orep.iterations
    for a, b in zip(rep.trace, orep.trace):
        assert a[1] == pytest.approx(b[1], rel=1e-5)   # objective per iteration
        assert a[4] == b[4]                              # same barrier sequence


def test_generated_pattern_kernels_match_interpreter():
    """The NVRTC pattern kernels (one straight-line function per pattern tape)
    against the generic tape interpreter and the oracle, on C1 and case118."""
    import os

    for tag in ("C1", "T4"):
        tiles = TILES[tag]
        outs = {}
        for mode in ("interp", "patterns"):
            if mode == "interp":
                os.environ["GN_AD_INTERPRETER"] = "1"
            m = build_acopf(parse_matpower(tiled_case(tiles))).model
            try:
                backend = ad.ad_backend(m)
            finally:
                os.environ.pop("GN_AD_INTERPRETER", None)
            assert backend.startswith("patterns" if mode == "patterns" else "interpreter"), backend
            rng = np.random.default_rng(3)
            x = m.start + 0.01 * rng.standard_normal(m.n_var)
            yv = rng.standard_normal(m.n_con)
            outs[mode] = (ad.eval_objective(m, x), ad.eval_constraints(m, x), ad.eval_gradient(m, x),
                          ad.eval_jacobian(m, x), ad.eval_lagrangian_hessian(m, x, yv, 0.7))
        om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
        ref = (OM.objective(om, x), OM.constraints(om, x), OM.gradient(om, x), OM.jacobian(om, x),
               OM.hessian(om, x, yv, 0.7))
        for a, b, r in zip(outs["patterns"], outs["interp"], ref):
            a, b, r = np.atleast_1d(a), np.atleast_1d(b), np.atleast_1d(r)
            scale = max(1.0, np.max(np.abs(r)))
            assert np.max(np.abs(a - b)) <= 1e-14 * scale
            assert np.max(np.abs(a - r)) <= 1e-12 * scale


@pytest.mark.gpu
def test_long_tape_runs_on_generated_kernels():
    """Tapes beyond the interpreter's 64 entries (the reference tape has no
    cap, expressions.py:147-219) run on the generated pattern kernels and
    match the oracle; with the interpreter forced, model upload fails loudly
    instead of truncating."""
    import os

    from paper_2307_16830_b200 import ModelBuilder
    from paper_2307_16830_b200.expressions import cos, param, sin, var

    k = 24   # ~150 tape entries: sum_k p_k sin(x0 p_k + x1) cos(x2 - p_k)
    expr = None
    for j in range(k):
        t = param(j) * sin(var(0) * param(j) + var(1)) * cos(var(2) - param(j))
        expr = t if expr is None else expr + t
    rng = np.random.default_rng(5)
    R, n = 40, 6
    vi = np.stack([rng.choice(n, 3, replace=False) for _ in range(R)])
    pa = rng.uniform(0.2, 1.5, (R, k))

    def build():
        b = ModelBuilder()
        b.add_variables(n, -np.ones(n) * 3, np.ones(n) * 3, np.zeros(n))
        b.add_objective(expr, vi, pa)
        b.add_constraints(expr, vi, pa)
        return b.finalize()

    m = build()
    assert len(m.pattern_blocks[0].tape.ops) > 64
    x = rng.uniform(-1, 1, n)
    yv = rng.standard_normal(m.n_con)
    om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
    got = (ad.eval_objective(m, x), ad.eval_constraints(m, x), ad.eval_gradient(m, x),
           ad.eval_jacobian(m, x), ad.eval_lagrangian_hessian(m, x, yv, 0.7))
    ref = (OM.objective(om, x), OM.constraints(om, x), OM.gradient(om, x), OM.jacobian(om, x),
           OM.hessian(om, x, yv, 0.7))
    for a, r in zip(got, ref):
        a, r = np.atleast_1d(a), np.atleast_1d(r)
        assert np.max(np.abs(a - r)) <= 1e-12 * max(1.0, np.max(np.abs(r)))
    os.environ["GN_AD_INTERPRETER"] = "1"
    try:
        m2 = build()
        with pytest.raises(Exception, match="interpreter"):
            ad.eval_gradient(m2, x)
    finally:
        os.environ.pop("GN_AD_INTERPRETER", None)
