"""Interior-point behaviour on small problems (GPU), after test_ipm_core.py:103-200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402
from paper_2307_16830_b200.expressions import log, param, var  # noqa: E402
from paper_2307_16830_b200.ipm import EVAL_ERROR, LINE_SEARCH_FAILURE, MAX_ITER, OPTIMAL  # noqa: E402
from paper_2307_16830_b200.model import ModelBuilder  # noqa: E402


def box(n, lo=-50.0, hi=50.0, start=0.0):
    b = ModelBuilder()
    b.add_variables(n, np.full(n, lo), np.full(n, hi), np.full(n, start))
    return b


def quadratic_model(n=4):
    b = box(n)
    b.add_objective((var(0) - param(0)) ** 2, np.arange(n).reshape(-1, 1),
                    np.arange(n, dtype=float).reshape(-1, 1))
    return b.finalize()


def eq_model():
    b = box(2, -10, 10, 0.5)
    b.add_objective(var(0) ** 2, np.array([[0], [1]]), np.zeros((2, 0)))
    b.add_constraints(var(0) + var(1) - 2.0, np.array([[0, 1]]), np.zeros((1, 0)))
    return b.finalize()


def test_unconstrained_quadratic():
    rep = solve(quadratic_model(), SolverOptions(tol=1e-6))
    assert rep.status == OPTIMAL and rep.iterations <= 15
    np.testing.assert_allclose(rep.x, np.arange(4.0), atol=1e-4)


def test_equality_constrained():
    rep = solve(eq_model(), SolverOptions(tol=1e-6))
    assert rep.status == OPTIMAL
    np.testing.assert_allclose(rep.x, [1.0, 1.0], atol=1e-4)


def test_infeasible_not_optimal():
    b = box(1, -5, 5, 0.4)
    b.add_constraints(var(0), np.array([[0]]), np.zeros((1, 0)))
    b.add_constraints(var(0) - 1.0, np.array([[0]]), np.zeros((1, 0)))
    rep = solve(b.finalize(), SolverOptions(tol=1e-4, max_iter=150))
    assert rep.status in (LINE_SEARCH_FAILURE, MAX_ITER)


def test_active_bound_and_range():
    b = box(1, -5.0, 1.0)
    b.add_objective((var(0) - 3.0) ** 2, np.array([[0]]), np.zeros((1, 0)))
    rep = solve(b.finalize(), SolverOptions(tol=1e-6))
    assert rep.status == OPTIMAL and rep.x[0] == pytest.approx(1.0, abs=1e-4)
    b = box(1, -20.0, 20.0)
    b.add_objective((var(0) - 5.0) ** 2, np.array([[0]]), np.zeros((1, 0)))
    b.add_constraints(var(0), np.array([[0]]), np.zeros((1, 0)))
    rep = solve(b.finalize(), SolverOptions(tol=1e-6), constraint_ranges=np.array([[-1.0, 2.0]]))
    assert rep.status == OPTIMAL and rep.x[0] == pytest.approx(2.0, abs=1e-3)


def test_eval_error_and_fixed_variable():
    b = box(1, -5.0, 5.0, start=-2.0)
    b.add_objective(log(var(0)), np.array([[0]]), np.zeros((1, 0)))
    assert solve(b.finalize(), SolverOptions(tol=1e-6)).status == EVAL_ERROR
    b = ModelBuilder()
    b.add_variables(2, np.array([-5.0, 2.0]), np.array([5.0, 2.0]), np.array([0.0, 2.0]))
    b.add_objective((var(0) - param(0)) ** 2, np.array([[0], [1]]), np.array([[1.0], [0.0]]))
    rep = solve(b.finalize(), SolverOptions(tol=1e-6))
    assert rep.status == OPTIMAL and rep.x[1] == pytest.approx(2.0, abs=1e-6)


def test_invariants_determinism_mu_alpha_filter():
    r1 = solve(eq_model(), SolverOptions(tol=1e-8))
    r2 = solve(eq_model(), SolverOptions(tol=1e-8))
    assert r1.trace == r2.trace and r1.objective == r2.objective
    mus = [row[4] for row in r1.trace]
    assert all(b <= a for a, b in zip(mus, mus[1:])) and min(mus) >= 1e-8 / 10.0
    assert all(0.0 < row[5] <= 1.0 for row in r1.trace)
    for theta, phi, entries in r1.debug.get("accepted", []):
        for th, ph in entries[:-1]:
            assert theta < th or phi < ph
    sec = r1.seconds
    assert sec["ad"] + sec["linear"] + sec["internal"] <= sec["total"] * 1.001


def nonconvex_model():
    """Concave objective (negative curvature at the start) with one equality:
    the speculative delta_w = 0 factorisation is not positive definite, so
    the inertia correction of kkt.py:424-447 runs inside the solve."""
    b = box(3, -1.0, 2.0, 0.0)
    b.add_objective(-(var(0) - param(0)) ** 2 + 0.5 * var(0) * var(1),
                    np.array([[0, 1], [1, 2], [2, 0]]), np.array([[0.3], [0.1], [-0.2]]))
    b.add_constraints(var(0) + var(1) + var(2) - 1.0, np.array([[0, 1, 2]]), np.zeros((1, 0)))
    return b.finalize()


@pytest.mark.parametrize("tol", (1e-4, 1e-8))
def test_regularization_inside_solve_matches_oracle(tol):
    """delta_w schedule inside the IPM (ipm.py:441-447): every iteration's
    delta_w, the iteration count and the solution equal the oracle's (which
    restates the reference loop with the dense-free condensed backend)."""
    from oracle import ipm as OI
    from oracle import model as OM

    m = nonconvex_model()
    rep = solve(m, SolverOptions(tol=tol))
    om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
    orep = OI.solve(om, m.lower, m.upper, m.start, OI.Options(tol=tol))
    assert rep.status == orep.status
    assert rep.iterations == orep.iterations
    dws = [row[6] for row in rep.trace]
    assert any(dw > 0 for dw in dws), "the correction path was not exercised"
    assert dws == [row[6] for row in orep.trace]
    assert rep.objective == pytest.approx(orep.objective, rel=1e-9, abs=1e-12)
    np.testing.assert_allclose(rep.x, orep.x, atol=1e-7)


@pytest.mark.parametrize("scaling", (True, False))
def test_native_setup_matches_oracle(networks_json, scaling):
    """gn_ipm_setup / gn_ipm_init_slacks vs the oracle's restatement of the
    _Problem scaling, relax_equalities and the initial slacks
    (ipm.py:112-123, 179-193, 371-380): bitwise for the scales, bounds,
    duals and slacks; theta0 (a sum) within 1e-14."""
    import torch

    from oracle import ipm as OI
    from oracle import model as OM
    from paper_2307_16830_b200.acopf import build_acopf
    from paper_2307_16830_b200.matpower import network_from_tables

    am = build_acopf(network_from_tables(networks_json["case118"]))
    m_ = am.model
    opts = SolverOptions(tol=1e-6, max_iter=0, scaling=scaling, keep_workspace=True)
    rep = solve(m_, opts, constraint_ranges=am.ranges)
    P = rep.debug["problem"]
    om = OM.expand(m_.n_var, m_.n_con, OM.from_model(m_))
    xl, xu, x0 = P.xl_h, P.xu_h, P.x0
    n, m = m_.n_var, m_.n_con
    if scaling:
        g0 = OM.gradient(om, x0)
        j0 = OM.jacobian(om, x0)
        gm = np.abs(g0).max()
        osc = min(1.0, 100.0 / gm) if gm > 0 else 1.0
        rmax = np.zeros(m)
        np.maximum.at(rmax, om.jac_rows, np.abs(j0))
        csc = np.ones(m)
        pos = rmax > 0
        csc[pos] = np.minimum(1.0, 100.0 / rmax[pos])
    else:
        osc, csc = 1.0, np.ones(m)
    host = lambda t: t.detach().cpu().numpy()[:m]
    # the scales from device AD values (AD parity is 1e-12, not bitwise)
    assert P.obj_scale == pytest.approx(osc, rel=1e-12)
    np.testing.assert_allclose(host(P.con_scale), csc, rtol=1e-12)
    # the rest bitwise from the device's own scales and g(x0)
    csc_d = host(P.con_scale)
    ranges = np.asarray(am.ranges, float)
    sl, su = OI.relax_equalities(m, np.column_stack([ranges[:, 0] * csc_d, ranges[:, 1] * csc_d]), P.tol_r)
    np.testing.assert_array_equal(host(P.sl), sl)
    np.testing.assert_array_equal(host(P.su), su)
    np.testing.assert_array_equal(P.x.cpu().numpy(), x0)
    np.testing.assert_array_equal(host(P.zsl), np.isfinite(sl).astype(float))
    np.testing.assert_array_equal(P.zxu.cpu().numpy(), np.isfinite(xu).astype(float))
    g = host(P.c)
    s0 = OI.initial_slacks(g, sl, su, P.tol_r, opts.bound_push)
    np.testing.assert_array_equal(host(P.s), s0)
    theta0 = float(P.scal[60].item())
    assert theta0 == pytest.approx(float(np.abs(g - s0).sum()), rel=1e-14)
    torch.cuda.synchronize()


def test_resolve_after_input_changes_matches_fresh_model(networks_json):
    """Cached per-model state (prepared inputs, symbolic plans keyed on the
    ordering's content) is invalidated by changed inputs: re-solving the same
    model object after changing its start point, its ranges, or mutating the
    ordering array in place equals a solve of a freshly built model."""
    from paper_2307_16830_b200 import kkt as K
    from paper_2307_16830_b200 import sparse as S
    from paper_2307_16830_b200.acopf import build_acopf
    from paper_2307_16830_b200.matpower import network_from_tables

    build = lambda: build_acopf(network_from_tables(networks_json["case30"]))
    am = build()
    opts = SolverOptions(tol=1e-6)
    solve(am.model, opts, constraint_ranges=am.ranges)
    rng = np.random.default_rng(5)
    am.model.start[:] = am.model.start + 0.01 * rng.random(am.model.n_var)
    ranges2 = np.array(am.ranges, dtype=float)
    ineq = ranges2[:, 0] != ranges2[:, 1]
    ranges2[ineq] *= 0.9
    r1 = solve(am.model, opts, constraint_ranges=ranges2)
    fresh = build()
    fresh.model.start[:] = am.model.start
    r2 = solve(fresh.model, opts, constraint_ranges=ranges2)
    assert (r1.status, r1.iterations) == (r2.status, r2.iterations)
    assert r1.objective == r2.objective
    np.testing.assert_array_equal(r1.x, r2.x)
    # ordering: the same array object mutated in place is a new ordering
    m_ = am.model
    cs = K.symbolic_condense(m_.hess_rows, m_.hess_cols, m_.jac_rows, m_.jac_cols, m_.n_var)
    perm = S.amd_order(cs.matrix)
    solve(m_, SolverOptions(tol=1e-6, ordering=perm), constraint_ranges=ranges2)
    perm[[0, -1]] = perm[[-1, 0]]
    r3 = solve(m_, SolverOptions(tol=1e-6, ordering=perm), constraint_ranges=ranges2)
    r4 = solve(fresh.model, SolverOptions(tol=1e-6, ordering=perm.copy()), constraint_ranges=ranges2)
    assert (r3.status, r3.iterations) == (r4.status, r4.iterations)
    assert r3.objective == r4.objective
    np.testing.assert_array_equal(r3.x, r4.x)
