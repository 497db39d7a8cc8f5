"""GPU ports of the reference suite's behavioural tests, through the C-ABI.

* objective of case14 against a symbolic (sympy) sum of generator costs
  (pkg/tests/test_autodiff.py:48-60);
* the constraint tape at a converged Newton power-flow point
  (pkg/tests/test_autodiff.py:76-83; oracle/powerflow.py, pinned in
  tests/test_reference_suite.py);
* finite-difference checks of the gradient, Jacobian and Lagrangian Hessian
  of the random model (pkg/tests/test_autodiff.py:102-140), zero-weight and
  multiplier-linearity properties of the Hessian (:160-185);
* Sylvester equivalence: the device factorisation of the condensed matrix
  succeeds iff the augmented KKT matrix has inertia (n+m, 0, m)
  (pkg/tests/test_kkt_condensed.py:298-314);
* iterative refinement behaviour (pkg/tests/test_kkt_condensed.py:318-352):
  consistent steps need at most one round, a perturbed step is recovered by
  six orders of magnitude, and refinement never refactorises.
"""
import numpy as np
import pytest
import torch

from oracle import powerflow as PF

from test_gpu_parity import product_model, random_model

pytestmark = pytest.mark.gpu

from paper_2307_16830_b200 import autodiff as ad  # noqa: E402
from paper_2307_16830_b200 import kkt as K  # noqa: E402


# ------------------------------------------------------------------ AD
def test_case14_objective_against_sympy(networks_json):
    sympy = pytest.importorskip("sympy")
    am = product_model("case14", networks_json)
    x = am.model.start
    pg = sympy.Symbol("pg")
    base = am.network.base_mva
    total = sympy.Integer(0)
    for gi, g in enumerate(am.network.generators):
        cost = g.cost[0] * base ** 2 * pg ** 2 + g.cost[1] * base * pg + g.cost[2]
        total += cost.subs(pg, sympy.Float(float(x[am.variables.pg[gi]]), 30))
    assert ad.eval_objective(am.model, x) == pytest.approx(float(total), rel=1e-12)


@pytest.mark.parametrize("tag", ("case14", "case30", "case57", "case118"))
def test_power_flow_point_satisfies_equalities(networks_json, tag):
    am = product_model(tag, networks_json)
    x = PF.power_flow_point(am.network, am.variables, am.model.n_var)
    g = ad.eval_constraints(am.model, x)
    eq = (am.ranges[:, 0] == 0) & (am.ranges[:, 1] == 0)
    assert np.max(np.abs(g[eq])) <= 1e-8


def _central(f, x, h):
    cols = []
    for j in range(x.size):
        e = np.zeros_like(x)
        e[j] = h
        cols.append((np.asarray(f(x + e), float) - np.asarray(f(x - e), float)) / (2 * h))
    return np.stack(cols, axis=-1)


def _dense(rows, cols, vals, shape, symmetric=False):
    out = np.zeros(shape)
    np.add.at(out, (rows, cols), vals)
    if symmetric:
        off = rows != cols
        np.add.at(out, (cols[off], rows[off]), vals[off])
    return out


def test_random_model_gradient_matches_fd():
    rng = np.random.default_rng(11)
    m = random_model(rng)
    for _ in range(5):
        x = rng.uniform(-0.8, 0.8, m.n_var)
        gf = _central(lambda z: ad.eval_objective(m, z), x, 1e-6)
        np.testing.assert_allclose(ad.eval_gradient(m, x), gf, rtol=1e-6, atol=1e-7)


def test_random_model_jacobian_matches_fd():
    rng = np.random.default_rng(12)
    m = random_model(rng)
    for _ in range(5):
        x = rng.uniform(-0.8, 0.8, m.n_var)
        J = _dense(m.jac_rows, m.jac_cols, ad.eval_jacobian(m, x), (m.n_con, m.n_var))
        Jf = _central(lambda z: ad.eval_constraints(m, z), x, 1e-6)
        np.testing.assert_allclose(J, Jf, rtol=1e-6, atol=1e-7)


def test_random_model_hessian_matches_fd():
    """Lagrangian Hessian vs central differences of w*grad f + J^T y."""
    rng = np.random.default_rng(15)
    m = random_model(rng)
    for _ in range(3):
        x = rng.uniform(-0.6, 0.6, m.n_var)
        y = rng.normal(size=m.n_con)
        w = 0.7

        def grad_l(z):
            J = _dense(m.jac_rows, m.jac_cols, ad.eval_jacobian(m, z), (m.n_con, m.n_var))
            return w * ad.eval_gradient(m, z) + J.T @ y

        H = _dense(m.hess_rows, m.hess_cols, ad.eval_lagrangian_hessian(m, x, y, w),
                   (m.n_var, m.n_var), symmetric=True)
        Hf = _central(grad_l, x, 1e-5)
        np.testing.assert_allclose(H, (Hf + Hf.T) / 2, rtol=1e-5, atol=1e-6)


def test_hessian_zero_weights_and_multiplier_linearity():
    rng = np.random.default_rng(14)
    m = random_model(rng)
    x = rng.uniform(-0.5, 0.5, m.n_var)
    assert np.all(ad.eval_lagrangian_hessian(m, x, np.zeros(m.n_con), 0.0) == 0.0)
    y1, y2 = rng.normal(size=m.n_con), rng.normal(size=m.n_con)
    h = lambda y, w: ad.eval_lagrangian_hessian(m, x, y, w)
    np.testing.assert_allclose(h(y1 + 2.0 * y2, 0.7), h(y1, 0.7) + 2.0 * h(y2, 0.0),
                               rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ KKT
def random_instance(rng, n=None, m=None):
    """Random interior KKT instance (the suite's random_kkt_instance)."""
    n = int(rng.integers(1, 9)) if n is None else n
    m = int(rng.integers(0, 6)) if m is None else m
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
    zxl, zxu, zsl, zsu = duals(dxl), duals(dxu), duals(dsl), duals(dsu)
    ws = K.KKTWorkspace(n, m, hr, hc, jr, jc)
    ws.set_iterate(W[hr, hc], A[jr, jc], dxl, dxu, zxl, zxu, dsl, dsu, zsl, zsu)
    pv = K.PVec(rng.normal(size=n), rng.normal(size=m), rng.normal(size=m),
                np.where(np.isfinite(dxl), rng.normal(size=n), 0.0),
                np.where(np.isfinite(dxu), rng.normal(size=n), 0.0),
                rng.normal(size=m), rng.normal(size=m))
    inv = lambda d: np.where(np.isfinite(d), 1.0 / d, 0.0)
    dense = dict(W=_dense(hr, hc, W[hr, hc], (n, n), symmetric=True), A=A,
                 sx=zxl * inv(dxl) + zxu * inv(dxu), ss=zsl * inv(dsl) + zsu * inv(dsu))
    return ws, pv, dense


def augmented(d, n, m, dw, dc):
    """[[W+Sx+dw, 0, A^T], [0, Ss+dw, -I], [A, -I, -dc]] (the bound blocks
    eliminated exactly as in the seven-block residual)."""
    M = np.zeros((n + 2 * m, n + 2 * m))
    M[:n, :n] = d["W"] + np.diag(d["sx"] + dw)
    M[n:n + m, n:n + m] = np.diag(d["ss"] + dw)
    M[:n, n + m:] = d["A"].T
    M[n + m:, :n] = d["A"]
    M[n:n + m, n + m:] = M[n + m:, n:n + m] = -np.eye(m)
    M[n + m:, n + m:] = -dc * np.eye(m)
    return M


def test_sylvester_equivalence():
    rng = np.random.default_rng(200)
    checked = agree_pd = 0
    while checked < 100:
        ws, _, d = random_instance(rng)
        back = K.CondensedBackend(ws)
        dw = float(rng.choice([0.0, 1e-3, 0.1]))
        dc = float(rng.choice([0.0, 1e-8]))
        eig = np.linalg.eigvalsh(augmented(d, ws.n, ws.m, dw, dc))
        if np.min(np.abs(eig)) < 1e-8:
            continue
        checked += 1
        ws.delta_w, ws.delta_c = dw, dc
        inertia = (int((eig > 0).sum()), 0, int((eig < 0).sum()))
        ok = back.try_factorize()
        assert ok == (inertia == (ws.n + ws.m, 0, ws.m)), (ws.n, ws.m, dw, dc, inertia)
        agree_pd += ok
    assert 0 < agree_pd < 100   # both outcomes exercised


def _solved(seed, n, m):
    rng = np.random.default_rng(seed)
    ws, pv, _ = random_instance(rng, n=n, m=m)
    back = K.CondensedBackend(ws)
    (dx, ds, dy), _ = K.solve_with_regularization(ws, back, pv, K.RegState())
    return rng, ws, back, pv, K.assemble_steps(ws, pv, dx, ds, dy)


def test_consistent_steps_need_no_rounds():
    _, ws, back, pv, steps = _solved(30, 4, 2)
    stats = K.iterative_refinement(ws, back, steps, pv)
    assert stats.rounds <= 1
    assert stats.final_residual <= 20 * np.finfo(float).eps * stats.scale


def test_perturbed_step_recovers():
    rng, ws, back, pv, steps = _solved(31, 6, 4)
    steps.x += torch.as_tensor(1e-3 * rng.normal(size=6), device=steps.x.device)
    r0 = K.residual_norm(ws.residual_full(steps, pv))
    stats = K.iterative_refinement(ws, back, steps, pv)
    assert stats.final_residual <= r0 / 1e6


def test_refinement_never_refactorises():
    _, ws, back, pv, steps = _solved(32, 5, 3)
    count = back.n_factorizations
    steps.x += 1e-4
    stats = K.iterative_refinement(ws, back, steps, pv)
    assert stats.rounds >= 1
    assert back.n_factorizations == count
