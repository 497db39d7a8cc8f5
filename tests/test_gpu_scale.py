"""Parity and size-independent properties at the headline size (C3: 9,996
buses, 89,748 variables, 129,571 constraints).

* End to end against the reference itself (tests/golden/end_to_end.json +
  C3_1e-06_x.npz, produced by tests/golden/make_golden.py): status,
  objective (rel 1e-6), iteration count (exact here, +-2 allowed by the
  contract), the per-iteration objective / barrier trace, and x.
* Determinism: two solves give bitwise-identical iterates and factors.
* Linearity of the Lagrangian Hessian in the multipliers (1e-12).
* The refactorisation solves the assembled K (residual 1e-10) and two
  refactorisations of the same values are bitwise identical.
"""
import numpy as np
import pytest

from conftest import golden_x

pytestmark = pytest.mark.gpu

import paper_2307_16830_b200 as gp  # noqa: E402
from paper_2307_16830_b200 import autodiff as ad  # noqa: E402
from paper_2307_16830_b200 import sparse as S  # noqa: E402
from paper_2307_16830_b200.acopf import build_acopf  # noqa: E402
from paper_2307_16830_b200.grids import tiled_case  # noqa: E402
from paper_2307_16830_b200.matpower import parse_matpower  # noqa: E402


@pytest.fixture(scope="module")
def c3():
    return build_acopf(parse_matpower(tiled_case(714)))


def test_c3_end_to_end_matches_reference(c3, end_to_end):
    ref = end_to_end["C3@1e-06"]
    rep = gp.solve(c3.model, gp.SolverOptions(tol=1e-6), constraint_ranges=c3.ranges)
    assert rep.status == ref["status"] == "optimal"
    assert rep.objective == pytest.approx(ref["objective"], rel=1e-6)
    assert rep.iterations == ref["iterations"]
    for a, b in zip(rep.trace, ref["trace"]):
        assert a[1] == pytest.approx(b[1], rel=1e-5)   # objective per iteration
        assert a[4] == pytest.approx(b[4], rel=1e-12)   # barrier parameter sequence
    assert np.max(np.abs(rep.x - golden_x("C3", 1e-6))) <= 1e-4
    # determinism of the whole GPU solve
    rep2 = gp.solve(c3.model, gp.SolverOptions(tol=1e-6), constraint_ranges=c3.ranges)
    np.testing.assert_array_equal(rep.x, rep2.x)


def test_c3_hessian_linear_in_multipliers(c3):
    m = c3.model
    rng = np.random.default_rng(0)
    x = m.start + 0.01 * rng.standard_normal(m.n_var)
    y1, y2 = rng.standard_normal(m.n_con), rng.standard_normal(m.n_con)
    h12 = ad.eval_lagrangian_hessian(m, x, y1 + y2, 0.5)
    h1 = ad.eval_lagrangian_hessian(m, x, y1, 0.0)
    h2 = ad.eval_lagrangian_hessian(m, x, y2, 0.5)
    assert np.max(np.abs(h12 - (h1 + h2))) <= 1e-12 * np.max(np.abs(h12))


def test_c3_refactor_bitwise_and_solve_residual(c3):
    import scipy.sparse as sp

    rep = gp.solve(c3.model, gp.SolverOptions(tol=1e-6, max_iter=5, keep_workspace=True),
                   constraint_ranges=c3.ranges)
    be = rep.debug["backend"]
    be.assemble()
    f1 = S.factorize_device(be.symbolic, be.kvals)
    assert f1.ok
    l1 = f1.values
    l2 = S.factorize_device(be.symbolic, be.kvals).values
    np.testing.assert_array_equal(l1, l2)
    mat = be.structure.matrix
    kv = be.kvals.cpu().numpy()
    n = mat.n
    r, c = mat.coords()
    Kl = sp.csc_matrix((kv, (r, c)), shape=(n, n))
    K = Kl + Kl.T - sp.diags(Kl.diagonal())
    b = np.random.default_rng(1).standard_normal(n)
    xs = S.solve(f1, b)
    # the condensed matrix is badly conditioned; the residual is relative to
    # |K| |x| (componentwise backward error)
    res = np.abs(K @ xs - b)
    scale = np.abs(K) @ np.abs(xs) + np.abs(b)
    assert np.max(res / scale) <= 1e-10
