"""C4 (BASELINE configs[3]): the 78,484-bus synthetic ACOPF (5,606 IEEE-14
tiles, 705,756 variables, 1,019,243 constraints) against the reference.

The golden (tests/golden/end_to_end_C4.json, C4_1e-06_x.npz, C4_perm.npz)
was produced by running the reference's ipm.solve (src/gridnlp/ipm.py:
301-563) on its own build_acopf (src/acopf.py:68) with the heap minimum
degree injected (tests/golden/make_golden_r2.py; the shipped O(n^2) scan
is infeasible at this size).  The same permutation is injected here, so
the solves factor the same pivot sequence; the permutation itself is
checked against our native minimum degree (bit-identical).

Tolerances: status equal, objective <= 1e-6
relative, iterations within +-2, ||x - x_ref||_inf <= 1e-3 (the converged
points of two tol-1e-6 solves differ by O(tol) in the flat directions).
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

import paper_2307_16830_b200 as gp  # noqa: E402
from paper_2307_16830_b200 import kkt, sparse  # noqa: E402
from paper_2307_16830_b200.acopf import build_acopf  # noqa: E402
from paper_2307_16830_b200.grids import tiled_case  # noqa: E402
from paper_2307_16830_b200.matpower import parse_matpower  # noqa: E402


@pytest.fixture(scope="module")
def c4():
    return build_acopf(parse_matpower(tiled_case(5606)))


@pytest.fixture(scope="module")
def c4_perm():
    return np.load(os.path.join(GOLDEN, "C4_perm.npz"))["perm"].astype(np.int64)


def test_c4_ordering_bit_identical(c4, c4_perm):
    m = c4.model
    cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    np.testing.assert_array_equal(sparse.amd_order(cs.matrix), c4_perm)


def test_c4_end_to_end_matches_reference(c4, c4_perm):
    with open(os.path.join(GOLDEN, "end_to_end_C4.json")) as fh:
        ref = json.load(fh)["C4@1e-06"]
    x_ref = np.load(os.path.join(GOLDEN, "C4_1e-06_x.npz"))["x"]
    rep = gp.solve(c4.model, gp.SolverOptions(tol=1e-6, ordering=c4_perm),
                   constraint_ranges=c4.ranges)
    assert rep.status == ref["status"] == "optimal"
    assert rep.objective == pytest.approx(ref["objective"], rel=1e-6)
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert np.max(np.abs(rep.x - x_ref)) <= 1e-3
    # the barrier parameter follows the same schedule while the iterations agree
    for a, b in zip(rep.trace[:10], ref["trace"][:10]):
        assert a[4] == pytest.approx(b[4], rel=1e-12)
