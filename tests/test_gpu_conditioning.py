"""Conditioning diagnostics on the device factor.

* ``sparse.estimate_condition`` (cholesky.py:220-241): Hager's lower
  estimate within a factor of ten of the true 1-norm condition number on
  random SPD matrices (the reference's own bound, test_sparse_linear.py:
  256-267), exact on the identity, bracketing a diagonal spread.
* ``report.diagnose_conditioning`` (src/bench.py:113-135): condensed and
  augmented estimates (and the dense oracle value when small) at the final
  iterate of case14/30/118 against the reference's values
  (tests/golden/conditioning.json, make_golden_r2.py) within a factor of
  ten -- the same bound, since the two solves' final iterates agree only
  to the IPM tolerance and kappa is 1e14..1e18 there.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

from paper_2307_16830_b200 import SolverOptions, solve  # noqa: E402
from paper_2307_16830_b200 import sparse as S  # noqa: E402
from paper_2307_16830_b200.acopf import build_acopf  # noqa: E402
from paper_2307_16830_b200.matpower import network_from_tables  # noqa: E402
from paper_2307_16830_b200.report import SKIPPED_TOO_LARGE, diagnose_conditioning  # noqa: E402


def random_spd(rng, n, density=0.2, shift=1.0):
    A = np.zeros((n, n))
    for _ in range(max(1, int(density * n * n / 2))):
        i, j = rng.integers(0, n, 2)
        A[max(i, j), min(i, j)] = A[min(i, j), max(i, j)] = rng.normal()
    A += np.diag(np.abs(A).sum(axis=1) + shift)
    return A


def factor_of(A):
    ri, ci = np.nonzero(np.tril(A))
    m, _ = S.coo_to_csc(A.shape[0], ri, ci, A[ri, ci])
    f = S.factorize(S.symbolic_cholesky(m, S.amd_order(m)), m.values)
    assert f.ok
    return f, m


def test_condensed_estimate_identity_and_spread():
    f, m = factor_of(np.eye(3))
    assert S.estimate_condition(f, m) == pytest.approx(1.0)
    f, m = factor_of(np.diag([1.0, 1e6]))
    assert 0.5e6 <= S.estimate_condition(f, m) <= 2e6


def test_condensed_estimate_random_spd_within_factor_ten():
    rng = np.random.default_rng(9)
    for _ in range(5):
        A = random_spd(rng, 30, density=0.3)
        f, m = factor_of(A)
        est = S.estimate_condition(f, m)
        true = np.linalg.cond(A, 1)
        assert true / 10.0 <= est <= true * 1.01


@pytest.mark.parametrize("case", ("case14", "case30", "case118"))
def test_diagnose_conditioning_matches_reference(networks_json, case):
    with open(os.path.join(GOLDEN, "conditioning.json")) as fh:
        ref = json.load(fh)[case]
    am = build_acopf(network_from_tables(networks_json[case]))
    rep = solve(am.model, SolverOptions(tol=1e-6, keep_workspace=True), constraint_ranges=am.ranges)
    d = diagnose_conditioning(rep)
    for key in ("condensed_condition", "augmented_condition"):
        assert ref[key] / 10.0 <= d[key] <= ref[key] * 10.0, (key, d[key], ref[key])
    if ref["augmented_condition_dense"] == SKIPPED_TOO_LARGE:
        assert d["augmented_condition_dense"] == SKIPPED_TOO_LARGE
    else:
        r = float(ref["augmented_condition_dense"])
        assert r / 10.0 <= d["augmented_condition_dense"] <= r * 10.0
        # the estimate is a lower bound of the dense value (Hager)
        assert d["augmented_condition"] <= d["augmented_condition_dense"] * 1.01
