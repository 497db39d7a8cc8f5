"""CPU ports of the reference suite's property tests (no GPU needed).

* COO -> lower-CSC conversion: the small-pattern, duplicate, upper-triangle,
  slot-map and hypothesis dense-roundtrip properties of
  pkg/tests/test_sparse_linear.py:46-87, against the native host routine
  behind ``sparse.coo_to_csc`` (gn_coo_to_csc);
* the power-flow oracle (oracle/powerflow.py) pinned against the oracle
  model's constraint evaluation on the four IEEE cases, so the GPU test that
  uses it (tests/test_gpu_reference_suite.py) compares against a checked
  point (pkg/tests/test_autodiff.py:76-83).
"""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import model as OM
from oracle import powerflow as PF
from paper_2307_16830_b200 import sparse as S
from paper_2307_16830_b200.acopf import build_acopf
from paper_2307_16830_b200.matpower import network_from_tables


class TestCooToCsc:
    def test_small_pattern(self):
        m, _ = S.coo_to_csc(2, np.array([0, 1, 1]), np.array([0, 0, 1]), np.array([1.0, 2.0, 3.0]))
        assert m.nnz == 3
        np.testing.assert_array_equal(m.indptr, [0, 2, 3])
        np.testing.assert_array_equal(m.indices, [0, 1, 1])

    def test_duplicates_accumulate(self):
        m, slot = S.coo_to_csc(1, np.array([0, 0]), np.array([0, 0]), np.array([1.0, 2.0]))
        assert m.nnz == 1 and m.values[0] == 3.0
        np.testing.assert_array_equal(slot, [0, 0])

    def test_upper_triangle_rejected(self):
        with pytest.raises(S.UpperTriangleEntry):
            S.coo_to_csc(2, np.array([0]), np.array([1]), np.array([1.0]))

    def test_slot_map_reassembles_values(self):
        rows, cols = np.array([0, 1, 1, 0]), np.array([0, 0, 1, 0])
        vals = np.array([1.0, 2.0, 3.0, 4.0])
        m, slot = S.coo_to_csc(2, rows, cols, vals)
        rebuilt = np.zeros(m.nnz)
        np.add.at(rebuilt, slot, vals)
        np.testing.assert_array_equal(rebuilt, m.values)

    @given(st.integers(1, 8), st.integers(0, 30), st.integers(0, 2 ** 32 - 1))
    @settings(max_examples=60, deadline=None)
    def test_dense_roundtrip(self, n, nnz, seed):
        rng = np.random.default_rng(seed)
        rows = rng.integers(0, n, nnz)
        cols = np.minimum(rows, rng.integers(0, n, nnz))
        vals = rng.normal(size=nnz)
        m, slot = S.coo_to_csc(n, rows, cols, vals)
        want = np.zeros((n, n))
        np.add.at(want, (rows, cols), vals)
        got = np.zeros((n, n))
        r, c = m.coords()
        got[r, c] = m.values
        np.testing.assert_allclose(got, want, atol=1e-14)
        # CSC invariants: sorted strictly increasing rows per column, lower only
        assert m.indptr[0] == 0 and m.indptr[-1] == m.nnz
        for j in range(n):
            col = m.indices[m.indptr[j]:m.indptr[j + 1]]
            assert np.all(np.diff(col) > 0) and np.all(col >= j)
        assert slot.size == nnz and (nnz == 0 or slot.max() < m.nnz)


@pytest.mark.parametrize("tag", ("case14", "case30", "case57", "case118"))
def test_power_flow_oracle_satisfies_equalities(networks_json, tag):
    am = build_acopf(network_from_tables(networks_json[tag]))
    m = am.model
    x = PF.power_flow_point(am.network, am.variables, m.n_var)
    om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
    g = OM.constraints(om, x)
    eq = (am.ranges[:, 0] == 0) & (am.ranges[:, 1] == 0)
    assert eq.sum() > 0
    assert np.max(np.abs(g[eq])) <= 1e-10
