"""Pin the CPU oracle against the reference's own outputs (golden vectors).

The golden files were produced by running the reference package gridnlp
0.1.0 (tests/golden/make_golden.py).  The oracle restates the reference
algorithm with the same floating-point operation order, so integer arrays
must match bit for bit and most float arrays too; the remaining float
checks use 1e-14-relative tolerances.
"""
import numpy as np
import pytest

from oracle import kkt as OK
from oracle import model as OM
from oracle import ipm as OI
from oracle import sparse as OS
from oracle import tape as OT
from oracle.ordering import min_degree_order

from conftest import MODEL_TAGS, golden_x
from golden_io import oracle_blocks, oracle_model


def rel_close(a, b, tol):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(1.0, float(np.abs(b).max())) if b.size else 1.0
    assert a.shape == b.shape
    assert float(np.abs(a - b).max() if a.size else 0.0) <= tol * scale


@pytest.mark.parametrize("tag", MODEL_TAGS)
def test_template_and_expansion_bitexact(golden_models, tag):
    g = golden_models[tag]
    blocks = oracle_blocks(g)
    for b in blocks:
        fs, sp = OT.template(b.ops, b.consts, b.out)
        assert fs == b.first_slots and sp == b.second_pairs
    om = OM.expand(int(g["n"]), int(g["m"]), blocks)
    for f in ("jac_rows", "jac_cols", "hess_rows", "hess_cols"):
        np.testing.assert_array_equal(getattr(om, f), g[f])
    for bi, b in enumerate(om.blocks):
        for k, a in enumerate(b.jac_slots):
            np.testing.assert_array_equal(a, g[f"b{bi}_jac_slots{k}"])
        for k, a in enumerate(b.hess_slots):
            np.testing.assert_array_equal(a, g[f"b{bi}_hess_slots{k}"])
            np.testing.assert_array_equal(b.hess_factor[k], g[f"b{bi}_hess_factor{k}"])


@pytest.mark.parametrize("tag", MODEL_TAGS)
def test_canonical_order_is_fixed_point(golden_models, tag):
    g = golden_models[tag]
    for b in oracle_blocks(g):
        order = OM.canonical_order(b.var_idx, b.params, b.targets)
        np.testing.assert_array_equal(order, np.arange(b.n))


@pytest.mark.parametrize("tag", MODEL_TAGS)
@pytest.mark.parametrize("pt", (0, 1))
def test_ad_values(golden_models, tag, pt):
    g = golden_models[tag]
    om = oracle_model(g)
    x, y, w = g[f"ad{pt}_x"], g[f"ad{pt}_y"], float(g[f"ad{pt}_w"])
    assert OM.objective(om, x) == pytest.approx(float(g[f"ad{pt}_f"]), rel=1e-14)
    rel_close(OM.constraints(om, x), g[f"ad{pt}_c"], 1e-15)
    rel_close(OM.gradient(om, x), g[f"ad{pt}_grad"], 1e-15)
    rel_close(OM.jacobian(om, x), g[f"ad{pt}_jac"], 1e-15)
    rel_close(OM.hessian(om, x, y, w), g[f"ad{pt}_hess"], 1e-15)


@pytest.mark.parametrize("tag", MODEL_TAGS)
def test_condense_order_symbolic_bitexact(golden_models, tag):
    g = golden_models[tag]
    cs = OS.condense(g["hess_rows"], g["hess_cols"], g["jac_rows"], g["jac_cols"], int(g["n"]))
    np.testing.assert_array_equal(cs.matrix.indptr, g["cond_indptr"])
    np.testing.assert_array_equal(cs.matrix.indices, g["cond_indices"])
    for f in ("w_map", "diag_map", "ata_map", "ata_row", "ata_s1", "ata_s2"):
        np.testing.assert_array_equal(getattr(cs, f), g["cond_" + f])
    r, c = cs.matrix.coords()
    perm = min_degree_order(cs.matrix.n, r, c)
    np.testing.assert_array_equal(perm, g["sym_perm"])
    sym = OS.symbolic(cs.matrix, perm)
    for f in ("parent", "a_rowptr", "a_rowcol", "a_srcslot", "row_ptr", "row_cols",
              "l_colptr", "l_rowidx"):
        np.testing.assert_array_equal(getattr(sym, f), g["sym_" + f])


def _workspace(g):
    ws = OK.OWorkspace(int(g["n"]), int(g["m"]), g["hess_rows"], g["hess_cols"],
                       g["jac_rows"], g["jac_cols"])
    ws.set_iterate(*(g["ws_" + f] for f in ("w_vals", "a_vals", "dxl", "dxu", "zxl", "zxu",
                                             "dsl", "dsu", "zsl", "zsu")))
    ws.dw, ws.dc = float(g["ws_delta_w"]), float(g["ws_delta_c"])
    return ws


@pytest.mark.parametrize("tag", MODEL_TAGS)
def test_assembly_factor_solve(golden_models, tag):
    g = golden_models[tag]
    ws = _workspace(g)
    rel_close(ws.sx, g["ws_sigma_x"], 0)
    back = OK.OCondensedBackend(ws, ordering=g["sym_perm"])
    assert back.try_factorize()
    np.testing.assert_array_equal(back.cs.matrix.values, g["K_vals"])
    np.testing.assert_array_equal(back.l_vals, g["L_vals"])
    np.testing.assert_array_equal(OS.solve(back.sym, back.l_vals, g["solve_b"]), g["solve_x"])
    pv = OK.Vec7(*(g["pv_" + f] for f in OK.FIELDS))
    qx, qs, qy = ws.condense_pvec(pv)
    rel_close(qx, g["q_x"], 0)
    rel_close(ws.condensed_rhs(qx, qs, qy), g["rhs"], 1e-15)
    dx, ds, dy = back.solve3(qx, qs, qy)
    rel_close(dx, g["s3_dx"], 1e-15)
    st = OK.assemble_steps(ws, pv, dx, ds, dy)
    rel_close(st.zxl, g["st_zxl"], 1e-15)
    res = ws.residual_full(st, pv)
    for f in OK.FIELDS:
        rel_close(getattr(res, f).astype(float), g["res_" + f], 1e-15)
    assert ws.matrix_scale() == float(g["matrix_scale"])


@pytest.mark.parametrize("case,tol", [("case14", 1e-4), ("case14", 1e-6), ("case118", 1e-4),
                                      ("C1", 1e-6)])
def test_end_to_end_small(golden_models, end_to_end, case, tol):
    g = golden_models[case]
    om = oracle_model(g)
    rep = OI.solve(om, g["lower"], g["upper"], g["start"], OI.Options(tol=tol), g["ranges"])
    ref = end_to_end[f"{case}@{tol:g}"]
    assert rep.status == ref["status"]
    assert rep.iterations == ref["iterations"]
    assert rep.objective == ref["objective"]
    np.testing.assert_array_equal(rep.x, golden_x(case, tol))
    assert [list(map(float, t)) for t in rep.trace] == ref["trace"]


def test_known_answers_from_reference_tests():
    """KATs from the reference suite (test_sparse_linear.py:171-184)."""
    m, _ = OS.coo_to_csc(2, np.array([0, 1, 1]), np.array([0, 0, 1]), np.array([2.0, 1.0, 2.0]))
    sym = OS.symbolic(m, np.arange(2))
    l_vals, ok, _ = OS.factorize(sym, m.values)
    assert ok
    np.testing.assert_allclose(l_vals, [np.sqrt(2.0), 1.0 / np.sqrt(2.0), np.sqrt(1.5)])
    m, _ = OS.coo_to_csc(2, np.array([0, 1, 1]), np.array([0, 0, 1]), np.array([1.0, 2.0, 1.0]))
    _, ok, bad = OS.factorize(OS.symbolic(m, np.arange(2)), m.values)
    assert not ok and bad == 1
    # arrow matrix: centre eliminated last, factor nnz 2n-1 (test_sparse_linear.py:96-103)
    n = 10
    rows = [0] + list(range(1, n)) + list(range(1, n))
    cols = [0] + [0] * (n - 1) + list(range(1, n))
    m, _ = OS.coo_to_csc(n, np.array(rows), np.array(cols), np.ones(len(rows)))
    r, c = m.coords()
    perm = min_degree_order(n, r, c)
    assert perm[-1] == 0
    assert OS.symbolic(m, perm).l_rowidx.size == 2 * n - 1
    # delta_w schedule [0, 1e-4, 1e-2, 1.0] then [0, 1/3, 8/3] (test_kkt_condensed.py:246-277)
    calls = []

    class Fake:
        def __init__(self, ws, fails):
            self.ws, self.fails, self.k = ws, fails, 0

        def try_factorize(self):
            calls.append(self.ws.dw)
            self.k += 1
            return self.k > self.fails

        def solve3(self, qx, qs, qy):
            return np.zeros(1), np.zeros(1), np.zeros(1)

    ws = OK.OWorkspace(1, 1, np.zeros(1, np.int64), np.zeros(1, np.int64),
                       np.zeros(1, np.int64), np.zeros(1, np.int64))
    ws.set_iterate(np.ones(1), np.ones(1), np.ones(1), np.full(1, np.inf), np.ones(1),
                   np.zeros(1), np.ones(1), np.ones(1), np.ones(1), np.ones(1))
    pv = OK.Vec7(*(np.zeros(1) for _ in OK.FIELDS))
    reg = OK.RegState()
    OK.solve_with_regularization(ws, Fake(ws, 3), pv, reg)
    assert calls == [0.0, 1e-4, 1e-2, 1.0]
    calls.clear()
    OK.solve_with_regularization(ws, Fake(ws, 2), pv, reg)
    assert calls[0] == 0.0 and calls[1] == pytest.approx(1 / 3) and calls[2] == pytest.approx(8 / 3)
    # relaxation band and initial slack (test_ipm_core.py:42-80)
    sl, su = OI.relax_equalities(1, None, 1e-4)
    assert OI.initial_slacks(np.ones(1), sl, su, 1e-4, 0.01)[0] == pytest.approx(9.9e-5)
    assert OI.kkt_residual(np.array([1.0]), np.zeros(0), np.zeros(0), [np.zeros(1)], z_l1=1e6,
                           y_l1=0.0, m=0, n_bounds=1) == pytest.approx(1.0 / (1e6 / 100.0))
