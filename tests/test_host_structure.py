"""Native host structure vs the oracle and the reference's golden arrays (CPU).

Covers SURVEY.md §8(a) rows a1-a3 (record order, templates, COO expansion,
slot maps), a15 (symbolic condensation), a19 (ordering), a20 (symbolic
Cholesky): all must be bit-exact.
"""
import numpy as np
import pytest

from oracle import model as OM
from oracle import sparse as OS
from oracle.ordering import min_degree_order

from paper_2307_16830_b200 import kkt, sparse
from paper_2307_16830_b200.acopf import build_acopf
from paper_2307_16830_b200.grids import tiled_case
from paper_2307_16830_b200.matpower import network_from_tables, parse_matpower
from paper_2307_16830_b200.model import ModelBuilder
from paper_2307_16830_b200.expressions import param, sin, var

from conftest import MODEL_TAGS, TILES


def product_model(tag, networks_json):
    if tag.startswith("case"):
        return build_acopf(network_from_tables(networks_json[tag]))
    tiles = TILES[tag]
    return build_acopf(parse_matpower(tiled_case(tiles)))


@pytest.mark.parametrize("tag", MODEL_TAGS)
def test_acopf_model_matches_reference(golden_models, networks_json, tag):
    g = golden_models[tag]
    am = product_model(tag, networks_json)
    m = am.model
    assert (m.n_var, m.n_con) == (int(g["n"]), int(g["m"]))
    np.testing.assert_array_equal(m.lower, g["lower"])
    np.testing.assert_array_equal(m.upper, g["upper"])
    np.testing.assert_array_equal(m.start, g["start"])
    np.testing.assert_array_equal(am.ranges, g["ranges"])
    assert len(m.pattern_blocks) == int(g["n_blocks"]) == 15
    for bi, b in enumerate(m.pattern_blocks):
        p = f"b{bi}_"
        np.testing.assert_array_equal(np.asarray(b.tape.ops).reshape(-1, 3), g[p + "ops"])
        np.testing.assert_array_equal(np.asarray(b.tape.consts, float), g[p + "consts"])
        assert b.tape.first_slots == list(g[p + "first_slots"])
        assert b.tape.second_pairs == [tuple(r) for r in g[p + "second_pairs"].tolist()]
        np.testing.assert_array_equal(b.var_idx, g[p + "var_idx"])
        np.testing.assert_array_equal(b.params, g[p + "params"])
        if b.targets is not None:
            np.testing.assert_array_equal(b.targets, g[p + "targets"])
        for k, a in enumerate(b.jac_slots):
            np.testing.assert_array_equal(a, g[p + f"jac_slots{k}"])
        for k, a in enumerate(b.hess_slots):
            np.testing.assert_array_equal(a, g[p + f"hess_slots{k}"])
            np.testing.assert_array_equal(b.hess_factor[k], g[p + f"hess_factor{k}"])
    for f in ("jac_rows", "jac_cols", "hess_rows", "hess_cols"):
        np.testing.assert_array_equal(getattr(m, f), g[f])


@pytest.mark.parametrize("tag", MODEL_TAGS)
def test_condense_order_symbolic_native(golden_models, tag):
    g = golden_models[tag]
    n = int(g["n"])
    cs = kkt.symbolic_condense(g["hess_rows"], g["hess_cols"], g["jac_rows"], g["jac_cols"], n)
    np.testing.assert_array_equal(cs.matrix.indptr, g["cond_indptr"])
    np.testing.assert_array_equal(cs.matrix.indices, g["cond_indices"])
    for f in ("w_map", "diag_map", "ata_map", "ata_row", "ata_s1", "ata_s2"):
        np.testing.assert_array_equal(getattr(cs, f), g["cond_" + f])
    perm = sparse.amd_order(cs.matrix)
    np.testing.assert_array_equal(perm, g["sym_perm"])
    sym = sparse.symbolic_cholesky(cs.matrix, perm)
    for f in ("parent", "a_rowptr", "a_rowcol", "a_srcslot", "row_ptr", "row_cols",
              "l_colptr", "l_rowidx"):
        np.testing.assert_array_equal(getattr(sym, f), g["sym_" + f])
    info = sym.info
    assert info["nnz_l"] == g["sym_l_rowidx"].size
    assert info["n_fronts"] <= n


def _random_model(rng, n=8):
    b = ModelBuilder()
    b.add_variables(n, np.full(n, -10.0), np.full(n, 10.0), np.zeros(n))
    b.add_objective(param(0) * var(0) ** 2 + param(1) * sin(var(1)) * var(0),
                    rng.integers(0, n, (12, 2)), rng.normal(size=(12, 2)))
    b.add_constraints(var(0) * var(1) - param(0) * var(2), rng.integers(0, n, (6, 3)),
                      rng.normal(size=(6, 1)))
    b.add_constraint_increments(param(0) * var(0) * var(1), rng.integers(0, n, (9, 2)),
                                rng.normal(size=(9, 1)), rng.integers(0, 6, 9))
    return b.finalize()


def test_random_model_expansion_matches_oracle():
    rng = np.random.default_rng(5)
    for _ in range(5):
        m = _random_model(rng)
        om = OM.expand(m.n_var, m.n_con, OM.from_model(m))
        for f in ("jac_rows", "jac_cols", "hess_rows", "hess_cols"):
            np.testing.assert_array_equal(getattr(m, f), getattr(om, f))
        for b, ob in zip(m.pattern_blocks, om.blocks):
            for x, y in zip(b.jac_slots, ob.jac_slots):
                np.testing.assert_array_equal(x, y)
            for x, y in zip(b.hess_slots + b.hess_factor, ob.hess_slots + ob.hess_factor):
                np.testing.assert_array_equal(x, y)
            np.testing.assert_array_equal(
                OM.canonical_order(b.var_idx, b.params, b.targets), np.arange(b.n_records))


def test_canonical_order_matches_lexsort():
    rng = np.random.default_rng(9)
    vi = rng.integers(0, 4, (200, 3))
    pa = rng.integers(0, 3, (200, 2)).astype(float)
    tg = rng.integers(0, 5, 200)
    from paper_2307_16830_b200.model import canonical_order

    np.testing.assert_array_equal(canonical_order(vi, pa, tg), OM.canonical_order(vi, pa, tg))
    np.testing.assert_array_equal(canonical_order(vi, pa), OM.canonical_order(vi, pa))


def test_min_degree_matches_oracle_on_random_patterns():
    rng = np.random.default_rng(11)
    for n in (1, 5, 30, 120):
        A = rng.random((n, n)) < 0.08
        A = np.tril(A | A.T)
        np.fill_diagonal(A, True)
        r, c = np.nonzero(A)
        m, _ = sparse.coo_to_csc(n, r, c, np.ones(r.size))
        om, _ = OS.coo_to_csc(n, r, c, np.ones(r.size))
        np.testing.assert_array_equal(m.indptr, om.indptr)
        np.testing.assert_array_equal(m.indices, om.indices)
        rr, cc = m.coords()
        perm = sparse.amd_order(m)
        np.testing.assert_array_equal(perm, min_degree_order(n, rr, cc))
        sym = sparse.symbolic_cholesky(m, perm)
        osym = OS.symbolic(om, perm)
        np.testing.assert_array_equal(sym.l_rowidx, osym.l_rowidx)
        np.testing.assert_array_equal(sym.l_colptr, osym.l_colptr)


def test_larger_grid_structure_matches_oracle():
    am = build_acopf(parse_matpower(tiled_case(16)))
    m = am.model
    cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    ocs = OS.condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    np.testing.assert_array_equal(cs.ata_map, ocs.ata_map)
    r, c = cs.matrix.coords()
    perm = sparse.amd_order(cs.matrix)
    np.testing.assert_array_equal(perm, min_degree_order(m.n_var, r, c))
    sym = sparse.symbolic_cholesky(cs.matrix, perm)
    osym = OS.symbolic(ocs.matrix, perm)
    np.testing.assert_array_equal(sym.l_rowidx, osym.l_rowidx)
    np.testing.assert_array_equal(sym.parent, osym.parent)


def test_min_degree_matches_shipped_reference_at_2k_buses():
    """C2 (143 tiles, 17,922 columns): the permutation is bit-identical to the
    reference's own O(n^2) amd_order (amd.py:18-54), run by
    tests/golden/make_perm_golden.py."""
    import os

    from conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, "C2_perm.npz"))
    m = build_acopf(parse_matpower(tiled_case(143))).model
    cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    assert cs.matrix.indices.size == int(g["nnz_k"])
    np.testing.assert_array_equal(sparse.amd_order(cs.matrix), g["perm"].astype(np.int64))


@pytest.mark.parametrize("tiles", [1, 16])
@pytest.mark.parametrize("inject", [False, True])
def test_analyze_single_call_matches_separate_calls(tiles, inject):
    """gn_analyze (condense + ordering + symbolic + front plan in one native
    call, as the analysis worker can use it) equals the separate entry points."""
    import ctypes

    from paper_2307_16830_b200 import _lib as L

    m = build_acopf(parse_matpower(tiled_case(tiles))).model
    cs = kkt.symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    perm = sparse.amd_order(cs.matrix)
    sym = sparse.symbolic_cholesky(cs.matrix, perm)
    hr, hc, jr, jc = (L.i64(a) for a in (m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols))
    perm_out = np.empty(m.n_var, np.int64)
    hcs, hsym = ctypes.c_void_p(), ctypes.c_void_p()
    pin = L.i64(perm) if inject else None
    L.check(L.lib().gn_analyze(m.n_var, hr.size, L.ptr(hr), L.ptr(hc), jr.size, L.ptr(jr), L.ptr(jc),
                               None if pin is None else L.ptr(pin), L.ptr(perm_out),
                               ctypes.byref(hcs), ctypes.byref(hsym)))
    try:
        np.testing.assert_array_equal(perm_out, perm)
        nk, npr = ctypes.c_int64(), ctypes.c_int64()
        L.check(L.lib().gn_condense_info(hcs, ctypes.byref(nk), ctypes.byref(npr)))
        assert (nk.value, npr.value) == (cs.matrix.nnz, cs._np)
        maps = {k: np.empty(n, np.int64) for k, n in (
            ("indptr", m.n_var + 1), ("indices", nk.value), ("w_map", hr.size), ("diag_map", m.n_var),
            ("ata_map", npr.value), ("ata_row", npr.value), ("ata_s1", npr.value), ("ata_s2", npr.value))}
        L.check(L.lib().gn_condense_export(hcs, *(L.ptr(maps[k]) for k in (
            "indptr", "indices", "w_map", "diag_map", "ata_map", "ata_row", "ata_s1", "ata_s2"))))
        np.testing.assert_array_equal(maps["indptr"], cs.matrix.indptr)
        np.testing.assert_array_equal(maps["indices"], cs.matrix.indices)
        for f in ("w_map", "diag_map", "ata_map", "ata_row", "ata_s1", "ata_s2"):
            np.testing.assert_array_equal(maps[f], getattr(cs, f))
        info = L.SymbolicInfo()
        L.check(L.lib().gn_symbolic_info(hsym, ctypes.byref(info)))
        assert {f: getattr(info, f) for f, _ in L.SymbolicInfo._fields_} == sym.info
        nf = sym.info["n_fronts"]
        fa = {k: np.empty(nf, np.int32) for k in ("first", "ncols", "nrows", "parent", "order")}
        nsm = ctypes.c_int64()
        L.check(L.lib().gn_symbolic_fronts(hsym, *(L.ptr(fa[k]) for k in
                                                   ("first", "ncols", "nrows", "parent", "order")),
                                           ctypes.byref(nsm)))
        ref = sparse.front_plan(sym)
        for k in ("first", "ncols", "nrows", "parent", "order"):
            np.testing.assert_array_equal(fa[k], ref[k])
        assert nsm.value == ref["nf_small"]
    finally:
        L.lib().gn_condense_destroy(hcs)
        L.lib().gn_symbolic_destroy(hsym)
