"""Input formats and model construction around the path (CPU).

* The MATPOWER parser (src/matpower.py:156-279) on the reference's own IEEE
  case files: identical tables to the reference's parse (networks.json,
  written by tests/golden/make_golden.py).  The .m files are read from the
  reference checkout when it is mounted (the build container), and a
  writer -> parser round trip of the same tables runs everywhere.
* The oracle's ACOPF construction (oracle/acopf.py, used by the bench's
  reference arm) against the reference's golden arrays and against the
  product's native construction.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import acopf as OA
from paper_2307_16830_b200.acopf import build_acopf
from paper_2307_16830_b200.grids import tiled_case
from paper_2307_16830_b200.matpower import network_from_tables, parse_matpower, parse_matpower_file

REF_CASES = "/root/reference/pkg/src/gridnlp/cases"
CASES = ("case14", "case30", "case57", "case118")


def _tables(net):
    return dict(
        base_mva=net.base_mva,
        buses=[[b.id, b.type, b.pd, b.qd, b.gs, b.bs, b.vm, b.va, b.vmax, b.vmin] for b in net.buses],
        generators=[[g.bus, g.pg, g.qg, g.qmax, g.qmin, g.vg, g.pmax, g.pmin, *g.cost]
                    for g in net.generators],
        branches=[[br.from_bus, br.to_bus, br.r, br.x, br.b_charge, br.rate_a, br.tap, br.shift,
                   br.angmin, br.angmax] for br in net.branches])


@pytest.mark.skipif(not os.path.isdir(REF_CASES), reason="reference checkout not mounted")
@pytest.mark.parametrize("case", CASES)
def test_parse_ieee_files_like_the_reference(networks_json, case):
    net = parse_matpower_file(os.path.join(REF_CASES, f"{case}.m"))
    ref = networks_json[case]
    got = _tables(net)
    assert got["base_mva"] == ref["base_mva"]
    for key in ("buses", "generators", "branches"):
        assert len(got[key]) == len(ref[key])
        np.testing.assert_array_equal(np.array(got[key], float), np.array(ref[key], float))


def _matpower_text(t):
    """Minimal MATPOWER writer (per-unit fields back to MW / degrees)."""
    import math

    base = t["base_mva"]
    lines = ["function mpc = rt", "mpc.version = '2';", f"mpc.baseMVA = {base!r};", "mpc.bus = ["]
    for b in t["buses"]:
        lines.append(f"{int(b[0])} {int(b[1])} {b[2] * base!r} {b[3] * base!r} {b[4] * base!r} "
                     f"{b[5] * base!r} 1 {b[6]!r} {math.degrees(b[7])!r} 0 1 {b[8]!r} {b[9]!r};")
    lines += ["];", "mpc.gen = ["]
    for g in t["generators"]:
        lines.append(f"{int(g[0])} {g[1] * base!r} {g[2] * base!r} {g[3] * base!r} {g[4] * base!r} "
                     f"{g[5]!r} {base!r} 1 {g[6] * base!r} {g[7] * base!r};")
    lines += ["];", "mpc.branch = ["]
    for br in t["branches"]:
        lines.append(f"{int(br[0])} {int(br[1])} {br[2]!r} {br[3]!r} {br[4]!r} {br[5] * base!r} 0 0 "
                     f"{br[6]!r} {math.degrees(br[7])!r} 1 {math.degrees(br[8])!r} "
                     f"{math.degrees(br[9])!r};")
    lines += ["];", "mpc.gencost = ["]
    for g in t["generators"]:
        lines.append(f"2 0 0 3 {g[8]!r} {g[9]!r} {g[10]!r};")
    lines += ["];"]
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("case", CASES)
def test_writer_parser_round_trip(networks_json, case):
    ref = networks_json[case]
    net = parse_matpower(_matpower_text(ref))
    got = _tables(net)
    for key in ("buses", "generators", "branches"):
        np.testing.assert_allclose(np.array(got[key], float), np.array(ref[key], float),
                                   rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("case", ("case14", "case118"))
def test_oracle_acopf_matches_reference_golden(networks_json, golden_models, case):
    g = golden_models[case]
    oa = OA.build(network_from_tables(networks_json[case]))
    om = oa.model
    for f in ("jac_rows", "jac_cols", "hess_rows", "hess_cols"):
        np.testing.assert_array_equal(getattr(om, f), g[f])
    np.testing.assert_array_equal(oa.lower, g["lower"])
    np.testing.assert_array_equal(oa.upper, g["upper"])
    np.testing.assert_array_equal(oa.start, g["start"])
    np.testing.assert_array_equal(oa.ranges, g["ranges"])
    for bi, b in enumerate(om.blocks):
        np.testing.assert_array_equal(b.var_idx, g[f"b{bi}_var_idx"])
        np.testing.assert_array_equal(b.params, g[f"b{bi}_params"])
    np.testing.assert_array_equal(OA.ordering(oa), g["sym_perm"])


@pytest.mark.parametrize("tiles,seed", ((1, None), (97, 5)))
def test_oracle_acopf_matches_product(tiles, seed):
    net = parse_matpower(tiled_case(tiles, seed=seed))
    oa, am = OA.build(net), build_acopf(net)
    m = am.model
    for f in ("jac_rows", "jac_cols", "hess_rows", "hess_cols"):
        np.testing.assert_array_equal(getattr(oa.model, f), getattr(m, f))
    np.testing.assert_array_equal(oa.ranges, am.ranges)
    np.testing.assert_array_equal(oa.start, m.start)
    for a, b in zip(oa.model.blocks, m.pattern_blocks):
        np.testing.assert_array_equal(a.var_idx, b.var_idx)
        np.testing.assert_array_equal(a.params, b.params)
