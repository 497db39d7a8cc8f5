"""Synthetic ACOPF grids: IEEE-14 tiles on a near-square mesh.

The reference ships no grid generator (SURVEY.md §0 finding 7); the
benchmark configurations (BASELINE.json ``configs``) are produced by the
recipe in SURVEY.md Appendix B:

* ``k`` copies of the IEEE 14-bus system, bus ids offset by ``14*t``;
  only tile 0 keeps its type-3 reference bus, the others become PV;
* tiles laid out row-major in ``cols = ceil(sqrt(k))`` columns, tied
  bus 4(t) -> bus 5(t+1) to the right (r=0.01, x=0.05, b=0.02) and
  bus 9(t) -> bus 13(t+cols) downwards (r=0.02, x=0.08);
* optional limits: +-30 deg angle limits on every branch, per-branch
  rateA = 100*max(0.3, 1.5*S*_q) MVA on tile branches, 100 MVA on ties;
* optional load perturbation Pd/Qd * (1+eps), eps ~ U(-0.1, 0.1) per bus
  drawn from ``np.random.default_rng(seed)``.

The output is MATPOWER text, so the reference parser and ours read the
identical file (matpower.py).
"""
from __future__ import annotations

import math

import numpy as np

# IEEE 14-bus data (public domain test system).  Columns follow the
# MATPOWER v2 layout; only the fields the parser reads are kept.
#            id type   Pd     Qd    Gs   Bs    Vm     Va     Vmax  Vmin
_BUS14 = (
    (1, 3, 0.0, 0.0, 0.0, 0.0, 1.06, 0.0, 1.06, 0.94),
    (2, 2, 21.7, 12.7, 0.0, 0.0, 1.045, -4.98, 1.06, 0.94),
    (3, 2, 94.2, 19.0, 0.0, 0.0, 1.01, -12.72, 1.06, 0.94),
    (4, 1, 47.8, -3.9, 0.0, 0.0, 1.019, -10.33, 1.06, 0.94),
    (5, 1, 7.6, 1.6, 0.0, 0.0, 1.02, -8.78, 1.06, 0.94),
    (6, 2, 11.2, 7.5, 0.0, 0.0, 1.07, -14.22, 1.06, 0.94),
    (7, 1, 0.0, 0.0, 0.0, 0.0, 1.062, -13.37, 1.06, 0.94),
    (8, 2, 0.0, 0.0, 0.0, 0.0, 1.09, -13.36, 1.06, 0.94),
    (9, 1, 29.5, 16.6, 0.0, 19.0, 1.056, -14.94, 1.06, 0.94),
    (10, 1, 9.0, 5.8, 0.0, 0.0, 1.051, -15.1, 1.06, 0.94),
    (11, 1, 3.5, 1.8, 0.0, 0.0, 1.057, -14.79, 1.06, 0.94),
    (12, 1, 6.1, 1.6, 0.0, 0.0, 1.055, -15.07, 1.06, 0.94),
    (13, 1, 13.5, 5.8, 0.0, 0.0, 1.05, -15.16, 1.06, 0.94),
    (14, 1, 14.9, 5.0, 0.0, 0.0, 1.036, -16.04, 1.06, 0.94),
)
#          bus    Pg     Qg    Qmax  Qmin   Vg   Pmax  Pmin    c2            c1    c0
_GEN14 = (
    (1, 232.4, -16.9, 10.0, 0.0, 1.06, 332.4, 0.0, 0.0430292599, 20.0, 0.0),
    (2, 40.0, 42.4, 50.0, -40.0, 1.045, 140.0, 0.0, 0.25, 20.0, 0.0),
    (3, 0.0, 23.4, 40.0, 0.0, 1.01, 100.0, 0.0, 0.01, 40.0, 0.0),
    (6, 0.0, 12.2, 24.0, -6.0, 1.07, 100.0, 0.0, 0.01, 40.0, 0.0),
    (8, 0.0, 17.4, 24.0, -6.0, 1.09, 100.0, 0.0, 0.01, 40.0, 0.0),
)
#          f   t     r        x        b      ratio
_BRANCH14 = (
    (1, 2, 0.01938, 0.05917, 0.0528, 0.0),
    (1, 5, 0.05403, 0.22304, 0.0492, 0.0),
    (2, 3, 0.04699, 0.19797, 0.0438, 0.0),
    (2, 4, 0.05811, 0.17632, 0.034, 0.0),
    (2, 5, 0.05695, 0.17388, 0.0346, 0.0),
    (3, 4, 0.06701, 0.17103, 0.0128, 0.0),
    (4, 5, 0.01335, 0.04211, 0.0, 0.0),
    (4, 7, 0.0, 0.20912, 0.0, 0.978),
    (4, 9, 0.0, 0.55618, 0.0, 0.969),
    (5, 6, 0.0, 0.25202, 0.0, 0.932),
    (6, 11, 0.09498, 0.1989, 0.0, 0.0),
    (6, 12, 0.12291, 0.25581, 0.0, 0.0),
    (6, 13, 0.06615, 0.13027, 0.0, 0.0),
    (7, 8, 0.0, 0.17615, 0.0, 0.0),
    (7, 9, 0.0, 0.11001, 0.0, 0.0),
    (9, 10, 0.03181, 0.0845, 0.0, 0.0),
    (9, 14, 0.12711, 0.27038, 0.0, 0.0),
    (10, 11, 0.08205, 0.19207, 0.0, 0.0),
    (12, 13, 0.22092, 0.19988, 0.0, 0.0),
    (13, 14, 0.17093, 0.34802, 0.0, 0.0),
)
# case14 optimal apparent flows |S*_q| (p.u.) per tile branch, SURVEY.md App. B
_S_STAR = (1.298, 0.65, 0.556, 0.489, 0.373, 0.126, 0.506, 0.234, 0.149, 0.447,
           0.076, 0.081, 0.188, 0.119, 0.315, 0.072, 0.106, 0.037, 0.017, 0.055)

# named benchmark configurations
CONFIGS = {
    "C1": dict(tiles=1, limits=True),
    "C2": dict(tiles=143, limits=True),
    "C3": dict(tiles=714, limits=True),
    "C4": dict(tiles=5606, limits=True),
    "C5": dict(tiles=97, limits=True),
}


def _fmt(v: float) -> str:
    if float(v).is_integer() and abs(v) < 1e15:
        return str(int(v))
    return repr(float(v))


def tiled_case(tiles: int, limits: bool = True, seed: int | None = None,
               stress: bool = False) -> str:
    """MATPOWER text of a ``tiles``-copy IEEE-14 mesh (Appendix B recipe).

    ``seed=None`` leaves loads unperturbed; otherwise every bus's Pd/Qd is
    scaled by ``1+eps`` with ``eps = rng.uniform(-0.1, 0.1, nbus)``.
    """
    if tiles < 1:
        raise ValueError("tiles must be >= 1")
    cols = int(math.ceil(math.sqrt(tiles)))
    nb = 14 * tiles
    eps = np.zeros(nb)
    if seed is not None:
        eps = np.random.default_rng(seed).uniform(-0.1, 0.1, nb)
    ang = 30.0 if limits else 360.0

    bus_lines, gen_lines, cost_lines, br_lines = [], [], [], []
    for t in range(tiles):
        off = 14 * t
        for (bid, btype, pd, qd, gs, bs, vm, va, vmax, vmin) in _BUS14:
            k = off + bid - 1
            typ = btype if (t == 0 or btype != 3) else 2
            scale = 1.0 + eps[k]
            bus_lines.append("\t".join(_fmt(v) for v in (
                off + bid, typ, pd * scale, qd * scale, gs, bs, 1, vm, va, 0, 1,
                vmax, vmin)))
        for (gb, pg, qg, qmax, qmin, vg, pmax, pmin, c2, c1, c0) in _GEN14:
            gen_lines.append("\t".join(_fmt(v) for v in (
                off + gb, pg, qg, qmax, qmin, vg, 100, 1, pmax, pmin)))
            cost_lines.append("\t".join(_fmt(v) for v in (2, 0, 0, 3, c2, c1, c0)))
        for q, (f, tb, r, x, b, ratio) in enumerate(_BRANCH14):
            if limits:
                s = 0.9 * _S_STAR[q] if (stress and q == 0) else 1.5 * _S_STAR[q]
                rate = 100.0 * max(0.3, s)
            else:
                rate = 0.0
            br_lines.append("\t".join(_fmt(v) for v in (
                off + f, off + tb, r, x, b, rate, 0, 0, ratio, 0, 1, -ang, ang)))
    tie_rate = 100.0 if limits else 0.0
    for t in range(tiles):
        if (t % cols) + 1 < cols and t + 1 < tiles:
            br_lines.append("\t".join(_fmt(v) for v in (
                14 * t + 4, 14 * (t + 1) + 5, 0.01, 0.05, 0.02, tie_rate, 0, 0, 0, 0,
                1, -ang, ang)))
        if t + cols < tiles:
            br_lines.append("\t".join(_fmt(v) for v in (
                14 * t + 9, 14 * (t + cols) + 13, 0.02, 0.08, 0.0, tie_rate, 0, 0, 0,
                0, 1, -ang, ang)))

    def table(name, rows):
        return f"mpc.{name} = [\n" + "".join(f"\t{r};\n" for r in rows) + "];\n"

    return (f"function mpc = tiled{tiles}\n"
            f"% {tiles} IEEE-14 tiles, {cols} columns, limits={limits}, seed={seed}\n"
            "mpc.version = '2';\nmpc.baseMVA = 100;\n"
            + table("bus", bus_lines) + table("gen", gen_lines)
            + table("branch", br_lines) + table("gencost", cost_lines))


def config_case(name: str, seed: int | None = None) -> str:
    """MATPOWER text for a named configuration C1..C5."""
    cfg = CONFIGS[name]
    return tiled_case(cfg["tiles"], limits=cfg["limits"], seed=seed)
