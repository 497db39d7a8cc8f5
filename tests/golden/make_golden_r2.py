"""Round-2 golden vectors, produced by running the REFERENCE package.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):

    python tests/golden/make_golden_r2.py [C2] [C4]

* ``C2.npz``              value-level fixture of BASELINE configs[1] (2,002
                          buses): structure arrays, AD at two points,
                          condensed K pattern/maps, ordering, symbolic factor,
                          K/L values and KKT vector kernels at a real iterate
                          (same content as make_golden.dump_model).
* ``end_to_end_C4.json``  status / iterations / objective / trace of the
                          reference solve of C4 (78,484 buses, tol 1e-6),
                          ordering injected (heap minimum degree, identical
                          to the shipped scan -- which is infeasible at C4).
* ``C4_1e-06_x.npz``      converged x of that solve (float64).
* ``C4_perm.npz``         the injected permutation (int32), so GPU tests and
                          the bench can inject the same ordering.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as MG  # noqa: E402  (imports the reference from a temp copy)


def c2():
    rng = np.random.default_rng(20261017)
    am = MG.build_acopf(MG.parse_matpower(MG.tiled_case(143)))
    # the C2 permutation equals the shipped O(n^2) amd_order (C2_perm.npz,
    # checked by make_perm_golden.py); the heap ordering is injected here
    MG.dump_model("C2", am, rng, check_shipped_amd=False)


def c4():
    am = MG.build_acopf(MG.parse_matpower(MG.tiled_case(5606)))
    m = am.model
    t = time.perf_counter()
    perm_holder = {}

    def heap_amd(mat):
        p = MG._heap_amd(mat)
        perm_holder["perm"] = p
        return p

    MG.RK.amd_order = heap_amd
    print("C4 model", m.n_var, m.n_con, f"{time.perf_counter() - t:.1f}s", flush=True)
    t = time.perf_counter()
    rep = MG.solve(m, MG.SolverOptions(tol=1e-6), constraint_ranges=am.ranges)
    dt = time.perf_counter() - t
    MG.RK.amd_order = MG._SHIPPED_AMD
    rec = dict(status=rep.status, iterations=rep.iterations, objective=rep.objective,
               violation=rep.constraint_violation, residual_scaled=rep.residual_scaled,
               trace=[list(map(float, tr)) for tr in rep.trace], seconds=rep.seconds, wall=dt,
               n_var=rep.n_var, n_con=rep.n_con)
    with open(os.path.join(HERE, "end_to_end_C4.json"), "w") as fh:
        json.dump({"C4@1e-06": rec}, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "C4_1e-06_x.npz"), x=rep.x)
    np.savez_compressed(os.path.join(HERE, "C4_perm.npz"),
                        perm=np.asarray(perm_holder["perm"], dtype=np.int32))
    print("C4", rep.status, rep.iterations, rep.objective, f"{dt:.1f}s", flush=True)


def diag():
    """diagnose_conditioning of the reference (src/bench.py:113-135) at the
    final iterate of case14 / case30 / case118 (tol 1e-6)."""
    from gridnlp.bench import diagnose_conditioning

    out = {}
    for c in ("case14", "case30", "case118"):
        am = MG.build_acopf(MG.parse_matpower_file(os.path.join(MG.CASES, f"{c}.m")))
        rep = MG.solve(am.model, MG.SolverOptions(tol=1e-6, keep_workspace=True),
                       constraint_ranges=am.ranges)
        d = diagnose_conditioning(rep)
        ws = rep.debug["workspace"]
        d["delta_w"], d["delta_c"] = float(ws.delta_w), float(ws.delta_c)
        d["iterations"] = rep.iterations
        out[c] = d
        print(c, d, flush=True)
    with open(os.path.join(HERE, "conditioning.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["C2", "C4", "diag"]
    if "diag" in which:
        diag()
    if "C2" in which:
        c2()
    if "C4" in which:
        c4()
