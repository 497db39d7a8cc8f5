"""Helpers turning golden npz dumps into oracle inputs."""
import numpy as np

from oracle import model as OM

KINDS = (OM.OBJ, OM.DEF, OM.INC)


def oracle_blocks(g):
    blocks = []
    for b in range(int(g["n_blocks"])):
        p = f"b{b}_"
        ops = [tuple(int(v) for v in r) for r in g[p + "ops"]]
        blocks.append(OM.OBlock(
            KINDS[int(g[p + "kind"])], ops, [float(c) for c in g[p + "consts"]],
            int(g[p + "out"]), [int(s) for s in g[p + "first_slots"]],
            [tuple(int(v) for v in r) for r in g[p + "second_pairs"]],
            g[p + "var_idx"].astype(np.int64), g[p + "params"].astype(float),
            g[p + "targets"].astype(np.int64) if p + "targets" in g else None))
    return blocks


def oracle_model(g):
    return OM.expand(int(g["n"]), int(g["m"]), oracle_blocks(g))
