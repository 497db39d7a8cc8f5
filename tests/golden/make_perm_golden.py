"""Golden ordering at 2,002 buses from the REFERENCE's shipped amd_order.

Runs the unmodified O(n^2) ``gridnlp.sparse.amd.amd_order`` (amd.py:18-54,
~80 s) on the condensed pattern of config C2 (143 IEEE-14 tiles, SURVEY.md
Appendix B) and stores the permutation as ``C2_perm.npz`` (int32).  Build
container only: /root/reference does not exist on the GPU box.

    python tests/golden/make_perm_golden.py
"""
from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))


def main():
    tmp = tempfile.mkdtemp(prefix="gridnlp_ref_")
    shutil.copytree("/root/reference/pkg", os.path.join(tmp, "pkg"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba"))
    sys.path.insert(0, os.path.join(tmp, "pkg", "src"))
    from gridnlp.acopf import build_acopf
    from gridnlp.kkt import symbolic_condense
    from gridnlp.matpower import parse_matpower
    from gridnlp.sparse.amd import amd_order

    from paper_2307_16830_b200.grids import tiled_case

    m = build_acopf(parse_matpower(tiled_case(143))).model
    st = symbolic_condense(m.hess_rows, m.hess_cols, m.jac_rows, m.jac_cols, m.n_var)
    perm = np.asarray(amd_order(st.matrix))
    np.savez_compressed(os.path.join(HERE, "C2_perm.npz"), perm=perm.astype(np.int32),
                        nnz_k=np.int64(st.matrix.indices.size))
    print("C2 perm", perm.size, "nnzK", st.matrix.indices.size)


if __name__ == "__main__":
    main()
