"""The C-ABI boundary (include/gridopf.h) on CPU: the library loads, exports
every function the header declares, the ctypes signature table covers them,
and host-only entry points and error reporting work without a GPU."""
import ctypes
import os
import re

import numpy as np

from conftest import REPO

HEADER = os.path.join(REPO, "include", "gridopf.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2307_16830_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH) if hasattr(_lib, "LIB_PATH") else _lib.lib()
    names = declared_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_signature_table_covers_the_header():
    from paper_2307_16830_b200 import _lib

    table = set(_lib._SIGS) if hasattr(_lib, "_SIGS") else None
    if table is None:   # the table is the module-level dict of (restype, argtypes)
        table = {k for k, v in vars(_lib).items() if isinstance(v, dict)
                 for k in v if str(k).startswith("gn_")}
    missing = [n for n in declared_functions() if n not in table]
    assert not missing, missing


def test_host_entry_points_and_error_reporting():
    from paper_2307_16830_b200 import _lib, sparse

    lib = _lib.lib()
    assert lib.gn_version() > 0
    # error path: an upper-triangle coordinate is rejected with a message
    rows = np.array([0], np.int64)
    cols = np.array([1], np.int64)
    nnz = ctypes.c_int64()
    rc = lib.gn_coo_to_csc(2, 1, _lib.ptr(rows), _lib.ptr(cols), ctypes.byref(nnz), None, None, None)
    assert rc < 0
    assert b"above the diagonal" in lib.gn_last_error()
    # a host-only round trip: tridiagonal pattern, ordering, symbolic factor
    n = 6
    r = np.r_[np.arange(n), np.arange(1, n)]
    c = np.r_[np.arange(n), np.arange(n - 1)]
    m, _ = sparse.coo_to_csc(n, r, c, np.ones(r.size))
    perm = sparse.amd_order(m)
    assert sorted(perm.tolist()) == list(range(n))
    sym = sparse.symbolic_cholesky(m, perm)
    assert sym.factor_nnz == 2 * n - 1
