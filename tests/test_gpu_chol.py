"""GPU multifrontal Cholesky on matrices with LARGE fronts (CTA + DMMA path).

The ACOPF parity cases at 14-118 buses only produce warp-sized fronts
(<= 32 rows); these matrices force the CTA-per-front kernel, multi-panel
fronts (w > 32), the NB=16 panel variant (fronts > ~780 rows) and pivot
failures inside a large front.  Oracle: oracle/sparse.py (the reference's
up-looking kernel, cholesky.py:147-186, restated in C) on the same
symbolic structure, plus numpy dense checks.

Tolerances: ||L_gpu - L_oracle||_inf <= 1e-12 ||L_oracle||_inf; solves
<= 1e-10 relative residual; failing column identical to the oracle's.
"""
import numpy as np
import pytest

from oracle import sparse as OS

pytestmark = pytest.mark.gpu

from paper_2307_16830_b200 import sparse as S  # noqa: E402


def grid_laplacian(k, shift=0.1, seed=0):
    rng = np.random.default_rng(seed)
    n = k * k
    rows, cols, vals = [], [], []
    diag = np.full(n, shift)
    for i in range(k):
        for j in range(k):
            a = i * k + j
            for b in ([a + 1] if j + 1 < k else []) + ([a + k] if i + 1 < k else []):
                w = rng.uniform(0.5, 1.5)
                rows.append(b)
                cols.append(a)
                vals.append(-w)
                diag[a] += w
                diag[b] += w
    rows += list(range(n))
    cols += list(range(n))
    vals += list(diag)
    return S.coo_to_csc(n, np.array(rows), np.array(cols), np.array(vals))[0]


def dense_spd(n, seed):
    rng = np.random.default_rng(seed)
    M = rng.normal(size=(n, n))
    A = M @ M.T / n + np.eye(n)
    ri, ci = np.tril_indices(n)
    return S.coo_to_csc(n, ri, ci, A[ri, ci])[0], A


def check_against_oracle(m, perm):
    sym = S.symbolic_cholesky(m, perm)
    f = S.factorize(sym, m.values)
    om, _ = OS.coo_to_csc(m.n, *m.coords(), m.values)
    osym = OS.symbolic(om, perm)
    lo, ok, bad = OS.factorize(osym, om.values)
    assert f.ok == ok
    if not ok:
        assert f.failing_column == bad
        return sym, f
    lg = f.values
    assert np.max(np.abs(lg - lo)) <= 1e-12 * np.max(np.abs(lo))
    rng = np.random.default_rng(1)
    A = m.to_dense() if m.n <= 3000 else None
    for _ in range(3):
        b = rng.normal(size=m.n)
        x = S.solve(f, b)
        xo = OS.solve(osym, lo, b)
        assert np.max(np.abs(x - xo)) <= 1e-10 * max(1.0, np.max(np.abs(xo)))
        if A is not None:
            assert np.max(np.abs(A @ x - b)) <= 1e-10 * np.max(np.abs(b)) * max(1.0, np.abs(A).max())
    return sym, f


@pytest.mark.parametrize("k", [24, 60])
def test_grid_laplacian_min_degree(k):
    m = grid_laplacian(k)
    sym, _ = check_against_oracle(m, S.amd_order(m))
    if k == 60:
        assert sym.info["max_front"] > 32   # the CTA path ran


@pytest.mark.parametrize("n", [40, 200, 330])
def test_dense_front_multi_panel(n):
    m, A = dense_spd(n, n)
    sym, f = check_against_oracle(m, np.arange(n))
    assert sym.info["max_front"] == n
    L = np.zeros((n, n))
    r, c = sym.l_rowidx, np.repeat(np.arange(n), np.diff(sym.l_colptr))
    L[r, c] = f.values
    assert np.max(np.abs(L @ L.T - A)) <= 1e-12 * np.abs(A).max()


def test_dense_front_nb16_panel():
    m, _ = dense_spd(900, 9)   # 32-column panel would not fit in shared memory
    check_against_oracle(m, np.arange(900))


@pytest.mark.parametrize("shift_frac", [0.3, 0.9])
def test_failure_inside_large_front(shift_frac):
    m, A = dense_spd(150, 3)
    ev = np.linalg.eigvalsh(A)
    shift = ev.min() + shift_frac * (ev.max() - ev.min())
    ri, ci = np.tril_indices(150)
    B = A - shift * np.eye(150)
    mb = S.coo_to_csc(150, ri, ci, B[ri, ci])[0]
    _, f = check_against_oracle(mb, np.arange(150))
    assert not f.ok


def test_refactor_bitwise_large():
    m = grid_laplacian(50, seed=3)
    sym = S.symbolic_cholesky(m, S.amd_order(m))
    a = S.factorize(sym, m.values).values
    b = S.factorize(sym, m.values).values
    assert np.array_equal(a, b)


def test_dense_front_nb16_three_rows_per_thread():
    m, _ = dense_spd(700, 7)   # 16-column panels, 3 rows per thread, two panel buffers
    check_against_oracle(m, np.arange(700))


@pytest.mark.parametrize("n", [200, 330])
def test_double_buffered_panels_bitwise_equal_single_buffer(n, monkeypatch):
    """The next panel built in shared memory by the strip update (two panel
    buffers) is bitwise the one reloaded from the front (one buffer)."""
    m, _ = dense_spd(n, n + 1)
    sym = S.symbolic_cholesky(m, np.arange(n))
    two = S.factorize(sym, m.values).values
    monkeypatch.setenv("GN_SINGLE_PANEL_BUFFER", "1")
    one = S.factorize(sym, m.values).values
    assert np.array_equal(one, two)
    g = grid_laplacian(60, seed=5)   # CTA-per-front kernel below the top fronts
    gs = S.symbolic_cholesky(g, S.amd_order(g))
    one = S.factorize(gs, g.values).values
    monkeypatch.delenv("GN_SINGLE_PANEL_BUFFER")
    assert np.array_equal(one, S.factorize(gs, g.values).values)


def test_measured_dmma_peak_is_plausible():
    import ctypes

    import torch

    from paper_2307_16830_b200 import _lib as L

    tf = ctypes.c_double()
    L.check(L.lib().gn_measure_dmma_peak(ctypes.byref(tf), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    assert 5.0 < tf.value < 200.0   # B200 FP64 tensor cores: ~37 TFLOP/s
