"""`fdmd_rsvd` — the randomized SVD as one C-ABI call —
called through ctypes with raw device pointers, exactly as a flowdmd
maintainer would bind it, against the reference's golden
factors (tests/golden/small_cases.npz, written by the real reference) and
against the package's own randomized_svd at a config-1-like size."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2502_05339_b200 import _lib
    return _lib


def rsvd_abi(lib, X: torch.Tensor, T, r, l, q, omega):
    """X: (n, ld) device tensor, f32/f64 row-major; returns (S, V, U host)."""
    n = X.shape[0]
    S = np.zeros(r)
    V = np.zeros((T, r))
    U = torch.empty((r, n), dtype=torch.float64, device=X.device)
    om = np.ascontiguousarray(omega, dtype=np.float64)
    dt = lib.F32 if X.dtype == torch.float32 else lib.F64
    rc = lib.lib().fdmd_rsvd(ctypes.c_void_p(X.data_ptr()), dt, X.stride(0), n, T, r, l, q,
                             om.ctypes.data_as(ctypes.c_void_p), S.ctypes.data_as(ctypes.c_void_p),
                             V.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(U.data_ptr()), n,
                             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    lib.check(rc, "fdmd_rsvd")
    return S, V, U.t().cpu().numpy()


def _device(M, dtype=torch.float64):
    n, T = M.shape
    q = 16 // torch.empty((), dtype=dtype).element_size()
    ld = (T + q - 1) // q * q
    X = torch.zeros((n, ld), dtype=dtype, device="cuda")
    X[:, :T] = torch.as_tensor(M, dtype=dtype)
    return X


@pytest.mark.parametrize("case,r,p,q,seed", [("rsvd1", 20, 10, 2, 42), ("rsvd3", 5, 10, 2, 123),
                                             ("rsvd4", 12, 10, 1, 3)])
def test_rsvd_abi_matches_reference_goldens(lib, small_golden, case, r, p, q, seed):
    g = small_golden
    M = g[case + "_M"]
    T = M.shape[1]
    omega = np.random.default_rng(seed).standard_normal((T, r + p))
    S, V, U = rsvd_abi(lib, _device(M), T, r, r + p, q, omega)
    np.testing.assert_allclose(S, g[case + "_S"], rtol=1e-9, atol=1e-12 * g[case + "_S"][0])
    assert np.abs(U - g[case + "_U"]).max() <= 1e-7
    assert np.abs(V - g[case + "_V"]).max() <= 1e-7


def test_rsvd_abi_matches_python_path_at_scale(lib):
    """f32 snapshots, n = 500,000, T = 201, r = 150, l = 160, q = 1 (config 1's
    shape on fewer rows): same factors as fd.randomized_svd to rounding."""
    import paper_2502_05339_b200 as fd
    rng = np.random.default_rng(7)
    n, T, r, l = 500_000, 201, 150, 160
    k = 40
    base = (rng.standard_normal((n, k)) @ (rng.standard_normal((k, T)) * np.exp(-np.arange(k) / 8.0)[:, None])
            + 1e-3 * rng.standard_normal((n, T))).astype(np.float32)
    X = _device(base, torch.float32)
    omega = np.random.default_rng(11).standard_normal((T, l))
    S, V, U = rsvd_abi(lib, X, T, r, l, 1, omega)
    ref = fd.randomized_svd(X[:, :T], r, oversample=l - r, power_iters=1, seed=11)
    np.testing.assert_allclose(S, ref.S, rtol=1e-10)
    lead = 30   # well-separated leading factors (the tail sits at the noise floor)
    assert np.abs(U[:, :lead] - ref.U[:, :lead]).max() <= 1e-8
    assert np.abs(V[:, :lead] - ref.V[:, :lead]).max() <= 1e-8


def test_rsvd_abi_errors(lib):
    X = _device(np.eye(8))
    with pytest.raises(ValueError, match="rank"):
        rsvd_abi(lib, X, 8, 0, 4, 1, np.zeros((8, 4)))
    with pytest.raises(ValueError):
        rsvd_abi(lib, X, 8, 5, 10, 1, np.zeros((8, 10)))      # l > T
