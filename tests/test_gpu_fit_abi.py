"""The fit / model C ABI (include/fdmd.h: fdmd_ctx_*, fdmd_mat_*, fdmd_dmd_fit,
fdmd_model_*, fdmd_encode) driven through ctypes ALONE — numpy host buffers,
no torch and none of the package's Python layer — exactly as a flowdmd
maintainer would bind libfdmd, against the golden
outputs of the real reference (tests/golden/*.npz, oracle/gen_golden.py):
exact_dmd (dmd.py:240-274), optdmd (dmd.py:366-436), encode (runtime.py:47-52)
and decode (runtime.py:66-99). Tolerances: BASELINE north_star (sigma 1e-5
rel, lambda 1e-5 abs, frames 1e-4 rel-L2, modes up to phase)."""

import ctypes
import os
import threading

import numpy as np
import pytest

from conftest import ROOT, match_eigs, phase_aligned_error

pytestmark = pytest.mark.gpu

LIB = os.path.join(ROOT, "paper_2502_05339_b200", "libfdmd.so")
F32, F64 = 0, 1
EXACT, OPT = 0, 1
vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
PV = ctypes.POINTER(vp)


def _bind():
    if not os.path.exists(LIB):
        pytest.skip("libfdmd.so not built")
    L = ctypes.CDLL(LIB)
    sig = {
        "fdmd_last_error": (ctypes.c_char_p, []),
        "fdmd_ctx_create": (i32, [i32, i32, PV]),
        "fdmd_ctx_destroy": (i32, [vp]),
        "fdmd_mat_upload": (i32, [vp, vp, i32, i64, i64, i64, PV]),
        "fdmd_mat_free": (i32, [vp]),
        "fdmd_dmd_fit": (i32, [vp, vp, dbl, i32, i32, i32, vp, i32, i32, vp, vp, vp, vp, PV]),
        "fdmd_dmdc_fit": (i32, [vp, vp, vp, i32, dbl, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, PV]),
        "fdmd_model_info": (i32, [vp, ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(dbl),
                                  ctypes.POINTER(i32)]),
        "fdmd_model_history": (i32, [vp, vp, i32]),
        "fdmd_model_phi_to_host": (i32, [vp, vp, i64, i64, vp]),
        "fdmd_encode": (i32, [vp, vp, vp, vp]),
        "fdmd_model_decode": (i32, [vp, vp, vp, i32, vp]),
        "fdmd_model_free": (i32, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    return L


def _p(a):
    return a.ctypes.data_as(vp)


class Err(Exception):
    def __init__(self, rc, msg):
        super().__init__(f"rc={rc}: {msg}")
        self.rc = rc


@pytest.fixture(scope="module")
def abi():
    L = _bind()
    ctx = vp()
    rc = L.fdmd_ctx_create(0, 4, ctypes.byref(ctx))
    if rc != 0:
        pytest.skip("no CUDA device: " + L.fdmd_last_error().decode())
    yield L, ctx
    L.fdmd_ctx_destroy(ctx)


def chk(L, rc):
    if rc != 0:
        raise Err(rc, L.fdmd_last_error().decode())


def upload(abi, X):
    L, ctx = abi
    X = np.ascontiguousarray(X)
    dt = F32 if X.dtype == np.float32 else F64
    M = vp()
    chk(L, L.fdmd_mat_upload(ctx, _p(X), dt, X.shape[0], X.shape[1], X.shape[1], ctypes.byref(M)))
    return M


def fit(abi, X, r, seed, method=EXACT, p=10, q=2, lm_iters=0, dt=0.1):
    """The reference's _svd_of: oversample = min(p, min(n, T) - r), power_iters = q."""
    L, ctx = abi
    n, m = X.shape
    T = m - 1
    l = r + min(p, min(n, T) - r)
    omega = np.ascontiguousarray(np.random.default_rng(seed).standard_normal((T, l)))
    jitter = np.random.default_rng(0 if seed is None else seed).random(r)
    M = upload(abi, X)
    sig = np.zeros(r)
    lam = np.zeros(2 * r)
    model = vp()
    try:
        chk(L, L.fdmd_dmd_fit(ctx, M, dt, r, l, q, _p(omega), method, lm_iters, None, _p(jitter), _p(sig), _p(lam),
                              ctypes.byref(model)))
    finally:
        L.fdmd_mat_free(M)
    return model, sig, lam[0::2] + 1j * lam[1::2]


def phi_of(abi, model, n, r, row0=0, rows=None):
    L, ctx = abi
    rows = n - row0 if rows is None else rows
    out = np.zeros((rows, 2 * r))
    chk(L, L.fdmd_model_phi_to_host(ctx, model, row0, rows, _p(out)))
    return out[:, 0::2] + 1j * out[:, 1::2]


def encode(abi, model, u, r):
    L, ctx = abi
    z = np.zeros(2 * r)
    chk(L, L.fdmd_encode(ctx, model, _p(np.ascontiguousarray(u, dtype=np.float64)), _p(z)))
    return z[0::2] + 1j * z[1::2]


def decode(abi, model, Z, n):
    L, ctx = abi
    Z = np.atleast_2d(Z)
    zz = np.empty((Z.shape[0], 2 * Z.shape[1]))
    zz[:, 0::2], zz[:, 1::2] = Z.real, Z.imag
    out = np.zeros((Z.shape[0], n))
    chk(L, L.fdmd_model_decode(ctx, model, _p(zz), Z.shape[0], _p(out)))
    return out


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("case,r,seed", [("dmd_rand6", 6, 11), ("dmd_noisyrand", 8, 5)])
def test_exact_dmd_abi_small_goldens(abi, small_golden, case, r, seed):
    g = small_golden
    X = g[case + "_X"]
    n = X.shape[0]
    model, sig, lam = fit(abi, X, r, seed)
    try:
        np.testing.assert_allclose(sig, g[case + "_sigma"], rtol=1e-9)
        assert match_eigs(lam, g[case + "_lam"]) <= 1e-8
        phi = phi_of(abi, model, n, r)
        assert phase_aligned_error(phi, g[case + "_phi"]) <= 1e-7
        # the canonical phase is part of the contract: modes equal, not just up to phase
        assert np.abs(phi - g[case + "_phi"]).max() <= 1e-7 * np.abs(g[case + "_phi"]).max()
        z0 = encode(abi, model, X[:, 0], r)
        np.testing.assert_allclose(z0, g[case + "_z0"], rtol=1e-7, atol=1e-9 * np.abs(g[case + "_z0"]).max())
        f7 = decode(abi, model, lam ** 7 * z0, n)[0]
        assert rel(f7, g[case + "_frame7"]) <= 1e-8
        za = np.zeros(r, dtype=complex)
        za[0] = 1.0 + 0.5j
        assert rel(decode(abi, model, za, n)[0], g[case + "_frame_asym"]) <= 1e-8
        # chunked phi rows == the full read
        part = phi_of(abi, model, n, r, row0=7, rows=33)
        np.testing.assert_array_equal(part, phi[7:40])
    finally:
        abi[0].fdmd_model_free(model)


def test_optdmd_abi_small_golden(abi, small_golden):
    g = small_golden
    X = g["opt2_X"]
    n = X.shape[0]
    model, sig, lam = fit(abi, X, 8, 2, method=OPT, lm_iters=10)
    L = abi[0]
    try:
        np.testing.assert_allclose(sig, g["opt2_sigma"], rtol=1e-9)
        assert match_eigs(lam, g["opt2_lam"]) <= 1e-8
        assert phase_aligned_error(phi_of(abi, model, n, 8), g["opt2_phi"]) <= 1e-7
        k = L.fdmd_model_history(model, None, 0)
        hist = np.zeros(k)
        L.fdmd_model_history(model, _p(hist), k)
        np.testing.assert_allclose(hist, g["opt2_hist"], rtol=1e-8)
    finally:
        L.fdmd_model_free(model)


def test_config0_abi_full_size(abi, config_golden):
    """BASELINE config 0 exactly (n = 8192, m = 101, r = 20, p = 10, q = 2)."""
    from paper_2502_05339_b200 import synth   # the seeded host generator (input only)
    g = config_golden
    X = synth.generate_host(synth.config_params(0, seed=0))
    model, sig, lam = fit(abi, X, 20, 0)
    try:
        assert np.max(np.abs(sig - g["c0_sigma"]) / g["c0_sigma"]) <= 1e-5
        assert match_eigs(lam, g["c0_lam"]) <= 1e-5
        phi = phi_of(abi, model, X.shape[0], 20)
        assert phase_aligned_error(phi, g["c0_phi"]) <= 1e-5
        z0 = encode(abi, model, X[:, 0], 20)
        assert np.abs(z0 - g["c0_z0"]).max() <= 1e-5 * np.abs(g["c0_z0"]).max()
        fr = decode(abi, model, np.stack([lam ** k * z0 for k in (0, 1, 50, 100)]), X.shape[0])
        for j in range(4):
            assert rel(fr[j], g["c0_frames_sel"][:, j]) <= 1e-4
    finally:
        abi[0].fdmd_model_free(model)


def test_config3_shape_optdmd_abi(abi, config_golden):
    """The benched fit's shape (r = l = T = 200, q = 1, 10 LM iterations) on the
    reduced 16^3 x 3 grid, against the reference's OptDMD modes."""
    from paper_2502_05339_b200 import synth
    g = config_golden
    X = synth.generate_host(synth.config_params(3, seed=3, grid=16))
    model, sig, lam = fit(abi, X, 200, 3, method=OPT, q=1, lm_iters=10)
    try:
        assert np.max(np.abs(sig - g["c3s_opt_sigma"]) / g["c3s_opt_sigma"]) <= 1e-5
        assert match_eigs(lam, g["c3s_opt_lam"]) <= 1e-5
        head = phi_of(abi, model, X.shape[0], 200, rows=512)
        assert phase_aligned_error(head, g["c3s_opt_phi_head"]) <= 1e-5
    finally:
        abi[0].fdmd_model_free(model)


def _controlled(n, pairs, ell, m, seed, noise):
    """x_{j+1} = A x_j + B u_j with A = Psi Ablk Psi^T (known spectrum) and B in
    A's range — as BASELINE config 2 projects its control fields (synth.py). A
    B outside range(A) would add exact-zero eigenvalues whose exact-DMD modes
    Phi = X' V S^-1 U1^T U_hat W vanish (Phi = U_hat W Lambda), leaving
    pinv(Phi) undefined in those directions — for the reference algorithm too."""
    rng = np.random.default_rng(seed)
    Psi = np.linalg.qr(rng.standard_normal((n, 2 * pairs)))[0]
    rho = rng.uniform(0.9, 0.999, pairs)
    th = rng.uniform(0.05, 1.0, pairs)
    Ab = np.zeros((2 * pairs, 2 * pairs))
    eigs = []
    for i in range(pairs):
        c, s_ = np.cos(th[i]), np.sin(th[i])
        Ab[2 * i:2 * i + 2, 2 * i:2 * i + 2] = rho[i] * np.array([[c, -s_], [s_, c]])
        eigs += [rho[i] * np.exp(1j * th[i]), rho[i] * np.exp(-1j * th[i])]
    Bc = rng.standard_normal((2 * pairs, ell)) / np.sqrt(2 * pairs)
    U = rng.standard_normal((ell, m - 1))
    Z = np.empty((2 * pairs, m))
    Z[:, 0] = rng.standard_normal(2 * pairs)
    for j in range(m - 1):
        Z[:, j + 1] = Ab @ Z[:, j] + Bc @ U[:, j]
    X = Psi @ Z
    if noise:
        X = X + noise * rng.standard_normal(X.shape)
    return X, U, np.asarray(eigs)


@pytest.mark.parametrize("noise", [0.0, 1e-5])
def test_dmdc_abi_against_oracle_and_truth(abi, noise):
    """fdmd_dmdc_fit on a controlled system with known spectrum: eigenvalues
    against the oracle restatement (oracle.dmdc_fit, same Omegas) and the
    generator, and a controlled rollout z_{k+1} = lam z_k + reduced_b u_k dt
    (runtime.step_forced, runtime.py:164-200) through the model handle against
    the data."""
    import flowdmd_oracle as orc
    L, ctx = abi
    n, pairs, ell, m = 6000, 5, 3, 61
    X, U, true_eigs = _controlled(n, pairs, ell, m, seed=7, noise=noise)
    T = m - 1
    r_aug, r = 2 * pairs + ell, 2 * pairs
    l_aug, l = r_aug + 10, r + 10
    om_aug = np.random.default_rng(5).standard_normal((T, l_aug))
    om_out = np.random.default_rng(6).standard_normal((T, l))
    ref = orc.dmdc_fit(X, U, r_aug, r, seed=5, p=10, q=1)
    M = upload(abi, X)
    sig, lam, red = np.zeros(r_aug), np.zeros(2 * r), np.zeros(2 * r * ell)
    model = vp()
    try:
        chk(L, L.fdmd_dmdc_fit(ctx, M, _p(U), ell, 1.0, r_aug, l_aug, r, l, 1, _p(om_aug), _p(om_out), _p(sig),
                               _p(lam), _p(red), ctypes.byref(model)))
    finally:
        L.fdmd_mat_free(M)
    try:
        lam = lam[0::2] + 1j * lam[1::2]
        red = (red[0::2] + 1j * red[1::2]).reshape(r, ell)
        np.testing.assert_allclose(sig, ref["sigma_aug"][:r_aug], rtol=1e-9)
        assert match_eigs(lam, ref["lam"]) <= 1e-8
        d = np.array([np.abs(lam - t).min() for t in true_eigs])
        assert d.max() <= (1e-7 if noise == 0.0 else 1e-3), d.max()
        # controlled rollout through the model handle, from the data's first state
        z = encode(abi, model, X[:, 0], r)
        worst = 0.0
        for k in range(T):
            z = lam * z + red @ U[:, k]
            fr = decode(abi, model, z, n)[0]
            worst = max(worst, rel(fr, X[:, k + 1]))
        assert worst <= (1e-6 if noise == 0.0 else 1e-3), worst
    finally:
        L.fdmd_model_free(model)


def test_encode_ill_conditioned_modes_takes_qr_route(abi):
    """Two nearly parallel spatial modes (cond(phi) ~ 1e9 > 1e6): encode leaves
    the Gram route for a Householder QR of the table with the reference's SVD
    cut (pinv, linalg.py:93-104); the projection phi z matches numpy's
    pinv(phi, rcond=1e-12) u."""
    L, ctx = abi
    rng = np.random.default_rng(3)
    n, m = 400, 40
    a = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    b = a + 1e-9 * (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    lam = np.array([0.95 * np.exp(0.3j), 0.9 * np.exp(0.7j)])
    j = np.arange(m)
    X = (np.outer(a, lam[0] ** j) + np.outer(b, lam[1] ** j)).real
    X = X + 1e-12 * rng.standard_normal(X.shape)
    model, sig, lam_fit = fit(abi, X, 4, 1, p=10, q=2)
    try:
        phi = phi_of(abi, model, n, 4)
        sv = np.linalg.svd(phi, compute_uv=False)
        assert sv[0] / sv[-1] > 1e6
        u = X[:, 5]
        z = encode(abi, model, u, 4)
        z_np = np.linalg.pinv(phi, rcond=1e-12) @ u
        assert np.linalg.norm(phi @ z - phi @ z_np) <= 1e-6 * np.linalg.norm(u)
    finally:
        L.fdmd_model_free(model)


def test_abi_errors_and_concurrency(abi, small_golden):
    L, ctx = abi
    X = small_golden["dmd_rand6_X"]
    with pytest.raises(Err) as e:
        fit(abi, X, 0, 11)
    assert e.value.rc == -1
    with pytest.raises(Err) as e:
        fit(abi, X, 60, 11)
    assert e.value.rc == -1
    bad = X.copy()
    bad[3, 4] = np.nan
    with pytest.raises(Err) as e:
        upload(abi, bad)
    assert e.value.rc == -1
    with pytest.raises(Err):
        upload(abi, np.ones((4, 1)))
    # concurrent decodes on one shared model from 8 threads (server request threads)
    model, sig, lam = fit(abi, X, 6, 11)
    n = X.shape[0]
    z0 = encode(abi, model, X[:, 0], 6)
    want = decode(abi, model, z0, n)[0]
    errs = []

    def worker():
        try:
            for _ in range(20):
                got = decode(abi, model, z0, n)[0]
                if not np.array_equal(got, want):
                    errs.append("mismatch")
                zz = encode(abi, model, X[:, 0], 6)
                if not np.array_equal(zz, z0):
                    errs.append("encode mismatch")
        except Exception as exc:   # pragma: no cover - reported below
            errs.append(repr(exc))

    th = [threading.Thread(target=worker) for _ in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    L.fdmd_model_free(model)
    assert not errs, errs[:3]
