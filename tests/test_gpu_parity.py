"""Parity of the CUDA path (through the reference-mirroring API) against the
golden vectors produced by the real reference (`oracle/gen_golden.py`) and the
CPU oracle. Tolerances from BASELINE.json north_star: sigma rel <= 1e-5,
eigenvalues abs <= 1e-5, frames rel-L2 <= 1e-4, modes up to phase."""

import warnings

import numpy as np
import pytest

from conftest import aligned_coeff_error, checksum, match_eigs, phase_aligned_error

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SIG_TOL = 1e-5
LAM_TOL = 1e-5
FRAME_TOL = 1e-4


@pytest.fixture(scope="module")
def fd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_05339_b200 as fd
    return fd


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- rSVD
@pytest.mark.parametrize("case,r,p,q,seed", [("rsvd1", 20, 10, 2, 42), ("rsvd2", 2, 8, 2, 0),
                                             ("rsvd3", 5, 10, 2, 123), ("rsvd4", 12, 10, 1, 3)])
def test_randomized_svd_golden(fd, small_golden, case, r, p, q, seed):
    g = small_golden
    M = g[case + "_M"]
    res = fd.randomized_svd(M, r, oversample=p, power_iters=q, seed=seed)
    np.testing.assert_allclose(res.S, g[case + "_S"], rtol=1e-9, atol=1e-12 * g[case + "_S"][0])
    # canonicalised factors: identical up to rounding (sign convention mirrored)
    if case != "rsvd2":  # rsvd2 has a degenerate null space; only its leading factors are defined
        assert np.abs(res.U - g[case + "_U"]).max() <= 1e-7
        assert np.abs(res.V - g[case + "_V"]).max() <= 1e-7
    np.testing.assert_allclose(res.reconstruct(), (g[case + "_U"] * g[case + "_S"]) @ g[case + "_V"].T,
                               atol=1e-8 * g[case + "_S"][0])


def test_randomized_svd_deterministic(fd, small_golden):
    M = small_golden["rsvd3_M"]
    a = fd.randomized_svd(M, 5, seed=123)
    b = fd.randomized_svd(M, 5, seed=123)
    assert np.array_equal(a.U, b.U) and np.array_equal(a.S, b.S) and np.array_equal(a.V, b.V)


def test_randomized_svd_errors(fd):
    with pytest.raises(ValueError):
        fd.randomized_svd(np.eye(8), 5, oversample=10)
    with pytest.raises(ValueError):
        fd.randomized_svd(np.eye(8), 0)


def test_truncated_svd(fd):
    res = fd.truncated_svd(np.diag([3.0, 2.0, 1.0]), 2)
    np.testing.assert_allclose(res.S, [3.0, 2.0])
    with pytest.raises(ValueError):
        fd.truncated_svd(np.eye(3), 4)


# ---------------------------------------------------------------- exact DMD on the reference's test systems
SMALL = {
    "dmd_full8": dict(r=8, mode="full", seed=None),
    "dmd_rand6": dict(r=6, mode="randomized", seed=11),
    "dmd_noisy6": dict(r=6, mode="full", seed=None),
    "dmd_odd5": dict(r=5, mode="full", seed=None),
    "dmd_noisyrand": dict(r=8, mode="randomized", seed=5),
}


@pytest.mark.parametrize("case", list(SMALL))
def test_exact_dmd_golden(fd, small_golden, case):
    g, c = small_golden, SMALL[case]
    X = g[case + "_X"]
    model = fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), c["r"], svd_mode=c["mode"], seed=c["seed"])
    assert match_eigs(model.lam, g[case + "_lam"]) <= LAM_TOL * 1e-3
    np.testing.assert_allclose(model.sigma, g[case + "_sigma"], rtol=1e-9)
    assert phase_aligned_error(model.phi, g[case + "_phi"]) <= 1e-7
    np.testing.assert_array_equal(model.pair_partner, g[case + "_partner"])
    assert abs(model.provenance["residual_rel"] - g[case + "_residual_rel"]) <= 1e-9 + 1e-6 * g[case + "_residual_rel"]
    # decode table layout (dmd.py:92-120)
    table, re_idx, im_idx = model.decode_table()
    assert [tuple(x) for x in g[case + "_reidx"]] == [tuple(x) for x in re_idx]
    assert [tuple(x) for x in g[case + "_imidx"]] == [tuple(x) for x in im_idx]
    assert np.abs(table - g[case + "_table"]).max() <= 1e-7 * np.abs(g[case + "_table"]).max()
    # runtime on the device table
    z0 = fd.encode(model, X[:, 0])
    np.testing.assert_allclose(z0.z, g[case + "_z0"], rtol=1e-7, atol=1e-9 * np.abs(g[case + "_z0"]).max())
    assert rel(fd.decode(model, fd.step_k(model, z0, 7)), g[case + "_frame7"]) <= 1e-8
    zc = fd.eval_continuous(model, z0, 3.37 * 0.1)
    assert rel(fd.decode(model, zc), g[case + "_framec"]) <= 1e-8
    za = np.zeros(model.r, dtype=complex)
    za[0] = 1.0 + 0.5j
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert rel(fd.decode(model, za), g[case + "_frame_asym"]) <= 1e-8
    ctrl = fd.fit_control(model, [g[case + "_B"]])
    np.testing.assert_allclose(ctrl.reduced_b[0], g[case + "_redB"], atol=1e-8 * np.abs(g[case + "_redB"]).max())


def test_exact_dmd_determinism(fd, small_golden):
    X = small_golden["dmd_rand6_X"]
    a = fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 6, svd_mode="randomized", seed=11)
    b = fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 6, svd_mode="randomized", seed=11)
    assert np.array_equal(a.lam, b.lam)


def test_exact_dmd_errors(fd, small_golden):
    X = small_golden["dmd_full8_X"]
    with pytest.raises(ValueError):
        fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 0)
    with pytest.raises(ValueError):
        fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 60)
    with pytest.raises(ValueError):
        fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 20)   # rank-8 data: sigma_20 numerically zero
    with pytest.raises(ValueError):
        fd.SnapshotMatrix(np.ones((4, 1)), 0.1)
    bad = np.ones((4, 3))
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        fd.SnapshotMatrix(bad, 0.1)


def test_scalar_and_rotation(fd):
    m = fd.exact_dmd(fd.SnapshotMatrix(np.array([[1.0, 0.9, 0.81]]), 1.0), 1)
    np.testing.assert_allclose(m.lam, [0.9], atol=1e-12)
    th = 0.1
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    x = np.array([1.0, 0.3])
    cols = np.empty((2, 30))
    for k in range(30):
        cols[:, k] = x
        x = R @ x
    m = fd.exact_dmd(fd.SnapshotMatrix(cols, 1.0), 2)
    np.testing.assert_allclose(np.sort_complex(m.lam), np.sort_complex([np.exp(1j * th), np.exp(-1j * th)]), atol=1e-10)


# ---------------------------------------------------------------- OptDMD
@pytest.mark.parametrize("case,kw", [("opt", dict(r=6)),
                                     ("opt2", dict(r=8, iters=10, mode="randomized", seed=2))])
def test_optdmd_golden(fd, small_golden, case, kw):
    g = small_golden
    X = g[case + "_X"]
    cfg = fd.LMConfig(max_iters=kw.get("iters", 200))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        model = fd.optdmd(fd.SnapshotMatrix(X, 0.1), kw["r"], lm_config=cfg,
                          svd_mode=kw.get("mode", "full"), seed=kw.get("seed"))
    assert match_eigs(model.lam, g[case + "_lam"]) <= 1e-7
    hist = np.array(model.provenance["objective_history"])
    np.testing.assert_allclose(hist[0], g[case + "_hist"][0], rtol=1e-8)
    assert hist[-1] <= g[case + "_hist"][-1] * (1 + 1e-6)
    assert phase_aligned_error(model.phi, g[case + "_phi"]) <= 1e-5


# ---------------------------------------------------------------- BASELINE configs
def test_config0_full(fd, config_golden):
    from paper_2502_05339_b200 import synth
    g = config_golden
    p = synth.config_params(0, seed=0)
    X = synth.generate_host(p)
    np.testing.assert_allclose(checksum(X), g["c0_checksum"], rtol=1e-12)
    model = fd.exact_dmd(fd.SnapshotMatrix(X, synth.DT), 20, svd_mode="randomized", seed=0)
    assert np.abs(model.sigma - g["c0_sigma"]).max() <= SIG_TOL * g["c0_sigma"].min()
    assert match_eigs(model.lam, g["c0_lam"]) <= LAM_TOL
    assert phase_aligned_error(model.phi, g["c0_phi"]) <= 1e-4
    z0 = fd.encode(model, X[:, 0])
    assert aligned_coeff_error(model.phi, g["c0_phi"], z0.z, g["c0_z0"]) <= 1e-5
    Z = np.stack([fd.step_k(model, z0, k).z for k in range(101)], axis=1)
    frames = fd.decode_batch(model, Z).double().cpu().numpy().T
    sel = frames[:, [0, 1, 50, 100]]
    for j in range(4):
        assert rel(sel[:, j], g["c0_frames_sel"][:, j]) <= FRAME_TOL
    np.testing.assert_allclose(frames.sum(0), g["c0_frames_checksum"][0], rtol=1e-4, atol=1e-6)


def test_config1_reduced_grid(fd, config_golden):
    """Config 1's spectrum/rank/(p, q) on a 24^3 x 3 grid (reference run with q=1)."""
    from paper_2502_05339_b200 import synth
    g = config_golden
    p = synth.config_params(1, seed=1, grid=24)
    X = synth.generate_host(p)
    np.testing.assert_allclose(checksum(X), g["c1s_checksum"], rtol=1e-10)
    model = fd.exact_dmd(fd.SnapshotMatrix(X, synth.DT), 150, svd_mode="randomized", seed=1,
                         oversample=10, power_iters=1)
    assert np.abs(model.sigma - g["c1s_sigma"]).max() <= SIG_TOL * g["c1s_sigma"].min()
    assert match_eigs(model.lam, g["c1s_lam"]) <= LAM_TOL
    np.testing.assert_allclose(np.linalg.norm(model.phi, axis=0), 1.0, atol=1e-6)
    # modes up to phase (BASELINE tolerance), on the reference's first 512 rows
    assert phase_aligned_error(model.phi[:512], g["c1s_phi_head"]) <= 1e-5
    z0 = fd.encode(model, X[:, 0])
    assert aligned_coeff_error(model.phi[:512], g["c1s_phi_head"], z0.z, g["c1s_z0"]) <= 1e-5
    fr = np.stack([fd.decode(model, fd.step_k(model, z0, k)) for k in (1, 100, 200)], axis=1)
    for j in range(3):
        assert rel(fr[:4096, j], g["c1s_frames_head"][:, j]) <= FRAME_TOL
    np.testing.assert_allclose(fr.sum(0), g["c1s_frames_checksum"][0], rtol=1e-3, atol=1e-3)


def test_config3_reduced_grid_exact_and_opt(fd, config_golden):
    """Config 3's r = T = 200 (clamped l) on a 16^3 x 3 grid, exact DMD + 10 LM iterations."""
    from paper_2502_05339_b200 import synth
    g = config_golden
    p = synth.config_params(3, seed=3, grid=16)
    X = synth.generate_host(p)
    np.testing.assert_allclose(checksum(X), g["c3s_checksum"], rtol=1e-10)
    data = fd.SnapshotMatrix(X, synth.DT)
    model = fd.exact_dmd(data, 200, svd_mode="randomized", seed=3, oversample=10, power_iters=1)
    assert model.provenance["sketch"]["l"] == 200
    assert np.abs(model.sigma - g["c3s_sigma"]).max() <= SIG_TOL * g["c3s_sigma"].min()
    assert match_eigs(model.lam, g["c3s_lam"]) <= LAM_TOL
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mo = fd.optdmd(data, 200, lm_config=fd.LMConfig(max_iters=10), svd_mode="randomized", seed=3,
                       oversample=10, power_iters=1)
    assert match_eigs(mo.lam, g["c3s_opt_lam"]) <= LAM_TOL
    # the benched fit's modes (tcgen05 lift / modes path for fp32 tables), up to phase
    assert phase_aligned_error(mo.phi[:512], g["c3s_opt_phi_head"]) <= 1e-5
    # r = T: the varpro objective starts at round-off level in both implementations
    assert mo.provenance["objective_history"][0] <= 1e-12 * g["c3s_opt_sigma"][0]
    assert g["c3s_opt_hist"][0] <= 1e-12 * g["c3s_opt_sigma"][0]


# ---------------------------------------------------------------- reconstruct batch APIs
def test_reconstruct_matches_eval_continuous(fd, small_golden):
    X = small_golden["dmd_noisyrand_X"]
    model = fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 8, svd_mode="randomized", seed=5)
    z0 = fd.encode(model, X[:, 0])
    times = np.array([0.0, 0.05, 1.0, 2.37, 5.0])
    got = fd.reconstruct(model, z0, times).double().cpu().numpy()
    for j, t in enumerate(times):
        want = fd.decode(model, fd.eval_continuous(model, z0, t))
        assert rel(got[j], want) <= 1e-12


def test_rollout_matches_steps(fd, small_golden):
    X = small_golden["dmd_full8_X"]
    model = fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 8)
    z0 = fd.encode(model, X[:, 0])
    frames, dens = fd.rollout(model, z0, 25)
    assert dens is None and frames.shape == (model.n, 25)
    np.testing.assert_allclose(frames[:, -1], fd.decode(model, fd.step_k(model, z0, 25)), rtol=1e-10, atol=1e-13)


def test_modal_basis_config4_formula(fd):
    rng = np.random.default_rng(0)
    n, r, B = 50000, 24, 7
    Uh = np.linalg.qr(rng.standard_normal((n, r)))[0].astype(np.float32)
    from paper_2502_05339_b200.device import alloc_tall
    U = alloc_tall(n, r, torch.float32, "col")
    U.buf[:r, :n].copy_(torch.as_tensor(Uh.T))
    W = rng.standard_normal((r, r)) + 1j * rng.standard_normal((r, r))
    lam = 0.99 * np.exp(1j * rng.uniform(0, 3, r))
    b = rng.standard_normal(r) + 1j * rng.standard_normal(r)
    for B in (7, 64):                       # SIMT GEMV/GEMM path and the tcgen05 path
        t = rng.uniform(0, 300, B)
        mb = fd.ModalBasis(U, W, lam, b)
        got = mb.reconstruct(t).double().cpu().numpy()
        want = (Uh.astype(np.float64) @ np.real(W @ (lam[:, None] ** t[None, :] * b[:, None]))).T
        err = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
        assert err.max() <= FRAME_TOL


def test_optdmd_tcgen05_lift_and_modes_match_dmma(fd):
    """fp32 tables: the tcgen05 lift / modes (FP16 2-way split, FP32-accurate)
    against the FP64 DMMA path on the same fit — eigenvalues identical (they
    never touch the tall products), modes and frames to FP32 accuracy."""
    from conftest import phase_aligned_error
    from paper_2502_05339_b200 import dmd, synth
    p = synth.config_params(3, seed=3, grid=16)
    X = synth.generate_host(p)
    assert X.dtype == np.float32
    kw = dict(lm_config=fd.LMConfig(max_iters=10), svd_mode="randomized", seed=3, oversample=10, power_iters=1,
              keep_basis=True)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = fd.optdmd(fd.SnapshotMatrix(X, synth.DT), 200, **kw)
        old = dmd._TC_FIT
        dmd._TC_FIT = False
        try:
            b = fd.optdmd(fd.SnapshotMatrix(X, synth.DT), 200, **kw)
        finally:
            dmd._TC_FIT = old
    np.testing.assert_array_equal(a.lam, b.lam)
    assert phase_aligned_error(a.phi, b.phi) <= 1e-5
    Ua = a.basis_U.view().double().cpu().numpy()
    Ub = b.basis_U.view().double().cpu().numpy()
    assert np.abs(Ua - Ub).max() <= 5e-6 * np.abs(Ub).max()      # FP32-accurate products, fp32 storage
    z0 = fd.encode(b, X[:, 0])
    fa = fd.decode(a, fd.step_k(a, z0, 50))
    fb = fd.decode(b, fd.step_k(b, z0, 50))
    assert rel(fa, fb) <= 1e-5


def test_optdmd_basis_planes_match_fp32_basis(fd):
    """keep_basis="planes" (the lift writes the config-4 basis straight into
    the fp16 hi/lo planes, the bench's schedule) against keep_basis=True (fp32
    U, then the split): same eigenvalues, U to FP32 accuracy, and the same
    config-4 frames u(t) = U Re(W Lam^t b)."""
    from paper_2502_05339_b200 import synth
    from paper_2502_05339_b200.runtime import ModalBasis
    p = synth.config_params(3, seed=3, grid=16)
    X = synth.generate_host(p)
    kw = dict(lm_config=fd.LMConfig(max_iters=10), svd_mode="randomized", seed=3, oversample=10, power_iters=1)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        a = fd.optdmd(fd.SnapshotMatrix(X, synth.DT), 200, keep_basis=True, **kw)
        b = fd.optdmd(fd.SnapshotMatrix(X, synth.DT), 200, keep_basis="planes", **kw)
    np.testing.assert_array_equal(a.lam, b.lam)
    pl = b.basis_U
    Ua = a.basis_U.view().double().cpu().numpy()
    Ub = ((pl["uh"].double() + pl["ul"].double()) / pl["su"]).cpu().numpy()[:, :200]
    assert np.abs(Ua - Ub).max() <= 2e-6 * np.abs(Ua).max()
    rng = np.random.default_rng(4)
    lam4 = rng.uniform(0.9, 0.999, 200) * np.exp(1j * rng.uniform(0.05, 1.0, 200))
    W4 = (rng.standard_normal((200, 200)) + 1j * rng.standard_normal((200, 200))) / np.sqrt(400)
    b4 = rng.standard_normal(200) + 1j * rng.standard_normal(200)
    times = rng.uniform(0.0, 300.0, 300)
    fa = ModalBasis(a.basis_U, W4, lam4, b4).reconstruct(times).double()
    fb = ModalBasis(pl, W4, lam4, b4).reconstruct(times).double()
    err = torch.linalg.vector_norm(fa - fb, dim=1) / torch.linalg.vector_norm(fa, dim=1)
    assert float(err.max()) <= 4e-6
    f1 = ModalBasis(pl, W4, lam4, b4).reconstruct(times[:1]).double()     # B = 1 from the planes
    assert float(torch.linalg.vector_norm(f1[0] - fa[0]) / torch.linalg.vector_norm(fa[0])) <= 4e-6


# ---------------------------------------------------------------- frames of the benched fit vs the reference
@pytest.fixture(scope="module")
def frames_golden():
    import os
    from conftest import GOLDEN
    return dict(np.load(os.path.join(GOLDEN, "config_frames.npz")))


@pytest.mark.parametrize("tc_fit", [True, False], ids=["tcgen05_lift_modes", "dmma_lift_modes"])
@pytest.mark.parametrize("method", ["opt", "exact"])
def test_config3_shape_frames_match_reference(fd, frames_golden, method, tc_fit):
    """What a user of the benched fit sees — z0 = encode(x0), decode(step_k)
    and a continuous-time frame — against frames the reference decoded from
    its own model (oracle/gen_golden.py frame_cases), with the tcgen05 lift /
    modes path (fp32 tables, the bench) and the FP64 DMMA path."""
    from paper_2502_05339_b200 import dmd, synth
    g = frames_golden
    p = synth.config_params(3, seed=3, grid=16)
    X = synth.generate_host(p)
    np.testing.assert_allclose(checksum(X), g["c3s_checksum"], rtol=1e-10)
    old = dmd._TC_FIT
    dmd._TC_FIT = tc_fit
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            data = fd.SnapshotMatrix(X, synth.DT)
            kw = dict(svd_mode="randomized", seed=3, oversample=10, power_iters=1)
            if method == "opt":
                model = fd.optdmd(data, 200, lm_config=fd.LMConfig(max_iters=10), **kw)
            else:
                model = fd.exact_dmd(data, 200, **kw)
            z0 = fd.encode(model, X[:, 0])
            fr = np.stack([fd.decode(model, fd.step_k(model, z0, k)) for k in (1, 50, 199)]
                          + [fd.decode(model, fd.eval_continuous(model, z0, 12.37))], axis=1)
    finally:
        dmd._TC_FIT = old
    assert match_eigs(model.lam, g[f"c3s_{method}_lam"]) <= LAM_TOL
    np.testing.assert_allclose(np.linalg.norm(model.phi, axis=0), g[f"c3s_{method}_phi_norms"], atol=1e-6)
    head = g[f"c3s_{method}_frames_head"]
    for j in range(fr.shape[1]):
        assert rel(fr[:4096, j], head[:, j]) <= FRAME_TOL, j
    np.testing.assert_allclose(fr.sum(0), g[f"c3s_{method}_frames_checksum"][0], rtol=FRAME_TOL,
                               atol=FRAME_TOL * np.abs(fr).sum(0).max())
    np.testing.assert_allclose((fr * fr).sum(0), g[f"c3s_{method}_frames_checksum"][1], rtol=2 * FRAME_TOL)


# ---------------------------------------------------------------- which sketch route runs
def test_long_series_takes_explicit_sketch_route(fd):
    """T >> l: the snapshot Gram X^T X would cost n T^2 > 2 n T l (1 + q), so
    the explicit Y = X Omega / X^T Q route runs — with the reference's factors."""
    import flowdmd_oracle as orc
    from paper_2502_05339_b200 import linalg as la
    rng = np.random.default_rng(0)
    n, T, r, p, q = 20000, 1000, 10, 10, 2
    M = rng.standard_normal((n, 12)) @ rng.standard_normal((12, T)) + 1e-3 * rng.standard_normal((n, T))
    assert not la.gram_route_ok(T, r + p, q)
    f = la.sketch_factors(la.as_tall(M), T, r + p, q, la.draw_omega(T, r + p, 4))
    assert "implicit_sketch" not in f.stats and "gram_first_pass" not in f.stats
    res = fd.randomized_svd(M, r, oversample=p, power_iters=q, seed=4)
    _, S, _ = orc.sketch_svd(M, r, p, q, 4)
    np.testing.assert_allclose(res.S, S, rtol=1e-10)


def test_rank_deficient_sketch_falls_back_under_gram_route(fd):
    """Exactly rank-5 data sketched at l = 18 with the snapshot-Gram route
    available: chol(Omega^T G_X Omega) is singular, so the explicit route and
    its shifted-CholeskyQR3 / Householder fallbacks run; the 5 nonzero singular
    values still match the reference algorithm (Householder QR)."""
    import flowdmd_oracle as orc
    from paper_2502_05339_b200 import linalg as la
    rng = np.random.default_rng(1)
    n, T, r, p, q = 5000, 60, 8, 10, 1
    M = rng.standard_normal((n, 5)) @ rng.standard_normal((5, T))
    assert la.gram_route_ok(T, r + p, q)
    f = la.sketch_factors(la.as_tall(M), T, r + p, q, la.draw_omega(T, r + p, 9))
    assert "implicit_sketch" not in f.stats
    assert f.stats.get("householder_fallback", 0) + f.stats.get("shifted_cholqr3", 0) >= 1, f.stats
    res = fd.randomized_svd(M, r, oversample=p, power_iters=q, seed=9)
    _, S, _ = orc.sketch_svd(M, r, p, q, 9)
    np.testing.assert_allclose(res.S[:5], S[:5], rtol=1e-9)
    assert np.all(res.S[5:] <= 1e-9 * res.S[0])
