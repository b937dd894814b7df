"""Pin the CPU oracle (oracle/flowdmd_oracle.py) against the golden vectors
produced by the real reference in the build container (oracle/gen_golden.py)."""

import numpy as np
import pytest

import flowdmd_oracle as orc
from conftest import checksum, match_eigs


@pytest.mark.parametrize("case,r,p,q,seed", [("rsvd1", 20, 10, 2, 42), ("rsvd2", 2, 8, 2, 0),
                                             ("rsvd3", 5, 10, 2, 123), ("rsvd4", 12, 10, 1, 3)])
def test_sketch_svd_bitwise(small_golden, case, r, p, q, seed):
    g = small_golden
    U, S, V = orc.sketch_svd(g[case + "_M"], r, p, q, seed)
    np.testing.assert_allclose(S, g[case + "_S"], rtol=1e-13)
    np.testing.assert_allclose(U, g[case + "_U"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(V, g[case + "_V"], rtol=0, atol=1e-10)


def test_cholqr2_variant_close(small_golden):
    g = small_golden
    M = g["rsvd4_M"]
    U, S, V = orc.sketch_svd_cholqr2(M, 12, 10, 1, orc.draw_omega(M.shape[1], 22, 3))
    np.testing.assert_allclose(S, g["rsvd4_S"], rtol=1e-12)
    assert np.abs(U - g["rsvd4_U"]).max() < 1e-9


CASES = {
    "dmd_full8": dict(r=8, mode="full", seed=None),
    "dmd_rand6": dict(r=6, mode="randomized", seed=11),
    "dmd_noisy6": dict(r=6, mode="full", seed=None),
    "dmd_odd5": dict(r=5, mode="full", seed=None),
    "dmd_noisyrand": dict(r=8, mode="randomized", seed=5),
}


@pytest.mark.parametrize("case", list(CASES))
def test_exact_dmd_oracle(small_golden, case):
    g, c = small_golden, CASES[case]
    X = g[case + "_X"]
    o = orc.exact_dmd(X, c["r"], c["mode"], c["seed"])
    # bit-level agreement is not guaranteed across BLAS thread schedules; 1e-12 pins it
    np.testing.assert_allclose(o["lam"], g[case + "_lam"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(o["phi"], g[case + "_phi"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(o["sigma"], g[case + "_sigma"], rtol=1e-13)
    np.testing.assert_allclose(o["residual"], g[case + "_residual"], rtol=1e-9, atol=1e-11)
    np.testing.assert_array_equal(orc.partner_map(o["lam"]), g[case + "_partner"])
    table, re_idx, im_idx = orc.decode_columns(o["phi"], o["lam"])
    np.testing.assert_allclose(table, g[case + "_table"], rtol=0, atol=1e-10)
    assert [tuple(x) for x in g[case + "_reidx"]] == re_idx
    assert [tuple(x) for x in g[case + "_imidx"]] == im_idx
    z0 = orc.encode(o["phi"], X[:, 0])
    np.testing.assert_allclose(z0, g[case + "_z0"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(orc.decode(o["phi"], o["lam"], orc.step_k(o["lam"], z0, 7)), g[case + "_frame7"],
                               rtol=1e-10, atol=1e-12)
    zc = orc.eval_continuous(o["lam"], 0.1, z0, 0.337)
    np.testing.assert_allclose(zc, g[case + "_zc"], rtol=1e-10, atol=1e-13)
    za = np.zeros(c["r"], dtype=complex)
    za[0] = 1.0 + 0.5j
    np.testing.assert_allclose(orc.decode(o["phi"], o["lam"], za), g[case + "_frame_asym"], atol=1e-13)
    np.testing.assert_allclose(orc.reduced_control(o["phi"], [g[case + "_B"]])[0], g[case + "_redB"],
                               rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("case,kw", [("opt", dict(r=6)),
                                     ("opt2", dict(r=8, max_iters=10, svd_mode="randomized", seed=2))])
def test_optdmd_oracle(small_golden, case, kw):
    g = small_golden
    o = orc.optdmd(g[case + "_X"], **kw)
    np.testing.assert_allclose(o["lam"], g[case + "_lam"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(o["history"], g[case + "_hist"], rtol=1e-12)


def test_config0_oracle(config_golden):
    from paper_2502_05339_b200 import synth
    g = config_golden
    p = synth.config_params(0, seed=0)
    X = synth.generate_host(p)
    np.testing.assert_allclose(checksum(X), g["c0_checksum"], rtol=1e-13)
    o = orc.exact_dmd(X, 20, "randomized", 0)
    np.testing.assert_allclose(o["lam"], g["c0_lam"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(o["sigma"], g["c0_sigma"], rtol=1e-13)
    z0 = orc.encode(o["phi"], X[:, 0])
    fr = orc.decode(o["phi"], o["lam"], orc.step_k(o["lam"], z0, 50))
    np.testing.assert_allclose(fr, g["c0_frames_sel"][:, 2], rtol=1e-10, atol=1e-12)


def test_config1_small_oracle(config_golden):
    from paper_2502_05339_b200 import synth
    g = config_golden
    p = synth.config_params(1, seed=1, grid=24)
    X = synth.generate_host(p)
    np.testing.assert_allclose(checksum(X), g["c1s_checksum"], rtol=1e-12)
    o = orc.exact_dmd(X, 150, "randomized", 1, p=10, q=1, residual=False)
    assert match_eigs(o["lam"], g["c1s_lam"]) <= 1e-12
    np.testing.assert_allclose(o["sigma"], g["c1s_sigma"], rtol=1e-13)


def test_cholqr2_precision_on_config1_shape(config_golden):
    """The GPU orthonormalises with CholeskyQR2, not Householder; on the
    config-1 spectrum the algorithm change alone stays far inside 1e-5."""
    from paper_2502_05339_b200 import synth
    g = config_golden
    p = synth.config_params(1, seed=1, grid=24)
    X = synth.generate_host(p).astype(np.float64)
    Xx, Xp = X[:, :-1], X[:, 1:]
    om = orc.draw_omega(200, 160, 1)
    U, S, V = orc.sketch_svd_cholqr2(Xx, 150, 10, 1, om)
    np.testing.assert_allclose(S, g["c1s_sigma"], rtol=1e-10)
    K = U.T @ Xp @ (V / S)
    lam = np.linalg.eigvals(K)
    assert match_eigs(lam, g["c1s_lam"]) <= 1e-8
