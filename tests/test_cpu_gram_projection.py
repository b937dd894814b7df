"""Projection from the snapshot Gram (linalg.PROJ_GRAM_TOL):
the route decision and its accuracy against the REAL reference's goldens
(tests/golden/config_cases.npz, oracle/gen_golden.py), on CPU with the
checker standing in for libfdmd (tests/cpu_ops.py). Config 3's shape
(r = T = 200, the benched fit) must take the route and stay within 1e-7 of
the reference; config 1's (r = 150 inside the noise cluster) must keep the
direct Q^T S route and its 1e-10 agreement."""

import numpy as np
import pytest
import torch

from conftest import match_eigs, phase_aligned_error


def _fit(X, r, seed, method):
    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200 import device as dv
    from paper_2502_05339_b200 import synth
    from cpu_ops import CpuOps
    prev = dv.set_ops(CpuOps())
    try:
        data = fd.SnapshotMatrix(torch.as_tensor(X), synth.DT, device=torch.device("cpu"))
        if method == "opt":
            return fd.optdmd(data, r, svd_mode="randomized", seed=seed, oversample=10, power_iters=1,
                             lm_config=fd.LMConfig(max_iters=10))
        return fd.exact_dmd(data, r, svd_mode="randomized", seed=seed, oversample=10, power_iters=1)
    finally:
        dv.set_ops(prev)


@pytest.fixture(scope="module")
def c3s():
    from paper_2502_05339_b200 import synth
    return synth.generate_host(synth.config_params(3, seed=3, grid=16))


def test_config3_shape_takes_the_gram_projection(c3s, config_golden):
    g = config_golden
    model = _fit(c3s, 200, 3, "exact")
    st = model.provenance["sketch"]
    assert st.get("gram_projection") == 1 and st["proj_gram_bound"] <= 1e-7, st
    assert np.max(np.abs(model.sigma - g["c3s_sigma"]) / g["c3s_sigma"]) <= 1e-7
    assert match_eigs(model.lam, g["c3s_lam"]) <= 1e-7


def test_config3_optdmd_gram_projection_modes(c3s, config_golden):
    g = config_golden
    mo = _fit(c3s, 200, 3, "opt")
    assert mo.provenance["sketch"].get("gram_projection") == 1
    assert match_eigs(mo.lam, g["c3s_opt_lam"]) <= 1e-7
    assert phase_aligned_error(mo.phi[:512], g["c3s_opt_phi_head"]) <= 1e-6


def test_config1_shape_keeps_the_direct_projection(config_golden):
    from paper_2502_05339_b200 import synth
    g = config_golden
    X = synth.generate_host(synth.config_params(1, seed=1, grid=24))
    model = _fit(X, 150, 1, "exact")
    st = model.provenance["sketch"]
    assert "gram_projection" not in st and st["proj_gram_bound"] > 1e-7, st
    assert np.max(np.abs(model.sigma - g["c1s_sigma"]) / g["c1s_sigma"]) <= 1e-9
    assert match_eigs(model.lam, g["c1s_lam"]) <= 1e-7


def test_rank_deficient_sketch_span_only_pass_avoids_householder():
    """A numerically rank-deficient sketch (exactly rank-6 data, and rank-6 data
    stored in fp32, sketched at l = 18, q = 1): the span-only first pass takes
    its factor from the eigen-decomposition of the sketch Gram
    (linalg._span_from_gram) instead of a Householder QR of the tall buffer;
    the final orthonormalisation keeps its own fallbacks, and the identifiable
    singular values still match the reference algorithm (oracle.sketch_svd,
    Householder QR throughout)."""
    import flowdmd_oracle as orc
    from paper_2502_05339_b200 import device as dv
    from paper_2502_05339_b200 import linalg as la
    from cpu_ops import CpuOps
    rng = np.random.default_rng(5)
    n, T, r, p, q = 4000, 60, 8, 10, 1
    base = rng.standard_normal((n, 6)) @ rng.standard_normal((6, T))
    prev = dv.set_ops(CpuOps())
    try:
        for M, tol in ((base, 1e-9), (base.astype(np.float32).astype(np.float64), 1e-8)):
            Mt = dv.Tall(torch.as_tensor(M).contiguous(), "row", n, T)
            f = la.sketch_factors(Mt, T, r + p, q, la.draw_omega(T, r + p, 9))
            assert f.stats.get("eigh_span_fallback", 0) + f.stats.get("shifted_cholqr3", 0) \
                + f.stats.get("householder_fallback", 0) >= 1, f.stats
            _, S, _ = orc.sketch_svd(M, r, p, q, 9)
            got = f.s.cpu().numpy()
            np.testing.assert_allclose(got[:6], S[:6], rtol=tol)
        # exactly rank-deficient: the singular Gram takes the eigen route in the span-only pass
        Mt = dv.Tall(torch.as_tensor(base).contiguous(), "row", n, T)
        f = la.sketch_factors(Mt, T, r + p, q, la.draw_omega(T, r + p, 9))
        assert f.stats.get("eigh_span_fallback", 0) >= 1 and f.stats["span_rank"][0] == 6, f.stats
    finally:
        dv.set_ops(prev)
