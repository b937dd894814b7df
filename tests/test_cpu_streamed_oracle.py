"""Pins the streamed FP64 oracle (oracle/streamed_fit.py) — the checker for
the full-size configs — against the REAL reference's outputs
(tests/golden/streamed_cases.npz from oracle/gen_golden_streamed.py):
config 0 in full and 98,304-row blocks of configs 1 and 3 at their full grid
specs. Measured deltas (build container): sigma <= 3e-14 rel, lambda <= 2e-12,
modes <= 3e-11 up to phase, z0 <= 3e-11, frames <= 2e-12."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, aligned_coeff_error, checksum, match_eigs, phase_aligned_error

sf = pytest.importorskip("streamed_fit")

KS = (1, 50, 100)


@pytest.fixture(scope="module")
def g():
    return dict(np.load(os.path.join(GOLDEN, "streamed_cases.npz")))


def _check(g, tag, model, X, rows):
    RS, colsum = sf.snapshot_r(rows)
    z0 = sf.encode_x(RS, model, 0)
    head = X[:2048].astype(np.float64)
    fr = sf.frames_rows(model, head, z0, KS)
    nrm = sf.frame_norms(model, RS, colsum, z0, KS)
    phi_head = model.phi_rows(X[:512].astype(np.float64))
    np.testing.assert_allclose(model.sigma, g[tag + "_sigma"], rtol=1e-12)
    assert match_eigs(model.lam, g[tag + "_lam"]) <= 1e-11
    assert phase_aligned_error(phi_head, g[tag + "_phi_head"]) <= 1e-9
    assert aligned_coeff_error(phi_head, g[tag + "_phi_head"], z0, g[tag + "_z0"]) <= 1e-9
    ref = g[tag + "_frames_head"]
    assert np.linalg.norm(fr - ref) / np.linalg.norm(ref) <= 1e-10
    np.testing.assert_allclose(nrm, g[tag + "_frames_norms"], rtol=1e-7)
    if tag + "_residual_rel" in g:
        np.testing.assert_allclose(model.extra["residual_rel"], g[tag + "_residual_rel"], rtol=1e-9)


def test_streamed_oracle_config0(g):
    from paper_2502_05339_b200 import synth
    X = synth.generate_host(synth.config_params(0, seed=0))
    np.testing.assert_allclose(checksum(X), g["c0_checksum"], rtol=1e-13)
    rows = sf.Rows.from_array(X, block=3000)            # ragged last block
    model = sf.exact_dmd(rows, 20, 10, 2, 0)
    _check(g, "c0_exact", model, X, rows)


def test_streamed_oracle_config1_block(g):
    from paper_2502_05339_b200 import synth
    X = synth.generate_host(synth.config_params(1, seed=1), 0, 98304)
    np.testing.assert_allclose(checksum(X), g["c1b_checksum"], rtol=1e-12)
    rows = sf.Rows.from_array(X, block=40000)
    model = sf.exact_dmd(rows, 150, 10, 1, 1)
    _check(g, "c1b_exact", model, X, rows)


@pytest.mark.parametrize("method", ["exact", "opt"])
def test_streamed_oracle_config3_block(g, method):
    from paper_2502_05339_b200 import synth
    X = synth.generate_host(synth.config_params(3, seed=3), 0, 98304)
    np.testing.assert_allclose(checksum(X), g["c3b_checksum"], rtol=1e-12)
    rows = sf.Rows.from_array(X, block=40000)
    if method == "opt":
        model = sf.optdmd(rows, 200, 10, 1, 3, 10)
    else:
        model = sf.exact_dmd(rows, 200, 10, 1, 3)
    _check(g, f"c3b_{method}", model, X, rows)
