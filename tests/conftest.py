import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfdmd.so")


@pytest.fixture(scope="session")
def small_golden():
    return dict(np.load(os.path.join(GOLDEN, "small_cases.npz")))


@pytest.fixture(scope="session")
def config_golden():
    return dict(np.load(os.path.join(GOLDEN, "config_cases.npz")))


def checksum(X):
    X = np.asarray(X, dtype=np.float64)
    return np.array([X.sum(), (X * X).sum(), X[::97].sum(), X[:, ::7].sum()])


def match_eigs(a, b):
    """max |a_i - b_pi(i)| under min-cost matching (near-ties in the sort key
    can swap order)."""
    from scipy.optimize import linear_sum_assignment
    a = np.asarray(a); b = np.asarray(b)
    C = np.abs(a[:, None] - b[None, :])
    i, j = linear_sum_assignment(C)
    return float(C[i, j].max()) if len(i) else 0.0


def phase_aligned_error(phi, ref):
    """max over columns of ||phi_k e^{i theta} - ref_k|| / ||ref_k|| with the
    best phase theta (modes compare up to phase, BASELINE.json)."""
    phi = np.asarray(phi); ref = np.asarray(ref)
    worst = 0.0
    for k in range(ref.shape[1]):
        ip = np.vdot(phi[:, k], ref[:, k])
        ph = ip / abs(ip) if abs(ip) > 0 else 1.0
        e = np.linalg.norm(phi[:, k] * ph - ref[:, k]) / max(np.linalg.norm(ref[:, k]), 1e-300)
        worst = max(worst, e)
    return worst


def aligned_coeff_error(phi, ref_phi, z, zref):
    """Reduced coordinates compared with the per-mode phase that aligns phi
    to ref_phi (phi_k e^{i t} pairs with z_k e^{-i t}): max |z_k / p_k - zref_k|
    over max |zref|, p_k the unit phase rotating phi_k onto ref_phi_k."""
    phi = np.asarray(phi); ref_phi = np.asarray(ref_phi)
    z = np.asarray(z); zref = np.asarray(zref)
    h = ref_phi.shape[0]
    out = np.empty_like(zref)
    for k in range(zref.size):
        ip = np.vdot(phi[:h, k], ref_phi[:, k])
        ph = ip / abs(ip) if abs(ip) > 0 else 1.0
        out[k] = z[k] / ph
    return float(np.abs(out - zref).max() / max(np.abs(zref).max(), 1e-300))
