"""Generate golden vectors by running the REAL reference (`flowdmd`) here.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. \
        python oracle/gen_golden.py

Writes `tests/golden/*.npz`. Inputs that are cheap to regenerate (the
BASELINE-config snapshot matrices) are NOT stored: the fixture stores the
generator parameters' seed plus a checksum of the regenerated matrix, and
tests regenerate them with `paper_2502_05339_b200.synth`. Small test-style
inputs (from the reference's own `conftest.stable_linear_system`) are stored
verbatim.

The reference hard-codes q=2 and clamps p in `_svd_of` (dmd.py:216-222);
BASELINE configs 1-3 use q=1, so `_patched_svd_of` below honours explicit
(p, q) with l = min(r+p, T), mirroring the clamp at dmd.py:220.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

import flowdmd                                   # noqa: E402  (reference, read-only import)
import flowdmd.dmd as ref_dmd                    # noqa: E402
from flowdmd.dmd import LMConfig, ReducedModel, SnapshotMatrix, exact_dmd, fit_control, optdmd  # noqa: E402
from flowdmd.linalg import randomized_svd        # noqa: E402
from flowdmd.runtime import decode, encode, eval_continuous, step_k  # noqa: E402
from conftest import stable_linear_system        # noqa: E402  (reference test fixture)

from paper_2502_05339_b200 import synth          # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

_orig_svd_of = ref_dmd._svd_of


def _patched(p, q):
    def svd_of(X, r, svd_mode, seed):
        if svd_mode != "randomized":
            return _orig_svd_of(X, r, svd_mode, seed)
        T = min(X.shape)
        return randomized_svd(X, r, oversample=min(p, T - r), power_iters=q, seed=seed)
    return svd_of


def checksum(X):
    X = np.asarray(X, dtype=np.float64)
    return np.array([X.sum(), (X * X).sum(), X[::97].sum(), X[:, ::7].sum()])


def model_arrays(prefix, model, out):
    out[prefix + "lam"] = model.lam
    out[prefix + "sigma"] = model.sigma
    out[prefix + "phi"] = model.phi
    out[prefix + "partner"] = model.pair_partner
    if "residual" in model.provenance:
        out[prefix + "residual"] = model.provenance["residual"]
        out[prefix + "residual_rel"] = model.provenance["residual_rel"]


def small_cases():
    out = {}
    # --- randomized_svd (test_linalg.py:45-73; test_acceptance.py:257-275)
    rng = np.random.default_rng(5)
    M = rng.standard_normal((500, 20)) @ rng.standard_normal((20, 200)) + 1e-8 * rng.standard_normal((500, 200))
    res = randomized_svd(M, 20, oversample=10, power_iters=2, seed=42)
    out["rsvd1_M"], out["rsvd1_U"], out["rsvd1_S"], out["rsvd1_V"] = M, res.U, res.S, res.V
    M = np.zeros((10, 10)); M[:3, :3] = np.diag([3.0, 2.0, 1.0])
    res = randomized_svd(M, 2, oversample=8, seed=0)
    out["rsvd2_M"], out["rsvd2_U"], out["rsvd2_S"], out["rsvd2_V"] = M, res.U, res.S, res.V
    rng = np.random.default_rng(9)
    M = rng.standard_normal((40, 30))
    res = randomized_svd(M, 5, seed=123)
    out["rsvd3_M"], out["rsvd3_U"], out["rsvd3_S"], out["rsvd3_V"] = M, res.U, res.S, res.V
    # q = 1, p = 10 on a tall noisy matrix (BASELINE-style power count)
    rng = np.random.default_rng(11)
    M = rng.standard_normal((3000, 12)) @ rng.standard_normal((12, 80)) + 1e-3 * rng.standard_normal((3000, 80))
    res = randomized_svd(M, 12, oversample=10, power_iters=1, seed=3)
    out["rsvd4_M"], out["rsvd4_U"], out["rsvd4_S"], out["rsvd4_V"] = M, res.U, res.S, res.V

    # --- exact_dmd (test_dmd.py:30-106)
    cases = {
        "dmd_full8": dict(kw=dict(n=120, rank=8, frames=50, seed=3), r=8, mode="full", seed=None),
        "dmd_rand6": dict(kw=dict(n=200, rank=6, frames=60, seed=7), r=6, mode="randomized", seed=11),
        "dmd_noisy6": dict(kw=dict(n=60, rank=6, frames=40, seed=5, noise=0.01), r=6, mode="full", seed=None),
        "dmd_odd5": dict(kw=dict(n=80, rank=5, frames=50, seed=21), r=5, mode="full", seed=None),
        "dmd_noisyrand": dict(kw=dict(n=400, rank=10, frames=60, seed=4, noise=0.02), r=8,
                              mode="randomized", seed=5),
    }
    for name, c in cases.items():
        data, eigs = stable_linear_system(**c["kw"])
        model = exact_dmd(data, c["r"], svd_mode=c["mode"], seed=c["seed"])
        out[name + "_X"] = data.states
        out[name + "_true"] = eigs
        model_arrays(name + "_", model, out)
        table, re_idx, im_idx = model.decode_table()
        out[name + "_table"] = table
        out[name + "_reidx"] = np.array(re_idx, dtype=np.int64).reshape(-1, 2)
        out[name + "_imidx"] = np.array(im_idx, dtype=np.int64).reshape(-1, 2)
        # runtime: encode frame 0, step_k, decode, continuous time, asymmetric fallback
        z0 = encode(model, data.states[:, 0])
        out[name + "_z0"] = z0.z
        out[name + "_frame7"] = decode(model, step_k(model, z0, 7))
        zc = eval_continuous(model, z0, 3.37 * data.dt)
        out[name + "_zc"] = zc.z
        out[name + "_framec"] = decode(model, zc)
        za = np.zeros(model.r, dtype=complex); za[0] = 1.0 + 0.5j
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            out[name + "_frame_asym"] = decode(model, za)
        rng = np.random.default_rng(77)
        Bc = rng.standard_normal((model.n, 4))
        out[name + "_B"] = Bc
        out[name + "_redB"] = fit_control(model, [Bc]).reduced_b[0]

    # --- optdmd (test_dmd.py:123-159)
    data, eigs = stable_linear_system(n=60, rank=6, frames=40, seed=9, noise=0.01)
    model = optdmd(data, 6)
    out["opt_X"] = data.states
    model_arrays("opt_", model, out)
    out["opt_hist"] = np.array(model.provenance["objective_history"])
    data, eigs = stable_linear_system(n=300, rank=8, frames=60, seed=31, noise=0.005)
    model = optdmd(data, 8, lm_config=LMConfig(max_iters=10), svd_mode="randomized", seed=2)
    out["opt2_X"] = data.states
    model_arrays("opt2_", model, out)
    out["opt2_hist"] = np.array(model.provenance["objective_history"])
    return out


def config_cases():
    out = {}
    # Config 0 exactly as BASELINE.json states it (reference defaults p=10, q=2 apply).
    p = synth.config_params(0, seed=0)
    X = synth.generate_host(p)
    out["c0_checksum"] = checksum(X)
    model = exact_dmd(SnapshotMatrix(X, synth.DT), 20, svd_mode="randomized", seed=0)
    model_arrays("c0_", model, out)
    z0 = encode(model, X[:, 0])
    out["c0_z0"] = z0.z
    frames = np.stack([decode(model, step_k(model, z0, k)) for k in range(101)], axis=1)
    out["c0_frames_sel"] = frames[:, [0, 1, 50, 100]]
    out["c0_frames_checksum"] = np.stack([frames.sum(0), (frames * frames).sum(0)])
    # Config 1 shape at a reduced grid (24^3 x 3): same modes/m/r/p/q.
    ref_dmd._svd_of = _patched(10, 1)
    try:
        p = synth.config_params(1, seed=1, grid=24)
        X = synth.generate_host(p)
        out["c1s_checksum"] = checksum(X)
        model = exact_dmd(SnapshotMatrix(X, synth.DT), 150, svd_mode="randomized", seed=1)
        model_arrays("c1s_", model, out)
        del out["c1s_phi"]
        out["c1s_phi_head"] = model.phi[:512]
        out["c1s_phi_norms"] = np.linalg.norm(model.phi, axis=0)
        z0 = encode(model, X[:, 0])
        out["c1s_z0"] = z0.z
        fr = np.stack([decode(model, step_k(model, z0, k)) for k in (1, 100, 200)], axis=1)
        out["c1s_frames_checksum"] = np.stack([fr.sum(0), (fr * fr).sum(0)])
        out["c1s_frames_head"] = fr[:4096]
        # Config 3 shape at a reduced grid (16^3 x 3): r = T = 200 (l clamped), OptDMD 10 iters.
        p = synth.config_params(3, seed=3, grid=16)
        X = synth.generate_host(p)
        out["c3s_checksum"] = checksum(X)
        model = exact_dmd(SnapshotMatrix(X, synth.DT), 200, svd_mode="randomized", seed=3)
        model_arrays("c3s_", model, out)
        del out["c3s_phi"]
        out["c3s_phi_norms"] = np.linalg.norm(model.phi, axis=0)
        mo = optdmd(SnapshotMatrix(X, synth.DT), 200, lm_config=LMConfig(max_iters=10),
                    svd_mode="randomized", seed=3)
        out["c3s_opt_lam"] = mo.lam
        out["c3s_opt_sigma"] = mo.sigma
        out["c3s_opt_hist"] = np.array(mo.provenance["objective_history"])
        out["c3s_opt_phi_head"] = mo.phi[:512]
    finally:
        ref_dmd._svd_of = _orig_svd_of
    return out


def frame_cases():
    """Round-2 additions (tests/golden/config_frames.npz): frames decoded from
    the reference's OptDMD and exact-DMD models at the config-3 shape, so the
    benched fit (OptDMD, r = T = 200, fp32 snapshots) is pinned through what a
    user sees — z0 = encode(x0), decode(step_k(z0, k)) and a continuous-time
    frame — not only through lambda."""
    out = {}
    ref_dmd._svd_of = _patched(10, 1)
    try:
        p = synth.config_params(3, seed=3, grid=16)
        X = synth.generate_host(p)
        out["c3s_checksum"] = checksum(X)
        for tag, fit in (("opt", lambda: optdmd(SnapshotMatrix(X, synth.DT), 200, lm_config=LMConfig(max_iters=10),
                                                svd_mode="randomized", seed=3)),
                         ("exact", lambda: exact_dmd(SnapshotMatrix(X, synth.DT), 200, svd_mode="randomized",
                                                     seed=3))):
            model = fit()
            z0 = encode(model, X[:, 0])
            fr = np.stack([decode(model, step_k(model, z0, k)) for k in (1, 50, 199)]
                          + [decode(model, eval_continuous(model, z0, 12.37))], axis=1)
            out[f"c3s_{tag}_z0"] = z0.z
            out[f"c3s_{tag}_lam"] = model.lam
            out[f"c3s_{tag}_phi_norms"] = np.linalg.norm(model.phi, axis=0)
            out[f"c3s_{tag}_frames_head"] = fr[:4096]
            out[f"c3s_{tag}_frames_checksum"] = np.stack([fr.sum(0), (fr * fr).sum(0)])
            out[f"c3s_{tag}_frames_x0_rel"] = np.array([np.linalg.norm(fr[:, 0] - X[:, 1]) / np.linalg.norm(X[:, 1])])
    finally:
        ref_dmd._svd_of = _orig_svd_of
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1 and sys.argv[1] == "frames":
        f = frame_cases()
        np.savez_compressed(os.path.join(OUT, "config_frames.npz"), **f)
        print("config_frames.npz", os.path.getsize(os.path.join(OUT, "config_frames.npz")))
        return
    s = small_cases()
    np.savez_compressed(os.path.join(OUT, "small_cases.npz"), **s)
    c = config_cases()
    np.savez_compressed(os.path.join(OUT, "config_cases.npz"), **c)
    for f in ("small_cases.npz", "config_cases.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)))
    print("reference flowdmd", flowdmd.__version__, "numpy", np.__version__)


if __name__ == "__main__":
    main()
