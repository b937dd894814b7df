"""Golden vectors that pin oracle/streamed_fit.py to the REAL reference.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. \
        python oracle/gen_golden_streamed.py

Cases (tests/golden/streamed_cases.npz):
  * c0   — BASELINE config 0 in full (n = 8,192, m = 101, f64), exact DMD
           r = 20 with the reference's own randomized defaults (p = 10, q = 2)
  * c1b  — a contiguous 98,304-row block of BASELINE config 1 at its full
           128^3 x 3 grid spec (fp32 storage, m = 201), exact DMD at r = 150,
           p = 10, q = 1 (reference `_svd_of` patched to honour (p, q), as
           oracle/gen_golden.py)
  * c3b  — the same for BASELINE config 3 (256^3 x 3 spec): exact DMD and
           OptDMD (10 LM iterations) at r = T = 200 (l clamped to 200), the
           benched regime. (OptDMD at r < T is not a pin: its LM trajectory
           turns 1e-12 input differences — CholeskyQR2 vs Householder — into
           1e-3 eigenvalue differences within two steps; measured on c1b.)
For each: sigma, lambda, the first 512 rows of phi, every column norm of phi,
z0 = encode(x0), frames decode(step_k(z0, k)) for k in (1, 50, 100) — head
rows plus per-frame sum / sum of squares — and exact DMD's residual_rel.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import flowdmd.dmd as ref_dmd                    # noqa: E402  (reference, read-only import)
from flowdmd.dmd import LMConfig, SnapshotMatrix, exact_dmd, optdmd  # noqa: E402
from flowdmd.runtime import decode, encode, step_k  # noqa: E402

from gen_golden import _orig_svd_of, _patched, checksum  # noqa: E402
from paper_2502_05339_b200 import synth          # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "streamed_cases.npz")
KS = (1, 50, 100)
C1_ROWS = 98304


def _record(tag, model, X, out):
    out[f"{tag}_sigma"] = model.sigma
    out[f"{tag}_lam"] = model.lam
    out[f"{tag}_phi_head"] = model.phi[:512]
    out[f"{tag}_phi_norms"] = np.linalg.norm(model.phi, axis=0)
    z0 = encode(model, X[:, 0])
    out[f"{tag}_z0"] = z0.z
    fr = np.stack([decode(model, step_k(model, z0, k)) for k in KS], axis=1)
    out[f"{tag}_frames_head"] = fr[:2048]
    out[f"{tag}_frames_norms"] = np.stack([fr.sum(0), (fr * fr).sum(0)])
    if "residual_rel" in model.provenance:
        out[f"{tag}_residual_rel"] = np.array(model.provenance["residual_rel"])


def main():
    out = {}
    p = synth.config_params(0, seed=0)
    X = synth.generate_host(p)
    out["c0_checksum"] = checksum(X)
    _record("c0_exact", exact_dmd(SnapshotMatrix(X, synth.DT), 20, svd_mode="randomized", seed=0), X, out)
    ref_dmd._svd_of = _patched(10, 1)
    try:
        p = synth.config_params(1, seed=1)
        X = synth.generate_host(p, 0, C1_ROWS)
        out["c1b_checksum"] = checksum(X)
        _record("c1b_exact", exact_dmd(SnapshotMatrix(X, synth.DT), 150, svd_mode="randomized", seed=1), X, out)
        p = synth.config_params(3, seed=3)
        X = synth.generate_host(p, 0, C1_ROWS)
        out["c3b_checksum"] = checksum(X)
        _record("c3b_exact", exact_dmd(SnapshotMatrix(X, synth.DT), 200, svd_mode="randomized", seed=3), X, out)
        _record("c3b_opt", optdmd(SnapshotMatrix(X, synth.DT), 200, lm_config=LMConfig(max_iters=10),
                                  svd_mode="randomized", seed=3), X, out)
    finally:
        ref_dmd._svd_of = _orig_svd_of
    np.savez_compressed(OUT, **out)
    print(OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()
