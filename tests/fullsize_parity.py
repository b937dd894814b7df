"""Full-size parity of the device fit against the streamed FP64 oracle
(oracle/streamed_fit.py, pinned to the real reference by
tests/test_cpu_streamed_oracle.py) — TEST HARNESS (GPU box).

    python tests/fullsize_parity.py --config c3 [--out profiles/r02_fullsize_c3.json]
    python tests/fullsize_parity.py --config c1

The snapshot matrix is generated in HBM by the bench's device generator; the
oracle reads the very same fp32 bytes back in row blocks (so both sides fit
identical inputs), runs the reference algorithm in float64 on the host cores,
and the two are compared on:
  * sigma (relative), lambda (absolute, after min-cost matching);
  * modes up to phase on random row blocks (device table rows vs oracle rows);
  * z0 = encode(x0) (with the same per-mode phase);
  * frames decode(step_k(z0, k)) on the same random row blocks, plus the sum
    and squared norm of each full frame (oracle: from S^T S, no frame formed).
Tolerances (BASELINE north_star): sigma 1e-5 rel, lambda 1e-5 abs, frames
1e-4 rel-L2, modes up to phase.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

CASES = {
    "c1": dict(cfg=1, seed=1, r=150, p=10, q=1, method="exact"),
    "c3": dict(cfg=3, seed=3, r=200, p=10, q=1, method="opt", lm_iters=10),
}
KS = (1, 50, 200)


def run(case: str, n_blocks: int = 8, block_rows: int = 4096, oracle_block: int = 1 << 18, grid=None) -> dict:
    import torch

    import paper_2502_05339_b200 as fd
    import streamed_fit as sf
    from conftest import aligned_coeff_error, match_eigs, phase_aligned_error
    from paper_2502_05339_b200 import device as dv
    from paper_2502_05339_b200 import synth
    c = CASES[case]
    p = synth.config_params(c["cfg"], seed=c["seed"], grid=grid)
    n, m, r = p.n, p.m, c["r"]
    S = dv.alloc_tall(n, m, torch.float32, "row")
    S.buf[:, m:].zero_()
    tabs = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables()]
    dv.get_ops().synth3d(tabs, m, p.noise, synth.noise_key(p.seed), 0, n, S)
    torch.cuda.synchronize()
    out = {"case": case, "n": n, "m": m, "r": r, "p": c["p"], "q": c["q"], "method": c["method"]}
    # ---- device fit (the product path) ----
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        data = fd.SnapshotMatrix(S, synth.DT)
        kw = dict(svd_mode="randomized", seed=c["seed"], oversample=c["p"], power_iters=c["q"])
        if c["method"] == "opt":
            model = fd.optdmd(data, r, lm_config=fd.LMConfig(max_iters=c["lm_iters"]), **kw)
        else:
            model = fd.exact_dmd(data, r, residual=False, **kw)
        x0 = S.buf[:n, 0].clone()
        z0 = fd.encode(model, x0)
        frames = [fd.decode(model, fd.step_k(model, z0, k), to_host=False).double() for k in KS]
    torch.cuda.synchronize()
    out["device_fit_s"] = time.perf_counter() - t0
    rng = np.random.default_rng(11)
    starts = np.sort(rng.choice(n // block_rows, size=n_blocks, replace=False)) * block_rows
    rows = np.concatenate([np.arange(s0, s0 + block_rows) for s0 in starts])
    ridx = torch.as_tensor(rows, device="cuda")
    fr_dev = np.stack([f[ridx].cpu().numpy() for f in frames], axis=1)
    fr_norms_dev = np.array([[float(f.sum()), float((f * f).sum())] for f in frames]).T
    D, E = model.modes.basis()
    phi_dev = D.view()[ridx].double().cpu().numpy() @ E
    lam_dev, sig_dev, z0_dev = model.lam, model.sigma, z0.z
    del frames, model, data
    torch.cuda.empty_cache()

    # ---- streamed FP64 oracle over the same bytes ----
    def fetch(a, b):
        return S.buf[a:b, :m].double().cpu().numpy()

    t0 = time.perf_counter()
    R = sf.Rows(n, m, fetch, block=oracle_block)
    if c["method"] == "opt":
        om = sf.optdmd(R, r, c["p"], c["q"], c["seed"], c["lm_iters"])
    else:
        om = sf.exact_dmd(R, r, c["p"], c["q"], c["seed"], residual=False)
    RS, colsum = sf.snapshot_r(R)
    z0_or = sf.encode_x(RS, om, 0)
    Sb = S.buf[ridx, :m].double().cpu().numpy()
    phi_or = om.phi_rows(Sb)
    fr_or = sf.frames_rows(om, Sb, z0_or, KS)
    fr_norms_or = sf.frame_norms(om, RS, colsum, z0_or, KS)
    out["oracle_s"] = time.perf_counter() - t0
    out["oracle_passes"] = R.passes
    out["oracle_threads"] = os.cpu_count()

    def rel(a, b):
        return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

    out["sample_rows"] = int(rows.size)
    out["sigma_rel_max"] = float(np.abs(sig_dev / om.sigma - 1).max())
    out["lambda_abs_max"] = match_eigs(lam_dev, om.lam)
    out["modes_phase_aligned_max"] = phase_aligned_error(phi_dev, phi_or)
    out["z0_aligned_rel"] = aligned_coeff_error(phi_dev, phi_or, z0_dev, z0_or)
    out["frames_rel_l2"] = [rel(fr_dev[:, j], fr_or[:, j]) for j in range(len(KS))]
    out["frame_sum_rel"] = [float(abs(fr_norms_dev[0, j] / fr_norms_or[0, j] - 1)) for j in range(len(KS))]
    out["frame_sumsq_rel"] = [float(abs(fr_norms_dev[1, j] / fr_norms_or[1, j] - 1)) for j in range(len(KS))]
    out["ks"] = list(KS)
    out["tolerances"] = {"sigma_rel": 1e-5, "lambda_abs": 1e-5, "frames_rel_l2": 1e-4, "modes": "up to phase, 1e-5"}
    out["pass"] = bool(out["sigma_rel_max"] <= 1e-5 and out["lambda_abs_max"] <= 1e-5
                       and max(out["frames_rel_l2"]) <= 1e-4 and out["modes_phase_aligned_max"] <= 1e-5
                       and max(out["frame_sumsq_rel"]) <= 2e-4)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(CASES))
    ap.add_argument("--out", default=None)
    ap.add_argument("--grid", type=int, default=None)
    a = ap.parse_args()
    res = run(a.config, grid=a.grid)
    js = json.dumps(res, indent=1)
    print(js)
    if a.out:
        with open(a.out, "w") as f:
            f.write(js + "\n")


if __name__ == "__main__":
    main()
