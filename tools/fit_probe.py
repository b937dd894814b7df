"""Per-step stage times + caching-allocator counters of the config-3 fit.

    python tools/fit_probe.py [--config c3|c1] [--steps 4]

Prints one line per step: wall s, the stages that moved, and the deltas of
torch.cuda.memory_stats() counters that indicate allocator churn
(num_alloc_retries, num_device_alloc/free); also every CholQR cond value.
"""
import argparse
import json
import os
import sys
import time
import warnings

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--table", default=None, help="table dtype override: f32|f64")
    ap.add_argument("--smi", action="store_true", help="sample nvidia-smi like bench.py's ClockSampler")
    ap.add_argument("--nogc", action="store_true", help="gc.disable() during the steps")
    ap.add_argument("--recon", action="store_true", help="also build the reconstruct planes each step")
    args = ap.parse_args()
    import bench
    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200 import device as dv
    from paper_2502_05339_b200 import linalg as la
    from paper_2502_05339_b200 import synth, trace

    cfg = bench.CONFIGS[args.config]
    p = synth.config_params(cfg["cfg"], seed=cfg["seed"], grid=cfg["grid"])
    S = dv.alloc_tall(p.n, p.m, torch.float32, "row", zero=True)
    tabs = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables()]
    dv.get_ops().synth3d(tabs, p.m, p.noise, synth.noise_key(p.seed), 0, p.n, S)
    del tabs
    data = fd.SnapshotMatrix(S, synth.DT, check_finite=False)
    conds = []
    orig = la._cond_upper

    def cond_log(R):
        v = orig(R)
        conds.append(v)
        return v
    la._cond_upper = cond_log
    lm = fd.LMConfig(max_iters=cfg["lm_iters"])
    if args.nogc:
        import gc
        gc.collect()
        gc.disable()
    if args.smi:
        clk = bench.ClockSampler(0)
        clk.start()
    keys = ("num_alloc_retries", "num_device_alloc", "num_device_free", "num_sync_all_streams")
    for i in range(args.steps):
        conds.clear()
        torch.cuda.synchronize()
        m0 = torch.cuda.memory_stats()
        trace.enable()
        t0 = time.perf_counter()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model = fd.optdmd(data, cfg["r"], lm_config=lm, svd_mode="randomized", seed=cfg["seed"],
                              oversample=cfg["p"], power_iters=cfg["q"], keep_basis=True)
        if args.recon:
            from paper_2502_05339_b200.runtime import ModalBasis
            U = model.basis_U
            del model
            r = cfg["r"]
            mb = ModalBasis(U, np.eye(r, dtype=complex), np.ones(r, dtype=complex), np.ones(r, dtype=complex), dt=1.0)
            mb.tc_state()
            model = None
            del mb, U
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        rec = trace.disable()
        st = trace.summarize(rec)
        sth = trace.summarize_host(rec)
        m1 = torch.cuda.memory_stats()
        print(json.dumps({"step": i, "s": round(dt, 4),
                          "alloc": {k: m1.get(k, 0) - m0.get(k, 0) for k in keys},
                          "reserved_GB": round(torch.cuda.memory_reserved() / 1e9, 2),
                          "peak_GB": round(torch.cuda.max_memory_allocated() / 1e9, 2),
                          "conds": [float(f"{c:.3e}") for c in conds], "stages": st, "host": sth}), flush=True)
        del model
    if args.smi:
        print(json.dumps(clk.stop()))


if __name__ == "__main__":
    main()
