"""Benchmark of the B200 DMD hot path (BASELINE.json metric: DMD fit GFLOP/s +
reconstruct frames/s at 256^3, r=200, as % of roofline).

One step = the config-3 fit (randomized SVD r=200, p=10 (clamped: l=T=200),
q=1, CholeskyQR2, 10 OptDMD LM iterations, modes + POD basis U) followed by
the config-4 reconstruction u(t) = U Re(W Lam^t b) at 1024 seeded continuous
times in batches of 1, 32 and 1024 frames. Inputs are resident in HBM before
the timed region (`value`); `e2e` repeats the fit through the public API from
pinned host memory with the host<->device copies inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c1] [--impl fdmd|reference]

Multi-GPU (torchrun): rows are sharded across ranks (strong scaling, fixed
256^3 problem), the only collectives are NCCL all-reduces of the small
Gram/projection blocks; time = max over ranks of CUDA-event time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

METRIC = "DMD fit GFLOP/s + reconstruct frames/s (256³, r=200); % of roofline"
CONFIGS = {
    "c3": dict(cfg=3, grid=256, r=200, p=10, q=1, lm_iters=10, times=1024, seed=3),
    "c1": dict(cfg=1, grid=128, r=150, p=10, q=1, lm_iters=10, times=1024, seed=1),
    "c3s": dict(cfg=3, grid=64, r=200, p=10, q=1, lm_iters=10, times=1024, seed=3),
    # BASELINE config 1 as written: exact DMD r = 150 + 200 integer steps + 1 interactive frame (a side line)
    "c1x": dict(cfg=1, grid=128, r=150, p=10, q=1, steps=200, seed=1),
    # config 2 (DMDc): augmented fit r_aug = 158 + 200 controlled frames (a side line, not the headline)
    "c2": dict(cfg=2, grid=128, r=150, r_aug=158, p=10, q=1, ell=8, steps=200, seed=2),
}


def fit_flops(n, m, r, p, q, modes="optdmd"):
    """SURVEY.md §8(d) algorithmic flops (executed terms only)."""
    T = m - 1
    l = min(r + p, T)
    terms = {
        "sketch+power 2nTl(1+2q)": 2.0 * n * T * l * (1 + 2 * q),
        "CholQR2 4nl^2(1+q)": 4.0 * n * l * l * (1 + q),
        "projection 2nml": 2.0 * n * m * l,
        "lift U 2nlr": 2.0 * n * l * r,
        ("modes 4nr^2" if modes == "optdmd" else "modes 4nTr"): 4.0 * n * r * (r if modes == "optdmd" else T),
    }
    return sum(terms.values()), terms, l


def executed_terms(n, m, r, p, q, route="gram_projection"):
    """Flops libfdmd actually executes for the same fit (OptDMD, resident
    snapshots), split by arithmetic. Snapshot-Gram route
    (q >= 1): the sketch, every power pass Z = X^T Q and the first CholeskyQR
    pass of each orthonormalisation follow from one symmetric Gram X^T X
    (n T^2); the only tall GEMM is the final Q1 = X (W R1^-1) (2nTl);
    CholeskyQR2's second pass is one SYRK (n l^2) whose R2^-1 is folded into
    small matrices; the projection Q^T S (2nml). Those run in FP64 (DMMA).
    The lift U = Q Ub (2nlr) and the modes (one column per conjugate pair,
    ~2nr^2) run on tcgen05 with an FP16 2-way split, FP32-accurate, into the
    fp32 tables.

    route "gram_projection" (linalg.PROJ_GRAM_TOL: taken when the a-priori
    error bound allows, e.g. config 3 with r = T): B = Q^T S also follows from
    the snapshot Gram and its border X^T s_m (2nT, carried by the same panel
    kernel: fdmd_tall_gram_bordered), so there is no Q1 buffer, no second
    CholeskyQR pass and no direct projection; the only tall GEMM is the lift
    U = X (W R1^-1 Ub) (2nTr, FP64 DMMA, written as the fp16 planes of the
    tcgen05 modes product)."""
    T = m - 1
    l = min(r + p, T)
    if q >= 1 and route == "gram_projection":
        fp64 = {"snapshot Gram nT^2": 1.0 * n * T * T, "border X^T s_m 2nT (same kernel)": 2.0 * n * T,
                "lift U = S Umap 2nTr": 2.0 * n * T * r}
        return fp64, {"modes 2nr^2": 2.0 * n * r * r}
    if q == 0:   # explicit sketch: Y = X Omega, CholeskyQR2 (SYRK + TRSM + SYRK)
        fp64 = {"sketch 2nTl": 2.0 * n * T * l, "CholQR2 3nl^2": 3.0 * n * l * l, "projection 2nml": 2.0 * n * m * l}
    else:
        fp64 = {"snapshot Gram nT^2": 1.0 * n * T * T, "Q1 = X W R1^-1 2nTl": 2.0 * n * T * l,
                "CholQR2 second pass nl^2": 1.0 * n * l * l, "projection 2nml": 2.0 * n * m * l}
    tc = {"lift U 2nlr": 2.0 * n * l * r, "modes 2nr^2": 2.0 * n * r * r}
    return fp64, tc


def executed_flops(n, m, r, p, q, route="gram_projection"):
    fp64, tc = executed_terms(n, m, r, p, q, route)
    return sum(fp64.values()) + sum(tc.values())


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
def _dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _relaunch_distributed(args):
    """`bench.py --gpus N` outside torchrun: one process per GPU through
    torch.distributed.run (127.0.0.1 rendezvous), after checking that N GPUs
    are visible — never silently run fewer ranks than asked."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


class CpuArm:
    """The reference's own CPU implementation of the path, timed on the host.

    Preferred: the UNMODIFIED reference package `flowdmd` installed offline
    into baseline/_ref (pip --target) — `optdmd` from
    flowdmd/dmd.py:366-436 with its init exact_dmd (pinv + residual) — with
    only `_svd_of` (dmd.py:216-222) patched to honour the config's (p, q), as
    SURVEY §8(d) prescribes. Fallback when baseline/_ref is absent: the oracle
    port oracle/flowdmd_oracle.py (kind "port")."""

    def __init__(self):
        ref = os.path.join(ROOT, "baseline", "_ref")
        self.kind = "port"
        if os.path.isdir(os.path.join(ref, "flowdmd")):
            sys.path.insert(0, ref)
            try:
                import flowdmd.dmd as rdmd
                import flowdmd.linalg as rlin
                self.rdmd, self.rlin, self.kind = rdmd, rlin, "reference"
            except Exception:
                self.kind = "port"
        if self.kind == "port":
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import flowdmd_oracle as orc
            self.orc = orc

    def describe(self):
        return ("flowdmd (reference package, unmodified, baseline/_ref) optdmd" if self.kind == "reference"
                else "oracle port (oracle/flowdmd_oracle.py) optdmd")

    def fit(self, X, cfg):
        if self.kind == "port":
            return self.orc.optdmd(X, cfg["r"], max_iters=cfg["lm_iters"], svd_mode="randomized", seed=cfg["seed"],
                                   p=cfg["p"], q=cfg["q"])
        rdmd, rlin = self.rdmd, self.rlin
        orig = rdmd._svd_of

        def svd_of(Xm, r, svd_mode, seed):      # dmd.py:216-222 with the config's (p, q)
            T = min(Xm.shape)
            return rlin.randomized_svd(Xm, r, oversample=min(cfg["p"], T - r), power_iters=cfg["q"], seed=seed)

        rdmd._svd_of = svd_of
        try:
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                return rdmd.optdmd(rdmd.SnapshotMatrix(X, 0.1), cfg["r"],
                                   lm_config=rdmd.LMConfig(max_iters=cfg["lm_iters"]),
                                   svd_mode="randomized", seed=cfg["seed"])
        finally:
            rdmd._svd_of = orig


def run_reference(args, cfg):
    """--impl reference: the reference's CPU implementation (CpuArm) on a
    bounded row sample of the workload, all host cores."""
    world, rank, _ = _dist_init()
    if rank != 0:
        return
    from paper_2502_05339_b200 import synth
    arm = CpuArm()
    res = cpu_sample(arm, synth, cfg, args.cpu_rows)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        arm.fit(res["X"], cfg)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    tmed = float(np.median(times))
    val = res["flops"] / tmed / 1e9
    line = {
        "metric": METRIC, "value": round(val, 3), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tmed * 1e3, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": dict(arm_config(cfg, res["n"], res["m"], cfg["r"], res["l"], f"cpu{os.cpu_count()}threads"),
                       sample_rows=res["rows"]),
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": arm.kind,
                         "sample": res["sample"]},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def arm_config(cfg, n, m, r, l, parallelism):
    """The workload both bench arms report (the reference arm adds sample_rows)."""
    return {"workload": f"config{cfg['cfg']} fit (OptDMD, {cfg['lm_iters']} LM iters) + config4 reconstruct",
            "n": n, "m": m, "r": r, "l": l, "p": cfg["p"], "q": cfg["q"], "grid": f"{cfg['grid']}^3x3",
            "snapshot_dtype": "f32", "parallelism": parallelism, "l2": "inputs larger than L2 (X >= 3.8 GB)"}


def cpu_sample(arm, synth, cfg, rows):
    p = synth.config_params(cfg["cfg"], seed=cfg["seed"], grid=cfg["grid"])
    n_full = p.n
    rows = min(rows, p.n)
    X = synth.generate_host(p, 0, rows).astype(np.float64)
    flops, _, _ = fit_flops(rows, p.m, cfg["r"], cfg["p"], cfg["q"])
    sample = (f"config{cfg['cfg']} rows [0,{rows}) x {p.m} snapshots (same generator, first {rows} rows of the "
              f"{n_full}-row matrix); {arm.describe()} r={cfg['r']} p={cfg['p']} q={cfg['q']} "
              f"{cfg['lm_iters']} LM iters, numpy/OpenBLAS fp64, all host threads; GFLOP/s from the SURVEY "
              f"§8d formula at n={rows} (every n-dependent cost of the reference is linear in n)")
    _, _, l = fit_flops(n_full, p.m, cfg["r"], cfg["p"], cfg["q"])
    return {"X": X, "rows": rows, "flops": flops, "sample": sample, "n": n_full, "m": p.m, "l": l}


def dmdc_flops(n, m, r_aug, r, p, q, ell):
    """Config-2 fit work (SURVEY §8(d) formula for C2 plus the output-basis
    sketch that §8(c) leaves to the builder): the augmented sketch of
    [X; Upsilon] at l1 = r_aug + p, the rank-r sketch of X' at l2 = r + p,
    the cross product Q1^T Q2 and the modes X' V S^-1 (4nTr)."""
    T = m - 1
    l1, l2 = min(r_aug + p, T), min(r + p, T)
    na = n + ell
    terms = {"aug sketch+power 2nTl1(1+2q)": 2.0 * na * T * l1 * (1 + 2 * q),
             "aug CholQR2 4nl1^2(1+q)": 4.0 * na * l1 * l1 * (1 + q),
             "aug projection 2nml1": 2.0 * na * m * l1,
             "X' sketch+power 2nTl2(1+2q)": 2.0 * n * T * l2 * (1 + 2 * q),
             "X' CholQR2 4nl2^2(1+q)": 4.0 * n * l2 * l2 * (1 + q),
             "X' projection 2nml2": 2.0 * n * m * l2,
             "cross Q1^T Q2 2nl1l2": 2.0 * n * l1 * l2,
             "modes 4nTr": 4.0 * n * T * r}
    return sum(terms.values()), terms


def run_c1x(args, cfg):
    """BASELINE config 1 as written: exact DMD (randomized SVD r = 150, p = 10,
    q = 1) of the 128^3 x 3 matrix from HBM-resident snapshots, then 200 integer
    steps decoded in one batched device GEMM and one interactive single-frame
    GEMV. One JSON line (a side workload; full-size parity of this fit:
    tests/test_gpu_fullsize.py::test_config1_full_size_vs_streamed_oracle)."""
    import warnings

    import torch

    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200 import device as dv
    from paper_2502_05339_b200 import synth, trace
    torch.cuda.set_device(0)
    p = synth.config_params(cfg["cfg"], seed=cfg["seed"], grid=cfg["grid"])
    n, m, r = p.n, p.m, cfg["r"]
    S = dv.alloc_tall(n, m, torch.float32, "row")
    S.buf[:, m:].zero_()
    tabs = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables()]
    dv.get_ops().synth3d(tabs, m, p.noise, synth.noise_key(p.seed), 0, n, S)
    torch.cuda.synchronize()
    data = fd.SnapshotMatrix(S, synth.DT)
    x0 = S.buf[:n, 0].clone()
    F, terms, l = fit_flops(n, m, r, cfg["p"], cfg["q"], modes="exact")
    F -= terms.pop("lift U 2nlr")                       # exact DMD forms no POD lift (dmd.py:240-274)

    def one():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model = fd.exact_dmd(data, r, svd_mode="randomized", seed=cfg["seed"], oversample=cfg["p"],
                                 power_iters=cfg["q"])
            e[1].record()
            z0 = fd.encode(model, x0)
            frames = fd.rollout(model, z0, cfg["steps"], to_host=False)
            frames = frames[0] if isinstance(frames, tuple) else frames
            e[2].record()
            one_frame = fd.decode(model, fd.step_k(model, z0, 7), to_host=False)
        e[3].record()
        torch.cuda.synchronize()
        del frames, one_frame, model
        return [e[i].elapsed_time(e[i + 1]) / 1e3 for i in range(3)]

    for _ in range(args.warmup):
        one()
    trace.enable()
    ts = np.array([one() for _ in range(args.steps)])
    stages = trace.summarize(trace.disable(), args.steps)
    fit_t, roll_t, one_t = [float(x) for x in ts.mean(axis=0)]
    line = {"metric": "config-1 exact DMD fit GFLOP/s + rollout frames/s", "value": round(F / fit_t / 1e9, 1),
            "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round((fit_t + roll_t + one_t) * 1e3, 1), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config1 exact DMD (r=150, p=10, q=1) + 200 integer steps + 1 interactive frame",
                       "n": n, "m": m, "r": r, "l": l, "grid": "128^3x3", "snapshot_dtype": "f32",
                       "l2": "inputs larger than L2"},
            "fit": {"s": round(fit_t, 4), "flops": F, "terms": terms}, "fit_stages_ms": stages,
            "rollout": {"frames": cfg["steps"], "s": round(roll_t, 4),
                        "frames_per_s": round(cfg["steps"] / roll_t, 1),
                        "hbm_GBps": round((4.0 * n * r + 4.0 * n * cfg["steps"]) / roll_t / 1e9, 1)},
            "interactive_frame": {"ms": round(one_t * 1e3, 3),
                                  "hbm_GBps": round(4.0 * n * (r + 1) / one_t / 1e9, 1)}}
    print(json.dumps(line), flush=True)


def run_c2(args, cfg):
    """Config 2: the augmented DMDc fit of a 128^3 x 3 controlled system
    (synth.config2_params) from HBM-resident snapshots, then 200 controlled
    steps driven by a fresh seeded control sequence (rollout(q_seq=...)),
    all frames decoded on the device. One JSON line (a side workload)."""
    import warnings

    import torch

    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200 import device as dv
    from paper_2502_05339_b200 import synth
    torch.cuda.set_device(0)
    p = synth.config2_params(cfg["seed"], grid=cfg["grid"], ell=cfg["ell"])
    n, m = p.n, p.m

    def states(u):
        S = dv.alloc_tall(n, u.shape[1] + 1, torch.float32, "row")
        S.buf[:, u.shape[1] + 1:].zero_()
        tabs = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables(u)]
        dv.get_ops().synth3d(tabs, u.shape[1] + 1, 0.0, 0, 0, n, S)
        return S

    u = p.controls(5)
    S = states(u)
    u2 = p.controls(77, cfg["steps"])
    truth = states(u2)
    x0 = truth.buf[:n, 0].clone()
    q_seq = [[u2[:, k]] for k in range(cfg["steps"])]
    F, terms = dmdc_flops(n, m, cfg["r_aug"], cfg["r"], cfg["p"], cfg["q"], cfg["ell"])

    def one():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model, ctrl = fd.dmdc_fit(fd.SnapshotMatrix(S, 1.0), u, cfg["r_aug"], cfg["r"], seed=3,
                                      oversample=cfg["p"], power_iters=cfg["q"])
            e[1].record()
            z0 = fd.encode(model, x0)
            frames, _ = fd.rollout(model, z0, cfg["steps"], ctrl=ctrl, q_seq=q_seq, to_host=False)
        e[2].record()
        torch.cuda.synchronize()
        return e[0].elapsed_time(e[1]) / 1e3, e[1].elapsed_time(e[2]) / 1e3, frames

    from paper_2502_05339_b200 import trace
    for _ in range(args.warmup):
        one()
    trace.enable()
    ts = [one() for _ in range(args.steps)]
    stages = trace.summarize(trace.disable(), args.steps)
    fit_t = float(np.mean([t[0] for t in ts]))
    roll_t = float(np.mean([t[1] for t in ts]))
    frames = ts[-1][2]
    tr = truth.buf[:n, 1:cfg["steps"] + 1].t().double()
    err = float(((frames.double() - tr).norm(dim=1) / tr.norm(dim=1)).max())
    line = {"metric": "config-2 DMDc fit GFLOP/s + controlled rollout frames/s", "value": round(F / fit_t / 1e9, 1),
            "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round((fit_t + roll_t) * 1e3, 1), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2 DMDc fit ([X;Upsilon] r_aug=158, p=10, q=1; output basis r=150) + "
                                   "200 controlled steps with fresh seeded controls", "n": n, "m": m, "ell": cfg["ell"],
                       "grid": "128^3x3", "snapshot_dtype": "f32", "l2": "inputs larger than L2"},
            "fit": {"s": round(fit_t, 4), "flops": F, "terms": terms}, "fit_stages_ms": stages,
            "rollout": {"frames": cfg["steps"], "s": round(roll_t, 4), "frames_per_s": round(cfg["steps"] / roll_t, 1),
                        "max_rel_err_vs_generator": err}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="fdmd", choices=["fdmd", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=65536)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.config == "c2":
        return run_c2(args, cfg)
    if args.config == "c1x":
        return run_c1x(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    world, rank, local = _dist_init()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch_distributed(args)
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    from paper_2502_05339_b200 import shards
    # NCCL_ALGO / NCCL_PROTO pinned (deterministic sums). FDMD_DIST_BACKEND=gloo is a
    # functional check of the multi-rank path on a 1-GPU box (every rank on cuda:0,
    # host-staged collectives): its timings mean nothing
    shards.init_process_group(os.environ.get("FDMD_DIST_BACKEND", "nccl"))
    group = None
    if world > 1:
        import torch.distributed as dist
        group = dist.group.WORLD

    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200 import _lib, synth, trace
    from paper_2502_05339_b200 import device as dv
    from paper_2502_05339_b200.runtime import ModalBasis

    p = synth.config_params(cfg["cfg"], seed=cfg["seed"], grid=cfg["grid"])
    n, m, r = p.n, p.m, cfg["r"]
    bounds = np.linspace(0, n, world + 1).astype(np.int64)
    row0, row1 = int(bounds[rank]), int(bounds[rank + 1])
    n_loc = row1 - row0
    shard = dv.Shard(row0, n_loc, n, group, world) if world > 1 else None

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- inputs resident in HBM (device generator, synth.py recipe) ----
    S = dv.alloc_tall(n_loc, m, torch.float32, "row")
    S.buf[:, m:].zero_()
    tabs = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables()]
    dv.get_ops().synth3d(tabs, m, p.noise, synth.noise_key(p.seed), row0, n_loc, S)
    torch.cuda.synchronize()
    data = fd.SnapshotMatrix(S, synth.DT, shard=shard)
    # config 4: W (r x r complex), Lam and b from config 3's generator (conjugate-closed)
    rng = np.random.default_rng(4)
    lam4 = np.concatenate([p.lam, np.conj(p.lam)])[:r]
    b4 = np.concatenate([p.b, np.conj(p.b)])[:r]
    W4 = (rng.standard_normal((r, r)) + 1j * rng.standard_normal((r, r))) / np.sqrt(2 * r)
    times = rng.uniform(0.0, 300.0, cfg["times"])
    peak_burst = ctypes_peak(_lib, 0.4)
    peak = ctypes_peak(_lib, 8.0)                           # sustained: one ~2 s launch after ~2 s of ramp
    ops = dv.get_ops()
    F_fit, terms, l = fit_flops(n, m, r, cfg["p"], cfg["q"])
    lm = fd.LMConfig(max_iters=cfg["lm_iters"])

    route_used = [None]   # projection route the fit took (linalg.PROJ_GRAM_TOL)
    chunk_used = [None]   # frames per tcgen05 launch (U streamed once per launch; clusters multicast it)

    def one_step(record):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        import warnings
        with warnings.catch_warnings(), trace.stage("fit"):
            warnings.simplefilter("ignore")
            model = fd.optdmd(data, r, lm_config=lm, svd_mode="randomized", seed=cfg["seed"],
                              oversample=cfg["p"], power_iters=cfg["q"], keep_basis=BASIS_MODE)
        ev[1].record()
        route_used[0] = "gram_projection" if model.provenance["sketch"].get("gram_projection") else "direct"
        U = model.basis_U
        del model                                            # config 4 reconstructs from U, not the table
        mb = ModalBasis(U, W4, lam4, b4, dt=1.0)
        f1 = mb.reconstruct(times[:1])                       # interactive frame (one basis pass)
        ev[2].record()
        with trace.stage("reconstruct.basis_split"):
            mb.tc_state()                                    # fp16 hi/lo planes (written by the lift already)
        ev[3].record()
        mb.release_fp32()
        del U                                                # the planes carry the basis from here on
        if chunk_used[0] is None:                            # fixed at the first (warm-up) step:
            chunk_used[0] = frame_chunk(n_loc, len(times))   # S + planes resident, fp32 U released
        chunk = chunk_used[0]
        outb = torch.empty((chunk, n_loc), dtype=torch.float32, device="cuda")
        mb.reconstruct(times[:32], out=outb[:32])            # one 32-frame batch
        ev[4].record()
        for c0 in range(0, len(times), chunk):               # 1024 frames streamed through one buffer
            mb.reconstruct(times[c0:c0 + chunk], out=outb[: len(times[c0:c0 + chunk])])
        ev[5].record()
        torch.cuda.synchronize()
        t = [ev[0].elapsed_time(ev[i]) / 1e3 for i in range(1, 6)]
        del mb, f1, outb
        return {"fit": t[0], "rec1": t[1] - t[0], "split": t[2] - t[1], "rec32": t[3] - t[2],
                "rec1024": t[4] - t[3]}

    for _ in range(args.warmup):
        one_step(False)
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    ops.profile = []
    trace.enable()
    launches0 = ops.launches
    barrier()
    torch.cuda.synchronize()
    t0e = torch.cuda.Event(enable_timing=True)
    t1e = torch.cuda.Event(enable_timing=True)
    t0e.record()
    res = [one_step(True) for _ in range(args.steps)]
    t1e.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ops.launches - launches0
    prof = ops.profile
    ops.profile = None
    rec_raw = trace.disable()
    stages = trace.summarize(rec_raw, args.steps)
    if os.environ.get("FDMD_BENCH_DIAG"):
        # per-occurrence device / host ms of the first stages of each fit, then the
        # same snapshot Gram launched in isolation (first-kernel-of-step effects)
        for name, e0, e1, h in rec_raw:
            if name in ("power.XtX", "sketch.alloc_Q", "power.Y=XWR1^-1", "cholqr.gram2"):
                print(f"diag {name}: device {e0.elapsed_time(e1):.2f} ms host {h * 1e3:.2f} ms", file=sys.stderr)
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            ops.tall_gram(data.S, data.S, K1=m - 1, K2=m - 1, symmetric=True)
            e1.record()
            torch.cuda.synchronize()
            print(f"diag isolated XtX: {e0.elapsed_time(e1):.2f} ms", file=sys.stderr)
    # the two FP64 DMMA kernels of the fit launched ALONE (after the timed region,
    # GPU idle for 1 s first): inside the step the snapshot Gram is the first kernel
    # after the reconstruct phase and runs clock-capped (sw_power_cap)
    isolated = {}
    if route_used[0] == "gram_projection":
        T_ = m - 1
        Um_ = torch.randn((T_, r), dtype=torch.float64, device="cuda") / T_
        iso_cases = {
            "tall_gram_panel_kernel (bordered snapshot Gram)":
                (lambda: ops.tall_gram_bordered(data.S, T_), 1.0 * n_loc * T_ * T_ + 2.0 * n_loc * T_),
            "tall_gemm_tma_kernel (lift into planes)":
                (lambda: ops.tall_gemm_planes(data.S, Um_, bound=1e3), 2.0 * n_loc * T_ * r),
        }
        saved_prof, ops.profile = ops.profile, None
        for name, (fn, fl) in iso_cases.items():
            torch.cuda.synchronize()
            time.sleep(1.0)
            best = 1e9
            for _ in range(3):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                out_ = fn()
                e1.record()
                torch.cuda.synchronize()
                del out_
                best = min(best, e0.elapsed_time(e1))
            isolated[name] = {"ms": round(best, 2), "tflops": round(fl / best / 1e9, 2),
                              "frac": round(fl / best / 1e9 / peak, 4)}
        ops.profile = saved_prof
        del Um_
    total = max_over_ranks(t0e.elapsed_time(t1e) / 1e3)
    fit_t = max_over_ranks(float(np.mean([x["fit"] for x in res])))
    rec = {k: max_over_ranks(float(np.mean([x[k] for x in res]))) for k in ("rec1", "split", "rec32", "rec1024")}

    # roofline: FP64 DMMA contraction kernels (tall_gemm + tall_gram), CUDA events
    kt = {"tall_gemm": [0.0, 0.0, 0, 0.0], "tall_gram": [0.0, 0.0, 0, 0.0], "decode": [0.0, 0.0, 0, 0.0],
          "tc_decode": [0.0, 0.0, 0, 0.0]}
    for name, fl, e0, e1, nb in prof:
        kt.setdefault(name, [0.0, 0.0, 0, 0.0])
        kt[name][0] += e0.elapsed_time(e1) / 1e3
        kt[name][1] += fl
        kt[name][2] += 1
        kt[name][3] += nb
    fit_kernel_t = (kt["tall_gemm"][0] + kt["tall_gram"][0]) / args.steps
    # per-GPU TFLOP/s of all DMMA contraction launches (flops each launch executes)
    achieved_all = (kt["tall_gemm"][1] + kt["tall_gram"][1]) / args.steps / max(fit_kernel_t, 1e-12) / 1e12
    # dominant kernel of the step by device time among the fit's tensor-bound
    # FP64 kernels (the tcgen05 reconstruction kernels are HBM-bound, reported
    # under "reconstruct")
    dom = max(("tall_gemm", "tall_gram"), key=lambda k: kt[k][0])
    g = kt[dom]
    achieved = g[1] / max(g[0], 1e-12) / 1e12                         # executed flops / its launch time
    value = F_fit / fit_t / 1e9

    # reconstruct figures (config 4, HBM-bound)
    def rec_obj(B, t):
        byt = 4.0 * n * r + 4.0 * n * B + 8.0 * r * B
        gbs = byt / t / 1e9 / world
        return {"frames_per_s": round(B / t, 1), "ms": round(t * 1e3, 3), "hbm_GBps_per_gpu": round(gbs, 1),
                "frac_hbm": round(gbs / hbm_peak(), 3)}
    recon = {"B=1": rec_obj(1, rec["rec1"]), "B=32": rec_obj(32, rec["rec32"])}
    recon["B=1"]["kernel"] = ("tc_decode (tcgen05 over the basis planes, one basis pass)" if BASIS_MODE == "planes"
                              else "decode (SIMT GEMV over fp32 U)")
    recon["B=32"]["kernel"] = "tc_decode (tcgen05, FP16 2-way split)"
    b1024 = rec["rec1024"]
    CHUNK = chunk_used[0]
    B = len(times)
    # SURVEY §8(d) algorithmic bytes: the basis read ONCE + frames written (+ coefficients)
    alg = 4.0 * n * r + 4.0 * n * B + 8.0 * r * B
    # what the streamed schedule must move: the basis once per launch + frames
    sched = (4.0 * n * r) * math.ceil(B / CHUNK) + 4.0 * n * B
    recon["B=1024"] = {"frames_per_s": round(B / b1024, 1), "ms": round(b1024 * 1e3, 2),
                       "hbm_GBps_per_gpu": round(alg / b1024 / 1e9 / world, 1),
                       "frac_hbm": round(alg / b1024 / 1e9 / world / hbm_peak(), 3),
                       "frac_basis": "§8(d) bytes: basis read once + frames written",
                       "schedule_GBps_per_gpu": round(sched / b1024 / 1e9 / world, 1),
                       "schedule_bytes": sched,
                       "frames_per_launch": CHUNK,
                       "kernel": f"tc_decode2 (tcgen05 cta_group::2 CTA pairs, 256 frames per pair tile; the "
                                 f"launch's frame tiles interleaved with the row pairs so they share the basis "
                                 f"rows through one die's L2), {CHUNK}-frame launches "
                                 f"streamed through one buffer (1024 frames = {B * 4.0 * n / 1e9:.0f} GB > HBM)"}
    recon["basis_split_ms"] = round(rec["split"] * 1e3, 2)

    # ---- e2e through the public API from pinned host memory ----
    e2e = None
    if not args.no_e2e:
        host = torch.empty((n_loc, m), dtype=torch.float32, pin_memory=True)
        host.copy_(S.view().cpu())
        del data, S
        torch.cuda.empty_cache()
        e2e = run_e2e(args, fd, host, n_loc, m, r, cfg, lm, shard, F_fit, max_over_ranks, barrier)

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config(cfg, n, m, r, l, f"rows{world}"),
        "fit": {"s": round(fit_t, 4), "gflops": round(value, 1), "flops": F_fit,
                "per_step_s": [round(x["fit"], 4) for x in res],
                "terms": {k: v for k, v in terms.items()},
                "value_kind": "equivalent-work rate: SURVEY §8(d) reference-algorithm flops / fit time (an "
                              "algebraically equivalent restructuring counts as the terms it replaces); the "
                              "roofline-comparable rate is executed_tflops",
                "projection_route": route_used[0],
                "executed_flops": executed_flops(n, m, r, cfg["p"], cfg["q"], route_used[0]),
                "executed_terms_fp64_dmma": executed_terms(n, m, r, cfg["p"], cfg["q"], route_used[0])[0],
                "executed_terms_tcgen05_fp32_accurate": executed_terms(n, m, r, cfg["p"], cfg["q"], route_used[0])[1],
                "executed_tflops": round(executed_flops(n, m, r, cfg["p"], cfg["q"], route_used[0]) / fit_t / 1e12, 3)},
        "reconstruct": recon,
        "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "peak_burst": round(peak_burst, 2),
                     "frac_burst": round(achieved / peak_burst, 4),
                     "traffic": traffic_from_profiles(DOM_NAMES[dom], args.config),
                     "kernel": DOM_NAMES[dom] + " (FP64 DMMA m8n8k4, TMA-fed); achieved = flops its "
                               "launches execute (symmetric Gram / triangular apply as n*l^2) / their CUDA-event time",
                     "algorithmic_bytes_per_launch": round(g[3] / max(g[2], 1)),
                     "traffic_source": f"profiles/dominant_kernel_traffic.json[{args.config}] (ncu "
                                       "dram__bytes_read+write per launch of this kernel, this config, one bench "
                                       "step, same code)",
                     "peak_source": "in-run DMMA.8x8x4 throughput probe (fdmd_dmma_peak): `peak` sustained (one "
                                    "~2 s launch after ~2 s of ramp), `peak_burst` a ~0.1 s launch; spec 40 TF/s; "
                                    "MEASURED_PEAKS.json has no FP64 figure",
                     "contractions": {"kernels": "tall_gemm + tall_gram (all FP64 DMMA work of the fit)",
                                      "achieved": round(achieved_all, 3), "frac": round(achieved_all / peak, 4),
                                      "share_of_fit": round(fit_kernel_t / fit_t, 3)},
                     "in_step_tflops": {DOM_NAMES[k]: round(kt[k][1] / max(kt[k][0], 1e-12) / 1e12, 2)
                                        for k in ("tall_gemm", "tall_gram") if kt[k][2]},
                     "isolated": isolated,
                     "launches_per_step": {k: v[2] // args.steps for k, v in kt.items()},
                     "ms_per_step": {k: round(v[0] / args.steps * 1e3, 2) for k, v in kt.items()}},
        "fit_stages_ms": stages,
        "clocks": clk,
        "gpu_launches": launches,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if rank == 0 and not args.no_cpu:
        arm = CpuArm()
        s = cpu_sample(arm, synth, cfg, args.cpu_rows)
        t0 = time.perf_counter()
        arm.fit(s["X"], cfg)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": round(s["flops"] / dt / 1e9, 3), "unit": "GFLOP/s", "cores": os.cpu_count(),
                                "kind": arm.kind, "sample": s["sample"], "s": round(dt, 2)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_e2e(args, fd, host, n_loc, m, r, cfg, lm, shard, F_fit, max_over_ranks, barrier):
    import warnings

    import torch
    from paper_2502_05339_b200 import trace
    ts = []
    stages = {}
    inner = {}
    for i in range(1 + args.e2e_steps):
        barrier()
        torch.cuda.synchronize()
        if i >= 1:
            trace.enable()
        t0 = time.perf_counter()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            with trace.stage("e2e.upload"):   # streamed: the transfer overlaps the first sketch stage
                d2 = fd.SnapshotMatrix(host, 0.1, shard=shard, stream=True)
            with trace.stage("e2e.fit"):
                model = fd.optdmd(d2, r, lm_config=lm, svd_mode="randomized", seed=cfg["seed"],
                                  oversample=cfg["p"], power_iters=cfg["q"])
            with trace.stage("e2e.frame_d2h"):
                z0 = fd.ReducedState(np.ones(r, dtype=complex))
                frame = fd.decode(model, fd.step_k(model, z0, 10))        # D2H of one frame
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i >= 1:
            rec = trace.disable()
            for k, v in trace.summarize(rec).items():
                if k.startswith("e2e."):
                    stages[k] = stages.get(k, 0.0) + v / args.e2e_steps
                else:   # what the e2e fit is made of (the upload with the Gram under it, then the tail)
                    inner[k] = inner.get(k, 0.0) + v / args.e2e_steps
        del d2, model, frame
        if i >= 1:
            ts.append(max_over_ranks(dt))
    t = float(np.mean(ts))
    return {"value": round(F_fit / t / 1e9, 2), "unit": "GFLOP/s", "s_per_step": round(t, 3),
            "stages_ms": {k: round(v, 1) for k, v in stages.items()},
            "fit_stages_ms": {k: round(v, 1) for k, v in inner.items() if v >= 1.0},
            "h2d_bytes_per_step": int(n_loc * m * 4), "d2h_bytes_per_step": int(n_loc * 8 + 2 * r * 16),
            "api": "SnapshotMatrix(pinned host f32, stream=True) -> optdmd (H2D overlapped with the first "
                   "sketch stage) -> decode(step_k) to host"}


def frame_chunk(n_loc, total, keep=0.0, margin=3e9):
    """Frames per reconstruction launch: the widest 128 * 2^k batch whose
    frame buffer fits in free HBM after `keep` more bytes (the basis planes)
    with `margin` to spare. A launch's frame tiles walk the basis rows in
    lock-step, so the basis is fetched from DRAM ~once per launch (L2)."""
    import torch
    free = torch.cuda.mem_get_info()[0] + torch.cuda.memory_reserved() - torch.cuda.memory_allocated() - keep
    chunk = 128
    while chunk * 2 <= total and chunk * 2 * 4.0 * n_loc <= free - margin:
        chunk *= 2
    return min(chunk, total)


def ctypes_peak(_lib, seconds):
    """DMMA.8x8x4 throughput probe (fdmd_dmma_peak): the last launch of a
    growing series lasts ~seconds/4 (0.4 -> burst, 8 -> sustained)."""
    import ctypes
    v = ctypes.c_double(0.0)
    _lib.check(_lib.lib().fdmd_dmma_peak(float(seconds), ctypes.byref(v)), "dmma_peak")
    return v.value


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


# config-4 basis kept by the fit: "planes" = the lift writes the fp16 hi/lo planes
# the reconstruction streams (no fp32 U, no split pass); FDMD_BENCH_BASIS=fp32
# keeps the fp32 basis + a separate split (round-1 schedule)
BASIS_MODE = "planes" if os.environ.get("FDMD_BENCH_BASIS", "planes") == "planes" else True

DOM_NAMES = {"tall_gemm": "tall_gemm_tma_kernel", "tall_gram": "tall_gram_panel_kernel"}


def traffic_from_profiles(kernel, config="c3"):
    """dram bytes per launch of `kernel` for this config from the committed
    ncu summary (profiles/dominant_kernel_traffic.json, keyed by config),
    or None when that config/kernel was not profiled with the current code."""
    path = os.path.join(ROOT, "profiles", "dominant_kernel_traffic.json")
    try:
        js = json.load(open(path))
    except Exception:
        return None
    ent = js.get("configs", {}).get(config, {})
    return ent.get("kernels", {}).get(kernel, {}).get("traffic_bytes_per_launch")


if __name__ == "__main__":
    main()
