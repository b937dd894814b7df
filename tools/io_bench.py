"""Throughput of the streaming model/dataset I/O at BASELINE config-1 size
(n = 6,291,456, m = 201, r = 150): dataset write/read (10 GB f64) and model
write/read (15 GB c128 phi). Files go to --dir (default /tmp on the box).

    python tools/io_bench.py [--dir /tmp/fdmd_io] [--grid 128]
"""
import argparse
import json
import os
import shutil
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_05339_b200 as fd  # noqa: E402
from paper_2502_05339_b200 import device as dv, model_io as mio, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="/tmp/fdmd_io")
    ap.add_argument("--grid", type=int, default=128)
    a = ap.parse_args()
    os.makedirs(a.dir, exist_ok=True)
    p = synth.config_params(1, seed=1, grid=a.grid)
    S = dv.alloc_tall(p.n, p.m, torch.float64, "row", zero=True)
    tabs = [torch.as_tensor(np.ascontiguousarray(t), device="cuda") for t in p.sep_tables()]
    dv.get_ops().synth3d(tabs, p.m, p.noise, synth.noise_key(p.seed), 0, p.n, S)
    data = fd.SnapshotMatrix(S, synth.DT, check_finite=False)
    res = {"n": p.n, "m": p.m}
    ds = os.path.join(a.dir, "ds")
    torch.cuda.synchronize()
    t = time.perf_counter(); mio.save_dataset(ds, data); dt_w = time.perf_counter() - t
    nb = 8.0 * p.n * p.m
    t = time.perf_counter(); d2 = mio.load_dataset(ds, dtype=torch.float32); torch.cuda.synchronize()
    dt_r = time.perf_counter() - t
    res["dataset_write_GBps"] = round(nb / dt_w / 1e9, 2)
    res["dataset_read_GBps"] = round(nb / dt_r / 1e9, 2)
    model = fd.exact_dmd(d2, 150, svd_mode="randomized", seed=1, oversample=10, power_iters=1, residual=False)
    mp = os.path.join(a.dir, "m.kdmd")
    t = time.perf_counter(); mio.save_model(mp, model); dt_mw = time.perf_counter() - t
    mb = os.path.getsize(mp)
    t = time.perf_counter(); back = mio.load_model(mp); torch.cuda.synchronize(); dt_mr = time.perf_counter() - t
    res["model_bytes"] = mb
    res["model_write_GBps"] = round(mb / dt_mw / 1e9, 2)
    res["model_read_GBps"] = round(mb / dt_mr / 1e9, 2)
    res["roundtrip_lam_equal"] = bool(np.array_equal(back.lam, model.lam))
    print(json.dumps(res))
    shutil.rmtree(a.dir, ignore_errors=True)


if __name__ == "__main__":
    main()
