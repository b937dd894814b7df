"""Interactive-serving throughput: one request =
ModelServer.frame_payload(session, k, "speed", "bin") on a large 2-D MAC grid.

    python tools/serve_bench.py [--nx 2048 --ny 2048 --r 64 --threads 8]

Reports (JSON line):
  * mac_decode kernel: CUDA-event time, algorithmic bytes (table read once:
    8 * n_state * ncol for f64, + planes written) -> GB/s and fraction of the
    measured HBM peak (MEASURED_PEAKS.json);
  * frame_payload latency (host call incl. the f32 plane D2H) serial, and
    request throughput with T threads (one CUDA stream per thread);
  * the CPU oracle port of the same frame (numpy decode table @ c + centring,
    all host cores) for one request, as the reference's cost.
The model is synthetic (random conjugate-paired modes of the requested rank).
"""

import argparse
import json
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import paper_2502_05339_b200 as fd                     # noqa: E402
from paper_2502_05339_b200 import device as dv          # noqa: E402


def hbm_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("hbm_gbs",):
            if k in d:
                return float(d[k])
    except Exception:
        pass
    return 6550.7


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=2048)
    ap.add_argument("--ny", type=int, default=2048)
    ap.add_argument("--r", type=int, default=64)
    ap.add_argument("--threads", type=int, default=8)
    ap.add_argument("--requests", type=int, default=20)
    ap.add_argument("--cpu", action="store_true", help="also time the CPU oracle port")
    a = ap.parse_args()
    nx, ny, r = a.nx, a.ny, a.r
    g = fd.GridSpec(nx, ny, 1.0 / nx)
    n = g.n_state
    rng = np.random.default_rng(0)
    pairs = r // 2
    lam_h = 0.98 * np.exp(1j * rng.uniform(0.05, 1.0, pairs))
    lam = np.empty(r, dtype=np.complex128)
    lam[0::2], lam[1::2] = lam_h, np.conj(lam_h)
    # device table directly (the host phi of this size would be 8.6 GB complex)
    from paper_2502_05339_b200.modes import DeviceModes, TableLayout
    lay = TableLayout(lam)
    T = dv.alloc_tall(n, lay.ncol, torch.float64, "col")
    T.buf[: lay.ncol, :n].normal_()
    model = fd.ReducedModel(None, lam, np.ones(r), 0.1, g, {}, _modes=DeviceModes(T, lay))
    srv = fd.ModelServer(model)
    sess = srv.get_session(srv.create_session({}))
    ops = dv.get_ops()
    c = torch.randn(lay.ncol, dtype=torch.float64, device="cuda")
    for _ in range(3):
        ops.mac_decode(T, c, nx, ny, "speed")
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 20
    ev[0].record()
    for _ in range(reps):
        ops.mac_decode(T, c, nx, ny, "speed")
    ev[1].record()
    torch.cuda.synchronize()
    k_ms = ev[0].elapsed_time(ev[1]) / reps
    alg_bytes = 8.0 * n * lay.ncol + 8.0 * nx * ny
    gbs = alg_bytes / k_ms / 1e6
    # host-call latency (serial)
    for k in range(3):
        srv.frame_payload(sess, k, "speed", "bin")
    t0 = time.perf_counter()
    for k in range(a.requests):
        srv.frame_payload(sess, k, "speed", "bin")
    lat = (time.perf_counter() - t0) / a.requests
    # concurrent sessions
    sessions = [srv.get_session(srv.create_session({})) for _ in range(a.threads)]

    def work(s):
        for k in range(a.requests):
            srv.frame_payload(s, k, "speed", "bin")

    th = [threading.Thread(target=work, args=(s,)) for s in sessions]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    conc = a.threads * a.requests / (time.perf_counter() - t0)
    out = {"workload": f"frame_payload speed/bin, {nx}x{ny} MAC grid (n_state={n}), r={r}, f64 table",
           "mac_decode": {"ms": round(k_ms, 4), "alg_bytes": alg_bytes, "GBps": round(gbs, 1),
                          "frac_hbm": round(gbs / hbm_peak(), 3)},
           "frame_payload_ms_serial": round(lat * 1e3, 3),
           f"requests_per_s_{a.threads}_threads": round(conc, 1),
           "payload_bytes": 12 + 4 * nx * ny}
    if a.cpu:
        import flowdmd_oracle as orc
        D = T.buf[: lay.ncol, :n].t().cpu().numpy()
        cc = c.cpu().numpy()
        t0 = time.perf_counter()
        reps_c = 3
        for _ in range(reps_c):
            planes = orc.center_planes(D @ cc, nx, ny, "speed")
            orc.encode_planes(planes, "bin")
        out["cpu_oracle_ms"] = round((time.perf_counter() - t0) / reps_c * 1e3, 1)
        out["cpu_cores"] = os.cpu_count()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
