"""Device smoke-solver throughput: steps/s of the
reference plume scene at a larger grid, and CG iterations per step.

    python tools/solver_bench.py [--nx 64 --ny 128 --frames 20 --cg-max-iters 1000]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_05339_b200 import solver  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=64)
    ap.add_argument("--ny", type=int, default=128)
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--cg-max-iters", type=int, default=1000)
    a = ap.parse_args()
    scene = solver.SceneConfig(kind="plume", nx=a.nx, ny=a.ny, h=1.0 / a.nx, frames=3, cg_max_iters=a.cg_max_iters)
    solver.generate_dataset(scene)                      # warm-up (allocations, module load)
    scene = solver.SceneConfig(kind="plume", nx=a.nx, ny=a.ny, h=1.0 / a.nx, frames=a.frames,
                               cg_max_iters=a.cg_max_iters)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    data, dens = solver.generate_dataset(scene)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"workload": f"plume {a.nx}x{a.ny}, {a.frames} frames (reference solver pipeline)",
                      "s": round(dt, 3), "steps_per_s": round((a.frames - 1) / dt, 2),
                      "n_state": data.S.n}))


if __name__ == "__main__":
    main()
