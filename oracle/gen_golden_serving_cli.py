"""Golden outputs of the reference CLI commands that use editing, density
advection and guided upscaling (cli.py:138-234), run by the REAL reference
in this container.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_serving_cli.py

Writes tests/golden/serving_cli/: a plume dataset (reference solver, with
density frames) and its 2x-coarsened guide dataset, an exact-DMD model file,
an edit spec file, and the reference CLI's output datasets for
  rollout --edit --density, reverse --density, upres (project on / off)
plus outputs.txt (exit codes and stdout). Nothing here runs on the GPU box.
"""

from __future__ import annotations

import contextlib
import io
import os
import shutil

import numpy as np

from flowdmd import model_io                                   # reference, read-only import
from flowdmd.cli import cli_main
from flowdmd.dmd import SnapshotMatrix, exact_dmd
from flowdmd.editing import EditSpec, cluster_modes
from flowdmd.grid import build_downsample, coarse_grid
from flowdmd.solver import SceneConfig, generate_dataset

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "serving_cli")


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    scene = SceneConfig(kind="plume", nx=16, ny=32, h=1.0 / 16, frames=14)
    snap, dens = generate_dataset(scene)
    ds = os.path.join(OUT, "dataset")
    model_io.save_dataset(ds, snap, dens)
    model = exact_dmd(model_io.load_dataset(ds), 6)
    mpath = os.path.join(OUT, "model.kdmd")
    model_io.save_model(mpath, model)
    low_g = coarse_grid(snap.grid_meta, 2)
    A = build_downsample(snap.grid_meta, 2)
    low = SnapshotMatrix(A @ snap.states[:, :6], snap.dt, low_g, {"solver": "downsample"})
    lpath = os.path.join(OUT, "low")
    model_io.save_dataset(lpath, low)
    _, high = cluster_modes(model)
    spec = EditSpec.identity(model.r)
    spec.weights[high] = 0.6
    spec.growth_scale[high] = 0.8
    spec.freq_scale[high] = 1.25
    epath = os.path.join(OUT, "edit.kv")
    model_io.save_edit(epath, spec)
    spath = os.path.join(OUT, "scene.kv")
    model_io.save_scene(spath, SceneConfig(kind="plume", nx=16, ny=32, h=1.0 / 16, frames=6, warmup=2))
    runs = {
        "simulate": ["simulate", spath, "-o", os.path.join(OUT, "sim")],
        "rollout_edit_density": ["rollout", "--model", mpath, "--dataset", ds, "--start-frame", "1", "--k", "2",
                                 "--frames", "4", "--edit", epath, "--density",
                                 "--out", os.path.join(OUT, "rollout_ed")],
        "reverse_density": ["reverse", "--model", mpath, "--dataset", ds, "--start-frame", "8", "--frames", "3",
                            "--density", "--out", os.path.join(OUT, "reverse_d")],
        "upres_on": ["upres", "--low", lpath, "--model", mpath, "--split", "4", "--factor", "2",
                     "--out", os.path.join(OUT, "upres_on")],
        "upres_off": ["upres", "--low", lpath, "--model", mpath, "--split", "3", "--factor", "2",
                      "--project", "off", "--out", os.path.join(OUT, "upres_off")],
        "upres_bad_factor": ["upres", "--low", lpath, "--model", mpath, "--split", "4", "--factor", "3",
                             "--out", os.path.join(OUT, "nope")],
    }
    with open(os.path.join(OUT, "outputs.txt"), "w") as fh:
        for name, argv in runs.items():
            so, se = io.StringIO(), io.StringIO()
            with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
                rc = cli_main(argv)
            fh.write(f"## {name} rc={rc}\n{so.getvalue().replace(OUT, '<OUT>')}--stderr--\n"
                     f"{se.getvalue().replace(OUT, '<OUT>')}")
    total = 0
    for root, _, files in os.walk(OUT):
        for f in files:
            total += os.path.getsize(os.path.join(root, f))
    print("wrote", OUT, total, "bytes")


if __name__ == "__main__":
    main()
