"""Golden files for the on-disk formats, written by the REAL reference here.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:. python oracle/gen_golden_io.py

Writes tests/golden/io/: a model file saved by flowdmd.model_io.save_model
(exact DMD of a reference test system, with grid metadata and provenance),
a dataset directory saved by save_dataset (with grid + solid cells, density
frames and meta entries), a conjugate-pair-broken hand-built model, and
io_expect.npz with the values the reference's loaders return (phi, lam,
sigma, states, decoded frames) so the -m gpu tests can compare without the
reference. All files are small (< 200 kB).
"""

from __future__ import annotations

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from flowdmd import model_io                         # noqa: E402  (reference, read-only import)
from flowdmd.dmd import ReducedModel, SnapshotMatrix, exact_dmd  # noqa: E402
from flowdmd.grid import GridSpec                    # noqa: E402
from flowdmd.runtime import decode, encode, step_k   # noqa: E402
from conftest import stable_linear_system            # noqa: E402  (reference test fixture)

OUT = os.path.join(ROOT, "tests", "golden", "io")


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    # a 2D-grid-shaped state: nx = 6, ny = 5 MAC grid (n = (nx+1) ny + nx (ny+1) = 71)
    mask = np.zeros((5, 6), dtype=bool)
    mask[2, 3] = True
    grid = GridSpec(6, 5, 0.25, "open", mask)
    n = (6 + 1) * 5 + 6 * (5 + 1)
    rng = np.random.default_rng(11)
    X = np.asarray(stable_linear_system(n, 6, 40, 3)[0].states)
    snaps = SnapshotMatrix(X, 0.05, grid, {"solver": "test", "note": "golden", "cfl": 0.5})
    density = rng.standard_normal((5, 6, X.shape[1]))
    model_io.save_dataset(os.path.join(OUT, "dataset"), snaps, density)
    model = exact_dmd(snaps, 6, svd_mode="full")
    model_io.save_model(os.path.join(OUT, "model.kdmd"), model)
    # hand-built model whose partner columns are NOT exact conjugates
    lam = np.array([0.9 * np.exp(0.3j), 0.9 * np.exp(-0.3j), 0.5])
    phi = rng.standard_normal((n, 3)) + 1j * rng.standard_normal((n, 3))
    hb = ReducedModel(phi, lam, np.array([3.0, 2.0, 1.0]), 0.1, None, {"method": "hand", "k": 3})
    model_io.save_model(os.path.join(OUT, "handbuilt.kdmd"), hb)
    loaded = model_io.load_model(os.path.join(OUT, "model.kdmd"))
    z0 = encode(loaded, X[:, 0])
    np.savez(os.path.join(OUT, "io_expect.npz"),
             X=X, phi=loaded.phi, lam=loaded.lam, sigma=loaded.sigma, dt=loaded.dt,
             frame5=decode(loaded, step_k(loaded, z0, 5)), z0=z0.z,
             hb_phi=phi, hb_lam=lam, density=density,
             manifest=open(os.path.join(OUT, "dataset", "manifest")).read())
    # the reference CLI on the golden dataset (cli.py:126-270)
    import contextlib
    import io as _io
    from flowdmd.cli import cli_main
    cli = os.path.join(OUT, "cli")
    os.makedirs(cli)
    ds = os.path.join(OUT, "dataset")
    runs = {
        "train": ["train", ds, "-o", os.path.join(cli, "trained.kdmd"), "--rank", "6"],
        "train_opt": ["train", ds, "-o", os.path.join(cli, "trained_opt.kdmd"), "--rank", "6",
                      "--method", "optdmd", "--svd", "randomized", "--seed", "3"],
        "rollout": ["rollout", "--model", os.path.join(OUT, "model.kdmd"), "--dataset", ds, "--start-frame", "2",
                    "--k", "2", "--frames", "5", "--out", os.path.join(cli, "rollout")],
        "reverse": ["reverse", "--model", os.path.join(OUT, "model.kdmd"), "--dataset", ds, "--start-frame", "30",
                    "--frames", "3", "--out", os.path.join(cli, "reverse")],
        "eval": ["eval", "--model", os.path.join(OUT, "model.kdmd"), "--dataset", ds, "--stride", "3"],
        "bad_start": ["rollout", "--model", os.path.join(OUT, "model.kdmd"), "--dataset", ds, "--start-frame",
                      "99", "--out", os.path.join(cli, "nope")],
    }
    outs = {}
    for name, argv in runs.items():
        so, se = _io.StringIO(), _io.StringIO()
        with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
            rc = cli_main(argv)
        outs[name] = (rc, so.getvalue(), se.getvalue())
    with open(os.path.join(cli, "outputs.txt"), "w") as fh:
        for name, (rc, so, se) in outs.items():
            fh.write(f"## {name} rc={rc}\n{so}--stderr--\n{se}")
    for root, _, files in os.walk(OUT):
        for f in files:
            print(os.path.relpath(os.path.join(root, f), ROOT), os.path.getsize(os.path.join(root, f)))


if __name__ == "__main__":
    main()
