"""Multi-rank (row-sharded) fit orchestration on CPU: world_size 2 over gloo,
with the CPU checker standing in for libfdmd (tests/cpu_ops.py). Every
reduction over rows must be all-reduced, argmax pivots must resolve to the
lowest global row, and the result must equal the single-rank fit."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, match_eigs


def _fit(X, shard, device, mode="randomized", method="exact"):
    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200 import device as dv
    from cpu_ops import CpuOps
    prev = dv.set_ops(CpuOps())
    try:
        data = fd.SnapshotMatrix(torch.as_tensor(X), 0.1, shard=shard, device=device)
        if method == "opt":     # the bench's fit: OptDMD on a randomized basis
            model = fd.optdmd(data, 8, svd_mode=mode, seed=5, oversample=10, power_iters=1,
                              lm_config=fd.LMConfig(max_iters=10))
        else:
            model = fd.exact_dmd(data, 8, svd_mode=mode, seed=5, oversample=10, power_iters=1)
        z0 = fd.encode(model, torch.as_tensor(X[:, 0]))
        frame = fd.decode(model, fd.step_k(model, z0, 3))
        return model, z0.z, frame
    finally:
        dv.set_ops(prev)


def _worker(rank, world, X, out_path, port, method="exact"):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2502_05339_b200.device import Shard
    n = X.shape[0]
    bounds = np.linspace(0, n, world + 1).astype(int)
    r0, r1 = bounds[rank], bounds[rank + 1]
    shard = Shard(int(r0), int(r1 - r0), n, dist.group.WORLD, world)
    model, z0, frame = _fit(X[r0:r1], shard, torch.device("cpu"), method=method)
    frames = [None] * world
    dist.all_gather_object(frames, frame)
    if rank == 0:
        np.savez(out_path, lam=model.lam, sigma=model.sigma, res=model.provenance.get("residual_rel", 0.0),
                 z0=z0, frame=np.concatenate(frames))
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def data(small_golden):
    return small_golden["dmd_noisyrand_X"]


def test_single_rank_cpu_orchestration(data, small_golden):
    model, z0, frame = _fit(data, None, torch.device("cpu"))
    import flowdmd_oracle as orc
    ref = orc.exact_dmd(data, 8, "randomized", 5, p=10, q=1)
    assert match_eigs(model.lam, ref["lam"]) <= 1e-10
    np.testing.assert_allclose(model.sigma, ref["sigma"], rtol=1e-10)
    np.testing.assert_allclose(model.provenance["residual_rel"], ref["residual_rel"], rtol=1e-8)


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_optdmd_matches_single(data, world):
    """The bench's fit (OptDMD, randomized basis) row-sharded over 2 ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npz")
        mp.spawn(_worker, args=(world, data, out, port, "opt"), nprocs=world, join=True)
        got = dict(np.load(out))
    model, z0, frame = _fit(data, None, torch.device("cpu"), method="opt")
    assert match_eigs(got["lam"], model.lam) <= 1e-9
    np.testing.assert_allclose(got["sigma"], model.sigma, rtol=1e-12)
    np.testing.assert_allclose(got["z0"], z0, rtol=1e-7, atol=1e-10)
    np.testing.assert_allclose(got["frame"], frame, rtol=1e-7, atol=1e-9)


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_matches_single(data, world):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npz")
        mp.spawn(_worker, args=(world, data, out, port), nprocs=world, join=True)
        got = dict(np.load(out))
    model, z0, frame = _fit(data, None, torch.device("cpu"))
    assert match_eigs(got["lam"], model.lam) <= 1e-11
    np.testing.assert_allclose(got["sigma"], model.sigma, rtol=1e-12)
    np.testing.assert_allclose(got["res"], model.provenance["residual_rel"], rtol=1e-9)
    np.testing.assert_allclose(got["z0"], z0, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(got["frame"], frame, rtol=1e-9, atol=1e-11)


# ---------------------------------------------------------------- round 2: TSQR, DMDc, sharded writer
def _cpu_device(monkey=True):
    from paper_2502_05339_b200 import device as dv
    dv.default_device = lambda: torch.device("cpu")


def _fit_more(X, shard, out_dir=None):
    import warnings
    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200 import device as dv
    from cpu_ops import CpuOps
    prev = dv.set_ops(CpuOps())
    try:
        out = {}
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            data = fd.SnapshotMatrix(torch.as_tensor(X), 0.1, shard=shard, device=torch.device("cpu"))
            full = fd.exact_dmd(data, 8, svd_mode="full")                 # TSQR across shards
            out["full_lam"], out["full_sigma"] = full.lam, full.sigma
            u = np.random.default_rng(5).standard_normal((2, X.shape[1] - 1))
            mc, ctrl = fd.dmdc_fit(data, u, 10, 8, seed=3)                # control rows on the last rank
            out["dmdc_lam"], out["dmdc_B"] = mc.lam, ctrl.reduced_b[0]
            ex = fd.exact_dmd(data, 8, svd_mode="randomized", seed=5, oversample=10, power_iters=1)
            out["ex_lam"] = ex.lam
            if out_dir is not None:
                fd.model_io.save_model(os.path.join(out_dir, "m.kdmd"), ex)
        return out
    finally:
        dv.set_ops(prev)


def _worker_more(rank, world, X, out_dir, port):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _cpu_device()
    from paper_2502_05339_b200.shards import row_bounds, row_shard
    b = row_bounds(X.shape[0], world)
    out = _fit_more(np.ascontiguousarray(X[b[rank]:b[rank + 1]]), row_shard(X.shape[0]), out_dir)
    if rank == 0:
        np.savez(os.path.join(out_dir, "r.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_tsqr_dmdc_and_sharded_writer(data, monkeypatch):
    """svd_mode='full' (Householder TSQR over the shards), the augmented DMDc
    fit with its control rows on the last rank, and the sharded model writer,
    against the single-rank results on the same rows."""
    import socket
    from paper_2502_05339_b200 import device as dv
    monkeypatch.setattr(dv, "default_device", lambda: torch.device("cpu"))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_more, args=(2, data, d, port), nprocs=2, join=True)
        got = dict(np.load(os.path.join(d, "r.npz")))
        with tempfile.TemporaryDirectory() as d1:
            ref = _fit_more(data, None, d1)
            a = open(os.path.join(d, "m.kdmd"), "rb").read()
            b = open(os.path.join(d1, "m.kdmd"), "rb").read()
    assert match_eigs(got["full_lam"], ref["full_lam"]) <= 1e-10
    np.testing.assert_allclose(got["full_sigma"], ref["full_sigma"], rtol=1e-12)
    assert match_eigs(got["dmdc_lam"], ref["dmdc_lam"]) <= 1e-10
    np.testing.assert_allclose(got["dmdc_B"], ref["dmdc_B"], rtol=1e-6, atol=1e-8 * np.abs(ref["dmdc_B"]).max())
    assert match_eigs(got["ex_lam"], ref["ex_lam"]) <= 1e-11
    # same header and layout; phi (column-major c128 after sigma / lambda) equal to round-off
    n, r = data.shape[0], 8
    glen = int(np.frombuffer(a[32:36], dtype="<u4")[0])
    off = 36 + glen + 8 * r + 16 * r
    assert a[:36 + glen] == b[:36 + glen]
    pa = np.frombuffer(a[off:off + 16 * n * r], dtype="<c16")
    pb = np.frombuffer(b[off:off + 16 * n * r], dtype="<c16")
    assert np.abs(pa - pb).max() <= 1e-9 * np.abs(pb).max()
