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
