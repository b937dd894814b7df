"""The row-sharded CUDA path, executed: world_size 2 and 4 over gloo with
every rank on cuda:0 (this pool leases one GPU per call). Each rank runs the
real libfdmd kernels on its row block — the snapshot-Gram sketch, CholeskyQR2,
the tcgen05 lift / modes for fp32 tables, the pair-statistics all-gather, the
real-ification branch (real eigenvalues in the data), a streamed upload into
a Shard, ModalBasis reconstruction, DMDc and the sharded model writer — and
only the small blocks cross ranks (host-staged by `Shard` under gloo; NCCL
on a multi-GPU box). Results are compared with the single-rank fit of the
same data on the same device; a sharded fit must also repeat bit for bit.

No rank ever waits inside a kernel for another rank: the collectives are
host-side gloo calls between launches, so sharing one GPU cannot deadlock.
"""

import os
import socket
import tempfile
import warnings

import numpy as np
import pytest

from conftest import ROOT, match_eigs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

R = 22


def make_data(n=24000, m=61, seed=0):
    """Ten damped conjugate pairs plus two real decaying modes (rank 22),
    fp32 storage, noise 1e-4."""
    rng = np.random.default_rng(seed)
    K = 10
    lam = np.exp(rng.uniform(-0.03, 0.0, K) + 1j * np.sort(rng.uniform(0.3, 3.0, K)))
    phi = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
    b = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    j = np.arange(m)
    X = 2.0 * np.real(phi @ (b[:, None] * lam[:, None] ** j[None, :]))
    for lr, amp in ((0.95, 1.5), (0.8, 0.7)):
        X += amp * rng.standard_normal(n)[:, None] * (lr ** j)[None, :]
    X += 1e-4 * rng.standard_normal(X.shape)
    return X.astype(np.float32)


def _fit_all(fd, X_local, shard, stream=False):
    """Every sharded entry point on this rank's rows; returns host arrays."""
    from paper_2502_05339_b200.device import alloc_tall
    from paper_2502_05339_b200.runtime import ModalBasis
    out = {}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        if stream:
            host = torch.from_numpy(X_local).pin_memory()
            data = fd.SnapshotMatrix(host, 0.1, shard=shard, stream=True)
        else:
            data = fd.SnapshotMatrix(X_local, 0.1, shard=shard)
        mo = fd.optdmd(data, R, lm_config=fd.LMConfig(max_iters=10), svd_mode="randomized", seed=7,
                       oversample=10, power_iters=1, keep_basis=True)
        out["opt_lam"] = mo.lam
        out["opt_sigma"] = mo.sigma
        out["opt_sketch"] = dict(mo.provenance.get("sketch", {}))
        z0 = fd.encode(mo, X_local[:, 0])
        out["opt_z0"] = z0.z
        out["opt_frame"] = fd.decode(mo, fd.step_k(mo, z0, 5))
        out["opt_frames_tc"] = fd.reconstruct(mo, z0, np.linspace(0.0, 3.0, 40)).double().cpu().numpy()
        # config-4 style reconstruction from the sharded POD basis
        U = mo.basis_U
        rng = np.random.default_rng(3)
        W = rng.standard_normal((R, R)) + 1j * rng.standard_normal((R, R))
        mb = ModalBasis(U, W, mo.lam, np.ones(R, dtype=complex), dt=0.1)
        out["basis_frames"] = mb.reconstruct(np.linspace(0.0, 2.0, 48)).double().cpu().numpy()
        out["basis_frame1"] = mb.reconstruct(np.array([0.7])).double().cpu().numpy()
        del mo, U, mb
        ex = fd.exact_dmd(data, R, svd_mode="randomized", seed=7, oversample=10, power_iters=1)
        out["ex_lam"] = ex.lam
        out["ex_res"] = ex.provenance["residual_rel"]
        ze = fd.encode(ex, X_local[:, 0])
        out["ex_frame"] = fd.decode(ex, fd.step_k(ex, ze, 9))
        full = fd.exact_dmd(data, R, svd_mode="full")
        out["full_lam"] = full.lam
        out["full_sigma"] = full.sigma
    return out


def _worker(rank, world, X, out_dir, port):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2502_05339_b200 as fd
    from paper_2502_05339_b200.shards import row_bounds, row_shard
    n = X.shape[0]
    b = row_bounds(n, world)
    Xl = np.ascontiguousarray(X[b[rank]:b[rank + 1]])
    shard = row_shard(n)
    a = _fit_all(fd, Xl, shard)
    a2 = _fit_all(fd, Xl, shard)                     # bitwise repeatability
    s = _fit_all(fd, Xl, shard, stream=True)         # streamed upload into the shard
    # DMDc (control rows on the last rank) and the sharded model writer
    u = np.random.default_rng(5).standard_normal((2, X.shape[1] - 1))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mc, ctrl = fd.dmdc_fit(fd.SnapshotMatrix(Xl, 0.1, shard=shard), u, R + 2, R, seed=3)
        ex = fd.exact_dmd(fd.SnapshotMatrix(Xl, 0.1, shard=shard), R, svd_mode="randomized", seed=7,
                          oversample=10, power_iters=1)
    fd.model_io.save_model(os.path.join(out_dir, "sharded.kdmd"), ex)
    gathered = [None] * world
    dist.all_gather_object(gathered, {k: v for k, v in a.items() if k != "opt_sketch"})
    gathered_s = [None] * world
    dist.all_gather_object(gathered_s, {k: v for k, v in s.items() if k != "opt_sketch"})
    same = all(np.array_equal(a[k], a2[k]) for k in a if k != "opt_sketch")
    flags = [None] * world
    dist.all_gather_object(flags, same)
    if rank == 0:
        cat = {}
        for key in ("opt_frame", "ex_frame"):
            cat[key] = np.concatenate([g[key] for g in gathered])
            cat["s_" + key] = np.concatenate([g[key] for g in gathered_s])
        for key in ("opt_frames_tc", "basis_frames", "basis_frame1"):
            cat[key] = np.concatenate([g[key] for g in gathered], axis=1)
            cat["s_" + key] = np.concatenate([g[key] for g in gathered_s], axis=1)
        for key in ("opt_lam", "opt_sigma", "opt_z0", "ex_lam", "ex_res", "full_lam", "full_sigma"):
            cat[key] = a[key]
            cat["s_" + key] = s[key]
        cat["repeat_bitwise"] = np.array(all(flags))
        cat["implicit"] = np.array(a["opt_sketch"].get("implicit_sketch", 0))
        cat["dmdc_lam"] = mc.lam
        cat["dmdc_B"] = ctrl.reduced_b[0]
        np.savez(os.path.join(out_dir, "r.npz"), **cat)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def fd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_05339_b200 as fd
    return fd


@pytest.fixture(scope="module")
def single(fd):
    X = make_data()
    res = _fit_all(fd, X, None)
    u = np.random.default_rng(5).standard_normal((2, X.shape[1] - 1))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        mc, ctrl = fd.dmdc_fit(fd.SnapshotMatrix(X, 0.1), u, R + 2, R, seed=3)
        ex = fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), R, svd_mode="randomized", seed=7, oversample=10,
                          power_iters=1)
    res["dmdc_lam"] = mc.lam
    res["dmdc_B"] = ctrl.reduced_b[0]
    res["ex_model"] = ex
    return X, res


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_cuda_path_matches_single_rank(fd, single, world):
    import torch.multiprocessing as mp
    X, ref = single
    assert np.isreal(ref["opt_lam"]).sum() >= 2          # the real-ification branch runs
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, X, d, port), nprocs=world, join=True)
        got = dict(np.load(os.path.join(d, "r.npz"), allow_pickle=True))
        loaded = fd.model_io.load_model(os.path.join(d, "sharded.kdmd"))
    assert bool(got["repeat_bitwise"]), "a sharded fit must repeat bit for bit"
    assert int(got["implicit"]) == 1
    for pre in ("", "s_"):
        # reductions over rows are split differently across ranks: agreement to
        # round-off of the fp64 sums, fp32 tables / frames to fp32 accuracy
        np.testing.assert_allclose(got[pre + "opt_sigma"], ref["opt_sigma"], rtol=1e-10)
        assert match_eigs(got[pre + "opt_lam"], ref["opt_lam"]) <= 1e-9
        np.testing.assert_allclose(got[pre + "opt_z0"], ref["opt_z0"], rtol=1e-5, atol=1e-5 * np.abs(ref["opt_z0"]).max())
        assert rel(got[pre + "opt_frame"], ref["opt_frame"]) <= 1e-5
        assert rel(got[pre + "opt_frames_tc"], ref["opt_frames_tc"]) <= 1e-5
        assert rel(got[pre + "basis_frames"], ref["basis_frames"]) <= 1e-5
        assert rel(got[pre + "basis_frame1"], ref["basis_frame1"]) <= 1e-5
        assert match_eigs(got[pre + "ex_lam"], ref["ex_lam"]) <= 1e-9
        np.testing.assert_allclose(got[pre + "ex_res"], ref["ex_res"], rtol=1e-6)
        assert rel(got[pre + "ex_frame"], ref["ex_frame"]) <= 1e-5
        assert match_eigs(got[pre + "full_lam"], ref["full_lam"]) <= 1e-9
        np.testing.assert_allclose(got[pre + "full_sigma"], ref["full_sigma"], rtol=1e-10)
    assert match_eigs(got["dmdc_lam"], ref["dmdc_lam"]) <= 1e-8
    np.testing.assert_allclose(got["dmdc_B"], ref["dmdc_B"], rtol=1e-5, atol=1e-6 * np.abs(ref["dmdc_B"]).max())
    # the sharded writer: same file structure, phi equal to the single-rank model's
    ex = ref["ex_model"]
    assert loaded.n == ex.n and loaded.r == ex.r
    assert match_eigs(loaded.lam, ex.lam) <= 1e-9
    from conftest import phase_aligned_error
    assert phase_aligned_error(loaded.phi, ex.phi) <= 1e-5
