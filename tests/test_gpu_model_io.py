"""Model / dataset files on the GPU path: reference-
written files load into HBM tables and re-save byte-identically; a model
fitted on the device round-trips through save_model/load_model; datasets
stream into row-major HBM (f64 or f32)."""

import os

import numpy as np
import pytest

from conftest import ROOT, match_eigs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden", "io")


@pytest.fixture(scope="module")
def fd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_05339_b200 as fd
    return fd


@pytest.fixture(scope="module")
def expect():
    return np.load(os.path.join(GOLD, "io_expect.npz"))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["model.kdmd", "handbuilt.kdmd"])
def test_reference_model_roundtrip_on_device(fd, tmp_path, expect, name):
    from paper_2502_05339_b200 import model_io as mio
    m = mio.load_model(os.path.join(GOLD, name))
    assert m.modes.table.buf.is_cuda
    want = expect["phi"] if name == "model.kdmd" else expect["hb_phi"]
    np.testing.assert_array_equal(m.phi, want)
    out = tmp_path / name
    mio.save_model(out, m)
    assert out.read_bytes() == open(os.path.join(GOLD, name), "rb").read()
    if name == "model.kdmd":
        z0 = fd.encode(m, expect["X"][:, 0])
        np.testing.assert_allclose(z0.z, expect["z0"], rtol=1e-10, atol=1e-12)
        assert rel(fd.decode(m, fd.step_k(m, z0, 5)), expect["frame5"]) <= 1e-10


@pytest.mark.parametrize("method", ["exact", "optdmd"])
def test_fitted_model_save_load(fd, tmp_path, small_golden, method):
    from paper_2502_05339_b200 import model_io as mio
    X = small_golden["dmd_noisyrand_X"]
    data = fd.SnapshotMatrix(X, 0.1)
    if method == "exact":
        model = fd.exact_dmd(data, 8, svd_mode="randomized", seed=5, oversample=10, power_iters=1)
    else:
        model = fd.optdmd(data, 8, svd_mode="randomized", seed=5, oversample=10, power_iters=1,
                          lm_config=fd.LMConfig(max_iters=5))
    path = tmp_path / "fit.kdmd"
    mio.save_model(path, model)
    back = mio.load_model(path)
    np.testing.assert_array_equal(back.lam, model.lam)
    np.testing.assert_array_equal(back.sigma, model.sigma)
    assert rel(back.phi, model.phi) <= 1e-12
    z0 = fd.encode(model, X[:, 0])
    assert rel(fd.decode(back, fd.step_k(back, z0, 4)), fd.decode(model, fd.step_k(model, z0, 4))) <= 1e-10
    assert back.provenance["method"] == method


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_dataset_stream_to_device(fd, tmp_path, expect, dtype):
    from paper_2502_05339_b200 import model_io as mio
    td = torch.float64 if dtype == "f64" else torch.float32
    d = mio.load_dataset(os.path.join(GOLD, "dataset"), dtype=td)
    assert d.S.buf.is_cuda and d.S.dtype == td
    want = expect["X"] if dtype == "f64" else expect["X"].astype(np.float32)
    np.testing.assert_array_equal(d.S.view().cpu().numpy(), want)
    if dtype == "f64":
        out = tmp_path / "ds"
        mio.save_dataset(out, d, mio.load_dataset_density(os.path.join(GOLD, "dataset")))
        for name in ("manifest", "snapshots.bin", "density.bin"):
            assert (out / name).read_bytes() == open(os.path.join(GOLD, "dataset", name), "rb").read(), name
    # a fit straight from the loaded dataset matches the reference model file
    ref = mio.load_model(os.path.join(GOLD, "model.kdmd"))
    model = fd.exact_dmd(d, 6, svd_mode="full")
    assert match_eigs(model.lam, ref.lam) <= (1e-10 if dtype == "f64" else 1e-5)


def test_large_model_stream_blocks(fd, tmp_path):
    """More modes than one streaming block, odd r, n not a multiple of anything."""
    from paper_2502_05339_b200 import model_io as mio
    rng = np.random.default_rng(4)
    n, m = 100_003, 40
    X = rng.standard_normal((n, 12)) @ rng.standard_normal((12, m)) + 1e-3 * rng.standard_normal((n, m))
    model = fd.exact_dmd(fd.SnapshotMatrix(X, 0.1), 11, svd_mode="randomized", seed=1, oversample=5,
                         power_iters=1, table_dtype=torch.float64)
    path = tmp_path / "big.kdmd"
    mio.save_model(path, model)
    assert os.path.getsize(path) > 16 * n * 11
    back = mio.load_model(path)
    np.testing.assert_array_equal(back.lam, model.lam)
    assert rel(back.phi, model.phi) <= 1e-14
