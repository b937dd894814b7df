"""On-disk formats against files written by the REAL
reference (tests/golden/io, oracle/gen_golden_io.py): byte-identical
round trips, the reference's loaders' values, and its error behaviour
(model_io.py:206-251). CPU: device "cpu" with the CPU checker ops; the
same paths run on the GPU in test_gpu_model_io."""

import os
import shutil

import numpy as np
import pytest
import torch

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden", "io")


@pytest.fixture(scope="module")
def expect():
    return np.load(os.path.join(GOLD, "io_expect.npz"))


@pytest.fixture()
def cpu_ops():
    from paper_2502_05339_b200 import device as dv
    from cpu_ops import CpuOps
    prev = dv.set_ops(CpuOps())
    yield
    dv.set_ops(prev)


def test_kv_codec_roundtrip(expect):
    from paper_2502_05339_b200 import model_io as mio
    text = str(expect["manifest"])
    kv = mio.kv_loads(text)
    assert mio.kv_dumps(kv) == text
    assert mio.format_value(0.1) == "0.1" and mio.format_value(True) == "true"
    assert mio.format_value([1, 2.5]) == "1.0,2.5" and mio.format_value(None) == "none"   # np.asarray promotes
    with pytest.raises(ValueError):
        mio.kv_loads("no equals sign")
    with pytest.raises(ValueError):
        mio.kv_dumps({"a=b": 1})


def test_load_reference_model_and_resave_byte_identical(tmp_path, expect, cpu_ops):
    from paper_2502_05339_b200 import model_io as mio
    m = mio.load_model(os.path.join(GOLD, "model.kdmd"), device=torch.device("cpu"))
    np.testing.assert_array_equal(m.phi, expect["phi"])
    np.testing.assert_array_equal(m.lam, expect["lam"])
    np.testing.assert_array_equal(m.sigma, expect["sigma"])
    assert m.dt == float(expect["dt"])
    assert m.grid_meta.nx == 6 and m.grid_meta.boundary == "open" and m.grid_meta.solids()[2, 3]
    out = tmp_path / "resaved.kdmd"
    mio.save_model(out, m)
    assert out.read_bytes() == open(os.path.join(GOLD, "model.kdmd"), "rb").read()


def test_load_handbuilt_non_conjugate_model(tmp_path, expect, cpu_ops):
    from paper_2502_05339_b200 import model_io as mio
    m = mio.load_model(os.path.join(GOLD, "handbuilt.kdmd"), device=torch.device("cpu"))
    np.testing.assert_array_equal(m.phi, expect["hb_phi"])
    np.testing.assert_array_equal(m.lam, expect["hb_lam"])
    assert m.provenance == {"k": "3", "method": "hand"}
    out = tmp_path / "hb.kdmd"
    mio.save_model(out, m)
    assert out.read_bytes() == open(os.path.join(GOLD, "handbuilt.kdmd"), "rb").read()


def _corrupt(tmp_path, fn):
    src = open(os.path.join(GOLD, "model.kdmd"), "rb").read()
    p = tmp_path / "bad.kdmd"
    p.write_bytes(fn(bytearray(src)))
    return p


def test_model_file_errors(tmp_path):
    from paper_2502_05339_b200 import model_io as mio
    from paper_2502_05339_b200.errors import BadMagicError, BadVersionError, ChecksumError, SizeMismatchError
    cpu = torch.device("cpu")

    def bad_magic(b):
        b[0:4] = b"XXXX"
        return bytes(b)

    def bad_version(b):
        b[4:8] = np.asarray([2], dtype="<u4").tobytes()
        return bytes(b)

    def flip_phi(b):
        b[len(b) // 2] ^= 0x01
        return bytes(b)

    with pytest.raises(BadMagicError):
        mio.load_model(_corrupt(tmp_path, bad_magic), device=cpu)
    with pytest.raises(BadMagicError):
        mio.load_model(_corrupt(tmp_path, lambda b: bytes(b[:3])), device=cpu)
    with pytest.raises(BadVersionError):
        mio.load_model(_corrupt(tmp_path, bad_version), device=cpu)
    with pytest.raises(ChecksumError):
        mio.load_model(_corrupt(tmp_path, flip_phi), device=cpu)
    for cut in (6, 20, 40, 300, 2000, 7000, 7190):
        with pytest.raises(SizeMismatchError, match="truncated"):
            mio.load_model(_corrupt(tmp_path, lambda b: bytes(b[:cut])), device=cpu)
    with pytest.raises(SizeMismatchError, match="trailing bytes"):
        mio.load_model(_corrupt(tmp_path, lambda b: bytes(b) + b"\0\0"), device=cpu)


def test_dataset_load_and_resave_byte_identical(tmp_path, expect):
    from paper_2502_05339_b200 import model_io as mio
    d = mio.load_dataset(os.path.join(GOLD, "dataset"), device=torch.device("cpu"))
    np.testing.assert_array_equal(d.S.view().numpy(), expect["X"])
    assert d.dt == 0.05 and d.meta["note"] == "golden" and d.grid_meta.solids()[2, 3]
    dens = mio.load_dataset_density(os.path.join(GOLD, "dataset"))
    np.testing.assert_array_equal(dens, expect["density"])
    out = tmp_path / "ds"
    mio.save_dataset(out, d, dens)
    for name in ("manifest", "snapshots.bin", "density.bin"):
        assert (out / name).read_bytes() == open(os.path.join(GOLD, "dataset", name), "rb").read(), name


def test_dataset_errors(tmp_path):
    from paper_2502_05339_b200 import model_io as mio
    from paper_2502_05339_b200.errors import BadMagicError, ChecksumError, SizeMismatchError
    cpu = torch.device("cpu")
    src = os.path.join(GOLD, "dataset")
    d1 = tmp_path / "trunc"
    shutil.copytree(src, d1)
    with open(d1 / "snapshots.bin", "r+b") as fh:
        fh.truncate(100)
    with pytest.raises(SizeMismatchError):
        mio.load_dataset(d1, device=cpu)
    d2 = tmp_path / "crc"
    shutil.copytree(src, d2)
    with open(d2 / "snapshots.bin", "r+b") as fh:
        fh.seek(8)
        fh.write(b"\x01")
    with pytest.raises(ChecksumError):
        mio.load_dataset(d2, device=cpu)
    d3 = tmp_path / "kind"
    shutil.copytree(src, d3)
    (d3 / "manifest").write_text((d3 / "manifest").read_text().replace("kind = dataset", "kind = other"))
    with pytest.raises(BadMagicError):
        mio.load_dataset(d3, device=cpu)
    with pytest.raises(SizeMismatchError):
        mio.load_dataset(tmp_path / "missing", device=cpu)
