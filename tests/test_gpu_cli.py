"""CLI train / rollout / reverse / eval on the GPU against the REAL reference
CLI's outputs on the same files (tests/golden/io/cli, oracle/gen_golden_io.py)."""

import contextlib
import io
import os
import re

import numpy as np
import pytest

from conftest import ROOT, match_eigs, phase_aligned_error

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden", "io")
CLI = os.path.join(GOLD, "cli")


@pytest.fixture(scope="module")
def fd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_05339_b200 as fd
    return fd


@pytest.fixture(scope="module")
def ref_out():
    text = open(os.path.join(CLI, "outputs.txt")).read()
    out = {}
    for block in text.split("## ")[1:]:
        head, rest = block.split("\n", 1)
        name, rc = head.split(" rc=")
        so, se = rest.split("--stderr--\n", 1)
        out[name] = (int(rc), so, se)
    return out


def run(argv):
    from paper_2502_05339_b200.cli import cli_main
    so, se = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
        rc = cli_main(argv)
    return rc, so.getvalue(), se.getvalue()


def strip_paths(s):
    return re.sub(r"-> \S+|to \S+", "<path>", s)


@pytest.mark.parametrize("name,extra,tol", [("train", [], 1e-10),
                                            ("train_opt", ["--method", "optdmd", "--svd", "randomized",
                                                           "--seed", "3"], 1e-8)])
def test_train_matches_reference_cli(fd, tmp_path, ref_out, name, extra, tol):
    from paper_2502_05339_b200 import model_io as mio
    out = tmp_path / "m.kdmd"
    rc, so, se = run(["train", os.path.join(GOLD, "dataset"), "-o", str(out), "--rank", "6"] + extra)
    rrc, rso, _ = ref_out[name]
    assert rc == rrc == 0
    assert strip_paths(so.splitlines()[0]) == strip_paths(rso.splitlines()[0])
    assert len(so.splitlines()) == len(rso.splitlines())
    ours = mio.load_model(out)
    ref = mio.load_model(os.path.join(CLI, f"{'trained' if name == 'train' else 'trained_opt'}.kdmd"))
    assert match_eigs(ours.lam, ref.lam) <= tol
    np.testing.assert_allclose(ours.sigma, ref.sigma, rtol=1e-10)
    assert phase_aligned_error(ours.phi, ref.phi) <= 1e-6


@pytest.mark.parametrize("name,argv", [
    ("rollout", ["rollout", "--start-frame", "2", "--k", "2", "--frames", "5"]),
    ("reverse", ["reverse", "--start-frame", "30", "--frames", "3"])])
def test_rollout_reverse_match_reference_cli(fd, tmp_path, ref_out, name, argv):
    from paper_2502_05339_b200 import model_io as mio
    out = tmp_path / name
    rc, so, se = run(argv + ["--model", os.path.join(GOLD, "model.kdmd"), "--dataset",
                             os.path.join(GOLD, "dataset"), "--out", str(out)])
    rrc, rso, _ = ref_out[name]
    assert rc == rrc == 0 and strip_paths(so) == strip_paths(rso)
    got = np.fromfile(out / "snapshots.bin", dtype="<f8")
    want = np.fromfile(os.path.join(CLI, name, "snapshots.bin"), dtype="<f8")
    assert got.size == want.size
    assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)
    kg = mio.kv_loads((out / "manifest").read_text())
    kw = mio.kv_loads(open(os.path.join(CLI, name, "manifest")).read())
    kg.pop("snapshots_crc32"), kw.pop("snapshots_crc32")
    assert kg == kw


def test_eval_matches_reference_cli(fd, ref_out):
    from paper_2502_05339_b200 import model_io as mio
    rc, so, se = run(["eval", "--model", os.path.join(GOLD, "model.kdmd"), "--dataset",
                      os.path.join(GOLD, "dataset"), "--stride", "3"])
    assert rc == 0
    got, want = mio.kv_loads(so), mio.kv_loads(ref_out["eval"][1])
    assert list(got) == list(want)
    for k in got:
        if k in ("kind", "model_rank", "frames_compared", "stride"):
            assert got[k] == want[k]
        else:
            np.testing.assert_allclose(mio.parse_floats(got[k]), mio.parse_floats(want[k]), rtol=1e-8)


def test_cli_errors_match_reference(fd, tmp_path, ref_out):
    rc, so, se = run(["rollout", "--model", os.path.join(GOLD, "model.kdmd"), "--dataset",
                      os.path.join(GOLD, "dataset"), "--start-frame", "99", "--out", str(tmp_path / "x")])
    rrc, _, rse = ref_out["bad_start"]
    assert rc == rrc == 1 and se == rse
    assert run([])[0] == 2
    rc, _, se = run(["serve", "--model", os.path.join(GOLD, "model.kdmd")])
    assert rc == 1 and "outside the B200 hot path" in se


# ---- commands using editing / density / guided upscaling (§8(f) rows 2-3) ----
SCLI = os.path.join(ROOT, "tests", "golden", "serving_cli")


@pytest.fixture(scope="module")
def ref_out2():
    text = open(os.path.join(SCLI, "outputs.txt")).read()
    out = {}
    for block in text.split("## ")[1:]:
        head, rest = block.split("\n", 1)
        name, rc = head.split(" rc=")
        so, se = rest.split("--stderr--\n", 1)
        out[name] = (int(rc), so, se)
    return out


def _compare_dataset(mio, got_dir, want_dir, tol):
    got = np.fromfile(os.path.join(got_dir, "snapshots.bin"), dtype="<f8")
    want = np.fromfile(os.path.join(want_dir, "snapshots.bin"), dtype="<f8")
    assert got.size == want.size
    assert np.linalg.norm(got - want) <= tol * np.linalg.norm(want)
    kg = mio.kv_loads(open(os.path.join(got_dir, "manifest")).read())
    kw = mio.kv_loads(open(os.path.join(want_dir, "manifest")).read())
    for k in ("snapshots_crc32", "density_crc32"):
        kg.pop(k, None), kw.pop(k, None)
    assert kg == kw
    if os.path.exists(os.path.join(want_dir, "density.bin")):
        dg = np.fromfile(os.path.join(got_dir, "density.bin"), dtype="<f8")
        dw = np.fromfile(os.path.join(want_dir, "density.bin"), dtype="<f8")
        assert dg.size == dw.size and np.linalg.norm(dg - dw) <= tol * np.linalg.norm(dw)


@pytest.mark.parametrize("name,argv,sub", [
    ("rollout_edit_density", ["rollout", "--start-frame", "1", "--k", "2", "--frames", "4", "--edit",
                              "<SCLI>/edit.kv", "--density"], "rollout_ed"),
    ("reverse_density", ["reverse", "--start-frame", "8", "--frames", "3", "--density"], "reverse_d")])
def test_edit_density_commands_match_reference_cli(fd, tmp_path, ref_out2, name, argv, sub):
    from paper_2502_05339_b200 import model_io as mio
    argv = [a.replace("<SCLI>", SCLI) for a in argv]
    out = tmp_path / sub
    rc, so, se = run(argv + ["--model", os.path.join(SCLI, "model.kdmd"), "--dataset",
                             os.path.join(SCLI, "dataset"), "--out", str(out)])
    rrc, rso, _ = ref_out2[name]
    assert rc == rrc == 0, se
    assert strip_paths(so) == strip_paths(rso)
    _compare_dataset(mio, str(out), os.path.join(SCLI, sub), 1e-9)


@pytest.mark.parametrize("name,extra,sub", [("upres_on", ["--split", "4"], "upres_on"),
                                            ("upres_off", ["--split", "3", "--project", "off"], "upres_off")])
def test_upres_command_matches_reference_cli(fd, tmp_path, ref_out2, name, extra, sub):
    from paper_2502_05339_b200 import model_io as mio
    out = tmp_path / sub
    rc, so, se = run(["upres", "--low", os.path.join(SCLI, "low"), "--model", os.path.join(SCLI, "model.kdmd"),
                      "--factor", "2", "--out", str(out)] + extra)
    rrc, rso, _ = ref_out2[name]
    assert rc == rrc == 0, se
    assert strip_paths(so) == strip_paths(rso)
    _compare_dataset(mio, str(out), os.path.join(SCLI, sub), 1e-9)
    rc, so, se = run(["upres", "--low", os.path.join(SCLI, "low"), "--model", os.path.join(SCLI, "model.kdmd"),
                      "--split", "4", "--factor", "3", "--out", str(tmp_path / "nope")])
    assert (rc, se) == (ref_out2["upres_bad_factor"][0], ref_out2["upres_bad_factor"][2])


def test_simulate_matches_reference_cli(fd, tmp_path, ref_out2):
    from paper_2502_05339_b200 import model_io as mio
    out = tmp_path / "sim"
    rc, so, se = run(["simulate", os.path.join(SCLI, "scene.kv"), "-o", str(out)])
    rrc, rso, _ = ref_out2["simulate"]
    assert rc == rrc == 0, se
    assert strip_paths(so) == strip_paths(rso)
    _compare_dataset(mio, str(out), os.path.join(SCLI, "sim"), 1e-6)
