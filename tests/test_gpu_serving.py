"""Serving / editing / guided upscaling on the device (SURVEY.md §8(f) rows
2-3) against the reference's own outputs (tests/golden/serving_cases.npz,
written by oracle/gen_golden_serving.py) and the oracle.

Tolerances: f32 payload planes within 1e-6 of the plane maximum (one f32
rounding step), u8 rasters within one count, f64 fields / states within
1e-9 relative (decode sums in a different order than BLAS), eigenvalues of
an edit to 1e-12. The MAC kernels are checked against the oracle at large
grids: the stencils (inject, project, advect) bit-exactly on identical
inputs, decode planes to 1e-13."""

import json
import os

import numpy as np
import pytest

import flowdmd_oracle as orc
from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_05339_b200 as fd
    return fd


@pytest.fixture(scope="module")
def sg():
    return dict(np.load(os.path.join(GOLDEN, "serving_cases.npz")))


def _grid(fd, sg):
    nx, ny = (int(v) for v in sg["grid"])
    return fd.GridSpec(nx, ny, float(sg["h"]), json.loads(str(sg["model_info"]))["grid"]["boundary"])


@pytest.fixture(scope="module")
def model(fd, sg):
    return fd.ReducedModel(sg["phi"], sg["lam"], sg["sigma"], float(sg["dt"]), _grid(fd, sg))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def assert_payload(got, want):
    got = np.frombuffer(got, dtype=np.uint8)
    assert got.size == want.size
    np.testing.assert_array_equal(got[:12], want[:12])
    a, b = got[12:], want[12:]
    if a.size == 4 * int(np.prod(want[:12].view("<u4"))):
        a, b = a.view("<f4"), b.view("<f4")
        assert np.abs(a - b).max() <= 1e-6 * max(np.abs(b).max(), 1e-30), np.abs(a - b).max()
    else:
        d = np.abs(a.astype(int) - b.astype(int))
        assert d.max() <= 1 and (d > 0).mean() < 0.01


def _server(fd, sg, model):
    data = fd.SnapshotMatrix(sg["X"], float(sg["dt"]), model.grid_meta)
    return fd.ModelServer(model, dataset=data, density=sg["density"])


def _edit_body(sg, model):
    return {"weights": sg["edit_weights"].tolist(), "growth_scale": sg["edit_growth"].tolist(),
            "freq_scale": sg["edit_freq"].tolist(), "start_frame": 3}


def test_model_info_matches_reference(fd, sg, model):
    info = _server(fd, sg, model).model_info()
    want = json.loads(str(sg["model_info"]))
    assert info["grid"] == want["grid"] and info["clusters"] == want["clusters"]
    assert info["n"] == want["n"] and info["r"] == want["r"] and info["dt"] == want["dt"]
    for a, b in zip(info["eigenvalues"], want["eigenvalues"]):
        for key in ("re", "im", "modulus", "freq"):
            assert abs(a[key] - b[key]) <= 1e-13 * max(1.0, abs(b[key]))


@pytest.mark.parametrize("tag", ["base", "edit"])
def test_session_replay_matches_reference(fd, sg, model, tag):
    srv = _server(fd, sg, model)
    body = {} if tag == "base" else _edit_body(sg, model)
    sess = srv.get_session(srv.create_session(body))
    for k in (0, 4, -2):
        for field in ("velocity", "speed", "density"):
            for fmt in ("bin", "raster"):
                got, ctype = srv.frame_payload(sess, k, field, fmt)
                assert ctype == "application/octet-stream"
                assert_payload(got, sg[f"payload_frame_{tag}_{k}_{field}_{fmt}"])
    frame = srv.apply_force(sess, {"x": 0.5, "y": 0.6, "dx": 0.3, "dy": -0.2, "radius": 0.2, "scale": 2.0})
    assert frame == int(sg[f"force_frame_{tag}"])
    for dk in (0, 3):
        for field in ("speed", "density"):
            got, _ = srv.frame_payload(sess, frame + dk, field, "bin")
            assert_payload(got, sg[f"payload_forced_{tag}_{dk}_{field}_bin"])
    A = orc.build_downsample(model.grid_meta.nx, model.grid_meta.ny, 2)
    low = A @ sg["X"][:, 5]
    for proj in (True, False):
        got, _ = srv.upres_preview(sess, {"factor": 2, "split": 4, "low": low.tolist(), "project": proj,
                                          "field": "velocity"})
        assert_payload(got, sg[f"payload_upres_{tag}_{int(proj)}"])


def test_edit_folds_into_mix_without_copy(fd, sg, model):
    spec = fd.EditSpec(sg["edit_weights"], sg["edit_growth"], sg["edit_freq"])
    em = fd.apply_edit(model, spec)
    assert em.modes.table is model.modes.table          # shared HBM table, no n-sized copy
    assert np.abs(em.lam - sg["edit_lam"]).max() <= 1e-12
    assert rel(em.phi, sg["edit_phi"]) <= 1e-12
    ident = fd.apply_edit(model, fd.EditSpec.identity(model.r))
    assert ident.modes is model.modes and ident.provenance["edits"][-1] == "identity"
    z0 = sg["z0"]
    assert abs(fd.band_energy(model, z0, sg["cluster_low"]) - float(sg["band_low"])) <= 1e-9 * float(sg["band_low"])
    assert abs(fd.band_energy(model, z0, sg["cluster_high"]) - float(sg["band_high"])) <= \
        1e-9 * max(float(sg["band_high"]), 1e-30)


def test_edit_pair_mismatch_rejected(fd, model):
    w = np.ones(model.r)
    a = int(np.flatnonzero(model.pair_partner > np.arange(model.r))[0])
    w[a] = 0.5
    with pytest.raises(ValueError, match="differs across conjugate pair"):
        fd.apply_edit(model, fd.EditSpec(w, np.ones(model.r), np.ones(model.r)))


def test_upres_matches_reference(fd, sg, model):
    A = orc.build_downsample(model.grid_meta.nx, model.grid_meta.ny, 2)
    L = A @ sg["X"][:, 7]
    cfg = fd.UpresConfig(split=4, factor=2)
    st, H = fd.upres_step(model, fd.ReducedState(sg["z0"], 0), L, cfg)
    assert np.abs(st.z - sg["upres_z"]).max() <= 1e-9 * np.abs(sg["upres_z"]).max()
    assert rel(H, sg["upres_H"]) <= 1e-9
    proj = fd.build_projector(model.grid_meta, 2)
    x = fd.constrained_project(proj, sg["upres_H"], L)
    assert np.abs(x - sg["upres_x"]).max() <= 1e-14 * np.abs(sg["upres_x"]).max()
    b = fd.blend_fields(sg["upres_x"], sg["upres_H"], model, cfg)
    assert rel(b, sg["upres_blend"]) <= 1e-9


@pytest.mark.parametrize("which", ["guided", "guided_noproj", "guided_blend"])
def test_guided_rollout_matches_reference(fd, sg, model, which):
    import warnings
    blend = np.linspace(0.0, 1.0, model.r) if which == "guided_blend" else None
    cfg = fd.UpresConfig(split=4, factor=2, blend=blend)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        out = fd.guided_rollout(model, sg["X"][:, 10], sg["guide_frames"], cfg, project=which != "guided_noproj")
    assert out.shape == sg[which].shape
    assert rel(out, sg[which]) <= 1e-9


def test_rollout_edit_and_density_match_reference(fd, sg, model):
    nx, ny = (int(v) for v in sg["grid"])
    spec = fd.EditSpec(sg["edit_weights"], sg["edit_growth"], sg["edit_freq"])
    d0 = fd.ScalarField(model.grid_meta, sg["density"][:, :, 0])
    frames, dens = fd.rollout(model, sg["z0"], 6, edit=spec, density0=d0)
    assert rel(frames, sg["rollout_frames"]) <= 1e-9
    assert dens.shape == (ny, nx, 6) and rel(dens, sg["rollout_density"]) <= 1e-9
    fb, db = fd.rollout(model, sg["z0"], 4, density0=d0, backward=True)
    assert rel(fb, sg["rollout_back_frames"]) <= 1e-9 and rel(db, sg["rollout_back_density"]) <= 1e-9


def test_serving_on_device_fit(fd, sg):
    """End to end on the package's own fit: exact_dmd on the device, then
    frames within the payload tolerance of the reference session."""
    g = _grid(fd, sg)
    data = fd.SnapshotMatrix(sg["X"], float(sg["dt"]), g)
    m = fd.exact_dmd(data, 8)
    srv = fd.ModelServer(m, dataset=data, density=sg["density"])
    sess = srv.get_session(srv.create_session({}))
    got, _ = srv.frame_payload(sess, 4, "speed", "bin")
    want = sg["payload_frame_base_4_speed_bin"][12:].view("<f4")
    a = np.frombuffer(got, dtype=np.uint8)[12:].view("<f4")
    assert np.abs(a - want).max() <= 1e-5 * np.abs(want).max()


# --------------------------------------------------------------------------
# kernels vs oracle at larger grids
# --------------------------------------------------------------------------

@pytest.mark.parametrize("nx,ny,ncol,dtype", [(256, 192, 40, torch.float64), (97, 301, 13, torch.float64),
                                              (512, 64, 64, torch.float32), (2, 2, 1, torch.float64)])
def test_mac_decode_kernel(fd, nx, ny, ncol, dtype):
    from paper_2502_05339_b200 import device as dv
    n = (nx + 1) * ny + nx * (ny + 1)
    rng = np.random.default_rng(nx + ny)
    D = rng.standard_normal((ncol, n))
    if dtype == torch.float32:
        D = D.astype(np.float32).astype(np.float64)
    c = rng.standard_normal(ncol)
    T = dv.alloc_tall(n, ncol, dtype, "col")
    T.buf[:ncol, :n].copy_(torch.from_numpy(D))
    flat = D.T @ c
    for field in ("velocity", "speed"):
        got = dv.get_ops().mac_decode(T, torch.from_numpy(c), nx, ny, field).cpu().numpy()
        want = orc.center_planes(flat, nx, ny, field)
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max() * max(1, ncol ** 0.5)


@pytest.mark.parametrize("nx,ny,f", [(256, 128, 2), (96, 60, 3), (64, 64, 4)])
def test_mac_stencils_bit_exact(fd, nx, ny, f):
    from paper_2502_05339_b200 import device as dv
    ops = dv.get_ops()
    rng = np.random.default_rng(f)
    n = (nx + 1) * ny + nx * (ny + 1)
    nl = (nx // f + 1) * (ny // f) + (nx // f) * (ny // f + 1)
    H = rng.standard_normal(n)
    L = rng.standard_normal(nl)
    x = ops.mac_project(torch.from_numpy(H).cuda(), torch.from_numpy(L).cuda(), nx, ny, f,
                        __import__("paper_2502_05339_b200.grid", fromlist=["x"]).downsample_gram_diag(f))
    want = orc.constrained_project(nx, ny, f, H, L)
    assert np.abs(x.cpu().numpy() - want).max() <= 4e-16 * np.abs(want).max()
    fine = ops.mac_inject(torch.from_numpy(np.stack([L, 2 * L])).cuda(), nx, ny, f).cpu().numpy()
    P = orc.build_inject(nx, ny, f)
    np.testing.assert_array_equal(fine[0], P @ L)
    np.testing.assert_array_equal(fine[1], P @ (2 * L))
    h, dt = 1.0 / nx, 0.07
    vel = rng.standard_normal(n) * 3.0
    q = rng.standard_normal((ny, nx))
    got = ops.mac_advect(torch.from_numpy(vel).cuda(), nx, ny, h, dt, torch.from_numpy(q).cuda()).cpu().numpy()
    np.testing.assert_array_equal(got, orc.advect_density(vel, nx, ny, h, q, dt))


def test_mac_kernel_argument_errors(fd):
    from paper_2502_05339_b200 import device as dv
    ops = dv.get_ops()
    T = dv.alloc_tall(10, 2, torch.float64, "col")
    with pytest.raises(ValueError):
        ops.mac_decode(T, torch.ones(2), 3, 3, "velocity")   # n_state 24 > 10 rows
    with pytest.raises(ValueError):
        ops.mac_inject(torch.ones(5, device="cuda"), 7, 4, 2)  # 7 not divisible by 2


def test_concurrent_sessions_match_serial(fd, sg, model):
    """ThreadingHTTPServer-style concurrency (server.py:1-21, test_server.py:224):
    8 threads, each its own session (half edited, with forces), produce the
    same payload bytes as the same requests issued serially."""
    import threading
    srv = _server(fd, sg, model)
    bodies = [{} if i % 2 == 0 else _edit_body(sg, model) for i in range(8)]

    def script(sess):
        out = []
        for k in (0, 3, 7):
            out.append(srv.frame_payload(sess, k, "speed", "bin")[0])
            out.append(srv.frame_payload(sess, k, "density", "raster")[0])
        srv.apply_force(sess, {"x": 0.4, "y": 0.5, "dx": 0.2, "dy": 0.1})
        out.append(srv.frame_payload(sess, 2, "velocity", "bin")[0])
        return out

    serial = [script(srv.get_session(srv.create_session(b))) for b in bodies]
    results = [None] * len(bodies)
    errors = []

    def run(i):
        try:
            results[i] = script(srv.get_session(srv.create_session(bodies[i])))
        except Exception as exc:   # pragma: no cover - surfaced below
            errors.append(exc)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(bodies))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for a, b in zip(results, serial):
        assert a == b
