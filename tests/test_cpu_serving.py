"""Serving / editing / guided upscaling — CPU side.

1. The oracle restatements (oracle/flowdmd_oracle.py, bottom section) are
   pinned against tests/golden/serving_cases.npz, written by the REAL
   reference (oracle/gen_golden_serving.py).
2. Host logic of the package: the MAC index maps the kernels use equal the
   reference-order sparse operators; validation and error behaviour of
   EditSpec / UpresConfig / shift_state / payload encoding.
"""

import json
import os

import numpy as np
import pytest

import flowdmd_oracle as orc
from conftest import GOLDEN


@pytest.fixture(scope="module")
def sg():
    return dict(np.load(os.path.join(GOLDEN, "serving_cases.npz")))


def _session_z0(sg, phi, lam, start):
    return orc.encode(phi, sg["X"][:, start])


def test_oracle_edit_matches_reference(sg):
    phi, lam = orc.apply_edit(sg["phi"], sg["lam"], float(sg["dt"]), sg["edit_weights"], sg["edit_growth"],
                              sg["edit_freq"])
    np.testing.assert_array_equal(lam, sg["edit_lam"])
    np.testing.assert_array_equal(phi, sg["edit_phi"])


@pytest.mark.parametrize("tag", ["base", "edit"])
@pytest.mark.parametrize("k", [0, 4, -2])
@pytest.mark.parametrize("field", ["velocity", "speed"])
def test_oracle_frame_payload_matches_reference(sg, tag, k, field):
    nx, ny = (int(v) for v in sg["grid"])
    phi, lam = sg["phi"], sg["lam"]
    start = 0
    if tag == "edit":
        phi, lam = sg["edit_phi"], sg["edit_lam"]
        start = 3
    z = _session_z0(sg, phi, lam, start)
    z = lam ** k * z if k < 0 else orc.step_k(lam, z, k)
    planes = orc.center_planes(orc.decode(phi, lam, z), nx, ny, field)
    for fmt in ("bin", "raster"):
        got = np.frombuffer(orc.encode_planes(planes, fmt), dtype=np.uint8)
        want = sg[f"payload_frame_{tag}_{k}_{field}_{fmt}"]
        if fmt == "bin":
            a = got[12:].view("<f4")
            b = want[12:].view("<f4")
            np.testing.assert_array_equal(got[:12], want[:12])
            assert np.abs(a - b).max() <= 1e-6 * np.abs(b).max()
        else:
            assert np.abs(got.astype(int) - want.astype(int)).max() <= 1


def test_oracle_density_advection_matches_reference(sg):
    nx, ny = (int(v) for v in sg["grid"])
    phi, lam, h, dt = sg["phi"], sg["lam"], float(sg["h"]), float(sg["dt"])
    z = _session_z0(sg, phi, lam, 0)
    q = sg["density"][:, :, 0]
    for _ in range(4):
        z = lam * z
        q = orc.advect_density(orc.decode(phi, lam, z), nx, ny, h, q, dt)
    want = sg["payload_frame_base_4_density_bin"][12:].view("<f4")
    assert np.abs(q.astype("<f4").ravel() - want).max() <= 1e-6 * np.abs(want).max()


def test_oracle_upres_matches_reference(sg):
    nx, ny = (int(v) for v in sg["grid"])
    phi, lam = sg["phi"], sg["lam"]
    A = orc.build_downsample(nx, ny, 2)
    L = A @ sg["X"][:, 7]
    z, H = orc.upres_step(phi, lam, sg["z0"], L, nx, ny, 2, 4)
    assert np.abs(z - sg["upres_z"]).max() <= 1e-10 * np.abs(sg["upres_z"]).max()
    assert np.linalg.norm(H - sg["upres_H"]) <= 1e-10 * np.linalg.norm(sg["upres_H"])
    x = orc.constrained_project(nx, ny, 2, sg["upres_H"], L)
    np.testing.assert_allclose(x, sg["upres_x"], rtol=0, atol=1e-14 * np.abs(sg["upres_x"]).max())


# --------------------------------------------------------------------------
# host logic of the package
# --------------------------------------------------------------------------

@pytest.mark.parametrize("nx,ny,f", [(16, 32, 2), (12, 9, 3), (8, 8, 4), (20, 10, 5)])
def test_index_maps_equal_reference_operators(nx, ny, f):
    from paper_2502_05339_b200.grid import GridSpec, downsample_gram_diag, downsample_index, inject_index
    g = GridSpec(nx, ny, 1.0 / nx)
    A = orc.build_downsample(nx, ny, f).tocsr()
    idx = downsample_index(g, f)
    for l in range(A.shape[0]):
        cols = A.indices[A.indptr[l]:A.indptr[l + 1]]
        np.testing.assert_array_equal(cols, idx[l])
        assert np.all(A.data[A.indptr[l]:A.indptr[l + 1]] == 1.0 / f)
    P = orc.build_inject(nx, ny, f).tocsr()
    inj = inject_index(g, f)
    np.testing.assert_array_equal(P.indices, inj)
    assert np.all(np.diff(P.indptr) == 1)
    G = (A @ A.T).tocsr()
    assert G.nnz == A.shape[0] and np.all(G.diagonal() == downsample_gram_diag(f))
    # no fine face is covered twice (the stencil projection relies on it)
    assert np.unique(idx).size == idx.size


def test_grid_validation_matches_reference():
    from paper_2502_05339_b200.grid import GridSpec, coarse_grid, unflatten
    with pytest.raises(ValueError, match="at least 2x2"):
        GridSpec(1, 4, 0.1)
    with pytest.raises(ValueError, match="cell width"):
        GridSpec(4, 4, 0.0)
    with pytest.raises(ValueError, match="unknown boundary"):
        GridSpec(4, 4, 0.1, "periodic")
    assert GridSpec(4, 4, 0.1, "closed-box").boundary == "closed"
    with pytest.raises(ValueError, match="not divisible"):
        coarse_grid(GridSpec(6, 4, 0.1), 4)
    with pytest.raises(ValueError, match="factor must be >= 2"):
        coarse_grid(GridSpec(6, 4, 0.1), 1)
    g = GridSpec(4, 3, 0.1)
    with pytest.raises(ValueError, match="grid wants"):
        unflatten(np.zeros(5), g)
    v = np.arange(g.n_state, dtype=float)
    f = unflatten(v, g)
    assert f.u.shape == (3, 5) and f.v.shape == (4, 4)


def test_editspec_validation():
    from paper_2502_05339_b200.editing import EditSpec
    with pytest.raises(ValueError, match="share a length"):
        EditSpec(np.ones(3), np.ones(2), np.ones(3))
    with pytest.raises(ValueError, match="weights must be >= 0"):
        EditSpec(-np.ones(2), np.ones(2), np.ones(2))
    with pytest.raises(ValueError, match="non-finite"):
        EditSpec(np.ones(2), np.array([1.0, np.nan]), np.ones(2))
    with pytest.raises(ValueError, match="cluster_threshold"):
        EditSpec(np.ones(2), np.ones(2), np.ones(2), 0.0)
    assert EditSpec.identity(4).is_identity()


def test_upres_config_validation():
    from paper_2502_05339_b200.upres import UpresConfig
    with pytest.raises(ValueError, match="split must be"):
        UpresConfig(split=-1, factor=2)
    with pytest.raises(ValueError, match="factor must be"):
        UpresConfig(split=1, factor=1)
    with pytest.raises(ValueError, match="blend weights"):
        UpresConfig(split=1, factor=2, blend=[0.5, 1.5])


def test_encode_planes_host_matches_oracle():
    from paper_2502_05339_b200.serving import encode_planes
    rng = np.random.default_rng(0)
    p = rng.standard_normal((2, 5, 7))
    for fmt in ("bin", "raster"):
        assert encode_planes(p, fmt)[0] == orc.encode_planes(p, fmt)
    assert encode_planes(np.zeros((1, 3, 3)), "raster")[0] == orc.encode_planes(np.zeros((1, 3, 3)), "raster")
    with pytest.raises(ValueError, match="unknown format"):
        encode_planes(p, "png")


def test_impulse_vector_matches_reference_formula():
    from paper_2502_05339_b200.grid import GridSpec
    from paper_2502_05339_b200.serving import impulse_vector
    g = GridSpec(6, 5, 0.2)
    f = impulse_vector(g, 0.5, 0.4, 0.3, -0.2, 0.35, 2.0)
    assert f.shape == (g.n_state,)
    # bump support and direction per component
    fu, fv = f[: g.n_u], f[g.n_u:]
    assert np.all(fu >= 0) and np.all(fv <= 0) and fu.max() > 0


def test_shift_state_floor_error():
    from paper_2502_05339_b200.errors import EigenvalueFloorError
    from paper_2502_05339_b200.serving import shift_state

    class M:
        lam = np.array([0.9, 1e-9])

    z = np.array([1.0 + 0j, 1.0])
    with pytest.raises(EigenvalueFloorError) as ei:
        shift_state(M, z, -1)
    assert ei.value.mode_indices == [1]


def test_model_info_fields(sg):
    info = json.loads(str(sg["model_info"]))
    assert set(info) == {"n", "r", "dt", "grid", "eigenvalues", "clusters"}
    assert info["grid"]["kind"] == "grid"


def test_scene_and_edit_files_roundtrip_reference_bytes(tmp_path):
    """Scene / edit-spec files written by the reference (tests/golden/serving_cli)
    load into this package's SceneConfig / EditSpec and re-save byte-identically."""
    from paper_2502_05339_b200 import model_io as mio
    d = os.path.join(GOLDEN, "serving_cli")
    scene = mio.load_scene(os.path.join(d, "scene.kv"))
    assert (scene.kind, scene.nx, scene.ny, scene.frames, scene.warmup) == ("plume", 16, 32, 6, 2)
    mio.save_scene(tmp_path / "s.kv", scene)
    assert (tmp_path / "s.kv").read_bytes() == open(os.path.join(d, "scene.kv"), "rb").read()
    spec = mio.load_edit(os.path.join(d, "edit.kv"))
    mio.save_edit(tmp_path / "e.kv", spec)
    assert (tmp_path / "e.kv").read_bytes() == open(os.path.join(d, "edit.kv"), "rb").read()


def test_sim_params_validation():
    from paper_2502_05339_b200.solver import SimParams
    for kw, msg in [({"dt": 0.0}, "dt must be positive"), ({"dt": 0.1, "cg_tol": 1.0}, "cg_tol"),
                    ({"dt": 0.1, "cg_max_iters": 0}, "cg_max_iters"), ({"dt": 0.1, "vorticity_eps": -1}, "eps")]:
        with pytest.raises(ValueError, match=msg):
            SimParams(**kw)
