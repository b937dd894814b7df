"""Interactive serving of a device-resident 2-D model (reference server.py:1-443,
SURVEY.md §8(f) row 2).

`ModelServer` mirrors the reference's session logic — `model_info`,
`create_session`, `get_session`, `delete_session`, `projector_for`,
`frame_payload`, `apply_force`, `upres_preview` — with the same arguments,
payload bytes and exceptions. The reference's HTTP layer
(`server._make_handler`, ThreadingHTTPServer) only calls these methods, so it
binds to this class unchanged; this package does not
re-implement the transport.

Per request:
  * session state stays on the host (O(r) reduced coefficients, as the
    reference keeps it);
  * the frame is ONE fused kernel (fdmd_mac_decode): decode from the HBM table,
    MAC cell-centring and speed, written as f64 planes; only the ny x nx
    planes (f32 / u8 payload) cross PCIe;
  * density views advect on the device (fdmd_mac_advect) through per-step
    decoded velocities that never leave HBM;
  * spectral edits fold into the session model's mix (editing.apply_edit):
    creating a session writes no n-sized buffer.
Concurrent requests from server threads are safe: models are immutable, a
session's force path is serialised by its lock, and every request runs on
the calling thread's current CUDA stream.
"""

from __future__ import annotations

import contextlib
import functools
import threading
import uuid

import numpy as np
import torch

from . import device as dv
from .editing import DEFAULT_CLUSTER_THRESHOLD, EditSpec, apply_edit, cluster_modes
from .errors import EigenvalueFloorError
from .grid import ScalarField, component_positions, is_grid
from .runtime import INVERSE_FLOOR, ReducedState, _conjugate_symmetry_defect, encode, step_forced, step_k
from . import upres as _upres


_tls = threading.local()


@contextlib.contextmanager
def request_stream(device):
    """Each server thread issues its requests on its own CUDA stream: the
    stream-keyed scratch buffers (device.CudaOps workspaces) and the
    allocator's per-stream pools then never interleave between requests
    running concurrently on different threads."""
    streams = getattr(_tls, "streams", None)
    if streams is None:
        streams = _tls.streams = {}
    st = streams.get(str(device))
    if st is None:
        st = streams[str(device)] = torch.cuda.Stream(device=device)
    st.wait_stream(torch.cuda.default_stream(device))   # inputs staged on the default stream
    with torch.cuda.stream(st):
        yield st
    st.synchronize()   # synchronous on return: session tensors are complete for any thread


def _on_request_stream(fn):
    @functools.wraps(fn)
    def wrapper(self, *args, **kwargs):
        with request_stream(_device(self.model)):
            return fn(self, *args, **kwargs)
    return wrapper


def shift_state(model, z, delta, floor=INVERSE_FLOOR):
    """Move a coefficient vector by a signed number of frames (server.py:43-54)."""
    if delta >= 0:
        return step_k(model, ReducedState(z, 0), delta).z
    mods = np.abs(model.lam)
    bad = np.flatnonzero(mods < floor)
    if bad.size:
        raise EigenvalueFloorError(
            f"inverse stepping blocked: modes {bad.tolist()} have |lambda| below {floor:g}", bad)
    return model.lam ** float(delta) * z


class Session:
    """One edited model + reference reduced state (server.py:57-67). The
    density is a device tensor (ny x nx f64) or None."""

    def __init__(self, model, z_ref, frame_ref, density_ref):
        self.model = model
        self.z_ref = z_ref
        self.frame_ref = frame_ref
        self.density_ref = density_ref
        self.lock = threading.Lock()

    def snapshot(self):
        with self.lock:
            return self.z_ref.copy(), self.frame_ref, self.density_ref


def _default_density(grid):
    """Centred blob so density views work without a dataset (server.py:70-76)."""
    j, i = np.meshgrid(np.arange(grid.ny), np.arange(grid.nx), indexing="ij")
    x = (i + 0.5) / grid.nx
    y = (j + 0.5) / grid.ny
    return np.exp(-(((x - 0.5) ** 2 + (y - 0.35) ** 2) / 0.02))


def _device(model):
    return model.modes.table.buf.device


def table_coefficients(model, z) -> torch.Tensor:
    """Raw-table coefficients (device f64) of Re(phi z) for a conjugate-symmetric
    z, or None when z is not (the reference then takes Re(phi z) directly)."""
    modes = model.modes
    z = np.asarray(z, dtype=np.complex128).ravel()
    scale = max(float(np.abs(z).max()) if z.size else 0.0, 1e-300)
    if modes.general is not None or _conjugate_symmetry_defect(model, z) > 1e-9 * scale:
        return None
    c = modes.layout.coeff(z)[:, 0]
    if modes.mix is not None:
        c = modes.mix[:, : c.size] @ c
    return torch.as_tensor(c, device=_device(model))


def decode_planes(model, z, field):
    """(channels, ny, nx) f64 device planes of the decoded, cell-centred state."""
    grid = model.grid_meta
    c = table_coefficients(model, z)
    ops = dv.get_ops()
    if c is not None:
        return ops.mac_decode(model.modes.table, c, grid.nx, grid.ny, field)
    # asymmetric coefficients: Re(phi z) through the basis (runtime.decode), then centre
    from .runtime import decode
    flat = decode(model, z, to_host=False).to(torch.float64)
    return _center_planes(flat, grid, field)


def _center_planes(flat: torch.Tensor, grid, field):
    nx, ny = grid.nx, grid.ny
    u = flat[: grid.n_u].reshape(ny, nx + 1)
    v = flat[grid.n_u:].reshape(ny + 1, nx)
    uc = 0.5 * (u[:, :-1] + u[:, 1:])
    vc = 0.5 * (v[:-1, :] + v[1:, :])
    if field == "velocity":
        return torch.stack([uc, vc])
    return torch.sqrt(uc * uc + vc * vc)[None]


def _host(t: torch.Tensor) -> np.ndarray:
    """Device -> host through a pinned staging buffer (one DMA at link speed)."""
    if t.device.type != "cuda":
        return t.numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def encode_planes(planes, fmt):
    """12-byte header (u32 nx, ny, channels) + row-major f32 or u8 planes
    (server.py:288-302); planes may be a device tensor or a numpy array."""
    if isinstance(planes, np.ndarray):
        planes = torch.from_numpy(planes)
    channels, ny, nx = planes.shape
    header = np.asarray([nx, ny, channels], dtype="<u4").tobytes()
    if fmt == "bin":
        if planes.device.type == "cuda":
            # one pinned staging buffer laid out as the payload (header + f32
            # planes): a single DMA, then one copy into the returned bytes
            buf = torch.empty(3 + planes.numel(), dtype=torch.float32, pin_memory=True)
            buf[:3].view(torch.int32).copy_(torch.tensor([nx, ny, channels], dtype=torch.int32))
            buf[3:].copy_(planes.reshape(-1).to(torch.float32), non_blocking=True)
            torch.cuda.current_stream(planes.device).synchronize()
            return buf.numpy().tobytes(), "application/octet-stream"
        return header + _host(planes.to(torch.float32)).tobytes(), "application/octet-stream"
    if fmt == "raster":
        p = planes.to(torch.float64)
        lo = p.min()
        hi = p.max()
        span = hi - lo
        if float(span.item()) <= 0:
            data = torch.zeros(p.shape, dtype=torch.uint8)
        else:
            data = torch.clamp((p - lo) / span * 255.0, 0, 255).to(torch.uint8)
        return header + _host(data).tobytes(), "application/octet-stream"
    raise ValueError(f"unknown format {fmt!r}")


def impulse_vector(grid, x, y, dx, dy, radius, scale):
    """Flat force vector: a smooth bump of (dx, dy) * scale around (x, y)
    (server.py:305-317)."""
    xu, yu = component_positions(grid, "u")
    xv, yv = component_positions(grid, "v")
    r2 = radius * radius
    fall_u = np.maximum(0.0, 1.0 - ((xu - x) ** 2 + (yu - y) ** 2) / r2)
    fall_v = np.maximum(0.0, 1.0 - ((xv - x) ** 2 + (yv - y) ** 2) / r2)
    return np.concatenate([(dx * scale * fall_u).ravel(), (dy * scale * fall_v).ravel()])


def decoded_velocity(model, z) -> torch.Tensor:
    """Flat decoded state (device, table dtype) — the velocity a density step uses."""
    from .runtime import decode
    return decode(model, z, to_host=False)


def advect_density(model, density: torch.Tensor, z, dt) -> torch.Tensor:
    grid = model.grid_meta
    vel = decoded_velocity(model, z)
    return dv.get_ops().mac_advect(vel, grid.nx, grid.ny, grid.h, dt, density)


class ModelServer:
    """Session logic of the reference's threaded model server (server.py:79-285)
    over a device-resident model. `dataset` is a SnapshotMatrix (HBM) or a
    reference-style object with `.states`; `density` an (ny, nx, frames) array."""

    def __init__(self, model, dataset=None, density=None, host="127.0.0.1", port=0):
        self.model = model
        self.dataset = dataset
        self.density_frames = density
        self.host = host
        self.port = port
        self.sessions = {}
        self.sessions_lock = threading.Lock()
        self.projectors = {}
        self.projectors_lock = threading.Lock()

    # -- session logic (server.py:117-196) -----------------------------------
    def model_info(self):
        model = self.model
        lam = model.lam
        freq = np.angle(lam) / model.dt
        low, high = cluster_modes(model, DEFAULT_CLUSTER_THRESHOLD)
        if is_grid(model.grid_meta):
            g = model.grid_meta
            grid = {"kind": "grid", "nx": g.nx, "ny": g.ny, "h": g.h, "boundary": g.boundary}
        else:
            grid = {"kind": "none"}
        return {
            "n": model.n, "r": model.r, "dt": model.dt, "grid": grid,
            "eigenvalues": [{"re": float(v.real), "im": float(v.imag), "modulus": float(abs(v)),
                             "freq": float(f)} for v, f in zip(lam, freq)],
            "clusters": {"threshold": DEFAULT_CLUSTER_THRESHOLD, "low": low.tolist(), "high": high.tolist()},
        }

    def _dataset_frame(self, start):
        from .dmd import SnapshotMatrix
        ds = self.dataset
        if isinstance(ds, SnapshotMatrix):
            frames = ds.S.k
            if not 0 <= start < frames:
                raise ValueError(f"start_frame {start} outside dataset (0..{frames - 1})")
            return ds.S.view()[:, start]
        frames = ds.states.shape[1]
        if not 0 <= start < frames:
            raise ValueError(f"start_frame {start} outside dataset (0..{frames - 1})")
        return ds.states[:, start]

    @_on_request_stream
    def create_session(self, body):
        model = self.model
        r = model.r
        spec = EditSpec(body.get("weights", np.ones(r)), body.get("growth_scale", np.ones(r)),
                        body.get("freq_scale", np.ones(r)),
                        float(body.get("cluster_threshold", DEFAULT_CLUSTER_THRESHOLD)))
        edited = apply_edit(model, spec)
        start = int(body.get("start_frame", 0))
        if self.dataset is not None:
            z0 = encode(edited, self._dataset_frame(start)).z
        else:
            z0 = np.ones(r, dtype=np.complex128)
        density = None
        if is_grid(model.grid_meta):
            g = model.grid_meta
            if self.density_frames is not None:
                vals = ScalarField(g, self.density_frames[:, :, start]).values
            else:
                vals = _default_density(g)
            density = torch.as_tensor(vals, dtype=torch.float64, device=_device(model))
        sid = uuid.uuid4().hex
        with self.sessions_lock:
            self.sessions[sid] = Session(edited, z0, 0, density)
        return sid

    def get_session(self, sid):
        with self.sessions_lock:
            return self.sessions.get(sid)

    def delete_session(self, sid):
        with self.sessions_lock:
            return self.sessions.pop(sid, None) is not None

    def projector_for(self, factor):
        grid = self.model.grid_meta
        key = (grid.nx, grid.ny, factor)
        with self.projectors_lock:
            if key not in self.projectors:
                self.projectors[key] = _upres.build_projector(grid, factor)
            return self.projectors[key]

    # -- frames (server.py:198-235) --------------------------------------------
    def frame_planes(self, session, k, field):
        """(channels, ny, nx) f64 device planes of frame k (no encoding)."""
        model = session.model
        grid = model.grid_meta
        if not is_grid(grid):
            raise ValueError("model has no grid metadata; frames unavailable")
        z_ref, frame_ref, density_ref = session.snapshot()
        if field in ("velocity", "speed"):
            z = shift_state(model, z_ref, k - frame_ref)
            return decode_planes(model, z, field)
        if field == "density":
            if density_ref is None:
                raise ValueError("no density available for this session")
            return self._advected_density(model, z_ref, frame_ref, density_ref, k)[None]
        raise ValueError(f"unknown field {field!r}")

    @_on_request_stream
    def frame_payload(self, session, k, field, fmt):
        planes = self.frame_planes(session, k, field)   # decode first, then format errors (server.py:225)
        return encode_planes(planes, fmt)

    def _advected_density(self, model, z_ref, frame_ref, density_ref, k):
        density = density_ref
        z = z_ref
        steps = k - frame_ref
        sign = 1 if steps >= 0 else -1
        for _ in range(abs(steps)):
            z = shift_state(model, z, sign)
            density = advect_density(model, density, z, sign * model.dt)
        return density

    # -- force / upres (server.py:237-285) -------------------------------------
    @_on_request_stream
    def apply_force(self, session, body):
        model = session.model
        grid = model.grid_meta
        if not is_grid(grid):
            raise ValueError("model has no grid metadata; forcing unavailable")
        x = float(body["x"])
        y = float(body["y"])
        dx = float(body["dx"])
        dy = float(body["dy"])
        radius = float(body.get("radius", 4 * grid.h))
        scale = float(body.get("scale", 1.0))
        if radius <= 0:
            raise ValueError("radius must be positive")
        force = impulse_vector(grid, x, y, dx, dy, radius, scale)
        with session.lock:
            state = ReducedState(session.z_ref, session.frame_ref)
            new = step_forced(model, None, state, f=[force])
            session.z_ref = new.z
            session.frame_ref = new.frame
            if session.density_ref is not None:
                session.density_ref = advect_density(model, session.density_ref, new.z, model.dt)
            return session.frame_ref

    @_on_request_stream
    def upres_preview(self, session, body):
        model = session.model
        factor = int(body["factor"])
        split = int(body["split"])
        project = bool(body.get("project", True))
        low = np.asarray(body["low"], dtype=np.float64)
        cfg = _upres.UpresConfig(split=split, factor=factor)
        z_ref, frame_ref, _ = session.snapshot()
        state = ReducedState(z_ref, frame_ref)
        new_state, H = _upres.upres_step(model, state, low, cfg, to_host=False)
        if project:
            proj = self.projector_for(factor)
            xp = _upres.constrained_project(proj, H, low, to_host=False)
            H = _upres.blend_fields(xp, H, model, cfg, to_host=False)
        planes = _center_planes(H.to(torch.float64), model.grid_meta, body.get("field", "speed"))
        return encode_planes(planes, body.get("format", "bin"))
