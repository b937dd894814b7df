"""2-D smoke solver on the device (reference solver.py, SURVEY.md §8(f)
row 4: the data generator the fit consumes).

Same pipeline, parameters, scenes and errors as the reference — sources,
MacCormack advection with extrema clamping, buoyancy, vorticity confinement,
masked conjugate-gradient pressure projection — with every grid-sized
operation in libfdmd (csrc/fdmd_solver.cuh). The state lives in HBM for the
whole run; `generate_dataset` writes the snapshots straight into the
row-major device buffer the fit reads (no host round trip), and density
frames come back once at the end.

Parity: element arithmetic follows the reference's numpy expression order;
the CG dot products / means are fixed-order device reductions instead of
BLAS, so iterates differ at rounding level and the solve converges to the
same tolerance (tests compare against reference datasets).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from . import device as dv
from .device import _ptr, _stream
from .errors import ConvergenceError
from .grid import GridSpec, MacField, ScalarField, component_positions


def _dev():
    return dv.default_device()


def _sol(name, *args):
    _lib.check(getattr(_lib.lib(), name)(*args), name)


@dataclass
class Emitter:
    """Disk source (solver.py:26-34)."""

    cx: float
    cy: float
    radius: float
    density_rate: float = 1.0
    temperature_rate: float = 1.0


@dataclass
class SimParams:
    """solver.py:37-55, same validation."""

    dt: float
    buoyancy_alpha: float = 0.0
    buoyancy_beta: float = 0.0
    vorticity_eps: float = 0.0
    cg_tol: float = 1e-6
    cg_max_iters: int = 1000
    source: Optional[Emitter] = None

    def __post_init__(self):
        if not self.dt > 0:
            raise ValueError("dt must be positive")
        if not 0 < self.cg_tol < 1:
            raise ValueError("cg_tol must lie in (0, 1)")
        if self.cg_max_iters < 1:
            raise ValueError("cg_max_iters must be >= 1")
        if self.vorticity_eps < 0:
            raise ValueError("vorticity_eps must be >= 0")


class _Grid:
    """Device-side constants of a GridSpec: solid mask, fluid count, scratch."""

    def __init__(self, grid: GridSpec):
        self.g = grid
        self.nx, self.ny, self.h = grid.nx, grid.ny, grid.h
        dev = _dev()
        solids = np.asarray(grid.solids(), dtype=bool)
        self.solid = torch.as_tensor(solids.astype(np.uint8), device=dev) if solids.any() else None
        self.nfluid = int((~solids).sum())
        self.closed = 1 if grid.boundary == "closed" else 0
        self.cells = grid.n_cells
        self.n_state = grid.n_state
        self.part = torch.empty(296, dtype=torch.float64, device=dev)   # FDMD_SOL_REDUCE_BLOCKS
        self.scal = torch.zeros(4, dtype=torch.float64, device=dev)
        big = max(self.n_state, 3 * self.cells)
        self.scratch = torch.empty(3 * max(grid.n_u, grid.n_v, self.cells) + big, dtype=torch.float64, device=dev)

    @property
    def sp(self):
        return _ptr(self.solid)


_GRIDS = {}


def _grid_of(grid: GridSpec) -> _Grid:
    key = (grid.nx, grid.ny, grid.h, grid.boundary, np.asarray(grid.solids()).tobytes())
    g = _GRIDS.get(key)
    if g is None:
        g = _GRIDS[key] = _Grid(grid)
    return g


@dataclass
class SimState:
    """solver.py:58-70 with device arrays: vel (flat MAC state), density and
    temperature (ny x nx), pressure (ny x nx or None)."""

    vel: torch.Tensor
    density: torch.Tensor
    temperature: torch.Tensor
    grid: GridSpec
    pressure: Optional[torch.Tensor] = None
    frame: int = 0

    @classmethod
    def zeros(cls, grid):
        dev = _dev()
        return cls(torch.zeros(grid.n_state, dtype=torch.float64, device=dev),
                   torch.zeros((grid.ny, grid.nx), dtype=torch.float64, device=dev),
                   torch.zeros((grid.ny, grid.nx), dtype=torch.float64, device=dev), grid)

    def mac(self) -> MacField:
        v = self.vel.cpu().numpy()
        g = self.grid
        return MacField(g, v[: g.n_u].reshape(g.ny, g.nx + 1), v[g.n_u:].reshape(g.ny + 1, g.nx))


# ---------------------------------------------------------------------------
# operators (device)
# ---------------------------------------------------------------------------
def apply_solid_mask(vel: torch.Tensor, grid: GridSpec) -> torch.Tensor:
    """grid.py:264-272 on a flat device state (new tensor)."""
    G = _grid_of(grid)
    out = vel.clone()
    _sol("fdmd_sol_mask", _ptr(out), G.nx, G.ny, G.sp, G.closed, _stream())
    return out


def _advect(G: _Grid, vel, q, which, dt, maccormack=True):
    out = torch.empty_like(q)
    _sol("fdmd_sol_advect", _ptr(vel), _ptr(q), which, G.nx, G.ny, float(G.h), float(dt), 1 if maccormack else 0,
         _ptr(G.scratch), _ptr(out), _stream())
    return out


def advect_maccormack(vel: torch.Tensor, q, dt, grid: GridSpec):
    """solver.py:153-169: q is a flat MAC state or an ny x nx cell array."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    G = _grid_of(grid)
    if q.dim() == 2:
        return _advect(G, vel, q.contiguous(), 2, dt)
    u = _advect(G, vel, q[: grid.n_u].contiguous(), 0, dt)
    v = _advect(G, vel, q[grid.n_u:].contiguous(), 1, dt)
    return torch.cat([u, v])


def _project(vel: torch.Tensor, G: _Grid, cg_tol, cg_max_iters, p0=None):
    """solver.py:261-315 — masked CG on the device; the convergence checks
    read one or two scalars per iteration back to the host."""
    h = G.h
    h2 = h * h
    n = G.cells
    dev = vel.device
    b = torch.empty((G.ny, G.nx), dtype=torch.float64, device=dev)
    _sol("fdmd_sol_rhs", _ptr(vel), G.nx, G.ny, float(h), G.sp, G.closed, float(G.nfluid), _ptr(b), _ptr(G.part),
         _ptr(G.scal[1:]), _stream())
    if n <= _CG1_MAX_CELLS:
        return _project_single(vel, G, b, cg_tol, cg_max_iters, p0)
    red = lambda a, bb, op: _sol("fdmd_sol_reduce", _ptr(a), _ptr(bb), G.sp, n, op, _ptr(G.part), _ptr(G.scal),
                                 _stream())   # noqa: E731
    red(b, None, 1)
    bnorm = float(G.scal[0].item())
    p = torch.zeros_like(b) if p0 is None else p0.clone()
    if p0 is not None and G.solid is not None:
        p[G.solid.bool()] = 0.0
    if bnorm == 0.0:
        return vel.clone(), p, 0.0, 0
    tol_abs = cg_tol * bnorm
    Ap = torch.empty_like(b)
    _sol("fdmd_sol_poisson", _ptr(p), G.nx, G.ny, float(h2), G.sp, 1 - G.closed, _ptr(Ap), _stream())
    r = b - Ap
    red(r, None, 1)
    rmax = float(G.scal[0].item())
    iters = 0
    if rmax > tol_abs:
        d = r.clone()
        red(r, r, 0)
        rs = float(G.scal[0].item())
        Ad = Ap
        converged = False
        for iters in range(1, cg_max_iters + 1):
            _sol("fdmd_sol_poisson", _ptr(d), G.nx, G.ny, float(h2), G.sp, 1 - G.closed, _ptr(Ad), _stream())
            red(d, Ad, 0)
            dAd = float(G.scal[0].item())
            if dAd <= 0.0:
                break
            alpha = rs / dAd
            _sol("fdmd_sol_cg_step", _ptr(p), _ptr(r), _ptr(d), _ptr(Ad), float(alpha), n, _stream())
            red(r, None, 1)
            rmax = float(G.scal[0].item())
            if rmax <= tol_abs:
                converged = True
                break
            red(r, r, 0)
            rs_new = float(G.scal[0].item())
            _sol("fdmd_sol_cg_dir", _ptr(d), _ptr(r), float(rs_new / rs), n, _stream())
            rs = rs_new
        if not converged and iters == cg_max_iters and rmax > tol_abs:
            raise ConvergenceError(
                f"pressure solve stalled at residual {rmax:.3e} (target {tol_abs:.3e}) after {cg_max_iters} "
                "iterations", residual=rmax, iterations=cg_max_iters)
        if rmax > tol_abs:
            raise ConvergenceError(
                f"pressure solve stalled at residual {rmax:.3e} (target {tol_abs:.3e}) after {iters} iterations",
                residual=rmax, iterations=iters)
    out = vel.clone()
    _sol("fdmd_sol_pressure_apply", _ptr(out), _ptr(p), G.nx, G.ny, float(h), G.sp, 1 - G.closed, _stream())
    return out, p, rmax, iters


_CG1_MAX_CELLS = 1 << 17   # SOL_CG1_MAX_CELLS: one-CTA CG below this size


def _project_single(vel, G: _Grid, b, cg_tol, cg_max_iters, p0):
    """The CG loop in one 1024-thread CTA (fdmd_sol_cg_single): same
    iteration and stopping rules, one status read per solve."""
    p = torch.zeros_like(b) if p0 is None else p0.clone()
    if p0 is not None and G.solid is not None:
        p[G.solid.bool()] = 0.0
    r = torch.empty_like(b)
    d = torch.empty_like(b)
    Ad = torch.empty_like(b)
    _sol("fdmd_sol_cg_single", _ptr(b), _ptr(p), _ptr(r), _ptr(d), _ptr(Ad), G.nx, G.ny, float(G.h * G.h), G.sp,
         1 - G.closed, float(cg_tol), int(cg_max_iters), _ptr(G.scal), _stream())
    rmax, iters, ran_out, bnorm = (float(v) for v in G.scal.cpu())
    if bnorm == 0.0:
        return vel.clone(), p, 0.0, 0
    tol_abs = cg_tol * bnorm
    iters = int(iters)
    if ran_out:
        raise ConvergenceError(
            f"pressure solve stalled at residual {rmax:.3e} (target {tol_abs:.3e}) after {cg_max_iters} "
            "iterations", residual=rmax, iterations=cg_max_iters)
    if rmax > tol_abs:
        raise ConvergenceError(
            f"pressure solve stalled at residual {rmax:.3e} (target {tol_abs:.3e}) after {iters} iterations",
            residual=rmax, iterations=iters)
    out = vel.clone()
    _sol("fdmd_sol_pressure_apply", _ptr(out), _ptr(p), G.nx, G.ny, float(G.h), G.sp, 1 - G.closed, _stream())
    return out, p, rmax, iters


def project_pressure(vel: torch.Tensor, grid: GridSpec, cg_tol=1e-6, cg_max_iters=1000):
    """solver.py:318-330."""
    G = _grid_of(grid)
    masked = apply_solid_mask(vel, grid)
    out, _, _, _ = _project(masked, G, cg_tol, cg_max_iters)
    return apply_solid_mask(out, grid)


def step(state: SimState, params: SimParams) -> SimState:
    """solver.py:337-355."""
    g = state.grid
    G = _grid_of(g)
    dt = params.dt
    vel = apply_solid_mask(state.vel, g)
    density, temperature = state.density, state.temperature
    src = params.source
    if src is not None:
        density, temperature = density.clone(), temperature.clone()
        _sol("fdmd_sol_emit", _ptr(density), _ptr(temperature), G.nx, G.ny, float(G.h), float(src.cx), float(src.cy),
             float(src.radius ** 2), float(src.density_rate * dt), float(src.temperature_rate * dt), _stream())
    new_vel = apply_solid_mask(advect_maccormack(vel, vel, dt, g), g)
    density = advect_maccormack(vel, density, dt, g)
    temperature = advect_maccormack(vel, temperature, dt, g)
    _sol("fdmd_sol_buoyancy", _ptr(new_vel), _ptr(density), _ptr(temperature), G.nx, G.ny,
         float(params.buoyancy_alpha), float(params.buoyancy_beta), float(dt), _stream())
    if params.vorticity_eps < 0:
        raise ValueError("eps must be >= 0")
    if params.vorticity_eps != 0.0:
        _sol("fdmd_sol_vorticity", _ptr(new_vel), G.nx, G.ny, float(G.h), float(params.vorticity_eps), float(dt),
             _ptr(G.scratch), _stream())
    new_vel = apply_solid_mask(new_vel, g)
    new_vel, pressure, _, _ = _project(new_vel, G, params.cg_tol, params.cg_max_iters, state.pressure)
    new_vel = apply_solid_mask(new_vel, g)
    return SimState(new_vel, density, temperature, g, pressure, state.frame + 1)


# ---------------------------------------------------------------------------
# scenes and datasets (solver.py:358-505)
# ---------------------------------------------------------------------------
@dataclass
class SceneConfig:
    kind: str = "plume"
    nx: int = 64
    ny: int = 128
    h: float = 1.0 / 64
    boundary: str = "open"
    dt: float = 0.05
    frames: int = 120
    warmup: int = 0
    buoyancy_alpha: float = 0.05
    buoyancy_beta: float = 0.3
    vorticity_eps: float = 1.5
    cg_tol: float = 1e-6
    cg_max_iters: int = 1000
    emit_cx: float = 0.5
    emit_cy: float = 0.12
    emit_radius: float = 0.08
    emit_density: float = 2.0
    emit_temperature: float = 2.0
    region_disks: tuple = ((0.35, 0.45, 0.13), (0.62, 0.52, 0.11), (0.5, 0.3, 0.09))
    region_up: float = 0.3
    region_down: Optional[float] = None
    record_density: bool = True

    def grid(self):
        return GridSpec(self.nx, self.ny, self.h, self.boundary)

    def params(self):
        src = None
        if self.kind == "plume":
            src = Emitter(self.emit_cx * self.nx * self.h, self.emit_cy * self.ny * self.h,
                          self.emit_radius * self.nx * self.h, self.emit_density, self.emit_temperature)
        plume = self.kind == "plume"
        return SimParams(dt=self.dt, buoyancy_alpha=self.buoyancy_alpha if plume else 0.0,
                         buoyancy_beta=self.buoyancy_beta if plume else 0.0,
                         vorticity_eps=self.vorticity_eps if plume else 0.0,
                         cg_tol=self.cg_tol, cg_max_iters=self.cg_max_iters, source=src)


def _region_mask(scene, grid):
    x, y = component_positions(grid, "c")
    w = scene.nx * scene.h
    hgt = scene.ny * scene.h
    mask = np.zeros((grid.ny, grid.nx), dtype=bool)
    flat = []
    for d in scene.region_disks:
        flat.extend(d if isinstance(d, (tuple, list)) else [d])
    for k in range(0, len(flat), 3):
        cx, cy, r = flat[k] * w, flat[k + 1] * hgt, flat[k + 2] * min(w, hgt)
        mask |= (x - cx) ** 2 + (y - cy) ** 2 <= r ** 2
    return mask


def initial_state(scene) -> SimState:
    """solver.py:439-460 (host set-up of a few arrays, then device)."""
    grid = scene.grid()
    state = SimState.zeros(grid)
    if scene.kind == "buoyant_region":
        mask = _region_mask(scene, grid)
        up = scene.region_up
        down = scene.region_down
        if down is None:
            n_in = int(mask.sum())
            n_out = mask.size - n_in
            down = -up * n_in / max(n_out, 1)
        centered = np.where(mask, up, down)
        v = np.zeros((grid.ny + 1, grid.nx))
        v[1:-1, :] = 0.5 * (centered[:-1, :] + centered[1:, :])
        flat = np.concatenate([np.zeros(grid.n_u), v.ravel()])
        state.vel = apply_solid_mask(torch.as_tensor(flat, device=_dev()), grid)
        state.density = torch.as_tensor(mask.astype(np.float64), device=_dev())
    elif scene.kind != "plume":
        raise ValueError(f"unknown scene kind {scene.kind!r}")
    return state


def generate_dataset(scene, *, snapshot_dtype=torch.float64):
    """Run a scene; returns (SnapshotMatrix in HBM, density frames (ny, nx,
    frames) host array or None) — solver.py:463-505."""
    from .dmd import SnapshotMatrix
    if scene.frames < 2:
        raise ValueError("a dataset needs at least 2 frames")
    grid = scene.grid()
    params = scene.params()
    G = _grid_of(grid)
    state = initial_state(scene)
    if scene.kind == "buoyant_region":
        vel, pressure, _, _ = _project(state.vel, G, scene.cg_tol, scene.cg_max_iters)
        state.vel = apply_solid_mask(vel, grid)
        state.pressure = pressure
    for _ in range(scene.warmup):
        state = step(state, params)
    S = dv.alloc_tall(grid.n_state, scene.frames, snapshot_dtype, "row", device=_dev(), zero=True)
    dens = torch.empty((scene.frames, grid.ny, grid.nx), dtype=torch.float64, device=_dev()) \
        if scene.record_density else None
    S.buf[: grid.n_state, 0].copy_(state.vel)
    if dens is not None:
        dens[0].copy_(state.density)
    for k in range(1, scene.frames):
        state = step(state, params)
        S.buf[: grid.n_state, k].copy_(state.vel)
        if dens is not None:
            dens[k].copy_(state.density)
    data = SnapshotMatrix(S, scene.dt, grid, {"scene": scene, "solver": "maccormack_cg"})
    return data, (dens.permute(1, 2, 0).cpu().numpy() if dens is not None else None)
