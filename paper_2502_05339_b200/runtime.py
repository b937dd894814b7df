"""Reduced-space runtime, mirroring `flowdmd.runtime` (reference runtime.py:1-264).

Coefficient arithmetic (step, step_k, eval_continuous, inverse_step, forced
steps) is O(r) and stays host-side exactly as in the reference. Every
n-dimensional product — decode (runtime.py:66-99), encode (runtime.py:47-52),
force projection (runtime.py:199), rollout frames — runs on the device table.

Additions beyond the reference API (the reference decodes one frame per
Python call):
  * ``decode_batch(model, Z)``        Z: r x B coefficients -> B x n frames (device)
  * ``reconstruct(model, z0, times)`` frames at arbitrary continuous times
  * ``ModalBasis`` + ``reconstruct_basis`` for u(t) = U Re(W Lam^t b) (config 4)
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import device as dv
from .device import Tall
from .errors import EigenvalueFloorError, RolloutOverflowError

INVERSE_FLOOR = 1e-8
_EXP_OVERFLOW = 700.0


class ImaginaryResidueWarning(RuntimeWarning):
    """Decoded field had a non-negligible imaginary part (runtime.py:22-27)."""


@dataclass
class ReducedState:
    z: np.ndarray
    frame: int = 0

    def __post_init__(self):
        self.z = np.asarray(self.z, dtype=np.complex128).ravel()
        if not np.isfinite(self.z.view(np.float64)).all():
            raise ValueError("reduced state contains non-finite entries")


def _as_state(z, frame=0):
    return z if isinstance(z, ReducedState) else ReducedState(z, frame)


def _dev(model):
    return model.modes.table.buf.device


def encode(model, u, frame=0):
    """z = pinv(phi) @ u (runtime.py:47-52) via the device table."""
    if isinstance(u, torch.Tensor):
        ut = u.reshape(-1)
    else:
        ut = torch.as_tensor(np.asarray(u).ravel())
    if ut.numel() != model.modes.n_local:
        raise ValueError(f"state has {ut.numel()} entries, model wants {model.n}")
    ut = ut.to(_dev(model))
    if not ut.is_floating_point():
        ut = ut.to(torch.float64)
    z = model.modes.project(ut[None, :])[:, 0]
    return ReducedState(z, frame)


def _conjugate_symmetry_defect(model, z):
    """runtime.py:55-63."""
    partner = model.pair_partner
    defect = 0.0
    for a in range(model.r):
        b = partner[a]
        if b == a:
            defect = max(defect, abs(z[a].imag))
        elif b > a:
            defect = max(defect, abs(z[b] - np.conj(z[a])))
    return defect


def _to_host_f64(t: torch.Tensor) -> np.ndarray:
    """Device frame(s) -> host float64 through pinned memory: the upcast runs
    on the device and the copy is a single DMA at link speed (a pageable
    .cpu() of a 50M-row frame runs at ~2 GB/s). Torch's caching host
    allocator reuses the pinned block across calls; the returned array keeps
    its tensor alive."""
    t = t.to(torch.float64)
    if t.device.type != "cuda":
        return t.numpy()
    h = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def decode(model, z, *, out: Optional[torch.Tensor] = None, to_host: bool = True):
    """Re(phi @ z) (runtime.py:66-99): table GEMV when z is conjugate-symmetric,
    otherwise the complex product through the same table plus the
    ImaginaryResidueWarning check. Returns a host float64 array (as the
    reference) unless to_host=False (device tensor in the table dtype)."""
    if isinstance(z, ReducedState):
        z = z.z
    z = np.asarray(z, dtype=np.complex128).ravel()
    if z.size != model.r:
        raise ValueError(f"reduced state has {z.size} entries, model rank is {model.r}")
    modes = model.modes
    dev = _dev(model)
    scale = max(float(np.abs(z).max()) if z.size else 0.0, 1e-300)
    if _conjugate_symmetry_defect(model, z) <= 1e-9 * scale and modes.general is None:
        c = modes.layout.coeff(z)
        frame = modes.decode_coeff(torch.as_tensor(c, device=dev), out=out)[0]
    else:
        D, E = modes.basis()
        ez = E @ z
        C = np.stack([ez.real, ez.imag], axis=1)
        frames = modes.decode_coeff(torch.as_tensor(C, device=dev), general=modes.general is not None,
                                    basis_coords=True)
        yr, yi = frames[0], frames[1]
        y2 = float(torch.sum(yr.double() ** 2).item()) + float(torch.sum(yi.double() ** 2).item())
        yi2 = float(torch.sum(yi.double() ** 2).item())
        if modes.shard is not None and modes.shard.world > 1:
            t = modes.shard.allreduce(torch.tensor([y2, yi2], dtype=torch.float64, device=dev))
            y2, yi2 = float(t[0]), float(t[1])
        ynorm = np.sqrt(y2)
        if ynorm > 0 and np.sqrt(yi2) > 1e-6 * ynorm:
            warnings.warn(
                "decoded field has relative imaginary residue "
                f"{np.sqrt(yi2) / ynorm:.2e}; conjugate-pair bookkeeping looks broken",
                ImaginaryResidueWarning, stacklevel=2)
        frame = yr
        if out is not None:
            out[0].copy_(yr)
            frame = out[0]
    if to_host:
        return _to_host_f64(frame)
    return frame


def step(model, zstate):
    s = _as_state(zstate)
    return ReducedState(model.lam * s.z, s.frame + 1)


def step_k(model, zstate, k):
    """runtime.py:108-124."""
    if k < 0:
        raise ValueError("k must be >= 0; use inverse_step to go backward")
    s = _as_state(zstate)
    if k == 0:
        return ReducedState(s.z.copy(), s.frame)
    mods = np.abs(model.lam)
    grow = mods > 1.0
    if grow.any():
        logmag = k * np.log(mods[grow])
        if logmag.max() > _EXP_OVERFLOW:
            i = int(np.flatnonzero(grow)[np.argmax(logmag)])
            raise RolloutOverflowError(f"|lambda_{i}|^k = {mods[i]:.6f}^{k} overflows")
    return ReducedState(model.lam ** k * s.z, s.frame + k)


def eval_continuous(model, z0, t):
    """runtime.py:127-142."""
    s = _as_state(z0)
    zero = np.flatnonzero(model.lam == 0)
    if zero.size:
        raise ValueError(f"modes {zero.tolist()} have zero eigenvalue; no continuous log exists")
    omega = np.log(model.lam) / model.dt
    if t != 0.0 and (omega.real * t).max() > _EXP_OVERFLOW:
        raise RolloutOverflowError(f"exp(Re(Omega) * {t}) overflows")
    return ReducedState(np.exp(omega * t) * s.z, s.frame)


def inverse_step(model, zstate, floor=INVERSE_FLOOR):
    """runtime.py:145-161."""
    s = _as_state(zstate)
    mods = np.abs(model.lam)
    bad = np.flatnonzero(mods < floor)
    if bad.size:
        raise EigenvalueFloorError(
            f"inverse stepping blocked: modes {bad.tolist()} have |lambda| below {floor:g}", bad)
    return ReducedState(s.z / model.lam, s.frame - 1)


def step_forced(model, ctrl, zstate, q=None, f=None, dt=None):
    """z' = lam z + sum_i B~_i q_i dt + pinv(phi) sum_j f_j dt (runtime.py:164-200)."""
    s = _as_state(zstate)
    if dt is None:
        dt = model.dt
    if dt <= 0:
        raise ValueError("dt must be positive")
    z = model.lam * s.z
    if q is not None:
        if ctrl is None:
            raise ValueError("channel inputs given without a ControlOperator")
        if len(q) != len(ctrl.reduced_b):
            raise ValueError(f"{len(q)} channel inputs for {len(ctrl.reduced_b)} channels")
        for mat, qi in zip(ctrl.reduced_b, q):
            qi = np.asarray(qi).ravel()
            if qi.size != mat.shape[1]:
                raise ValueError(f"channel input has {qi.size} entries, channel wants {mat.shape[1]}")
            z = z + (mat @ qi) * dt
    if f is not None:
        fs = [f] if (isinstance(f, (np.ndarray, torch.Tensor)) and f.ndim == 1) else list(f)
        total = None
        for fj in fs:
            fj = fj.reshape(-1) if isinstance(fj, torch.Tensor) else np.asarray(fj).ravel()
            if fj.shape[0] != model.n:
                raise ValueError(f"force vector has {fj.shape[0]} entries, model wants {model.n}")
            ft = torch.as_tensor(fj, device=_dev(model), dtype=torch.float64)
            total = ft if total is None else total + ft
        z = z + model.modes.project(total[None, :])[:, 0] * dt
    return ReducedState(z, s.frame + 1)


def kinetic_energy(u_flat, h):
    u_flat = np.asarray(u_flat)
    return 0.5 * h * h * float(np.vdot(u_flat, u_flat).real)


def rollout(model, z0, frames, ctrl=None, q_seq=None, f_seq=None, edit=None, density0=None,
            backward=False, *, to_host=True):
    """Repeatedly step and decode (runtime.py:209-264). The per-frame states are
    advanced on the host (O(r)); all frames are then decoded in one batched
    device GEMM when every state is conjugate-symmetric (the invariant every
    path here preserves), else frame by frame. `edit` folds into the model's
    mix (editing.apply_edit); `density0` (ScalarField or ny x nx array) is
    advected on the device through the decoded frames and returned as an
    (ny, nx, frames) array."""
    if frames < 1:
        raise ValueError("frames must be >= 1")
    if edit is not None:
        from .editing import apply_edit
        model = apply_edit(model, edit)            # folds into the mix; no n-sized copy
    density = None
    if density0 is not None:
        from .grid import is_grid
        if not is_grid(model.grid_meta):
            raise ValueError("density advection needs grid metadata on the model")
        density = torch.as_tensor(np.asarray(getattr(density0, "values", density0), dtype=np.float64),
                                  device=_dev(model))
    s = _as_state(z0)
    Z = np.empty((model.r, frames), dtype=np.complex128)
    for k in range(frames):
        if backward:
            s = inverse_step(model, s)
        elif q_seq is not None or f_seq is not None:
            s = step_forced(model, ctrl, s, q=None if q_seq is None else q_seq[k],
                            f=None if f_seq is None else f_seq[k])
        else:
            s = step(model, s)
        Z[:, k] = s.z
    out = decode_batch(model, Z)
    densities = None
    if density is not None:
        # smoke advected through each decoded frame on the device (runtime.py:255-262)
        g = model.grid_meta
        ops = dv.get_ops()
        dt = -model.dt if backward else model.dt
        dens = torch.empty((frames, g.ny, g.nx), dtype=torch.float64, device=density.device)
        for k in range(frames):
            density = ops.mac_advect(out[k], g.nx, g.ny, g.h, dt, density)
            dens[k].copy_(density)
        densities = dens.permute(1, 2, 0).cpu().numpy() if to_host else dens
    if to_host:
        return _to_host_f64(out).T, densities
    return out, densities


def decode_batch(model, Z, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Frames (B x n, device, table dtype) for coefficient columns Z (r x B)."""
    Z = Z if isinstance(Z, np.ndarray) else np.asarray(Z)
    Z = np.asarray(Z, dtype=np.complex128).reshape(model.r, -1)
    scale = max(float(np.abs(Z).max()) if Z.size else 0.0, 1e-300)
    sym = all(_conjugate_symmetry_defect(model, Z[:, k]) <= 1e-9 * max(np.abs(Z[:, k]).max(), 1e-300)
              for k in range(Z.shape[1])) if scale > 0 else True
    modes = model.modes
    dev = _dev(model)
    if sym and modes.general is None:
        C = torch.as_tensor(modes.layout.coeff(Z), device=dev)
        return modes.decode_coeff(C, out=out)
    frames = [decode(model, Z[:, k], to_host=False) for k in range(Z.shape[1])]
    res = torch.stack(frames, dim=0)
    if out is not None:
        out.copy_(res)
        return out
    return res


def continuous_coefficients(model, z0, times) -> torch.Tensor:
    """Table coefficients (ncol x B) of eval_continuous(model, z0, t) for each t,
    computed on the device (complex exp of Omega t)."""
    s = _as_state(z0)
    if np.any(model.lam == 0):
        raise ValueError("zero eigenvalue; no continuous log exists")
    dev = _dev(model)
    omega = torch.as_tensor(np.log(model.lam) / model.dt, device=dev)
    t = torch.as_tensor(np.asarray(times, dtype=np.float64), device=dev)
    if t.numel() and float((omega.real[:, None] * t[None, :]).max().item()) > _EXP_OVERFLOW:
        raise RolloutOverflowError("exp(Re(Omega) * t) overflows")
    Z = torch.exp(omega[:, None] * t[None, :].to(torch.complex128)) * torch.as_tensor(s.z, device=dev)[:, None]
    lay = model.modes.layout
    C = torch.empty((lay.ncol_table, Z.shape[1]), dtype=torch.float64, device=dev)
    ks = torch.as_tensor([k for k, _ in lay.re_idx], device=dev, dtype=torch.long)
    aa = torch.as_tensor([a for _, a in lay.re_idx], device=dev, dtype=torch.long)
    C[ks] = Z[aa].real
    if lay.im_idx:
        ks = torch.as_tensor([k for k, _ in lay.im_idx], device=dev, dtype=torch.long)
        aa = torch.as_tensor([a for _, a in lay.im_idx], device=dev, dtype=torch.long)
        C[ks] = Z[aa].imag
    return C


def reconstruct(model, z0, times, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Frames at continuous times (seconds from z0): B x n device tensor.
    Equivalent to decode(eval_continuous(model, z0, t)) per t for
    conjugate-symmetric z0 (the table path, runtime.py:81-88)."""
    C = continuous_coefficients(model, z0, times)
    return model.modes.decode_coeff(C, out=out)


class ModalBasis:
    """u(t) = U Re(W Lam^t b) with a real device basis U (n x r, column-major)
    — BASELINE config 4's reconstruction (north_star third part)."""

    # batches at least this large go to the tcgen05 kernel (fp32 bases);
    # a single frame is a GEMV and stays on the HBM-streaming SIMT kernel
    TC_MIN_BATCH = 16

    def __init__(self, U, W, lam, b, dt=1.0, use_tc: Optional[bool] = None):
        """U: the real basis as a column-major Tall, or the fp16 hi/lo planes
        dict of a tcgen05 lift (optdmd(keep_basis="planes"))."""
        planes = U if isinstance(U, dict) else None
        if planes is not None:
            U = None
            dev = planes["uh"].device
            use_tc = True
        else:
            assert U.layout == "col"
            dev = U.buf.device
        self.U = U
        self.W = torch.as_tensor(np.asarray(W, dtype=np.complex128), device=dev)
        self.lam = np.asarray(lam, dtype=np.complex128)
        self.omega = torch.as_tensor(np.log(self.lam) / dt, device=dev)
        self.b = torch.as_tensor(np.asarray(b, dtype=np.complex128), device=dev)
        self.use_tc = (U.dtype == torch.float32 and U.buf.is_cuda) if use_tc is None else use_tc
        self._tc = planes

    def coefficients(self, times) -> torch.Tensor:
        t = torch.as_tensor(np.asarray(times, dtype=np.float64), device=self.W.device)
        Lt = torch.exp(self.omega[:, None] * t[None, :].to(torch.complex128)) * self.b[:, None]
        return (self.W @ Lt).real.contiguous()      # r x B

    def tc_state(self):
        if self._tc is None:
            self._tc = dv.get_ops().tc_basis(self.U)
        return self._tc

    def release_fp32(self):
        """Drop this object's reference to the fp32 basis once the tcgen05
        planes exist (same bytes): frees HBM for wider frame batches; every
        batch size then runs on the tcgen05 kernel."""
        if not self.use_tc:
            raise ValueError("release_fp32 needs the tcgen05 path (fp32 CUDA basis)")
        if self.U is not None:
            self.tc_state()
        self.U = None

    def reconstruct(self, times, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        C = self.coefficients(times)
        if self.use_tc and (C.shape[1] >= self.TC_MIN_BATCH or self.U is None):
            return dv.get_ops().tc_decode(self.tc_state(), C, out=out)
        return dv.get_ops().decode(self.U, C, out=out)
