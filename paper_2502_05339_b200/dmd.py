"""DMD trainers on the device, mirroring `flowdmd.dmd` (reference dmd.py:1-507).

Names, signatures, validation and provenance keys follow the reference; the
n-dimensional work runs in libfdmd (FP64 DMMA), the r-dimensional work stays
on the device (cuSOLVER) except O(r) ordering/pairing bookkeeping, which is
host logic exactly as in the reference.

Extensions (keyword-only): ``oversample``/``power_iters`` overrides (the
reference hard-codes q=2 and clamps p, dmd.py:216-222), ``residual`` to skip
the diagnostic, ``table_dtype`` for the decode table, ``timings`` dict.
"""

from __future__ import annotations

import contextlib
import os
import time
import warnings
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import device as dv
from . import linalg as la
from .device import Shard, Tall, allreduce, alloc_tall
from .errors import ConvergenceError
from .modes import DeviceModes, TableLayout, conjugate_pairs, modes_from_host_phi
from .trace import stage

UNSTABLE_MODULUS = 1.05
SIGMA_CUTOFF = 1e-14

__all__ = [
    "SnapshotMatrix", "ReducedModel", "conjugate_pairs", "exact_dmd", "optdmd", "vandermonde",
    "LMConfig", "ControlOperator", "fit_control", "dmdc_fit", "UNSTABLE_MODULUS", "SIGMA_CUTOFF",
]


# ---------------------------------------------------------------------------
# SnapshotMatrix (dmd.py:26-50)
# ---------------------------------------------------------------------------
class SnapshotMatrix:
    """Time-ordered flattened states, one per column, resident in HBM.

    ``states`` may be a host array (uploaded once; float32 stays float32 in
    HBM and is upcast exactly in-kernel, other dtypes become float64), a
    CUDA tensor, or an existing row-major ``Tall``. ``shard`` marks a row
    block of a row-sharded matrix (multi-GPU).

    ``stream=True`` (host torch tensor, ideally pinned): the upload is
    deferred and streamed in chunks by the first consumer — a randomized fit
    overlaps it with its first sketch stage (linalg.PendingUpload); any other
    access to ``S`` completes it first. The non-finite check then runs on
    the device per chunk and raises ValueError from the consumer.
    """

    def __init__(self, states, dt, grid_meta=None, meta=None, *, shard: Optional[Shard] = None,
                 device=None, check_finite=True, stream=False):
        self.pending = None
        if isinstance(states, Tall):
            S = states
        else:
            shape = getattr(states, "shape", None)
            if shape is None:
                states = np.asarray(states, dtype=np.float64)
                shape = states.shape
            if len(shape) != 2 or shape[1] < 2:
                raise ValueError("snapshot matrix needs at least 2 columns")
            if stream and isinstance(states, torch.Tensor) and states.device.type == "cpu" and shape[0] > 0:
                host = states if states.dtype in (torch.float32, torch.float64) else states.double()
                S = alloc_tall(int(shape[0]), int(shape[1]), host.dtype, "row", device=device or dv.default_device())
                if S.ld > S.k:
                    S.buf[:, S.k:].zero_()
                self.pending = la.PendingUpload(host, S)
            else:
                S = la.as_tall(states, device)
        if S.k < 2:
            raise ValueError("snapshot matrix needs at least 2 columns")
        if (self.pending is None and check_finite and S.n > 0
                and not bool(torch.isfinite(S.view()).all().item())):
            raise ValueError("snapshot matrix contains non-finite entries")
        if not dt > 0:
            raise ValueError("dt must be positive")
        self._S = S
        self.dt = float(dt)
        self.grid_meta = grid_meta
        self.meta = dict(meta or {})
        self.shard = shard
        self._host = None

    @property
    def S(self) -> Tall:
        """The device matrix; completes a streamed upload first."""
        if self.pending is not None:
            p, self.pending = self.pending, None
            p.run()
        return self._S

    @S.setter
    def S(self, value: Tall):
        self._S = value
        self.pending = None

    def take_pending(self):
        """(device Tall, PendingUpload or None) for a consumer that streams."""
        p, self.pending = self.pending, None
        return self._S, p

    @property
    def n(self):
        return self._S.n if self.shard is None else self.shard.n_global

    @property
    def n_transitions(self):
        return self._S.k - 1

    @property
    def states(self):
        """Host float64 copy (the reference keeps states as float64 numpy)."""
        if self._host is None:
            self._host = self.S.view().to(torch.float64).cpu().numpy()
        return self._host


def _as_snapshots(data) -> SnapshotMatrix:
    if isinstance(data, SnapshotMatrix):
        return data
    # a reference-style object (e.g. flowdmd.dmd.SnapshotMatrix): .states, .dt
    return SnapshotMatrix(data.states, data.dt, getattr(data, "grid_meta", None), getattr(data, "meta", None))


# ---------------------------------------------------------------------------
# ReducedModel (dmd.py:53-128)
# ---------------------------------------------------------------------------
class ReducedModel:
    """Trained artifact: mode basis (device decode table), eigenvalues, sigma,
    dt, provenance. ``phi`` (n x r complex128, host) is materialised lazily
    from the device table; decoding never needs it."""

    def __init__(self, phi, lam, sigma, dt, grid_meta=None, provenance=None, *, _modes=None):
        self.lam = np.ascontiguousarray(lam, dtype=np.complex128)
        self.sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        self.dt = float(dt)
        self.grid_meta = grid_meta
        self.provenance = dict(provenance or {})
        if _modes is None:
            phi = np.ascontiguousarray(phi, dtype=np.complex128)
            if phi.ndim != 2:
                raise ValueError("phi must be a 2D matrix")
            if phi.shape[1] != self.lam.size or self.lam.size != self.sigma.size:
                raise ValueError("phi, lam, sigma sizes disagree")
            if not self.dt > 0:
                raise ValueError("dt must be positive")
            self._phi = phi
            self.modes = modes_from_host_phi(phi, self.lam)
        else:
            if self.lam.size != self.sigma.size:
                raise ValueError("phi, lam, sigma sizes disagree")
            if not self.dt > 0:
                raise ValueError("dt must be positive")
            self._phi = None
            self.modes = _modes
        self.pair_partner = conjugate_pairs(self.lam)
        self._phi_pinv = None
        self._decode_table = None

    @property
    def n(self):
        m = self.modes
        return m.n_local if m.shard is None else m.shard.n_global

    @property
    def r(self):
        return self.lam.size

    @property
    def phi(self):
        if self._phi is None:
            self._phi = self.modes.host_phi()
        return self._phi

    def phi_pinv(self):
        """pinv(phi) as a host r x n complex matrix (linalg.py:93-104 semantics)."""
        if self._phi_pinv is None:
            D, E = self.modes.basis()
            M = D.buf[: E.shape[0], : D.n].to(torch.float64).cpu().numpy()   # ncol x n
            self._phi_pinv = self.modes.pinv_rows() @ M
        return self._phi_pinv

    def decode_table(self):
        """(cols n x k float64, re_idx, im_idx) — dmd.py:92-120."""
        if self._decode_table is None:
            lay = self.modes.layout
            self._decode_table = (self.modes.host_table(), list(lay.re_idx), list(lay.im_idx))
        return self._decode_table

    def with_modes(self, phi, lam, note=None):
        prov = dict(self.provenance)
        if note:
            prov.setdefault("edits", [])
            prov["edits"] = list(prov["edits"]) + [note]
        return ReducedModel(phi, lam, self.sigma, self.dt, self.grid_meta, prov)


# ---------------------------------------------------------------------------
# ordering / pairing plan (dmd.py:158-213), host bookkeeping on r values
# ---------------------------------------------------------------------------
def frequency_order(lam):
    """Permutation applied by _order_and_pair (dmd.py:158-187)."""
    lam = np.asarray(lam)
    partner = conjugate_pairs(lam)
    units, seen = [], np.zeros(lam.size, dtype=bool)
    for i in range(lam.size):
        if seen[i]:
            continue
        j = int(partner[i])
        seen[i] = seen[j] = True
        if i == j:
            units.append((i, -1))
        else:
            units.append((i, j) if lam[i].imag >= lam[j].imag else (j, i))
    units.sort(key=lambda u: (abs(np.angle(lam[u[0]])), -abs(lam[u[0]]), lam[u[0]].real))
    order = []
    for a, b in units:
        order.append(a)
        if b >= 0:
            order.append(b)
    return np.asarray(order, dtype=np.int64)


@dataclass
class PairPlan:
    lam: np.ndarray                 # final eigenvalues (sorted, locked, real-ified)
    src: list                       # per computed unit: source eigen-column index
    pos_unit: list                  # per sorted position: (unit, conj?) ; -1 unused
    locked: list                    # per unit: True if it is a locked conjugate pair start
    realify: dict = field(default_factory=dict)   # unit -> True if lam real-ified and not paired


def pair_plan(lam_raw) -> PairPlan:
    order = frequency_order(lam_raw)
    lam = np.asarray(lam_raw, dtype=np.complex128)[order].copy()
    r = lam.size
    src, pos_unit, locked, realify = [], [None] * r, [], {}
    k = 0
    while k < r:
        u = len(src)
        src.append(int(order[k]))
        pos_unit[k] = (u, False)
        paired = (k + 1 < r and lam[k].imag > 0 and
                  abs(lam[k + 1] - np.conj(lam[k])) <= 1e-6 * max(abs(lam[k]), 1e-300))
        locked.append(bool(paired))
        if paired:
            lam[k + 1] = np.conj(lam[k])
            pos_unit[k + 1] = (u, True)
            k += 2
            continue
        if abs(lam[k].imag) <= 1e-12 * max(abs(lam[k]), 1e-300):
            lam[k] = lam[k].real
            realify[u] = True
        k += 1
    return PairPlan(lam, src, pos_unit, locked, realify)


def _modes_pass(A: Tall, Cmap: torch.Tensor, plan: PairPlan, row_pad_top: int, shard: Optional[Shard],
                table_dtype, timings: Optional[dict] = None, a_orthonormal: bool = False,
                tc_src: Optional[dict] = None) -> DeviceModes:
    """phi_raw = A @ [0_top; Cmap] for every computed unit, with fused
    column statistics; then normalise + phase-canonicalise + lock conjugates
    + build the decode table (dmd.py:189-213 and 92-120) in one HBM pass.

    Cmap: K x r complex (device) with phi_raw[:, j] = A[:, top:top+K] @ Cmap[:, j].
    a_orthonormal: A's columns are orthonormal (the POD basis U), which bounds
    the real-ification test of dmd.py:210 without an extra pass.
    tc_src: {"planes": fp16 planes of Q, "Umap": l x r} with A = Q @ Umap —
    the raw modes are then Q @ (Umap [Re|Im]) on tcgen05 (FP32-accurate,
    fp32 table) and the statistics come from a streaming pass over the table.
    """
    ops = dv.get_ops()
    dev = Cmap.device
    U = len(plan.src)
    K = int(Cmap.shape[0])
    mA = K + row_pad_top if A is None else A.k
    Bm = torch.zeros((mA, 2 * U), dtype=torch.float64, device=dev)
    src_t = torch.as_tensor(plan.src, device=dev, dtype=torch.long)
    Cs = Cmap[:, src_t]
    Bm[row_pad_top:row_pad_top + K, 0::2] = Cs.real
    Bm[row_pad_top:row_pad_top + K, 1::2] = Cs.imag
    n_loc = tc_src["n"] if A is None else A.n
    with stage("modes.alloc_raw"):
        raw = alloc_tall(n_loc, 2 * U, table_dtype, "col", device=dev)
    row0 = 0 if shard is None else shard.row0
    t0 = time.perf_counter()
    # SURVEY §8d counts F_modes = 4 n K r (real n x K times complex K x r); only
    # one column of each conjugate pair is executed, so the kernel is credited
    # with its executed 2 n K (2U) flops (the fit-level metric keeps the formula)
    with stage("modes.raw+stats"):
        if tc_src is not None:
            M = Bm if tc_src.get("Umap") is None else tc_src["Umap"] @ Bm
            coef = M.to(torch.float32)                                       # (l | m) x 2U
            # sum / max / first argmax of |phi|^2 come out of the frame epilogue when
            # the CTA-pair kernel runs (> 128 columns); otherwise a statistics pass
            # reads the table back
            st = ops.tc_decode_pairstats(tc_src["planes"], coef, raw.buf[: 2 * U], U, row_offset=row0)
            if st is None:
                st = ops.pair_stats(raw, U, row_offset=row0)
        else:
            st = ops.tall_gemm(A, Bm, raw, stats=True, row_offset=row0,
                               alg_flops=2.0 * n_loc * K * 2 * U)  # (U, 3)
    post = stage("modes.post")
    post.__enter__()
    st = la._reduce_pair_stats(st, shard)
    nrm = torch.sqrt(st[:, 0])
    idx = st[:, 2].round().long()
    # pivot values raw[idx] (gathered from the owning shard)
    local = idx - row0
    if shard is not None and shard.world > 1:
        own = (local >= 0) & (local < n_loc)
        piv = torch.zeros((U, 2), dtype=torch.float64, device=dev)
        li = torch.where(own, local, torch.zeros_like(local))
        ar = torch.arange(U, device=dev)
        vals_re = raw.buf[2 * ar, li].to(torch.float64)
        vals_im = raw.buf[2 * ar + 1, li].to(torch.float64)
        piv[:, 0] = torch.where(own, vals_re, torch.zeros_like(vals_re))
        piv[:, 1] = torch.where(own, vals_im, torch.zeros_like(vals_im))
        piv = shard.allreduce(piv)
    else:
        ar = torch.arange(U, device=dev)
        li = local.clamp(min=0)
        piv = torch.stack([raw.buf[2 * ar, li], raw.buf[2 * ar + 1, li]], dim=1).to(torch.float64)
    pc = torch.complex(piv[:, 0], piv[:, 1])
    pab = pc.abs()
    phase = torch.where(pab > 0, pc.conj() / torch.where(pab > 0, pab, torch.ones_like(pab)),
                        torch.ones_like(pc))
    s = torch.where(nrm > 0, phase / torch.where(nrm > 0, nrm, torch.ones_like(nrm)), phase)
    s = s.cpu().numpy()
    Cs_h = Cs.cpu().numpy()
    # real-ification of phi for real-ified eigenvalues (dmd.py:208-211)
    realified_phi = set()
    check = []
    for u in plan.realify:
        im_col = (Cs_h[:, u] * s[u]).imag
        if not np.any(im_col):
            realified_phi.add(u)
            continue
        if a_orthonormal:
            # A has orthonormal columns (rows of norm <= 1): ||Im||_inf lies in
            # [||v||_2 / sqrt(n), ||v||_2] — decide without a pass when possible
            v2 = float(np.linalg.norm(im_col))
            n_glob = n_loc if shard is None else shard.n_global
            if v2 * (1 + 1e-5) <= 1e-10:
                realified_phi.add(u)
                continue
            if v2 * (1 - 1e-5) / np.sqrt(n_glob) > 1e-10:
                continue
        check.append((u, im_col))
    if check:
        # max_i |Im(phi_u s_u)_i| for every candidate in ONE statistics-only pass
        # (column pair (Im, 0) per unit: the pair max is max Im^2)
        Bq = torch.zeros((mA, 2 * len(check)), dtype=torch.float64, device=dev)
        for k, (u, im_col) in enumerate(check):
            Bq[row_pad_top:row_pad_top + K, 2 * k] = torch.as_tensor(im_col, device=dev)
        with stage("modes.realify_pass"):
            if A is not None:
                stq = la._reduce_pair_stats(ops.tall_gemm(A, Bq, None, stats=True, row_offset=row0), shard)
                mx = torch.sqrt(stq[:, 1]).cpu().numpy()
            else:
                # no basis buffer (tcgen05 modes straight from Q): Im(phi_u s_u) from
                # the raw table columns, re * Im(s) + im * Re(s) (rare path)
                vals = []
                for u, _ in check:
                    su = complex(s[u])
                    col = (raw.buf[2 * u, :n_loc].double() * su.imag + raw.buf[2 * u + 1, :n_loc].double() * su.real)
                    vals.append(col.abs().max())
                mxt = torch.stack(vals)
                if shard is not None and shard.world > 1:
                    shard.allreduce(mxt, op="max")
                mx = mxt.cpu().numpy()
        for k, (u, _) in enumerate(check):
            if mx[k] <= 1e-10:
                realified_phi.add(u)
    # phi at each sorted position: (unit, conj)
    lam = plan.lam
    partner = conjugate_pairs(lam)
    r = lam.size
    extra = []
    for a in range(r):
        u, cj = plan.pos_unit[a]
        if partner[a] == a and u not in realified_phi:
            im_nonzero = np.any((Cs_h[:, u] * s[u]).imag != 0.0)
            if im_nonzero:
                extra.append(a)
    lay = TableLayout(lam, extra)
    # exactness: every partner pair must be (unit, False)/(unit, True) of one locked unit
    exact = True
    for a in range(r):
        b = partner[a]
        if b > a:
            ua, ca = plan.pos_unit[a]
            ub, cb = plan.pos_unit[b]
            if not (ua == ub and ca != cb):
                exact = False
    # linear maps raw(Re,Im of unit) -> table columns
    t_src, t_al, t_be = [], [], []

    def re_of(u, cj, f):      # f * Re(phi)
        sr, si = s[u].real, s[u].imag
        return (u, f * sr, -f * si)

    def im_of(u, cj, f):      # f * Im(phi)
        sr, si = s[u].real, s[u].imag
        sign = -1.0 if cj else 1.0
        return (u, f * sign * si, f * sign * sr)

    cols = [None] * lay.ncol
    for k, a in lay.re_idx:
        u, cj = plan.pos_unit[a]
        cols[k] = re_of(u, cj, 1.0 if partner[a] == a else 2.0)
    for k, a in lay.im_idx:
        u, cj = plan.pos_unit[a]
        cols[k] = im_of(u, cj, -2.0)
    for a, k in lay.extra.items():
        u, cj = plan.pos_unit[a]
        cols[k] = im_of(u, cj, 1.0)
    for c in cols:
        t_src.append(c[0]); t_al.append(c[1]); t_be.append(c[2])
    post.__exit__(None, None, None)
    general = None
    if not exact:
        # only hand-built / degenerate spectra: keep an explicit [Re phi_a, Im phi_a] basis
        general = alloc_tall(n_loc, 2 * r, table_dtype, "col", device=dev)
        g_src, g_al, g_be = [], [], []
        for a in range(r):
            u, cj = plan.pos_unit[a]
            c1 = re_of(u, cj, 1.0)
            if u in realified_phi:
                c2 = (u, 0.0, 0.0)
            else:
                c2 = im_of(u, cj, 1.0)
            for c in (c1, c2):
                g_src.append(c[0]); g_al.append(c[1]); g_be.append(c[2])
        ops.table_apply(raw, g_src, g_al, g_be, general, 2 * r)
    # the decode table stays implicit: table = raw @ mix (nraw x ncol, host);
    # no n x r rewrite (DeviceModes folds mix into every small-matrix product)
    mix = np.zeros((raw.k, lay.ncol), dtype=np.float64)
    for k, (u, al, be) in enumerate(zip(t_src, t_al, t_be)):
        mix[2 * u, k] = al
        mix[2 * u + 1, k] = be
    if timings is not None:
        timings["modes_s"] = time.perf_counter() - t0
    return DeviceModes(raw, lay, shard, general, mix=mix)


# ---------------------------------------------------------------------------
# helpers shared by the trainers
# ---------------------------------------------------------------------------
def _check_sigma(S):
    if S[-1] <= SIGMA_CUTOFF * S[0]:
        raise ValueError(
            f"requested rank hits numerically zero singular value "
            f"(sigma_r / sigma_1 = {S[-1] / S[0]:.3e}); lower the rank")


def _stability_warnings(lam):
    worst = float(np.abs(lam).max()) if lam.size else 0.0
    if worst > UNSTABLE_MODULUS:
        return [f"unstable rollout: max |lambda| = {worst:.6f}"]
    return []


@dataclass
class _Basis:
    """Truncated SVD of X = S[:, :T] for the trainers: U = A @ Umap (A tall
    on device), sigma, V (T x r) and U^T S (r x m)."""
    A: Tall
    Umap: Optional[torch.Tensor]   # l x r (randomized) or None (A is U itself)
    S: torch.Tensor
    V: torch.Tensor
    UtS: torch.Tensor
    stats: dict
    pre: Optional[dict] = None
    implicit: bool = False         # A is the snapshot buffer S itself: U = S @ Umap (m x r)


def _fit_basis(data: SnapshotMatrix, r: int, svd_mode: str, seed, oversample, power_iters,
               timings: Optional[dict], pre_svd=None) -> _Basis:
    S, pending = data.take_pending() if svd_mode == "randomized" else (data.S, None)
    T = S.k - 1
    n_tot = data.n
    t0 = time.perf_counter()
    if svd_mode == "randomized":
        # dmd.py:219-221: oversample = min(10, min(X.shape) - r), power_iters = 2
        cap = min(n_tot, T) - r
        p = min(10, cap) if oversample is None else min(oversample, cap)
        q = 2 if power_iters is None else power_iters
        l = r + p
        if not 1 <= r <= min(n_tot, T):
            raise ValueError(f"rank {r} out of range [1, {min(n_tot, T)}]")
        omega = la.draw_omega(T, l, seed)
        try:
            f = la.sketch_factors(S, T, l, q, omega, data.shard, pending=pending, pre_svd=pre_svd, r=r)
        except BaseException:
            data.pending = pending      # a streamed upload that failed is redone by the next consumer
            raise
        Ub_r = f.Ub[:, :r].contiguous()
        UtS = Ub_r.t() @ f.QtS
        basis = _Basis(f.Q, f.right(Ub_r).contiguous(), f.s[:r].contiguous(), f.Vh[:r].t().contiguous(),
                       UtS, f.stats)
        basis.stats.update(l=l, p=p, q=q)
        basis.pre = getattr(f, "pre", None)
        basis.implicit = f.implicit
    elif svd_mode == "full":
        X = Tall(S.buf, "row", S.n, T)                       # X = states[:, :-1] (dmd.py:248)
        svd = la.truncated_svd(X, r, shard=data.shard, keep_device=True)
        Ud = svd.U_device
        UtS = allreduce(data.shard, dv.get_ops().tall_gram(Ud, S))
        basis = _Basis(Ud, None, torch.as_tensor(svd.S, device=S.buf.device),
                       torch.as_tensor(svd.V, device=S.buf.device), UtS, {})
    else:
        raise ValueError(f"unknown svd mode {svd_mode!r}")
    if timings is not None:
        torch.cuda.synchronize()
        timings["svd_s"] = time.perf_counter() - t0
    return basis


_SIDE = {}

# OptDMD on fp32 tables: lift and modes on tcgen05 (FDMD_TC_FIT=0 keeps them on FP64 DMMA)
_TC_FIT = os.environ.get("FDMD_TC_FIT", "1") != "0"


def _side_stream(dev) -> torch.cuda.Stream:
    """Per-device stream for r x r work that overlaps a tall kernel."""
    key = str(dev)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=dev, priority=-1)   # small solves go first
    return _SIDE[key]


def _eig_device(Khat: torch.Tensor):
    """eig_small (linalg.py:107-133) on the device: cuSOLVER Xgeev + residual check."""
    w, V = dv.get_ops().geev(Khat)
    return la._check_eig(Khat.cpu().numpy(), w, V)


def _residual_diag(data: SnapshotMatrix, modes: DeviceModes, lam: np.ndarray):
    """||X' - Re(phi Lam pinv(phi) X)||_F and the relative value (dmd.py:269-272)."""
    S = data.S
    T = S.k - 1
    D, E = modes.basis()
    DtS = allreduce(data.shard, dv.get_ops().tall_gram(D, S, K1=E.shape[0]))   # ncol x m
    Z = modes.pinv_rows() @ DtS[:, :T].cpu().numpy()                           # pinv(phi) X
    F = np.real(E @ (lam[:, None] * Z))                                         # ncol x T
    out = dv.get_ops().residual(S, D, torch.as_tensor(F, device=S.buf.device), E.shape[0], T)
    out = allreduce(data.shard, out)
    res2, xp2 = out.cpu().numpy()
    res = float(np.sqrt(max(res2, 0.0)))
    return res, res / max(float(np.sqrt(xp2)), 1e-300)


def _default_table_dtype(data: SnapshotMatrix):
    return data._S.dtype


# ---------------------------------------------------------------------------
# exact DMD (dmd.py:240-274)
# ---------------------------------------------------------------------------
def exact_dmd(data, r, svd_mode="full", seed=None, *, oversample=None, power_iters=None,
              residual=True, table_dtype=None, timings=None):
    """One-shot fit of the reduced step operator (dmd.py:240-274)."""
    data = _as_snapshots(data)
    n, T = data.n, data.n_transitions
    if not 1 <= r <= min(n, T):
        raise ValueError(f"rank {r} out of range [1, {min(n, T)}]")
    basis = _fit_basis(data, r, svd_mode, seed, oversample, power_iters, timings)
    Sv = basis.S.cpu().numpy()
    _check_sigma(Sv)
    t0 = time.perf_counter()
    VS = basis.V / basis.S[None, :]                          # V / S   (T x r)
    Khat = basis.UtS[:, 1:] @ VS                             # U^H X' V S^-1 (dmd.py:255-256)
    lam_raw, W = _eig_device(Khat)
    plan = pair_plan(lam_raw)
    Wt = torch.as_tensor(W, device=VS.device)
    if timings is not None:
        timings["small_s"] = time.perf_counter() - t0
    # phi = X' (V/S) W  (dmd.py:255,258) = S [0; (V/S) W]; the sketch basis is no
    # longer needed, so it is released before the mode buffers are allocated.
    Cmap = VS.to(torch.complex128) @ Wt
    A, top = data.S, 1
    basis.A = None
    tdt = table_dtype or _default_table_dtype(data)
    # (stays on FP64 DMMA: Phi = X' V S^-1 W amplifies the operand error by
    # sigma_1 / sigma_r, so an FP32-accurate product is not enough here —
    # measured 5% on a cancellation-prone frame checksum of config 1; the
    # OptDMD modes U B^T have no such amplification and run on tcgen05)
    modes = _modes_pass(A, Cmap, plan, top, data.shard, tdt, timings)
    model = ReducedModel(None, plan.lam, Sv, data.dt, grid_meta=data.grid_meta,
                         provenance={"method": "exact", "svd": svd_mode, "seed": seed}, _modes=modes)
    if svd_mode == "randomized":
        model.provenance["sketch"] = {k: v for k, v in basis.stats.items()}
    if residual:
        t0 = time.perf_counter()
        res, rel = _residual_diag(data, modes, plan.lam)
        model.provenance["residual"] = res
        model.provenance["residual_rel"] = rel
        if timings is not None:
            timings["residual_s"] = time.perf_counter() - t0
    model.provenance["warnings"] = _stability_warnings(plan.lam)
    return model


# ---------------------------------------------------------------------------
# OptDMD (dmd.py:277-455), LM on the device
# ---------------------------------------------------------------------------
def vandermonde(alpha, T):
    """T x r matrix with entry (i, j) = alpha_j ** i (dmd.py:277-282)."""
    if T < 1:
        raise ValueError("T must be >= 1")
    alpha = np.asarray(alpha, dtype=np.complex128)
    return alpha[None, :] ** np.arange(T)[:, None]


@dataclass
class LMConfig:
    max_iters: int = 200
    init_damping: float = 1.0
    damping_up: float = 2.0
    damping_down: float = 3.0
    rel_tol: float = 1e-8
    collapse_tol: float = 1e-12


class _AlphaCollapse(Exception):
    pass


def _vander_t(alpha: torch.Tensor, T: int) -> torch.Tensor:
    t = torch.arange(T, device=alpha.device, dtype=torch.float64)
    return alpha[None, :] ** t[:, None].to(alpha.dtype)


def _min_sep_t(alpha: torch.Tensor) -> float:
    if alpha.numel() < 2:
        return float("inf")
    d = (alpha[:, None] - alpha[None, :]).abs()
    d.fill_diagonal_(float("inf"))
    return float(d.min().item())


def _objective_t(alpha, D, T):
    P = _vander_t(alpha, T)
    q = []
    B = la.lstsq_minnorm(P, D, qr_out=q)  # gelsd semantics (linalg.py:136-141)
    R = D - P @ B
    # P carries its orthonormal factor when the QR path ran (reused by the LM step)
    return float(torch.linalg.vector_norm(R).item()), B, (P, q[0] if q else None), R


def _varpro_lm_device(D: torch.Tensor, alpha0: np.ndarray, cfg: LMConfig):
    """dmd.py:314-363 on device tensors (complex128)."""
    T = D.shape[0]
    dev = D.device
    t = torch.arange(T, device=dev, dtype=torch.float64).to(torch.complex128)
    alpha = torch.as_tensor(np.asarray(alpha0, dtype=np.complex128), device=dev).clone()
    if _min_sep_t(alpha) < cfg.collapse_tol:
        raise _AlphaCollapse
    f, B, P, R = _objective_t(alpha, D, T)
    floor = 1e-14 * float(torch.linalg.vector_norm(D).item())
    history = [f]
    if cfg.max_iters == 0:
        return alpha, B, history, True
    mu = cfg.init_damping
    converged = False
    eye = torch.eye(alpha.numel(), dtype=torch.complex128, device=dev)
    jac = None
    for _ in range(cfg.max_iters):
        if f <= floor:
            converged = True
            break
        if jac is None:                   # a rejected step only changes mu: same J^H J and g
            Pm, Qp = P
            if Qp is None:
                Qp, _ = torch.linalg.qr(Pm, mode="reduced")
            dphi = torch.zeros_like(Pm)
            dphi[1:, :] = t[1:, None] * alpha[None, :] ** (t[1:, None] - 1)
            Wk = dphi - Qp @ (Qp.mH @ dphi)
            jac = ((Wk.mH @ Wk) * (B @ B.mH).conj(), torch.diagonal(Wk.mH @ (R @ B.mH)))
        JHJ, g = jac
        delta, info = torch.linalg.solve_ex(JHJ + mu * eye, g)
        if int(info.item()) != 0:
            mu *= cfg.damping_up
            continue
        cand = alpha + delta
        if _min_sep_t(cand) < cfg.collapse_tol:
            raise _AlphaCollapse
        f_new, B_new, P_new, R_new = _objective_t(cand, D, T)
        if f_new < f:
            rel = (f - f_new) / max(f, 1e-300)
            alpha, f, B, P, R = cand, f_new, B_new, P_new, R_new
            jac = None
            history.append(f)
            mu /= cfg.damping_down
            if rel < cfg.rel_tol or f <= floor:
                converged = True
                break
        else:
            mu *= cfg.damping_up
    return alpha, B, history, converged


def _symmetrize(alpha: np.ndarray, B: np.ndarray):
    """dmd.py:439-455."""
    partner = conjugate_pairs(alpha)
    alpha = alpha.copy()
    B = B.copy()
    for i in range(alpha.size):
        j = partner[i]
        if j > i:
            a = 0.5 * (alpha[i] + np.conj(alpha[j]))
            alpha[i] = a
            alpha[j] = np.conj(a)
            row = 0.5 * (B[i, :] + np.conj(B[j, :]))
            B[i, :] = row
            B[j, :] = np.conj(row)
        elif j == i and abs(alpha[i].imag) <= 1e-8 * max(abs(alpha[i]), 1e-300):
            alpha[i] = alpha[i].real
            B[i, :] = B[i, :].real
    return alpha, B


def optdmd(data, r, init=None, lm_config=None, svd_mode="full", seed=None, *, oversample=None,
           power_iters=None, table_dtype=None, timings=None, keep_basis=False):
    """Variable-projection refit of the eigenvalues (dmd.py:366-436)."""
    cfg = lm_config or LMConfig()
    data = _as_snapshots(data)
    n, T = data.n, data.n_transitions
    if not 1 <= r <= min(n, T):
        raise ValueError(f"rank {r} out of range [1, {min(n, T)}]")
    use_tc = (_TC_FIT and svd_mode == "randomized" and torch.cuda.is_available()
              and (table_dtype or _default_table_dtype(data)) == torch.float32 and data._S.buf.is_cuda)

    def _pre_svd(Q, fix):
        # the fp16 split of the CholeskyQR2 buffer (|entries| <= ~1: no scan)
        # is issued under svd(B); Q = buffer @ fix, and fix is folded into Umap
        if Q.dtype != torch.float64 or Q.layout != "row" or Q.k > 256:
            return None
        return dv.get_ops().tc_rows(Q, bound=2.0)

    with stage("optdmd.basis"):
        basis = _fit_basis(data, r, svd_mode, seed, oversample, power_iters, timings,
                           pre_svd=_pre_svd if use_tc else None)
    Sv = basis.S.cpu().numpy()
    _check_sigma(Sv)
    t0 = time.perf_counter()
    tdt = table_dtype or _default_table_dtype(data)
    dev = basis.V.device
    on_cuda = dev.type == "cuda"
    ready = torch.cuda.Event() if on_cuda else None
    if ready is not None:
        ready.record()
    # phi = U @ B.T (dmd.py:414). The POD basis U = Q Ub_r is lifted once into
    # a column-major table (the north_star reconstruction basis), Q is released,
    # and the modes are formed from U — peak HBM stays S + Q + U at config 3.
    # The lift does not depend on the eigenvalues: it is launched first, on all
    # but 8 SMs, and the r x r work below (eig, variable projection) runs on a
    # side stream in its shadow.
    tc_src = None
    if basis.Umap is None:
        U = basis.A
    elif basis.implicit and _TC_FIT and on_cuda and tdt == torch.float32 and r <= 256:
        # projection from the snapshot Gram: no sketch buffer exists, U = S Umap
        # is one FP64 DMMA pass over the snapshots (its error is O(u cond) —
        # it cannot go through a 22-bit split of S), written as fp32 and split
        # once into the fp16 planes the tcgen05 modes product (and the config-4
        # reconstruction) stream; |U| <= 1 (orthonormal columns)
        ops = dv.get_ops()
        S_ = basis.A
        n_loc = S_.n
        U = None
        # rows >= T of the m x r map are zero (X = S[:, :T]): the product runs over
        # K = T columns, and the kernel skips the empty half of the last k-chunk
        Um = basis.Umap[:T].contiguous()
        if keep_basis and keep_basis != "planes":
            with stage("lift.U=SM"):
                U = alloc_tall(n_loc, r, torch.float32, "col", device=dev)
                ops.tall_gemm(S_, Um, U, alg_flops=2.0 * n_loc * T * r, share_sms=True)
            with stage("lift.split_U"):
                qt = ops.tc_basis(U, bound=2.0)
        else:
            # the DMMA epilogue writes the fp16 planes directly (no fp32 U)
            with stage("lift.U=SM"):
                qt = ops.tall_gemm_planes(S_, Um, bound=2.0, alg_flops=2.0 * n_loc * T * r, share_sms=True)
            if keep_basis == "planes":
                U = qt
        basis.A = None
        tc_src = {"planes": qt, "Umap": None, "n": n_loc}
    elif (_TC_FIT and on_cuda and tdt == torch.float32 and basis.A.dtype == torch.float64
          and basis.A.layout == "row" and basis.A.k <= 256):
        # fp32 tables: the lift U = Q Ub and the modes Q (Ub B^T) run on tcgen05
        # (FP16 2-way split, FP32-accurate — the precision of the fp32 tables
        # they fill) from one fp16 copy of Q; Q itself is released before U
        # is allocated (peak S + Q + planes = S + U + planes + table)
        ops = dv.get_ops()
        with stage("lift.split_Q"):
            # the buffer holds (near-)orthonormal columns (CholeskyQR2 output,
            # Q = buffer @ fix with fix ~ I): |entries| <= ~1, no scan needed;
            # normally already issued under svd(B) (sketch_factors pre_svd)
            qt = getattr(basis, "pre", None) or ops.tc_rows(basis.A, bound=2.0)
        n_loc = basis.A.n
        basis.A = None
        U = None
        if keep_basis == "planes":
            # the config-4 basis as the fp16 hi/lo planes the batched
            # reconstruction streams, written by the lift itself (|U| <= 1)
            with stage("lift.U=QUb"):
                U = ops.tc_decode_planes(qt, basis.Umap.to(torch.float32), bound=2.0, share_sms=True)
        elif keep_basis:        # the config-4 basis; the model itself never needs U
            with stage("lift.U=QUb"):
                U = alloc_tall(n_loc, r, tdt, "col", device=dev)
                ops.tc_decode(qt, basis.Umap.to(torch.float32), out=U.buf[:r], share_sms=True)
        tc_src = {"planes": qt, "Umap": basis.Umap, "n": n_loc}
    else:
        with stage("lift.U=QUb"):
            U = alloc_tall(basis.A.n, r, tdt, "col", device=basis.A.buf.device)
            nl = float(basis.A.n)
            dv.get_ops().tall_gemm(basis.A, basis.Umap, U, alg_flops=2 * nl * basis.A.k * r,   # linalg.py:88
                                   share_sms=True)
    side = _side_stream(dev) if on_cuda else None
    if side is not None:
        side.wait_event(ready)
    with (torch.cuda.stream(side) if side is not None else contextlib.nullcontext()):
        Dm = (basis.V.conj() * basis.S[None, :]).to(torch.complex128)      # dmd.py:384
        if init is None:
            # alpha0 = exact_dmd(data, r, svd_mode, seed).lam (dmd.py:387): the same
            # seed reproduces the same SVD, so the eigenvalues come from it directly.
            # eigenvalues only: the init needs lam, not the residual-checked vectors
            # of eig_small (linalg.py:107-133) that exact_dmd would also build
            with stage("small.eig(Khat)"):
                VS = basis.V / basis.S[None, :]
                Khat = basis.UtS[:, 1:] @ VS
                with stage("small.geev"):
                    lam_raw, _ = dv.get_ops().geev(Khat, vectors=False)
                alpha0 = pair_plan(lam_raw).lam
        else:
            alpha0 = np.asarray(init, dtype=np.complex128)
            if alpha0.size != r:
                raise ValueError(f"init has {alpha0.size} eigenvalues, expected {r}")
        try:
            with stage("small.varpro_lm"):
                alpha, B, history, converged = _varpro_lm_device(Dm, alpha0, cfg)
        except _AlphaCollapse:
            rng = np.random.default_rng(0 if seed is None else seed)
            jitter = 1e-10 * (1.0 + np.abs(alpha0)) * np.exp(2j * np.pi * rng.random(alpha0.size))
            try:
                alpha, B, history, converged = _varpro_lm_device(Dm, alpha0 + jitter, cfg)
            except _AlphaCollapse:
                raise ConvergenceError("eigenvalue iterates collapsed below separation tolerance twice") from None
        alpha_h = alpha.cpu().numpy()
        B_h = B.cpu().numpy()
        Dh = Dm.cpu().numpy()
    if side is not None:
        torch.cuda.current_stream().wait_stream(side)
    a_s, B_s = _symmetrize(alpha_h, B_h)
    f_sym = float(np.linalg.norm(Dh - vandermonde(a_s, T) @ B_s))
    if f_sym <= history[-1] * (1 + 1e-9) and f_sym <= history[0] * (1 + 1e-12):
        alpha_h, B_h = a_s, B_s
    if timings is not None:
        timings["lm_s"] = time.perf_counter() - t0
    plan = pair_plan(alpha_h)
    Bt = torch.as_tensor(B_h.T.copy(), device=dev)                          # r x r
    if basis.Umap is not None:
        basis.A = None                                                       # release Q
    with stage("optdmd.modes_total"):
        modes = _modes_pass(U if tc_src is None else None, Bt, plan, 0, data.shard, tdt, timings,
                            a_orthonormal=True, tc_src=tc_src)
    tc_src = None
    model = ReducedModel(None, plan.lam, Sv, data.dt, grid_meta=data.grid_meta,
                         provenance={"method": "optdmd", "svd": svd_mode, "seed": seed,
                                     "objective_history": history, "converged": converged},
                         _modes=modes)
    model.basis_U = U if keep_basis else None
    if svd_mode == "randomized":
        model.provenance["sketch"] = {k: v for k, v in basis.stats.items()}
    warns = _stability_warnings(plan.lam)
    if not converged and cfg.max_iters > 0:
        warns.append(f"variable projection hit max_iters={cfg.max_iters}")
        warnings.warn(warns[-1], RuntimeWarning, stacklevel=2)
    model.provenance["warnings"] = warns
    return model


# ---------------------------------------------------------------------------
# control channels (dmd.py:458-491)
# ---------------------------------------------------------------------------
@dataclass
class ControlOperator:
    reduced_b: list
    labels: list

    def __post_init__(self):
        if len(self.reduced_b) != len(self.labels):
            raise ValueError("one label per channel required")
        self.reduced_b = [np.asarray(m, dtype=np.complex128) for m in self.reduced_b]


def fit_control(model, channels, labels=None):
    """Project each force-response matrix into the trained basis:
    reduced_b_i = pinv(phi) @ B_i (dmd.py:471-491), via the device table."""
    labels = labels or [f"channel_{k}" for k in range(len(channels))]
    reduced = []
    dev = model.modes.table.buf.device
    for mat in channels:
        if mat.shape[0] != model.n:
            raise ValueError(f"channel has {mat.shape[0]} rows, model state length is {model.n}")
        if hasattr(mat, "toarray") and not isinstance(mat, np.ndarray):
            mat = mat.toarray()
        if isinstance(mat, torch.Tensor):
            Bt = mat.to(dev)
        else:
            Bt = torch.as_tensor(np.asarray(mat, dtype=np.float64), device=dev)
        if Bt.is_complex():
            re = model.modes.project(Bt.real.t().contiguous())
            im = model.modes.project(Bt.imag.t().contiguous())
            red = re + 1j * im
        else:
            red = model.modes.project(Bt.t().contiguous())
        reduced.append(red)
    return ControlOperator(reduced, list(labels))


# ---------------------------------------------------------------------------
# Control-augmented DMDc (BASELINE config 2). No reference implementation:
# the reference's DMDc is fit_control with known B (dmd.py:471-491), joint
# identification is a declared non-goal. Parity unpinned;
# restated from Proctor et al. 2016 as cited at PAPER.md:420.
# ---------------------------------------------------------------------------
def dmdc_fit(data, controls, r_aug, r, seed=None, *, oversample=10, power_iters=1,
             table_dtype=None, timings=None):
    """Returns (ReducedModel, ControlOperator) for x_{j+1} = A x_j + B u_j.

    controls: ell x T host array (u_j for j < T). The augmented matrix
    [X; Upsilon] is sketched at rank r_aug; the output basis U_hat is a rank-r
    sketch of X' (seed + 1). reduced_b is scaled by 1/dt so that
    runtime.step_forced (which multiplies by dt, runtime.py:188) reproduces
    B u_j exactly.

    Row-sharded data (``data.shard``): the ell control rows of [X; Upsilon]
    live on the last rank; every reduction over rows is all-reduced.
    """
    data = _as_snapshots(data)
    shard = data.shard if (data.shard is not None and data.shard.world > 1) else None
    S = data.S
    n_loc, m = S.n, S.k
    n = data.n
    T = m - 1
    Ups = np.asarray(controls, dtype=np.float64)
    if Ups.ndim != 2 or Ups.shape[1] != T:
        raise ValueError(f"controls must be ell x {T}")
    ell = Ups.shape[0]
    dev = S.buf.device
    last = shard is None or shard.row0 + n_loc == n
    extra = ell if last else 0
    # augmented tall matrix: rows [S; Upsilon | 0] (the control rows on the last shard)
    with stage("dmdc.aug_copy"):
        Aug = alloc_tall(n_loc + extra, m, S.dtype, "row", device=dev, zero=False)
        Aug.buf[:n_loc].copy_(S.buf[:n_loc])
        if extra:
            tail = torch.zeros((ell, Aug.ld), dtype=S.dtype, device=dev)
            tail[:, :T] = torch.as_tensor(Ups, dtype=S.dtype, device=dev)
            Aug.buf[n_loc:n_loc + ell].copy_(tail)
    aug_shard = None
    if shard is not None:
        aug_shard = Shard(shard.row0, n_loc + extra, n + ell, shard.group, shard.world)
    t0 = time.perf_counter()
    p1 = min(oversample, min(n + ell, T) - r_aug)
    with stage("dmdc.sketch_aug"):
        f1 = la.sketch_factors(Aug, T, r_aug + p1, power_iters, la.draw_omega(T, r_aug + p1, seed), aug_shard)
    p2 = min(oversample, min(n, T) - r)
    # rank-r sketch of X' = S[:, 1:] (column window c0 = 1 of the same resident S)
    with stage("dmdc.sketch_Xp"):
        f2 = la.sketch_factors(S, T, r + p2, power_iters,
                               la.draw_omega(T, r + p2, None if seed is None else seed + 1), shard, c0=1)
    Ub1 = f1.Ub[:, :r_aug]
    s1 = f1.s[:r_aug]
    V1 = f1.Vh[:r_aug].t()
    Ub2 = f2.Ub[:, :r]
    # U1^T Uhat = Ub1^T (Q1[:n]^T Q2) Ub2
    Q1top = Tall(f1.Q.buf, "row", n_loc, f1.Q.k)
    with stage("dmdc.cross_Q1tQ2"):
        M12 = allreduce(shard, dv.get_ops().tall_gram(Q1top, f2.Q))       # l1 x l2
    if f1.fix is not None:
        M12 = f1.fix.t() @ M12
    if f2.fix is not None:
        M12 = M12 @ f2.fix
    U1tUh = Ub1.t() @ M12 @ Ub2                                        # r_aug x r
    U2 = torch.zeros((ell, r_aug), dtype=torch.float64, device=dev)   # control rows of U1
    if extra:
        U2 = f1.Q.buf[n_loc:n_loc + ell, : f1.Q.k].to(torch.float64) @ f1.right(Ub1)
    U2 = allreduce(shard, U2.contiguous())                             # ell x r_aug
    UhtXp = Ub2.t() @ f2.QtS[:, 1:]                                    # r x T
    core = UhtXp @ (V1 / s1[None, :])                                  # r x r_aug
    Atil = core @ U1tUh                                                # r x r
    Btil = core @ U2.t()                                               # r x ell
    with stage("small.eig(Atil)"):
        lam_raw, W = _eig_device(Atil)
    plan = pair_plan(lam_raw)
    Wt = torch.as_tensor(W, device=dev)
    Cmap = ((V1 / s1[None, :]) @ U1tUh).to(torch.complex128) @ Wt     # T x r
    del Aug, f1
    if timings is not None:
        torch.cuda.synchronize()
        timings["svd_s"] = time.perf_counter() - t0
    tdt = table_dtype or S.dtype
    with stage("dmdc.modes"):
        modes = _modes_pass(S, Cmap, plan, 1, shard, tdt, timings)
    model = ReducedModel(None, plan.lam, s1.cpu().numpy()[:r] if r <= r_aug else s1.cpu().numpy(),
                         data.dt, grid_meta=data.grid_meta,
                         provenance={"method": "dmdc", "svd": "randomized", "seed": seed,
                                     "r_aug": r_aug}, _modes=modes)
    # reduced_b = pinv(phi) U_hat B~ / dt, U_hat = Q2 Ub2
    with stage("dmdc.reduced_b"):
        D, E = modes.basis()
        DtQ2 = allreduce(shard, dv.get_ops().tall_gram(D, f2.Q, K1=E.shape[0]))   # ncol x l2
        y = (DtQ2 @ f2.right(Ub2) @ Btil).cpu().numpy()                    # ncol x ell
        with stage("dmdc.pinv_rows"):
            red = modes.pinv_rows() @ y / data.dt
    ctrl = ControlOperator([red], ["augmented"])
    model.provenance["A_tilde"] = Atil.cpu().numpy()
    model.provenance["B_tilde"] = Btil.cpu().numpy()
    return model, ctrl
