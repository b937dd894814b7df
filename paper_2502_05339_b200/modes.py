"""Device-resident mode basis: the pair-aware real decode table.

A fitted model never materialises the complex n x r mode matrix on the
device. It stores the reference's real decode table (dmd.py:92-120) column-
major in HBM:

    self-paired mode a : column  Re(phi_a)            [+ Im(phi_a) "extra" column if complex]
    conjugate pair a<b : columns 2 Re(phi_a), -2 Im(phi_a)

so phi = D @ E for a fixed sparse complex map E (ncol x r). Decode, encode
(pinv via the Gram D^T D), control projection and the residual diagnostic
all run on D. Models whose partner columns are not exact conjugates (only
possible for hand-built models) additionally keep a general basis
[Re phi_a, Im phi_a]_a.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import device as dv
from .device import Shard, Tall, allreduce, alloc_tall

# fp32 tables: batches of at least this many frames decode on tcgen05
TC_MIN_FRAMES = 16
_TC_DECODE = __import__("os").environ.get("FDMD_TC_DECODE", "1") != "0"


def conjugate_pairs(lam, tol=1e-8):
    """partner[i] = j with lam[j] ~ conj(lam[i]); i itself if real or unmatched
    (reference dmd.py:131-155, same greedy order and thresholds)."""
    lam = np.asarray(lam)
    r = lam.size
    scale = max(float(np.abs(lam).max()), 1e-300) if r else 1.0
    partner = np.full(r, -1, dtype=np.int64)
    for i in range(r):
        if partner[i] >= 0:
            continue
        if abs(lam[i].imag) <= tol * scale:
            partner[i] = i
            continue
        cand = np.flatnonzero(partner < 0)
        cand = cand[cand != i]
        if cand.size:
            d = np.abs(lam[cand] - np.conj(lam[i]))
            j = int(np.argmin(d))          # first minimum, as the reference's strict '<' scan
            if d[j] <= 10 * tol * scale + tol:
                partner[i] = cand[j]
                partner[cand[j]] = i
                continue
        partner[i] = i
    return partner


class TableLayout:
    """Host bookkeeping of the decode table for a given eigenvalue vector."""

    def __init__(self, lam, extra_modes=()):
        self.lam = np.asarray(lam, dtype=np.complex128)
        self.partner = conjugate_pairs(self.lam)
        r = self.lam.size
        self.re_idx, self.im_idx = [], []
        k = 0
        for a in range(r):
            b = self.partner[a]
            if b < a:
                continue
            if b == a:
                self.re_idx.append((k, a))
                k += 1
            else:
                self.re_idx.append((k, a))
                self.im_idx.append((k + 1, a))
                k += 2
        self.ncol_table = k
        self.extra = {}
        for a in extra_modes:
            self.extra[int(a)] = k
            k += 1
        self.ncol = k

    def E(self) -> np.ndarray:
        """phi = D @ E (ncol x r complex)."""
        r = self.lam.size
        E = np.zeros((self.ncol, r), dtype=np.complex128)
        col_re = {a: k for k, a in self.re_idx}
        col_im = {a: k for k, a in self.im_idx}
        for a in range(r):
            b = self.partner[a]
            if b == a:
                E[col_re[a], a] = 1.0
                if a in self.extra:
                    E[self.extra[a], a] = 1.0j
            elif b > a:
                E[col_re[a], a] = 0.5
                E[col_im[a], a] = -0.5j
                E[col_re[a], b] = 0.5
                E[col_im[a], b] = 0.5j
        return E

    def coeff(self, Z: np.ndarray) -> np.ndarray:
        """Table coefficients (ncol_table x B) for conjugate-symmetric states Z (r x B)."""
        Z = np.asarray(Z, dtype=np.complex128).reshape(self.lam.size, -1)
        c = np.empty((self.ncol_table, Z.shape[1]))
        for k, a in self.re_idx:
            c[k] = Z[a].real
        for k, a in self.im_idx:
            c[k] = Z[a].imag
        return c


def _pinv_svd(M: torch.Tensor, rel_tol: float) -> torch.Tensor:
    """SVD pseudo-inverse of a small device matrix (linalg.py:93-104)."""
    U, s, Vh = torch.linalg.svd(M, full_matrices=False)
    if s.numel() == 0 or float(s[0]) == 0.0:
        return torch.zeros((M.shape[1], M.shape[0]), dtype=M.dtype, device=M.device)
    keep = s > rel_tol * s[0]
    inv = torch.where(keep, 1.0 / torch.where(keep, s, torch.ones_like(s)), torch.zeros_like(s))
    return (Vh.mH * inv.to(Vh.dtype)) @ U.mH


class DeviceModes:
    """Decode table in HBM (+ optional general basis) and its cached Gram.

    ``mix`` (nraw x ncol, host float64): the table is implicit, table =
    table_buf @ mix — the fit keeps the raw [Re, Im] mode columns and folds
    the reference's normalisation / phase canonicalisation / pair locking
    (dmd.py:189-213) into this small matrix instead of rewriting n x r
    values (every consumer multiplies the table by a small matrix)."""

    def __init__(self, table: Tall, layout: TableLayout, shard: Optional[Shard] = None,
                 general: Optional[Tall] = None, mix: Optional[np.ndarray] = None):
        assert table.layout == "col"
        self.table = table
        self.layout = layout
        self.shard = shard
        self.general = general
        self.mix = None if mix is None else np.asarray(mix, dtype=np.float64)
        self._pinv_small = None
        self._pinv_cond2 = np.inf
        self._pinv_rows = None
        self._tc_planes = None     # fp16 hi/lo planes of the table for batched decodes
        # Gram of the raw table (D^T D, all raw columns): shared by every model
        # derived from the same table (editing.apply_edit folds into the mix)
        self.raw_gram = None

    @property
    def n_local(self) -> int:
        return self.table.n

    @property
    def dtype(self):
        return self.table.dtype

    # -- basis used for exact complex products: (Tall, E) -------------------
    def basis(self):
        if self.general is not None:
            r = self.layout.lam.size
            E = np.zeros((2 * r, r), dtype=np.complex128)
            for a in range(r):
                E[2 * a, a] = 1.0
                E[2 * a + 1, a] = 1.0j
            return self.general, E
        if self.mix is not None:
            return self.table, self.mix @ self.layout.E()
        return self.table, self.layout.E()

    def pinv_small(self) -> np.ndarray:
        """P such that pinv(phi) = P @ E^H @ D^T (r x r complex), from the
        Hermitian Gram phi^H phi = E^H (D^T D) E (eigh on the device). Only
        valid for a well-conditioned phi; `pinv_rows` is the general form."""
        if self._pinv_small is None:
            D, E = self.basis()
            G = self._gram(D)
            Et = torch.as_tensor(E, device=G.device)
            H = Et.mH @ G.to(torch.complex128) @ Et
            H = 0.5 * (H + H.mH)
            mu, V = torch.linalg.eigh(H)
            mu_max = float(mu.max().item()) if mu.numel() else 0.0
            keep = mu > max(1e-14 * mu_max, 0.0)
            inv = torch.where(keep, 1.0 / torch.where(keep, mu, torch.ones_like(mu)), torch.zeros_like(mu))
            P = (V * inv.to(V.dtype)) @ V.mH
            self._pinv_small = P.cpu().numpy()
            self._pinv_cond2 = (mu_max / float(mu.min().item())) if mu.numel() and float(mu.min()) > 0 else np.inf
        return self._pinv_small

    def _gram(self, D: Tall) -> torch.Tensor:
        if self.general is None and self.raw_gram is not None:
            return self.raw_gram
        G = allreduce(self.shard, dv.get_ops().tall_gram(D, D, symmetric=True))
        if self.general is None:
            self.raw_gram = G
        return G

    def pinv_rows(self) -> np.ndarray:
        """M (r x ncol complex) with pinv(phi) = M @ D^T — the reference's SVD
        pseudo-inverse (linalg.py:93-104: sigma > 1e-12 sigma_max kept).

        Well-conditioned phi (cond <= 1e6): M = (phi^H phi)^-1 E^H from the
        Gram (eigh), exact to O(u cond^2). Otherwise the Gram cannot resolve
        the reference's cut (it sees sigma ratios only down to ~1e-7): the
        table is orthonormalised on the device (CholeskyQR2 with its shifted /
        Householder / TSQR fallbacks, D = Q R), and M = pinv(R E) R^-T with
        the reference's SVD cut on the small R E, plus a RuntimeWarning."""
        if getattr(self, "_pinv_rows", None) is not None:
            return self._pinv_rows
        D, E = self.basis()
        P = self.pinv_small()
        if self._pinv_cond2 <= 1e12:
            self._pinv_rows = P @ E.conj().T
            return self._pinv_rows
        import warnings

        from . import linalg as la
        warnings.warn(f"ill-conditioned mode basis (cond(phi) ~ {np.sqrt(self._pinv_cond2):.1e}): "
                      "pseudo-inverse through a QR of the table", RuntimeWarning, stacklevel=3)
        ncol = E.shape[0]
        dev = D.buf.device
        Y = dv.alloc_tall(D.n, ncol, torch.float64, "row", device=dev)
        Y.view().copy_(D.view()[:, :ncol])
        # Householder QR of the table (TSQR across row shards): D = Q R, R may be
        # singular (a real mode's zero imaginary column)
        R = la._householder_inplace(Y, self.shard if (self.shard is not None and self.shard.world > 1) else None,
                                    None)
        del Y
        # phi = Q (R E): pinv(phi) = pinv(R E) Q^T, and on range(D) Q^T = (R^+)^T D^T
        RE = R.to(torch.complex128) @ torch.as_tensor(E, device=dev)
        self._pinv_rows = (_pinv_svd(RE, 1e-12) @ _pinv_svd(R, 1e-12).t().to(torch.complex128)).cpu().numpy()
        return self._pinv_rows

    def project(self, U: torch.Tensor) -> np.ndarray:
        """pinv(phi) @ U for U (nv x n_local) device rows -> (r x nv) complex host."""
        D, E = self.basis()
        ys = []
        ops = dv.get_ops()
        for v0 in range(0, U.shape[0], 8):
            ys.append(ops.colmajor_dot(D, U[v0:v0 + 8]))
        y = allreduce(self.shard, torch.cat(ys, dim=1)).cpu().numpy()   # ncol x nv
        return self.pinv_rows() @ y

    # -- decode ------------------------------------------------------------
    def decode_coeff(self, C: torch.Tensor, out: Optional[torch.Tensor] = None, general=False,
                     basis_coords=False) -> torch.Tensor:
        """frames (B x n_local) = table[:, :ncol] @ C (ncol x B) — or, with
        basis_coords, D @ C for C in the coordinates of basis()'s D."""
        if general and self.general is not None:
            return dv.get_ops().decode(self.general, C, out=out, ncols=int(C.shape[0]))
        if self.mix is not None and not basis_coords:
            M = torch.as_tensor(self.mix[:, : int(C.shape[0])], device=C.device)
            C = M @ C.to(torch.float64)
        k = int(C.shape[0])
        if (C.dim() == 2 and int(C.shape[1]) >= TC_MIN_FRAMES and self.table.dtype == torch.float32
                and self.table.buf.is_cuda and k <= 256 and _TC_DECODE):
            # frame batches on tcgen05 (FP32-accurate 2-way FP16 split): the
            # table is read once per 256 frames instead of once per 32
            if self._tc_planes is None or self._tc_planes["r"] != k:
                self._tc_planes = dv.get_ops().tc_basis(self.table, ncols=k)
            return dv.get_ops().tc_decode(self._tc_planes, C, out=out)
        return dv.get_ops().decode(self.table, C, out=out, ncols=k)

    def host_table(self) -> np.ndarray:
        """n x ncol_table float64 (the reference's decode_table cols)."""
        if self.mix is not None:
            nraw = self.mix.shape[0]
            v = self.table.buf[:nraw, : self.table.n].t().to(torch.float64)
            M = torch.as_tensor(self.mix[:, : self.layout.ncol_table], device=v.device)
            return (v @ M).cpu().numpy()
        v = self.table.buf[: self.layout.ncol_table, : self.table.n]
        return v.t().to(torch.float64).cpu().numpy().copy()

    def host_phi(self) -> np.ndarray:
        D, E = self.basis()
        M = D.buf[: E.shape[0], : D.n].t().to(torch.float64).cpu().numpy()
        return np.ascontiguousarray(M @ E)


def modes_from_host_phi(phi: np.ndarray, lam: np.ndarray, dtype=torch.float64, device=None) -> DeviceModes:
    """Build the device table from a host complex mode matrix (the
    ReducedModel(phi, lam, ...) constructor path, dmd.py:62-77)."""
    device = device or dv.default_device()
    phi = np.asarray(phi, dtype=np.complex128)
    lam = np.asarray(lam, dtype=np.complex128)
    n, r = phi.shape
    part = conjugate_pairs(lam)
    extra = [a for a in range(r) if part[a] == a and np.any(phi[:, a].imag != 0.0)]
    lay = TableLayout(lam, extra)
    cols = np.empty((lay.ncol, n))
    for k, a in lay.re_idx:
        cols[k] = phi[:, a].real if part[a] == a else 2.0 * phi[:, a].real
    for k, a in lay.im_idx:
        cols[k] = -2.0 * phi[:, a].imag
    for a, k in lay.extra.items():
        cols[k] = phi[:, a].imag
    T = alloc_tall(n, lay.ncol, dtype, "col", device=device)
    T.buf[: lay.ncol, :n].copy_(torch.from_numpy(cols))
    general = None
    exact = all(np.array_equal(phi[:, part[a]], np.conj(phi[:, a])) for a in range(r) if part[a] > a)
    if not exact:
        G = alloc_tall(n, 2 * r, dtype, "col", device=device)
        g = np.empty((2 * r, n))
        g[0::2] = phi.real.T
        g[1::2] = phi.imag.T
        G.buf[: 2 * r, :n].copy_(torch.from_numpy(g))
        general = G
    return DeviceModes(T, lay, None, general)
