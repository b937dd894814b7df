"""Device linear algebra for the DMD fit, mirroring `flowdmd.linalg`
(reference linalg.py:1-141) with the same names and semantics.

Tall work (n rows) runs in libfdmd FP64 DMMA kernels; small factors
(<= a few hundred on a side) stay on the device in cuSOLVER/cuBLAS via
torch.linalg (preferred library forced to cuSOLVER). The orthonormalisation
of the sketch is CholeskyQR2 (two Gram + Cholesky + triangular-apply passes)
instead of Householder (linalg.py:82,85), falling back to shifted CholeskyQR3
when the sketch is ill-conditioned and to a device Householder QR when it is
numerically rank deficient.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import device as dv
from .device import Shard, Tall, allreduce, alloc_tall
from .errors import ConvergenceError
from .trace import stage

if torch.cuda.is_available():
    try:
        torch.backends.cuda.preferred_linalg_library("cusolver")
    except Exception:  # pragma: no cover
        pass

# condition number of R1 above which CholeskyQR2 is replaced by shifted CholeskyQR3
CHOLQR2_COND_LIMIT = 3e7


# ---------------------------------------------------------------------------
# result type (linalg.py:17-26)
# ---------------------------------------------------------------------------
class SvdResult:
    """Truncated SVD factors ``M ~ U @ diag(S) @ V.conj().T``.

    ``U`` may live on the device (``U_device``, a column-major n x r table);
    the host array is materialised on first access, as the reference returns
    numpy arrays (linalg.py:17-26).
    """

    def __init__(self, U, S, V, U_device: Optional[Tall] = None, shard: Optional[Shard] = None):
        self._U = U
        self.S = np.asarray(S)
        self.V = np.asarray(V)
        self.U_device = U_device
        self.shard = shard

    @property
    def U(self):
        if self._U is None:
            self._U = self.U_device.view().double().cpu().numpy().copy()
        return self._U

    @U.setter
    def U(self, value):
        self._U = value

    def reconstruct(self):
        return (self.U * self.S) @ self.V.conj().T


# ---------------------------------------------------------------------------
# upload helpers
# ---------------------------------------------------------------------------
def as_tall(M, device=None) -> Tall:
    """Host (numpy) or device (torch) 2-D matrix -> row-major device Tall.
    fp32 stays fp32 (it is upcast exactly inside the kernels); everything
    else becomes fp64, as the reference coerces to float64 (dmd.py:36)."""
    if isinstance(M, Tall):
        return M
    device = device or dv.default_device()
    if isinstance(M, torch.Tensor):
        t = M
        dtype = torch.float32 if t.dtype == torch.float32 else torch.float64
    else:
        a = np.asarray(M)
        if np.iscomplexobj(a):
            raise ValueError("complex snapshot matrices are not supported on the device path")
        dtype = torch.float32 if a.dtype == np.float32 else torch.float64
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32 if dtype == torch.float32 else np.float64))
    if t.ndim != 2:
        raise ValueError("matrix must be 2-D")
    n, k = int(t.shape[0]), int(t.shape[1])
    T = alloc_tall(n, k, dtype, "row", device=device)
    if T.ld > k:
        T.buf[:, k:].zero_()
    copy_rows_h2d(T, t)
    return T


class PendingUpload:
    """A host snapshot matrix being streamed into a row-major device Tall.

    The copy runs in ~512 MB row chunks on a copy stream (pinned host memory
    -> contiguous staging buffer, double-buffered), each chunk re-pitched into
    S on the compute stream; `run(on_chunk)` calls on_chunk(r0, rows) in
    compute-stream order as soon as a chunk has landed, so row-separable work
    (the first sketch stage) overlaps the rest of the transfer. Every chunk
    is also checked for non-finite entries (SnapshotMatrix validation,
    dmd.py:26-50): `run` raises ValueError once the upload completes."""

    def __init__(self, host: torch.Tensor, S: Tall, chunk_bytes: int = 512 << 20):
        self.host = host
        self.S = S
        self.k = int(host.shape[1])
        self.chunk = max(1, chunk_bytes // (self.k * host.element_size()))

    def run(self, on_chunk=None):
        S, k, host = self.S, self.k, self.host
        dev = S.buf.device
        comp = torch.cuda.current_stream(dev)
        copy = torch.cuda.Stream(device=dev)
        rows = S.n
        nst = min(self.chunk, rows)
        staging = [torch.empty(nst * k, dtype=S.dtype, device=dev) for _ in range(2)]
        # the staging blocks come from the compute stream's pool: they may be
        # blocks freed there while queued kernels still read them, so the copy
        # stream starts behind everything already queued on the compute stream
        copy.wait_stream(comp)
        freed = [None, None]
        ok = torch.ones((), dtype=torch.bool, device=dev)
        for i, r0 in enumerate(range(0, rows, self.chunk)):
            rr = min(self.chunk, rows - r0)
            b = i & 1
            with torch.cuda.stream(copy):
                if freed[b] is not None:
                    copy.wait_event(freed[b])
                staging[b][: rr * k].copy_(host[r0:r0 + rr].reshape(-1), non_blocking=True)
                landed = torch.cuda.Event()
                landed.record(copy)
            comp.wait_event(landed)
            dst = S.buf[r0:r0 + rr, :k]
            dst.copy_(staging[b][: rr * k].view(rr, k))
            ok &= torch.isfinite(dst).all()
            freed[b] = torch.cuda.Event()
            freed[b].record(comp)
            if on_chunk is not None:
                on_chunk(r0, rr)
        for st in staging:
            st.record_stream(comp)
        if not bool(ok.item()):
            raise ValueError("snapshot matrix contains non-finite entries")


def copy_rows_h2d(T: Tall, t: torch.Tensor, row0: int = 0):
    """Copy a (rows x k) host/device tensor into rows [row0, row0+rows) of a
    row-major Tall with a pitched 2-D copy (no staging buffer)."""
    import ctypes

    from . import _lib
    rows, k = int(t.shape[0]), int(t.shape[1])
    if t.dtype != T.dtype:
        t = t.to(T.dtype)
    t = t.contiguous()
    if not T.buf.is_cuda:   # host-resident Tall (CPU test harness only)
        T.buf[row0:row0 + rows, :k].copy_(t)
        return
    elt = t.element_size()
    dst = T.buf.data_ptr() + row0 * T.ld * elt
    kind = 4  # cudaMemcpyDefault (UVA)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if t.device.type == "cpu" and T.ld != k and rows * k * elt > (64 << 20):
        # A host->device DMA with a short row pitch is slow (one descriptor per
        # row); stream contiguous chunks through a staging buffer and re-pitch
        # them on the device instead.
        chunk = max(1, (512 << 20) // (k * elt))
        staging = torch.empty(min(chunk, rows) * k, dtype=T.dtype, device=T.buf.device)
        for r0 in range(0, rows, chunk):
            rr = min(chunk, rows - r0)
            staging[: rr * k].copy_(t[r0:r0 + rr].reshape(-1), non_blocking=True)
            T.buf[row0 + r0:row0 + r0 + rr, :k].copy_(staging[: rr * k].view(rr, k))
        return
    _lib.check(_lib.lib().fdmd_copy2d(ctypes.c_void_p(dst), T.ld * elt, ctypes.c_void_p(t.data_ptr()),
                                      k * elt, k * elt, rows, kind, stream), "copy2d")


# ---------------------------------------------------------------------------
# CholeskyQR2 / shifted CholeskyQR3 (replaces np.linalg.qr at linalg.py:82,85)
# ---------------------------------------------------------------------------
def _chol_upper(G: torch.Tensor):
    L, info = torch.linalg.cholesky_ex(G)
    if int(info.item()) != 0:
        return None
    return L.mH


def _cond_upper(R: torch.Tensor) -> float:
    """2-norm condition number of the triangular factor for the CholQR2 /
    shifted-CholQR3 switch. The Frobenius bound ||R||_F ||R^-1||_F >= cond_2
    (two reductions) decides when it is clearly below the limit; only
    otherwise are the singular values computed (svdvals, ~9 ms at l = 200)."""
    l = R.shape[0]
    eye = torch.eye(l, dtype=R.dtype, device=R.device)
    Rinv = torch.linalg.solve_triangular(R, eye, upper=True)
    bound = float((torch.linalg.matrix_norm(R) * torch.linalg.matrix_norm(Rinv)).item())
    if not bound <= CHOLQR2_COND_LIMIT:      # also catches inf/nan
        return float(torch.linalg.cond(R).item())
    return bound


def _apply_rinv(Y: Tall, R: torch.Tensor, shard: Optional[Shard]):
    """Y <- Y R^-1 in place (R upper triangular, l x l)."""
    l = R.shape[0]
    eye = torch.eye(l, dtype=torch.float64, device=R.device)
    Rinv = torch.linalg.solve_triangular(R, eye, upper=True)
    n_tot = Y.n                                               # algorithmic TRSM: n l^2
    dv.get_ops().tall_gemm(Y, Rinv, Y, alg_flops=float(n_tot) * l * l, upper=True)


def cholqr2_inplace(Y: Tall, shard: Optional[Shard] = None, stats: Optional[dict] = None) -> torch.Tensor:
    """Orthonormalise the columns of Y in place. Returns R (Y_in = Q R)."""
    R, fix = cholqr2_deferred(Y, shard, stats)
    if fix is not None:
        l = fix.shape[0]
        dv.get_ops().tall_gemm(Y, fix, Y, alg_flops=float(Y.n) * l * l, upper=True)
    return R


def cholqr2_deferred(Y: Tall, shard: Optional[Shard] = None, stats: Optional[dict] = None,
                     passes: int = 2, G: Optional[torch.Tensor] = None):
    """CholeskyQR2 without the final tall triangular apply: Y is left holding
    Q1 and the orthonormal factor is Q = Y @ fix (fix = R2^-1, upper
    triangular, ~I). Every consumer of Q in the fit is linear, so `fix` is
    folded into small matrices instead of a second n*l^2 pass. Returns
    (R, fix) with Y_in = Q R; fix is None when Y already holds Q.

    passes=1 stops after the first CholeskyQR: Q1 = Y R1^-1 spans range(Y)
    to O(u kappa(Y)) and has cond(Q1) = 1 + O(u kappa^2) (~1.003 at
    kappa = 5e6), which is all a power iteration needs (it only uses the
    span: the next step is Z = X^T Q1 -> qr(Z)); Q1 is not even formed
    (fix = R1^-1) unless the shifted variant ran. The last orthonormalisation
    before the projection keeps both passes."""
    ops = dv.get_ops()
    l = Y.k
    if G is None:   # (a streamed first stage hands in Y^T Y, already all-reduced)
        with stage("cholqr.gram"):
            G = allreduce(shard, ops.tall_gram(Y, Y, symmetric=True))
    with stage("cholqr.chol+cond"):
        R1 = _chol_upper(G)
        if R1 is None:
            if passes == 1:
                ef = _span_from_gram(G, stats)
                if ef is not None:
                    return ef
            return _householder_inplace(Y, shard, stats), None
        cond = _cond_upper(R1)
    if stats is not None:
        stats.setdefault("cond_R1", []).append(cond)
    if cond > CHOLQR2_COND_LIMIT:
        # shifted CholeskyQR3 (Fukaya et al. 2020): shift makes the first
        # factorisation succeed with kappa(Q1) ~ sqrt(1/u); two CholQR passes follow.
        u = np.finfo(np.float64).eps / 2
        nrm2 = float(torch.linalg.matrix_norm(G, ord=2).item())
        n_tot = Y.n if shard is None else shard.n_global
        s = 11.0 * (n_tot * l + l * (l + 1)) * u * nrm2
        R0 = _chol_upper(G + s * torch.eye(l, dtype=G.dtype, device=G.device))
        if R0 is None:
            return _householder_inplace(Y, shard, stats), None
        _apply_rinv(Y, R0, shard)
        G = allreduce(shard, ops.tall_gram(Y, Y, symmetric=True))
        R1b = _chol_upper(G)
        if R1b is None:      # Y now holds Y_in R0^-1: its Householder R times R0 is Y_in's
            return _householder_inplace(Y, shard, stats) @ R0, None
        _apply_rinv(Y, R1b, shard)
        R1 = R1b @ R0
        if stats is not None:
            stats["shifted_cholqr3"] = stats.get("shifted_cholqr3", 0) + 1
    elif passes == 1:
        # single pass, nothing applied to the tall buffer: Q1 = Y @ R1^-1 is
        # left implicit (fix = R1^-1); X^T Q1 = (X^T Y) R1^-1 has the same
        # O(u kappa(Y)) error as a product with an explicitly formed Q1
        eye = torch.eye(l, dtype=torch.float64, device=R1.device)
        return R1, torch.linalg.solve_triangular(R1, eye, upper=True)
    else:
        _apply_rinv(Y, R1, shard)
    if passes == 1:
        return R1, None
    with stage("cholqr.gram2"):
        G2 = allreduce(shard, ops.tall_gram(Y, Y, symmetric=True))
    R2 = _chol_upper(G2)
    if R2 is None:
        raise ConvergenceError("CholeskyQR2: second Gram not positive definite")
    eye = torch.eye(l, dtype=torch.float64, device=R2.device)
    return R2 @ R1, torch.linalg.solve_triangular(R2, eye, upper=True)


# eigenvalues of a sketch Gram below this fraction of the largest are rounding
# noise of the Gram itself (u l w_max): those directions carry no information
SPAN_EIG_CUT = 1e-12


def _span_from_gram(G: torch.Tensor, stats: Optional[dict]):
    """Span-only orthonormalisation of a numerically rank-deficient sketch Y
    from its Gram G = Y^T Y = V diag(w) V^T: Q = Y fix, fix = [V_k w_k^-1/2 | 0]
    over the k eigen-directions above SPAN_EIG_CUT, nothing applied to the
    tall buffer. A power iteration only uses span(Q) (the next step is
    qr(X^T Q), whose Householder QR completes the zero columns), so the
    O(u cond^2) orthogonality of a one-pass factor is enough — and an exactly
    rank-deficient snapshot matrix (the noise-free controlled system of config
    2, rank 158 sketched at l = 168) no longer pays a Householder QR of the
    tall buffer (360 ms at n = 6.3 M) per sketch. The last orthonormalisation
    keeps CholeskyQR2 / shifted CholeskyQR3 / Householder.
    Returns (R, fix) with Y ~ (Y fix) R on the kept span (R is singular: the
    Gram route's Z = G_X M R^-1 shortcut is skipped for it), or None."""
    l = G.shape[0]
    w, V = torch.linalg.eigh(0.5 * (G + G.t()))
    wh = w.cpu()
    if not bool(torch.isfinite(wh).all()) or float(wh[-1]) <= 0.0:
        return None
    keep = wh > SPAN_EIG_CUT * float(wh[-1])
    k = int(keep.sum())
    if k == 0:
        return None
    idx = torch.arange(l - 1, l - 1 - k, -1, device=G.device)      # kept directions, largest first
    sq = torch.sqrt(w[idx])
    fix = torch.zeros((l, l), dtype=torch.float64, device=G.device)
    fix[:, :k] = V[:, idx] / sq[None, :]
    R = torch.zeros((l, l), dtype=torch.float64, device=G.device)
    R[:k] = sq[:, None] * V[:, idx].t()
    if stats is not None:
        stats["eigh_span_fallback"] = stats.get("eigh_span_fallback", 0) + 1
        stats.setdefault("span_rank", []).append(k)
    return R, fix


def _householder_inplace(Y: Tall, shard: Optional[Shard], stats: Optional[dict]) -> torch.Tensor:
    """Numerically rank-deficient sketch: Householder QR on the device
    (cuSOLVER geqrf/orgqr), matching the reference's np.linalg.qr."""
    if stats is not None:
        stats["householder_fallback"] = stats.get("householder_fallback", 0) + 1
    if shard is not None and shard.world > 1:
        return _tsqr_inplace(Y, shard)
    Q, R = torch.linalg.qr(Y.view().to(torch.float64), mode="reduced")
    Y.view().copy_(Q.to(Y.dtype))
    return R


def _tsqr_inplace(Y: Tall, shard: Shard) -> torch.Tensor:
    """Householder TSQR over the row shards (one level: every rank factors its
    block, the stacked l x l R factors are all-gathered and factored again).
    Every rank factors the same gathered stack in rank order, so the small R
    and the combine blocks are identical on all ranks; each rank then applies
    its own l x l block to its local Q. Returns R (Y_in = Q R)."""
    l = Y.k
    dev = Y.buf.device
    Yl = Y.view().to(torch.float64)
    if Y.n >= l:
        Ql, Rl = torch.linalg.qr(Yl, mode="reduced")                       # n_loc x l, l x l
    else:   # a shard shorter than the sketch width: pad its R with zero rows
        Ql, Rs = torch.linalg.qr(Yl, mode="complete")                      # n_loc x n_loc, n_loc x l
        Rl = torch.zeros((l, l), dtype=torch.float64, device=dev)
        Rl[: Rs.shape[0]] = Rs
        Ql = torch.cat([Ql, torch.zeros((Y.n, l - Y.n), dtype=torch.float64, device=dev)], dim=1)
    stack = torch.cat(shard.all_gather(Rl.contiguous()), dim=0)          # (world l) x l, rank order
    Q2, R = torch.linalg.qr(stack, mode="reduced")
    blk = Q2[shard_rank(shard) * l:(shard_rank(shard) + 1) * l]            # this rank's l x l combine block
    Y.view().copy_((Ql @ blk).to(Y.dtype))
    return R


def shard_rank(shard: Shard) -> int:
    import torch.distributed as dist
    return dist.get_rank(shard.group)


# ---------------------------------------------------------------------------
# randomized SVD core (linalg.py:62-90) over the first T columns of S
# ---------------------------------------------------------------------------
def draw_omega(cols: int, l: int, seed) -> np.ndarray:
    """Exactly linalg.py:80-81: the host-drawn float64 Gaussian test matrix."""
    return np.random.default_rng(seed).standard_normal((cols, l))


@dataclass
class SketchFactors:
    Q: Tall            # n x l fp64 buffer; the orthonormal basis is Q @ fix
    Ub: torch.Tensor   # l x l
    s: torch.Tensor    # l
    Vh: torch.Tensor   # l x T
    QtS: torch.Tensor  # l x m (Q^T S: both Q^T X and Q^T X'), fix already applied
    stats: dict
    fix: Optional[torch.Tensor] = None   # l x l upper triangular (None = identity)
    # implicit: no sketch buffer — Q is S @ fix with fix the m x l map
    # [W R1^-1; 0] (projection from the snapshot Gram); Q above is S itself
    implicit: bool = False

    def right(self, M: torch.Tensor) -> torch.Tensor:
        """Small matrix to multiply the stored buffer by to get (Q @ M)."""
        return M if self.fix is None else self.fix @ M


def _pad_rows(Bsmall: torch.Tensor, rows: int) -> torch.Tensor:
    if Bsmall.shape[0] == rows:
        return Bsmall.contiguous()
    out = torch.zeros((rows, Bsmall.shape[1]), dtype=torch.float64, device=Bsmall.device)
    out[: Bsmall.shape[0]] = Bsmall
    return out


def _rows(T: Tall, r0: int, rr: int) -> Tall:
    return Tall(T.buf[r0:r0 + rr], "row", rr, T.k)


# Snapshot-Gram route. X^T X costs n T^2 flops and T^2
# doubles; it replaces the sketch Y = X Omega, every power pass Z = X^T Q and
# the first CholeskyQR pass of each orthonormalisation (~2nTl(1+q) + nl^2(1+q)),
# so it is taken only when it is the cheaper side and its T x T block is small
# (a long series, T >> l, or a wide matrix keeps the explicit path).
GRAM_ROUTE_MAX_BYTES = 2 << 30


def gram_route_ok(T: int, l: int, q: int) -> bool:
    if q < 1 or 8.0 * T * T > GRAM_ROUTE_MAX_BYTES:
        return False
    return float(T) * T <= 2.0 * T * l * (1 + q) + float(l) * l * (1 + q)


def _inv_upper(R: torch.Tensor) -> torch.Tensor:
    eye = torch.eye(R.shape[0], dtype=torch.float64, device=R.device)
    return torch.linalg.solve_triangular(R, eye, upper=True)


def _gram_factor(GX: torch.Tensor, M: torch.Tensor):
    """R = chol(M^T (X^T X) M): the CholeskyQR factor of the tall X M taken
    from the snapshot Gram, and its condition bound; (None, cond) when X M is
    too ill-conditioned for CholeskyQR (the explicit path and its shifted /
    Householder fallbacks then run on the tall buffer)."""
    G = M.t() @ GX @ M
    R = _chol_upper(0.5 * (G + G.t()))
    if R is None:
        return None, float("inf")
    cond = _cond_upper(R)
    if not cond <= CHOLQR2_COND_LIMIT:
        return None, cond
    return R, cond


# Projection from the snapshot Gram: with Q1 = X W R1^-1 and
# R1 = chol(W^T G_X W), B = Q1^T S = (W R1^-1)^T (X^T S) follows from the
# m x m Gram S^T S — no Q1 buffer, no second CholeskyQR pass, no direct Q^T S.
# The price is accuracy: B's error grows from O(u ||S||) to O(u ||S|| cond(R1)),
# and the rank-r subspace moves by that over the singular-value gap at r. The
# route is taken only when the a-priori bound u cond(R1) sigma_1 / (sigma_r -
# sigma_{r+1}) is below PROJ_GRAM_TOL (sigma from R1; sigma_{r+1} = 0 when
# r = T, the whole row space). Measured against the reference (CPU probe,
# configs 0/1/3 recipes): bound 1.6e-8 (config 3, r = T) -> sigma 2e-9,
# lambda 4e-9; configs 0 / 1 (r inside the noise cluster) give bounds
# 8e-7 .. 1e-5 and keep the direct route.
PROJ_GRAM_TOL = float(os.environ.get("FDMD_PROJ_GRAM_TOL", "1e-7"))
_PROJ_GRAM = os.environ.get("FDMD_PROJ_GRAM", "1") != "0"


def _proj_gram_bound(R1: torch.Tensor, r: int, T: int) -> float:
    """u cond(R1) sigma_1 / (sigma_r - sigma_{r+1}) with sigma = sv(R1) =
    sv(X W) (exact 2-norm values: the Frobenius bound used for the CholeskyQR
    switch overestimates cond by up to ~l)."""
    u = np.finfo(np.float64).eps / 2
    l = R1.shape[0]
    if l <= r and r < T:
        return float("inf")               # no estimate of the gap at r
    sv = np.linalg.svd(R1.cpu().numpy(), compute_uv=False)
    if not (sv[-1] > 0 and np.all(np.isfinite(sv))):
        return float("inf")
    nxt = float(sv[r]) if r < l else 0.0  # r = l = T: the whole row space, sigma_{r+1} = 0
    gap = float(sv[r - 1]) - nxt
    return u * float(sv[0] / sv[-1]) * float(sv[0]) / gap if gap > 0 else float("inf")


def _cholqr_second_pass(Q: Tall, shard: Optional[Shard], stats: dict):
    """CholeskyQR2's second pass over a buffer that already holds Q1 (its
    first pass came from the snapshot Gram): R2 = chol(Q1^T Q1) and
    fix = R2^-1, never applied to the tall buffer. Falls back to the full
    CholeskyQR2 / shifted CholeskyQR3 / Householder chain on the buffer."""
    ops = dv.get_ops()
    with stage("cholqr.gram2"):
        G2 = allreduce(shard, ops.tall_gram(Q, Q, symmetric=True))
    R2 = _chol_upper(G2)
    if R2 is None:
        stats["gram_first_pass_fallback"] = stats.get("gram_first_pass_fallback", 0) + 1
        return cholqr2_deferred(Q, shard, stats, passes=2, G=G2)
    return R2, _inv_upper(R2)


def _place_rows(Bsmall: torch.Tensor, rows: int, r0: int) -> torch.Tensor:
    """Bsmall placed at rows [r0, r0 + K) of a zero rows x N matrix (the small
    operand of S @ [0; B; 0] for a column window of S)."""
    if r0 == 0:
        return _pad_rows(Bsmall, rows)
    out = torch.zeros((rows, Bsmall.shape[1]), dtype=torch.float64, device=Bsmall.device)
    out[r0:r0 + Bsmall.shape[0]] = Bsmall
    return out


def sketch_factors(S: Tall, T: int, l: int, q: int, omega: np.ndarray, shard: Optional[Shard] = None,
                   Q: Optional[Tall] = None, pending: Optional[PendingUpload] = None,
                   pre_svd=None, c0: int = 0, r: Optional[int] = None) -> SketchFactors:
    """Range finder + power passes + projection for X = S[:, c0:c0+T]
    (linalg.py:62-90 with Householder QR replaced by CholeskyQR2).

    Kernel sequence, snapshot-Gram route (q >= 1):
      G_X = X^T X (one symmetric tall Gram; streamed: accumulated chunk by
      chunk under the host->device transfer) -> R0 = chol(Omega^T G_X Omega)
      -> q x {Z = G_X M R^-1 -> W = qr(Z); R1 = chol(W^T G_X W)} (non-final
      stages never touch the tall data) -> Q1 = S [W R1^-1; 0] (the only tall
      GEMM) -> R2 = chol(Q1^T Q1) (CholeskyQR2's second pass; fix = R2^-1 is
      folded into every consumer) -> Q^T S -> svd(Q^T X) on the device.
    Explicit route (q = 0, T >> l, or an ill-conditioned factor): Y = S[Omega;0]
    -> CholQR -> q x {Z = S^T Q -> W = qr(Z) -> Y = S[W;0] -> CholQR} -> Q^T S.

    With `pending` (S still streaming in from the host) the row-separable
    first stage (G_X, or Y / Y^T Y / X^T Y on the explicit route) runs chunk by
    chunk as rows land, in the shadow of the transfer.
    The returned QtS is Q^T S over all m columns of S.

    `r` (the rank the caller truncates to) enables the projection from the
    snapshot Gram (PROJ_GRAM_TOL): the Gram is then taken over all m columns
    (S^T S), B = (W R1^-1)^T (X^T S) comes from it, and no n x l buffer is
    ever written (the result has implicit=True: Q = S @ fix).
    """
    if pending is not None and c0 != 0:
        raise ValueError("a streamed upload sketches the leading columns only")
    ops = dv.get_ops()
    dev = S.buf.device
    m = S.k
    stats: dict = {}
    Qbox = [Q]

    def _Q() -> Tall:
        # the n x l sketch buffer, allocated only when a route writes it
        if Qbox[0] is None:
            with stage("sketch.alloc_Q"):
                # slack rows: once Q is released, the two fp32 tables that follow it
                # (basis U, n x r, and the raw modes, n x (r + #real modes)) fit in
                # its block — together Q's size plus a few fp32 columns
                slack = (16 * S.n + (64 << 20)) // (8 * max(l, 1)) + 1
                Qb = alloc_tall(S.n + slack, l, torch.float64, "row", device=dev)
                Qbox[0] = Tall(Qb.buf, "row", S.n, l)
        return Qbox[0]

    Om = torch.as_tensor(np.asarray(omega, dtype=np.float64), device=dev)
    Omp = _place_rows(Om, m, c0)
    nl = float(S.n)
    Tc = c0 + T
    use_gram = gram_route_ok(T, l, q)
    # the projection route needs X^T S = [X^T X | X^T s_m] for a snapshot matrix
    # (m = T + 1): the bordered symmetric Gram (fdmd_tall_gram_bordered: the border
    # rides in the panel kernel's diagonal warp tiles; a plain 201 x 201 panel
    # plan would pad to 240 and cost 3 partitions)
    full = use_gram and r is not None and c0 == 0 and m - T in (0, 1)
    border = full and m == T + 1
    GX = XtS = bd = G0 = Zp = None
    if pending is not None and use_gram:
        # bordered: [X^T X | X^T s_m] accumulates in one T x (T + 1) block, one
        # kernel per chunk (the border rides in the symmetric panel Gram)
        GXb = torch.zeros((T, T + 1 if border else T), dtype=torch.float64, device=dev)

        def gram_stage(r0, rr):
            Sc = _rows(S, r0, rr)
            if border:
                ops.tall_gram_bordered(Sc, T, out=GXb, beta=1.0, alg_flops=1.0 * rr * T * T + 2.0 * rr * T)
            else:
                ops.tall_gram(Sc, Sc, K1=T, K2=T, symmetric=True, out=GXb, beta=1.0, alg_flops=1.0 * rr * T * T)

        with stage("sketch.stream_upload+XtX"):
            pending.run(gram_stage)
        GXb = allreduce(shard, GXb)
        GX = GXb[:, :T].contiguous()
        bd = GXb[:, T].contiguous() if border else None
    elif pending is not None:
        G0 = torch.zeros((l, l), dtype=torch.float64, device=dev)
        Zp = torch.zeros((T, l), dtype=torch.float64, device=dev) if q > 0 else None

        def first_stage(r0, rr):
            Sc, Yc = _rows(S, r0, rr), _rows(_Q(), r0, rr)
            ops.tall_gemm(Sc, Omp, Yc, alg_flops=2.0 * rr * T * l)
            ops.tall_gram(Yc, Yc, symmetric=True, out=G0, beta=1.0)
            if Zp is not None:
                ops.tall_gram(Sc, Yc, K1=T, out=Zp, beta=1.0, alg_flops=2.0 * rr * T * l)

        with stage("sketch.stream_upload+Y+G+XtY"):
            pending.run(first_stage)
        G0 = allreduce(shard, G0)
        if Zp is not None:
            Zp = allreduce(shard, Zp)
    elif use_gram and border:
        with stage("power.XtX+Xts_m"):
            # [X^T X | X^T s_m] in one pass (c0 = 0 on this route)
            GXb = allreduce(shard, ops.tall_gram_bordered(S, T, alg_flops=1.0 * nl * T * T + 2.0 * nl * T))
            GX = GXb[:, :T].contiguous()
            bd = GXb[:, T].contiguous()
    elif use_gram:
        with stage("power.XtX"):
            GX = allreduce(shard, ops.tall_gram(S, S, K1=Tc, K2=Tc, symmetric=True,
                                                alg_flops=1.0 * nl * T * T))   # (c0+T)^2
            if c0:
                GX = GX[c0:, c0:].contiguous()                               # T x T block of X
    implicit = False
    if GX is not None:
        # the sketch enters the algorithm only through Z = X^T Q1, Q1 = X Omega R0^-1,
        # R0 = chol((X Omega)^T (X Omega)): all of it follows from G_X, so Y = X Omega
        # and its Gram are never formed (counted as the terms they replace)
        with stage("sketch.implicit"):
            R0, _ = _gram_factor(GX, Om)
        if R0 is not None:
            implicit = True
            R, fix = R0, None
            stats["implicit_sketch"] = 1
    if not implicit:
        if G0 is None:
            with stage("sketch.Y=XOmega"):
                ops.tall_gemm(S, Omp, _Q(), alg_flops=2 * nl * T * l)
        with stage("sketch.cholqr2"):
            # power iterations only need the span: one CholeskyQR pass unless this
            # is the last orthonormalisation (q = 0)
            R, fix = cholqr2_deferred(_Q(), shard, stats, passes=2 if q == 0 else 1, G=G0)
    M = Om
    for it in range(q):
        final = it == q - 1
        with stage("power.Z=XtQ"):
            Z = None
            if it == 0 and Zp is not None and fix is not None:
                Z = Zp @ fix            # streamed X^T Y, buffer untouched (R1^-1 folded)
            elif GX is not None:
                # Q = X M R^-1 whatever CholeskyQR variant ran, so Z = X^T Q =
                # G_X M R^-1; needs an invertible R (a rank-deficient sketch takes
                # the Householder fallback, whose R may be singular: direct pass then)
                dR = torch.diagonal(R).abs()
                if float(dR.min()) > 1e-10 * float(dR.max()):
                    Z = GX @ (M @ _inv_upper(R))                          # T x l = X^T Q
            if Z is None:
                Z = allreduce(shard, ops.tall_gram(S, _Q(), K1=Tc, alg_flops=2 * nl * T * l))[c0:]   # X^T Q
                if fix is not None:
                    Z = Z @ fix
        with stage("power.qr(Z)"):
            W, _ = torch.linalg.qr(Z[:T], mode="reduced")    # T x l (Householder, device)
        M = W
        R1 = None
        if GX is not None:
            with stage("power.chol(WtGW)"):
                R1, _ = _gram_factor(GX, W)
        if R1 is not None and not final:
            # a non-final power stage is span-only: Q = X W R1^-1 stays implicit and
            # the next Z = G_X W R1^-1 needs no tall pass
            R, fix = R1, None
            stats["gram_power_stages"] = stats.get("gram_power_stages", 0) + 1
            continue
        if R1 is not None and full and _PROJ_GRAM:
            with stage("power.proj_bound"):
                bound = _proj_gram_bound(R1, r, T)
            stats["proj_gram_bound"] = bound
            if bound <= PROJ_GRAM_TOL:
                # B = Q1^T S = (W R1^-1)^T (X^T S) from the snapshot Gram: Q stays
                # implicit (Q = S [W R1^-1; 0]); no tall pass at all
                with stage("project.QtS_from_gram"):
                    M1 = W @ _inv_upper(R1)
                    XtS = GX if bd is None else torch.cat([GX, bd[:, None]], dim=1)   # T x m
                    QtS = M1.t() @ XtS                                       # l x m
                stats["gram_projection"] = 1
                return _svd_tail(S, QtS, c0, T, None, stats, _place_rows(M1, m, 0), implicit=True)
        if R1 is not None:
            # CholeskyQR2 with its first pass from the snapshot Gram: the tall GEMM
            # writes Q1 = X (W R1^-1) directly (no Y^T Y Gram, no triangular apply)
            with stage("power.Y=XWR1^-1"):
                ops.tall_gemm(S, _place_rows(W @ _inv_upper(R1), m, c0), _Q(), alg_flops=2 * nl * T * l)
            with stage("power.cholqr2"):
                R2, fix = _cholqr_second_pass(_Q(), shard, stats)
            R = R2 @ R1
            stats["gram_first_pass"] = 1
        else:
            with stage("power.Y=XW"):
                ops.tall_gemm(S, _place_rows(W, m, c0), _Q(), alg_flops=2 * nl * T * l)
            with stage("power.cholqr2"):
                R, fix = cholqr2_deferred(_Q(), shard, stats, passes=2 if final else 1)
    Q = _Q()
    with stage("project.QtS"):
        QtS = allreduce(shard, ops.tall_gram(Q, S, alg_flops=2 * nl * m * l))     # l x m
        if fix is not None:
            QtS = fix.t() @ QtS
    return _svd_tail(Q, QtS, c0, T, pre_svd, stats, fix)


def _svd_tail(Q: Tall, QtS: torch.Tensor, c0: int, T: int, pre_svd, stats: dict, fix,
              implicit: bool = False) -> SketchFactors:
    """svd(B), B = Q^T X (the leading block of Q^T S), on the device — on a side
    stream under the caller's Q-only tall work (`pre_svd`) when given."""
    pre = None
    with stage("small.svd(B)"):
        B = QtS[:, c0:c0 + T]
        if pre_svd is not None and B.is_cuda:
            # tall work that needs only Q (the caller's fp16 split of it) runs on
            # the main stream while the small SVD runs on a side stream
            main = torch.cuda.current_stream(B.device)
            ready = torch.cuda.Event()
            ready.record(main)
            pre = pre_svd(Q, fix)
            side = _svd_stream(B.device)
            side.wait_event(ready)
            with torch.cuda.stream(side):
                Ub, s, Vh = _svd_small(B)
            main.wait_stream(side)
            for t in (B, Ub, s, Vh):
                t.record_stream(side)
        else:
            Ub, s, Vh = _svd_small(B)
    f = SketchFactors(Q, Ub, s, Vh, QtS, stats, fix, implicit)
    f.pre = pre
    return f


def _svd_small(B: torch.Tensor):
    """np.linalg.svd(B, full_matrices=False) of linalg.py:87 on the device:
    cuSOLVER gesvdp through libfdmd (5.8 ms at 200 x 200 against 13-15 ms for the
    one-sided Jacobi gesvdj, profiles/r02_svd_probe.txt); gesvdj when gesvdp
    reports a failure, for wide-over-tall blocks and for the CPU test harness."""
    ops = dv.get_ops()
    if B.is_cuda and B.shape[0] <= B.shape[1] and hasattr(ops, "svd_small") and _SVD_GESVDP:
        Ub, s, Vh, info = ops.svd_small(B)
        if int(info.item()) == 0 and bool(torch.isfinite(s).all()):
            return Ub, s, Vh
    return torch.linalg.svd(B, full_matrices=False, driver="gesvdj" if B.is_cuda else None)


_SVD_GESVDP = os.environ.get("FDMD_SVD", "gesvdp") != "gesvdj"
_SVD_STREAMS = {}


def _svd_stream(dev) -> torch.cuda.Stream:
    key = str(dev)
    if key not in _SVD_STREAMS:
        # high priority: its latency-bound small kernels take SMs ahead of the
        # bulk split kernel queued on the main stream
        _SVD_STREAMS[key] = torch.cuda.Stream(device=dev, priority=-1)
    return _SVD_STREAMS[key]


def _canonical_signs(Q: Tall, Ub_r: torch.Tensor, shard: Optional[Shard]) -> torch.Tensor:
    """Sign of U = Q Ub_r at each column's first largest-|.| entry
    (linalg.py:29-44 for real U), found by a statistics-only DMMA pass."""
    ops = dv.get_ops()
    r = Ub_r.shape[1]
    Bp = torch.zeros((Ub_r.shape[0], 2 * r), dtype=torch.float64, device=Ub_r.device)
    Bp[:, 0::2] = Ub_r
    row0 = 0 if shard is None else shard.row0
    st = ops.tall_gemm(Q, Bp, None, stats=True, row_offset=row0)   # (r, 3)
    st = _reduce_pair_stats(st, shard)
    if not bool(torch.isfinite(st[:, :2]).all()):
        raise ConvergenceError("randomized SVD: non-finite basis (degenerate sketch)")
    idx = st[:, 2].round().long()
    local = idx - row0
    if shard is not None and shard.world > 1:
        own = (local >= 0) & (local < Q.n)
        rows = torch.zeros((r, Q.k), dtype=torch.float64, device=Ub_r.device)
        rows[own] = Q.view()[local[own]].to(torch.float64)
        rows = shard.allreduce(rows)
    else:
        rows = Q.view()[local].to(torch.float64)
    piv = (rows * Ub_r.t()).sum(dim=1)
    return torch.where(piv < 0, -1.0, 1.0).to(torch.float64)


def _reduce_pair_stats(st: torch.Tensor, shard: Optional[Shard]) -> torch.Tensor:
    """Combine per-rank [sumsq, max, argmax] (argmax ties -> lowest global row)."""
    if shard is None or shard.world <= 1:
        return st
    gathered = shard.all_gather(st)
    out = gathered[0].clone()
    out[:, 0] = 0.0
    for g in gathered:                                       # fixed rank order
        out[:, 0] += g[:, 0]
    best = gathered[0][:, 1].clone()
    bidx = gathered[0][:, 2].clone()
    for g in gathered[1:]:
        better = (g[:, 1] > best) | ((g[:, 1] == best) & (g[:, 2] < bidx))
        best = torch.where(better, g[:, 1], best)
        bidx = torch.where(better, g[:, 2], bidx)
    out[:, 1], out[:, 2] = best, bidx
    return out


def _validate_rank(rows, cols, r, l=None):
    if not 1 <= r <= min(rows, cols):
        raise ValueError(f"rank {r} out of range [1, {min(rows, cols)}]")
    if l is not None and l > min(rows, cols):
        raise ValueError(f"rank + oversample = {l} exceeds min dimension {min(rows, cols)}")


def randomized_svd(M, r, oversample=10, power_iters=2, seed=None, *, omega=None,
                   shard: Optional[Shard] = None, keep_device=False) -> SvdResult:
    """Sketched SVD (linalg.py:62-90): same Omega (default_rng(seed)), same
    power count, same canonicalisation; CholeskyQR2 replaces Householder QR."""
    A = as_tall(M)
    n_tot = A.n if shard is None else shard.n_global
    rows, cols = n_tot, A.k
    l = r + oversample
    _validate_rank(rows, cols, r, l)
    G = draw_omega(cols, l, seed) if omega is None else np.asarray(omega, dtype=np.float64)
    f = sketch_factors(A, cols, l, power_iters, G, shard, r=r)
    Ub_r = f.Ub[:, :r].contiguous()
    sgn = _canonical_signs(f.Q, f.right(Ub_r), shard)
    Ub_r = Ub_r * sgn[None, :]
    V = (f.Vh[:r].t() * sgn[None, :]).contiguous()
    U = alloc_tall(A.n, r, torch.float64, "col", device=A.buf.device)
    dv.get_ops().tall_gemm(f.Q, f.right(Ub_r), U)            # lift U = Q Ub_r (linalg.py:88)
    res = SvdResult(None, f.s[:r].cpu().numpy().copy(), V.cpu().numpy(), U_device=U, shard=shard)
    if not keep_device:
        _ = res.U
    return res


def truncated_svd(M, r, *, shard: Optional[Shard] = None, keep_device=False) -> SvdResult:
    """Dense truncated SVD (linalg.py:47-59) of a tall matrix on the device:
    Householder QR (cuSOLVER; TSQR across row shards) then the SVD of the
    small R factor; signs canonicalised as linalg.py:29-44."""
    A = as_tall(M)
    sharded = shard is not None and shard.world > 1
    rows, cols = (shard.n_global if sharded else A.n), A.k
    if not 1 <= r <= min(rows, cols):
        raise ValueError(f"rank {r} out of range [1, {min(rows, cols)}]")
    if sharded:
        if rows < cols:
            raise ValueError("svd_mode='full' on row-sharded data needs at least as many rows as columns")
        Y = alloc_tall(A.n, cols, torch.float64, "row", device=A.buf.device)
        Y.view().copy_(A.view())
        Rf = _tsqr_inplace(Y, shard)
        Ur, s, Vh = torch.linalg.svd(Rf, full_matrices=False, driver="gesvdj" if Rf.is_cuda else None)
        Ufull = Y.view() @ Ur
        del Y
    else:
        X = A.view().to(torch.float64)
        if rows >= cols:
            Qf, Rf = torch.linalg.qr(X, mode="reduced")
            Ur, s, Vh = torch.linalg.svd(Rf, full_matrices=False, driver="gesvdj" if Rf.is_cuda else None)
            Ufull = Qf @ Ur
        else:
            Ufull, s, Vh = torch.linalg.svd(X, full_matrices=False, driver="gesvd" if X.is_cuda else None)
    U = Ufull[:, :r]
    V = Vh[:r].t()
    ar = torch.arange(r, device=U.device)
    if sharded:
        # first largest |U| entry per column over all shards (ties -> lowest global row)
        mx, idx = U.abs().max(dim=0)
        st = torch.stack([torch.zeros_like(mx), mx, (idx + shard.row0).to(torch.float64)], dim=1)
        st = _reduce_pair_stats(st, shard)
        local = st[:, 2].round().long() - shard.row0
        own = (local >= 0) & (local < A.n)
        vals = U[local.clamp(0, max(A.n - 1, 0)), ar]
        piv = shard.allreduce(torch.where(own, vals, torch.zeros_like(vals)).contiguous())
    else:
        idx = torch.argmax(U.abs(), dim=0)
        piv = U[idx, ar]
    sgn = torch.where(piv < 0, -1.0, 1.0).to(torch.float64)
    U = U * sgn[None, :]
    V = V * sgn[None, :]
    Ut = alloc_tall(A.n, r, torch.float64, "col", device=A.buf.device)
    Ut.view().copy_(U)
    res = SvdResult(None, s[:r].cpu().numpy().copy(), V.cpu().numpy(), U_device=Ut, shard=shard)
    if not keep_device:
        _ = res.U
    return res


# ---------------------------------------------------------------------------
# small dense helpers (linalg.py:93-141)
# ---------------------------------------------------------------------------
def pinv(M, rel_tol=1e-12):
    """SVD pseudo-inverse (linalg.py:93-104) of a small matrix, on the device."""
    if not 0 < rel_tol < 1:
        raise ValueError(f"rel_tol must lie in (0, 1), got {rel_tol}")
    A = np.asarray(M)
    dev = dv.default_device()
    t = torch.as_tensor(A, device=dev)
    U, s, Vh = torch.linalg.svd(t, full_matrices=False)
    if s.numel() == 0 or float(s[0]) == 0.0:
        return np.zeros((A.shape[1], A.shape[0]), dtype=A.dtype)
    keep = s > rel_tol * s[0]
    inv = torch.where(keep, 1.0 / torch.where(keep, s, torch.ones_like(s)), torch.zeros_like(s))
    return ((Vh.mH * inv.to(Vh.dtype)) @ U.mH).cpu().numpy()


def eig_small(M, max_dim=2000):
    """Eigendecomposition with residual check (linalg.py:107-133); real
    input runs cuSOLVER Xgeev on the device."""
    A = np.asarray(M)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError(f"matrix must be square, got {A.shape}")
    if A.shape[0] > max_dim:
        raise ValueError(f"dense eig limited to {max_dim}, got {A.shape[0]}")
    dev = dv.default_device()
    if np.iscomplexobj(A):
        raise ValueError("eig_small on the device path takes real matrices (the DMD operator is real)")
    w, V = dv.get_ops().geev(torch.as_tensor(A, dtype=torch.float64, device=dev))
    return _check_eig(A, w, V)


def _check_eig(A, w, V):
    norms = np.linalg.norm(V, axis=0)
    norms[norms == 0.0] = 1.0
    V = V / norms
    scale = np.linalg.norm(A)
    resid = np.linalg.norm(A @ V - V * w)
    if scale > 0 and resid > 1e-8 * scale:
        raise ConvergenceError(f"eigendecomposition residual {resid:.3e} exceeds 1e-8 * ||M||",
                               residual=resid)
    return w, V


# CholeskyQR2 is used for the small tall factors (T x r Vandermonde of the
# variable projection) while cond(A) stays below this bound: u cond^2 <= 1e-4,
# so the second pass restores orthogonality to O(u)
SMALL_CHOLQR_COND = 1e6


def thin_qr_fullrank(A: torch.Tensor):
    """(Q, R^-1) of a numerically full-column-rank tall A (M >= N) = Q R, or
    None when A is too close to rank deficient for the unique least-squares
    solution to equal gelsd's minimum-norm one (the caller then takes the SVD).

    On the device a Householder QR of a 200 x 150 complex128 matrix is ~150
    latency-bound panel steps (10-15 ms; the LM loop of config 1 spent 42 ms
    per iteration in two of them). CholeskyQR2 — Gram, potrf, triangular
    inverse, twice — is a dozen small kernels; it runs while the Frobenius
    bound ||R||_F ||R^-1||_F >= cond_2(A) stays under SMALL_CHOLQR_COND,
    otherwise Householder QR decides."""
    M, N = int(A.shape[0]), int(A.shape[1])
    rcond = torch.finfo(torch.float64).eps * max(M, N)
    eye = torch.eye(N, dtype=A.dtype, device=A.device)
    G = A.mH @ A
    L, info = torch.linalg.cholesky_ex(0.5 * (G + G.mH))
    R1 = L.mH
    Ri1 = torch.linalg.solve_triangular(R1, eye, upper=True)
    bound = torch.linalg.matrix_norm(R1) * torch.linalg.matrix_norm(Ri1)
    chk = torch.stack([info.to(torch.float64), bound.real.to(torch.float64)]).cpu()
    if int(chk[0]) == 0 and float(chk[1]) <= SMALL_CHOLQR_COND:
        Q1 = A @ Ri1
        G2 = Q1.mH @ Q1
        L2, info2 = torch.linalg.cholesky_ex(0.5 * (G2 + G2.mH))
        if int(info2.item()) == 0:
            Ri2 = torch.linalg.solve_triangular(L2.mH, eye, upper=True)
            return Q1 @ Ri2, Ri1 @ Ri2
    Qa, Ra = torch.linalg.qr(A, mode="reduced")
    Ri = torch.linalg.solve_triangular(Ra, eye, upper=True)
    hb = float((torch.linalg.matrix_norm(Ra) * torch.linalg.matrix_norm(Ri)).item())
    if hb * rcond < 1e-3:
        return Qa, Ri
    return None


def lstsq_minnorm(A: torch.Tensor, B: torch.Tensor, qr_out: Optional[list] = None) -> torch.Tensor:
    """Minimum-norm least-squares solution of A X = B with numpy's default
    cut (np.linalg.lstsq(rcond=None) -> LAPACK gelsd: singular values at or
    below eps * max(M, N) * s_max are treated as zero), as linalg.py:136-141.
    CUDA `gels` is a plain QR that assumes full rank, so a rank-deficient A
    goes through its SVD on the device instead. `qr_out` (a list) receives the
    orthonormal factor Q of A when the QR path ran (the LM step reuses it)."""
    if A.shape[0] == 0 or A.shape[1] == 0:
        return torch.zeros((A.shape[1],) + tuple(B.shape[1:]), dtype=torch.result_type(A, B), device=A.device)
    M, N = int(A.shape[0]), int(A.shape[1])
    rcond = torch.finfo(torch.float64).eps * max(M, N)
    if M >= N:
        # fast path: when R of A = QR is provably well inside the cut
        # (||R||_F ||R^-1||_F >= cond_2(A)), A has full column rank numerically,
        # the least-squares solution is unique and equals the min-norm one
        fac = thin_qr_fullrank(A)
        if fac is not None:
            Qa, Ri = fac
            if qr_out is not None:
                qr_out.append(Qa)
            return Ri @ (Qa.mH @ B.to(Qa.dtype))
    U, s, Vh = torch.linalg.svd(A, full_matrices=False, driver="gesvdj" if A.is_cuda else None)
    keep = s > rcond * s[0]
    inv = torch.where(keep, 1.0 / torch.where(keep, s, torch.ones_like(s)), torch.zeros_like(s))
    UhB = U.mH @ B.to(U.dtype)
    if UhB.dim() == 1:
        return Vh.mH @ (inv.to(U.dtype) * UhB)
    return Vh.mH @ (inv.to(U.dtype)[:, None] * UhB)


def lstsq(A, B):
    """Minimum-norm least-squares solve (linalg.py:136-141) on the device."""
    dev = dv.default_device()
    At = torch.as_tensor(np.asarray(A), device=dev)
    Bt = torch.as_tensor(np.asarray(B), device=dev)
    if At.is_complex() or Bt.is_complex():
        ct = torch.complex128
        At, Bt = At.to(ct), Bt.to(ct)
    else:
        At, Bt = At.to(torch.float64), Bt.to(torch.float64)
    return lstsq_minnorm(At, Bt).cpu().numpy()
