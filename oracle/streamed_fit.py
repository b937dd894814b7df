"""Streamed FP64 oracle for the full-size BASELINE configs — TEST
INFRASTRUCTURE ONLY ("C3 restatement").

The reference keeps every n-row matrix in RAM as float64/complex128
(config 3: an 81 GB X, a 161 GB phi, an n x r pinv), so it cannot run at
n = 50.3 M. This module restates the same algorithm over row blocks of the
snapshot matrix S (n x m), in float64 on the host, never materialising an
n-row matrix: every tall quantity (the sketch Q, the POD basis U, the modes
phi) is carried as `S[:, window] @ small`, and each pass over S recomputes its
row block from the X block and the replicated small factors.

Restated functions (paths relative to /root/reference/pkg/src/flowdmd/):
  * randomized_svd            linalg.py:62-90  (range finder, q power passes,
                              B = Q^T M, svd(B), lift) with np.linalg.qr of the
                              tall sketch replaced by CholeskyQR2 (shifted
                              CholeskyQR3 when the sketch is ill-conditioned);
                              the small qr(M^T Q) stays Householder
  * _canonicalize             linalg.py:29-44  (first largest |U| entry positive)
  * exact_dmd                 dmd.py:240-274   (K^ = U^H X' V S^-1, eig, phi = X' V S^-1 W)
  * _order_and_pair           dmd.py:158-213   (order, unit norm, phase at the first
                              |max| entry, conjugate lock, real-ification)
  * optdmd                    dmd.py:366-436   (D = conj(V) S, varpro LM, symmetrize,
                              phi = U B^T)
  * ReducedModel.phi_pinv /   dmd.py:87-90, runtime.py:47-52 (z0 = pinv(phi) x0 with
    encode                    the SVD cut 1e-12, through a streamed Householder TSQR of S)
  * decode / step_k           runtime.py:66-124 (frames Re(phi lam^k z0) on row blocks)
  * residual diagnostic       dmd.py:269-272
The small r x r / T x r work reuses flowdmd_oracle (itself pinned against the
reference's goldens in tests/test_cpu_oracle_golden.py).

Pinning: tests/test_cpu_streamed_oracle.py checks this module against the
REAL reference's outputs on config 0 (full) and on a contiguous 98,304-row
block of config 1 (oracle/gen_golden_streamed.py, tests/golden/streamed_cases.npz).

The module never imports torch: the caller hands in `fetch(r0, r1)`
returning rows [r0, r1) of S as a float64 array (the GPU tests read the very
bytes the device fit consumed, so both sides see identical inputs).
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import flowdmd_oracle as orc  # noqa: E402

U_ROUND = np.finfo(np.float64).eps / 2


class Rows:
    """Row-block access to an n x m snapshot matrix S."""

    def __init__(self, n: int, m: int, fetch: Callable[[int, int], np.ndarray], block: int = 1 << 17):
        self.n, self.m, self.fetch, self.block = int(n), int(m), fetch, int(block)
        self.passes = 0

    @classmethod
    def from_array(cls, S, block: int = 1 << 17):
        S = np.asarray(S)
        return cls(S.shape[0], S.shape[1], lambda a, b: np.asarray(S[a:b], dtype=np.float64), block)

    def blocks(self):
        self.passes += 1
        for r0 in range(0, self.n, self.block):
            r1 = min(self.n, r0 + self.block)
            yield r0, self.fetch(r0, r1)


# --------------------------------------------------------------------------
# CholeskyQR2 of X M, carried as the small map M -> M R^-1
# --------------------------------------------------------------------------

def _gram_of(rows: Rows, c0: int, T: int, M: np.ndarray) -> np.ndarray:
    G = np.zeros((M.shape[1], M.shape[1]))
    for _, Sb in rows.blocks():
        Y = Sb[:, c0:c0 + T] @ M
        G += Y.T @ Y
    return G


def _chol_upper(G):
    try:
        return np.linalg.cholesky(0.5 * (G + G.T)).T
    except np.linalg.LinAlgError:
        return None


def cholqr2_map(rows: Rows, c0: int, T: int, M: np.ndarray) -> np.ndarray:
    """Returns M' with Q = X M' orthonormal (X = S[:, c0:c0+T]): two
    CholeskyQR passes, each a pass over S; shifted CholeskyQR3 (Fukaya et al.
    2020) when the first Gram is too ill-conditioned for Cholesky."""
    G = _gram_of(rows, c0, T, M)
    R1 = _chol_upper(G)
    if R1 is None or np.linalg.cond(R1) > 1e7:
        l = M.shape[1]
        s = 11.0 * (rows.n * l + l * (l + 1)) * U_ROUND * np.linalg.norm(G, 2)
        R0 = _chol_upper(G + s * np.eye(l))
        M = np.linalg.solve(R0.T, M.T).T                       # M R0^-1
        G = _gram_of(rows, c0, T, M)
        R1 = _chol_upper(G)
    M = np.linalg.solve(R1.T, M.T).T                           # M R1^-1
    G2 = _gram_of(rows, c0, T, M)
    R2 = _chol_upper(G2)
    return np.linalg.solve(R2.T, M.T).T                        # M R1^-1 R2^-1


# --------------------------------------------------------------------------
# randomized SVD (linalg.py:62-90)
# --------------------------------------------------------------------------

@dataclass
class StreamedSvd:
    Umap: np.ndarray      # T x r: U = X @ Umap
    S: np.ndarray         # r
    V: np.ndarray         # T x r
    QtS: np.ndarray       # l x m: Q^T S over all columns (Q = X M)
    Ub_r: np.ndarray      # l x r (canonical signs applied)
    M: np.ndarray         # T x l: Q = X M
    c0: int = 0


def randomized_svd(rows: Rows, T: int, r: int, p: int, q: int, seed, c0: int = 0) -> StreamedSvd:
    """linalg.py:62-90 over X = S[:, c0:c0+T] with oversample p (clamped to
    min dimension as dmd.py:219-221) and q power iterations."""
    l = r + min(p, min(rows.n, T) - r)
    Om = np.random.default_rng(seed).standard_normal((T, l))      # linalg.py:80-81
    M = cholqr2_map(rows, c0, T, Om)                              # Q = qr(X Omega)
    for _ in range(q):
        Z = np.zeros((T, l))
        for _, Sb in rows.blocks():
            Xb = Sb[:, c0:c0 + T]
            Z += Xb.T @ (Xb @ M)                                  # X^H Q
        W, _ = np.linalg.qr(Z)                                    # linalg.py:85
        M = cholqr2_map(rows, c0, T, W)                           # Q = qr(X W)
    QtS = np.zeros((l, rows.m))
    for _, Sb in rows.blocks():
        QtS += (Sb[:, c0:c0 + T] @ M).T @ Sb                      # B = Q^H M (all columns)
    Ub, s, Vh = np.linalg.svd(QtS[:, c0:c0 + T], full_matrices=False)
    Ub_r = Ub[:, :r].copy()
    V = Vh[:r].conj().T.copy()
    Umap = M @ Ub_r                                               # U = Q Ub (linalg.py:88)
    # _canonicalize (linalg.py:29-44): first largest |U| entry per column positive
    best = np.full(r, -1.0)
    sign = np.ones(r)
    for _, Sb in rows.blocks():
        Ub_blk = Sb[:, c0:c0 + T] @ Umap
        a = np.abs(Ub_blk)
        i = np.argmax(a, axis=0)
        v = a[i, np.arange(r)]
        upd = v > best                                            # strictly greater: first occurrence wins
        best[upd] = v[upd]
        sign[upd] = np.where(Ub_blk[i[upd], np.arange(r)[upd]] < 0, -1.0, 1.0)
    return StreamedSvd(Umap * sign, s[:r].copy(), V * sign, QtS, Ub_r * sign, M, c0)


# --------------------------------------------------------------------------
# modes: phi = S[:, c0:c0+T] @ C, ordered / normalised / locked (dmd.py:158-213)
# --------------------------------------------------------------------------

@dataclass
class StreamedModes:
    lam: np.ndarray
    C: np.ndarray         # T x r complex: phi = S[:, c0:c0+T] @ C (final, unit norm, canonical phase)
    c0: int
    sigma: np.ndarray
    extra: dict = field(default_factory=dict)

    def phi_rows(self, Sb: np.ndarray) -> np.ndarray:
        return Sb[:, self.c0:self.c0 + self.C.shape[0]] @ self.C


def order_and_pair(rows: Rows, lam, C, c0: int):
    """dmd.py:158-213 with phi = S[:, c0:c0+T] C: the column norms, the first
    |max| pivots and (for real-ified modes) max |Im| come from passes over S."""
    order = orc.frequency_order(lam)
    lam = np.array(lam, dtype=np.complex128)[order]
    C = np.array(C, dtype=np.complex128)[:, order]
    r = lam.size
    T = C.shape[0]
    nrm2 = np.zeros(r)
    best = np.full(r, -1.0)
    piv = np.zeros(r, dtype=np.complex128)
    for _, Sb in rows.blocks():
        P = Sb[:, c0:c0 + T] @ C
        a = np.abs(P)
        nrm2 += (a * a).sum(axis=0)
        i = np.argmax(a, axis=0)
        v = a[i, np.arange(r)]
        upd = v > best
        best[upd] = v[upd]
        piv[upd] = P[i[upd], np.arange(r)[upd]]
    nrm = np.sqrt(nrm2)
    out = C.copy()
    realify_check = []
    k = 0
    while k < r:
        s = 1.0 / nrm[k] if nrm[k] > 0 else 1.0
        pk = piv[k] * s
        if abs(pk) > 0:
            s = s * (np.conj(pk) / abs(pk))
        ck = C[:, k] * s
        out[:, k] = ck
        pair = (k + 1 < r and lam[k].imag > 0 and
                abs(lam[k + 1] - np.conj(lam[k])) <= 1e-6 * max(abs(lam[k]), 1e-300))
        if pair:
            lam[k + 1] = np.conj(lam[k])
            out[:, k + 1] = np.conj(ck)
            k += 2
            continue
        if abs(lam[k].imag) <= 1e-12 * max(abs(lam[k]), 1e-300):
            lam[k] = lam[k].real
            realify_check.append(k)
        k += 1
    if realify_check:
        mx = np.zeros(len(realify_check))
        idx = np.asarray(realify_check)
        for _, Sb in rows.blocks():
            mx = np.maximum(mx, np.abs((Sb[:, c0:c0 + T] @ out[:, idx]).imag).max(axis=0))
        for j, k in enumerate(realify_check):
            if mx[j] <= 1e-10:
                out[:, k] = out[:, k].real
    return lam, out


# --------------------------------------------------------------------------
# snapshot factor R_S (S = Q_S R_S, Householder TSQR) for pinv / frame norms
# --------------------------------------------------------------------------

def snapshot_r(rows: Rows):
    """One pass: R_S (m x m) of a streamed Householder TSQR of S (so
    S^T S = R_S^T R_S) and the column sums of S."""
    R = np.zeros((0, rows.m))
    colsum = np.zeros(rows.m)
    for _, Sb in rows.blocks():
        R = np.linalg.qr(np.vstack([R, Sb]), mode="r")
        colsum += Sb.sum(axis=0)
    if R.shape[0] < rows.m:
        R = np.vstack([R, np.zeros((rows.m - R.shape[0], rows.m))])
    return R, colsum


def encode_x(RS: np.ndarray, model: StreamedModes, col: int) -> np.ndarray:
    """z = pinv(phi) S[:, col] (runtime.py:47-52, pinv as linalg.py:93-104):
    phi = Q_S (R_S[:, window] C), so pinv(phi) = pinv(R_S[:, window] C) Q_S^T
    and Q_S^T S[:, col] = R_S[:, col]."""
    T = model.C.shape[0]
    A = RS[:, model.c0:model.c0 + T] @ model.C
    return orc.pinv_svd(A) @ RS[:, col]


# --------------------------------------------------------------------------
# trainers
# --------------------------------------------------------------------------

def exact_dmd(rows: Rows, r: int, p: int, q: int, seed, residual: bool = True) -> StreamedModes:
    """dmd.py:240-274 over X = S[:, :T], X' = S[:, 1:]."""
    T = rows.m - 1
    svd = randomized_svd(rows, T, r, p, q, seed)
    if svd.S[-1] <= orc.SIGMA_CUTOFF * svd.S[0]:
        raise ValueError("numerically zero singular value")
    VS = svd.V / svd.S
    UtXp = svd.Ub_r.T @ svd.QtS[:, 1:1 + T]                       # U^H X'
    Khat = UtXp @ VS                                              # dmd.py:255-256
    lam, W = orc.eig_checked(Khat)
    lam, C = order_and_pair(rows, lam, VS @ W, 1)                 # phi = X' V S^-1 W
    model = StreamedModes(lam, C, 1, svd.S, {"svd": svd, "khat": Khat})
    if residual:
        RS, colsum = snapshot_r(rows)
        model.extra["RS"], model.extra["colsum"] = RS, colsum
        # ||X' - Re(phi Lam pinv(phi) X)||: everything is S @ (m x T small)
        A = RS[:, 1:1 + T] @ C
        Z = orc.pinv_svd(A) @ RS[:, :T]                           # pinv(phi) X
        F = np.real(C @ (lam[:, None] * Z))                       # T x T
        H = np.zeros((rows.m, T))
        H[1:, :] = np.eye(T) - F                                  # X' - S[:,1:] F = S H
        res = float(np.linalg.norm(RS @ H))
        xp = float(np.linalg.norm(RS[:, 1:]))
        model.extra["residual"] = res
        model.extra["residual_rel"] = res / max(xp, 1e-300)
    return model


def optdmd(rows: Rows, r: int, p: int, q: int, seed, max_iters: int = 10) -> StreamedModes:
    """dmd.py:366-436 (init = the exact-DMD eigenvalues of the same seed)."""
    T = rows.m - 1
    ex = exact_dmd(rows, r, p, q, seed, residual=False)
    svd = ex.extra["svd"]
    D = np.conj(svd.V) * svd.S                                    # dmd.py:384
    try:
        alpha, B, hist, conv = orc.varpro_lm(D, ex.lam, max_iters)
    except orc._Collapse:
        rng = np.random.default_rng(0 if seed is None else seed)
        jit = 1e-10 * (1.0 + np.abs(ex.lam)) * np.exp(2j * np.pi * rng.random(ex.lam.size))
        alpha, B, hist, conv = orc.varpro_lm(D, ex.lam + jit, max_iters)
    a_s, B_s = orc.symmetrize(alpha, B)
    f_s = float(np.linalg.norm(D - orc.vandermonde(a_s, T) @ B_s))
    if f_s <= hist[-1] * (1 + 1e-9) and f_s <= hist[0] * (1 + 1e-12):
        alpha, B = a_s, B_s
    lam, C = order_and_pair(rows, alpha, svd.Umap @ B.T, 0)       # phi = U B^T
    return StreamedModes(lam, C, 0, svd.S, {"svd": svd, "history": hist, "converged": conv, "alpha0": ex.lam})


def frames_rows(model: StreamedModes, Sb: np.ndarray, z0: np.ndarray, ks) -> np.ndarray:
    """decode(step_k(z0, k)) restricted to the rows of Sb (runtime.py:66-124)."""
    P = model.phi_rows(Sb)
    return np.stack([np.real(P @ (model.lam ** k * z0)) for k in ks], axis=1)


def frame_norms(model: StreamedModes, RS: np.ndarray, colsum: np.ndarray, z0: np.ndarray, ks):
    """Sum and squared norm of every full frame Re(phi lam^k z0) = S_w Re(C z):
    from the column sums of S and S^T S = R_S^T R_S (no pass)."""
    T = model.C.shape[0]
    w = slice(model.c0, model.c0 + T)
    out = []
    for k in ks:
        c = np.real(model.C @ (model.lam ** k * z0))
        out.append((float(colsum[w] @ c), float(np.linalg.norm(RS[:, w] @ c) ** 2)))
    return np.array(out).T
