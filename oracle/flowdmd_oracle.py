"""CPU oracle for the DMD hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference algorithm of `flowdmd`
(arXiv 2502.05339 reference package, `/root/reference/pkg/src/flowdmd`).
It is the checker for the CUDA path; nothing in `paper_2502_05339_b200`
imports it. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
CPU-baseline leg may use it.

Pinning: `tests/test_oracle_golden.py` checks every function here against
golden vectors produced by running the *real* reference in the build
container (`oracle/gen_golden.py`, fixtures under `tests/golden/`), so the
oracle is pinned, not self-referential. The control-augmented DMDc fit
(`dmdc_fit`) has no reference implementation and is marked
"parity unpinned" below.

Every function cites the reference file:line it restates (paths relative to
`/root/reference/pkg/src/flowdmd/`).
"""

from __future__ import annotations

import numpy as np

# Thresholds restated from the reference (dmd.py:22-23, runtime.py:18-19).
UNSTABLE_MODULUS = 1.05
SIGMA_CUTOFF = 1e-14
INVERSE_FLOOR = 1e-8
EXP_OVERFLOW = 700.0


class OracleConvergenceError(RuntimeError):
    pass


# --------------------------------------------------------------------------
# linalg.py
# --------------------------------------------------------------------------

def canonicalize_columns(U, V):
    """linalg.py:29-44 — per column, divide U[:,k] and V[:,k] by the unit
    phase of U's first largest-magnitude entry."""
    U = np.array(U, copy=True)
    V = np.array(V, copy=True)
    piv_rows = np.argmax(np.abs(U), axis=0)            # first maximum, like np.argmax per column
    for k, i in enumerate(piv_rows):
        p = U[i, k]
        a = abs(p)
        if a == 0.0:
            continue
        ph = p / a
        U[:, k] /= ph
        V[:, k] /= ph
    return U, V


def dense_truncated_svd(M, r):
    """linalg.py:47-59 — top-r factors of a dense SVD, canonicalized."""
    M = np.asarray(M)
    if not 1 <= r <= min(M.shape):
        raise ValueError("rank out of range")
    U, s, Vh = np.linalg.svd(M, full_matrices=False)
    U, V = canonicalize_columns(U[:, :r], Vh[:r].conj().T)
    return U, s[:r].copy(), V


def sketch_svd(M, r, p, q, seed, omega=None):
    """linalg.py:62-90 — Gaussian range finder with q re-orthonormalised
    power passes (Householder QR), projection, small SVD, lift, canonicalize.

    `omega` may be supplied (cols x (r+p)); otherwise it is drawn exactly as
    linalg.py:80-81 does: default_rng(seed).standard_normal((cols, r+p)).
    """
    M = np.asarray(M)
    rows, cols = M.shape
    l = r + p
    if not 1 <= r <= min(rows, cols):
        raise ValueError("rank out of range")
    if l > min(rows, cols):
        raise ValueError("rank + oversample exceeds min dimension")
    G = draw_omega(cols, l, seed) if omega is None else np.asarray(omega)
    Q = np.linalg.qr(M @ G)[0]
    for _ in range(q):
        W = np.linalg.qr(M.conj().T @ Q)[0]
        Q = np.linalg.qr(M @ W)[0]
    B = Q.conj().T @ M
    Ub, s, Vh = np.linalg.svd(B, full_matrices=False)
    U, V = canonicalize_columns((Q @ Ub)[:, :r], Vh[:r].conj().T)
    return U, s[:r].copy(), V


def draw_omega(cols, l, seed):
    """linalg.py:80-81 — the Gaussian test matrix, float64, host-drawn."""
    return np.random.default_rng(seed).standard_normal((cols, l))


def pinv_svd(M, rel_tol=1e-12):
    """linalg.py:93-104 — SVD pseudo-inverse dropping s < rel_tol*s_max."""
    M = np.asarray(M)
    U, s, Vh = np.linalg.svd(M, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((M.shape[1], M.shape[0]), dtype=M.dtype)
    inv = np.where(s > rel_tol * s[0], 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return (Vh.conj().T * inv) @ U.conj().T


def eig_checked(M):
    """linalg.py:107-133 — eig with unit-norm vectors and residual check."""
    w, V = np.linalg.eig(M)
    nv = np.linalg.norm(V, axis=0)
    nv[nv == 0.0] = 1.0
    V = V / nv
    scale = np.linalg.norm(M)
    res = np.linalg.norm(M @ V - V * w)
    if scale > 0 and res > 1e-8 * scale:
        raise OracleConvergenceError("eig residual")
    return w, V


# --------------------------------------------------------------------------
# dmd.py
# --------------------------------------------------------------------------

def partner_map(lam, tol=1e-8):
    """dmd.py:131-155 — greedy conjugate matching; real (|Im| <= tol*scale)
    or unmatched eigenvalues are self-paired."""
    lam = np.asarray(lam)
    r = lam.size
    scale = max(float(np.abs(lam).max()), 1e-300) if r else 1.0
    out = -np.ones(r, dtype=np.int64)
    for i in range(r):
        if out[i] >= 0:
            continue
        if abs(lam[i].imag) <= tol * scale:
            out[i] = i
            continue
        free = [j for j in range(r) if j != i and out[j] < 0]
        if free:
            d = np.abs(lam[free] - np.conj(lam[i]))
            jj = int(np.argmin(d))
            if d[jj] <= 10 * tol * scale + tol:
                out[i] = free[jj]
                out[free[jj]] = i
                continue
        out[i] = i
    return out


def frequency_order(lam):
    """dmd.py:158-187 — the column permutation of _order_and_pair: units
    (self-paired or representative-with-partner, representative = larger Im)
    sorted by (|arg|, -|lam|, Re) of the representative."""
    lam = np.asarray(lam)
    part = partner_map(lam)
    seen = np.zeros(lam.size, dtype=bool)
    units = []
    for i in range(lam.size):
        if seen[i]:
            continue
        j = int(part[i])
        seen[i] = seen[j] = True
        if i == j:
            units.append((i, -1))
        elif lam[i].imag >= lam[j].imag:
            units.append((i, j))
        else:
            units.append((j, i))
    units.sort(key=lambda u: (abs(np.angle(lam[u[0]])), -abs(lam[u[0]]), lam[u[0]].real))
    order = []
    for a, b in units:
        order.append(a)
        if b >= 0:
            order.append(b)
    return np.asarray(order, dtype=np.int64)


def order_and_pair(lam, phi):
    """dmd.py:158-213 — sort, unit-normalise, canonicalise the
    representative's phase at its first |max| entry, lock exact conjugates,
    real-ify near-real eigenvalues/modes."""
    order = frequency_order(lam)
    lam = np.array(lam, dtype=np.complex128)[order]
    phi = np.array(phi, dtype=np.complex128)[:, order]
    k = 0
    r = lam.size
    while k < r:
        c = phi[:, k]
        nrm = np.linalg.norm(c)
        if nrm > 0:
            c = c / nrm
        i = int(np.argmax(np.abs(c)))
        if abs(c[i]) > 0:
            c = c * (np.conj(c[i]) / abs(c[i]))
        phi[:, k] = c
        pair = (k + 1 < r and lam[k].imag > 0 and
                abs(lam[k + 1] - np.conj(lam[k])) <= 1e-6 * max(abs(lam[k]), 1e-300))
        if pair:
            lam[k + 1] = np.conj(lam[k])
            phi[:, k + 1] = np.conj(c)
            k += 2
            continue
        if abs(lam[k].imag) <= 1e-12 * max(abs(lam[k]), 1e-300):
            lam[k] = lam[k].real
            if np.abs(c.imag).max() <= 1e-10:
                phi[:, k] = c.real
        k += 1
    return lam, phi


def svd_for_fit(X, r, svd_mode, seed, p=None, q=None):
    """dmd.py:216-222 with the oracle's (p, q) override: the reference
    clamps p = min(10, T - r) and hard-codes q = 2 for randomized mode."""
    if svd_mode == "full":
        return dense_truncated_svd(X, r)
    if svd_mode != "randomized":
        raise ValueError(svd_mode)
    T = min(X.shape)
    pp = min(10, T - r) if p is None else min(p, T - r)
    qq = 2 if q is None else q
    return sketch_svd(X, r, pp, qq, seed)


def exact_dmd(states, r, svd_mode="full", seed=None, p=None, q=None, residual=True):
    """dmd.py:240-274 — returns dict(lam, phi, sigma, residual, residual_rel)."""
    states = np.asarray(states, dtype=np.float64)
    X, Xp = states[:, :-1], states[:, 1:]
    n, T = X.shape
    if not 1 <= r <= min(n, T):
        raise ValueError("rank out of range")
    U, S, V = svd_for_fit(X, r, svd_mode, seed, p, q)
    if S[-1] <= SIGMA_CUTOFF * S[0]:
        raise ValueError("numerically zero singular value")
    P = Xp @ (V / S)
    Khat = U.conj().T @ P
    lam, W = eig_checked(Khat)
    lam, phi = order_and_pair(lam, P @ W)
    out = dict(lam=lam, phi=phi, sigma=S, U=U, V=V, khat=Khat)
    if residual:
        rec = (phi * lam) @ (pinv_svd(phi) @ X)
        res = float(np.linalg.norm(Xp - rec.real))
        out["residual"] = res
        out["residual_rel"] = res / max(np.linalg.norm(Xp), 1e-300)
    return out


def vandermonde(alpha, T):
    """dmd.py:277-282."""
    alpha = np.asarray(alpha, dtype=np.complex128)
    return alpha[None, :] ** np.arange(T)[:, None]


def _varpro_fit(alpha, D):
    P = vandermonde(alpha, D.shape[0])
    B = np.linalg.lstsq(P, D, rcond=None)[0]
    R = D - P @ B
    return float(np.linalg.norm(R)), B, P, R


def _min_sep(a):
    if a.size < 2:
        return np.inf
    d = np.abs(a[:, None] - a[None, :])
    np.fill_diagonal(d, np.inf)
    return float(d.min())


class _Collapse(Exception):
    pass


def varpro_lm(D, alpha0, max_iters=200, init_damping=1.0, up=2.0, down=3.0,
              rel_tol=1e-8, collapse_tol=1e-12):
    """dmd.py:314-363 — LM on the eigenvalues with the Kaufman projected
    Jacobian; returns (alpha, B, history, converged)."""
    T = D.shape[0]
    t = np.arange(T)
    alpha = np.array(alpha0, dtype=np.complex128)
    if _min_sep(alpha) < collapse_tol:
        raise _Collapse
    f, B, P, R = _varpro_fit(alpha, D)
    floor = 1e-14 * np.linalg.norm(D)
    hist = [f]
    if max_iters == 0:
        return alpha, B, hist, True
    mu = init_damping
    conv = False
    for _ in range(max_iters):
        if f <= floor:
            conv = True
            break
        Qp = np.linalg.qr(P)[0]
        dP = np.zeros_like(P)
        dP[1:, :] = t[1:, None] * alpha[None, :] ** (t[1:, None] - 1)
        Wk = dP - Qp @ (Qp.conj().T @ dP)
        JHJ = (Wk.conj().T @ Wk) * np.conj(B @ B.conj().T)
        g = np.diag(Wk.conj().T @ (R @ B.conj().T))
        try:
            step = np.linalg.solve(JHJ + mu * np.eye(alpha.size), g)
        except np.linalg.LinAlgError:
            mu *= up
            continue
        cand = alpha + step
        if _min_sep(cand) < collapse_tol:
            raise _Collapse
        f2, B2, P2, R2 = _varpro_fit(cand, D)
        if f2 < f:
            rel = (f - f2) / max(f, 1e-300)
            alpha, f, B, P, R = cand, f2, B2, P2, R2
            hist.append(f)
            mu /= down
            if rel < rel_tol or f <= floor:
                conv = True
                break
        else:
            mu *= up
    return alpha, B, hist, conv


def symmetrize(alpha, B):
    """dmd.py:439-455."""
    part = partner_map(alpha)
    alpha = alpha.copy()
    B = B.copy()
    for i in range(alpha.size):
        j = part[i]
        if j > i:
            a = 0.5 * (alpha[i] + np.conj(alpha[j]))
            alpha[i], alpha[j] = a, np.conj(a)
            row = 0.5 * (B[i, :] + np.conj(B[j, :]))
            B[i, :], B[j, :] = row, np.conj(row)
        elif j == i and abs(alpha[i].imag) <= 1e-8 * max(abs(alpha[i]), 1e-300):
            alpha[i] = alpha[i].real
            B[i, :] = B[i, :].real
    return alpha, B


def optdmd(states, r, init=None, max_iters=200, svd_mode="full", seed=None, p=None, q=None):
    """dmd.py:366-436 — returns dict(lam, phi, sigma, history, converged)."""
    states = np.asarray(states, dtype=np.float64)
    X = states[:, :-1]
    n, T = X.shape
    U, S, V = svd_for_fit(X, r, svd_mode, seed, p, q)
    if S[-1] <= SIGMA_CUTOFF * S[0]:
        raise ValueError("numerically zero singular value")
    D = np.conj(V) * S
    if init is None:
        alpha0 = exact_dmd(states, r, svd_mode, seed, p, q, residual=False)["lam"]
    else:
        alpha0 = np.asarray(init, dtype=np.complex128)
    try:
        alpha, B, hist, conv = varpro_lm(D, alpha0, max_iters)
    except _Collapse:
        rng = np.random.default_rng(0 if seed is None else seed)
        jit = 1e-10 * (1.0 + np.abs(alpha0)) * np.exp(2j * np.pi * rng.random(alpha0.size))
        alpha, B, hist, conv = varpro_lm(D, alpha0 + jit, max_iters)
    a_s, B_s = symmetrize(alpha, B)
    f_s = float(np.linalg.norm(D - vandermonde(a_s, T) @ B_s))
    if f_s <= hist[-1] * (1 + 1e-9) and f_s <= hist[0] * (1 + 1e-12):
        alpha, B = a_s, B_s
    lam, phi = order_and_pair(alpha, U @ B.T)
    return dict(lam=lam, phi=phi, sigma=S, history=hist, converged=conv)


def reduced_control(phi, channels):
    """dmd.py:471-491 — B~_i = pinv(phi) @ B_i."""
    pp = pinv_svd(phi)
    return [pp @ np.asarray(Bm) for Bm in channels]


# --------------------------------------------------------------------------
# ReducedModel decode table (dmd.py:92-120) and runtime.py
# --------------------------------------------------------------------------

def decode_columns(phi, lam):
    """dmd.py:92-120 — real table [Re phi_a] / [2 Re phi_a, -2 Im phi_a]
    with (column, mode) index maps for Re and Im coefficient parts."""
    part = partner_map(lam)
    n, r = phi.shape
    cols, re_idx, im_idx = [], [], []
    for a in range(r):
        b = part[a]
        if b < a:
            continue
        if b == a:
            re_idx.append((len(cols), a))
            cols.append(phi[:, a].real)
        else:
            re_idx.append((len(cols), a))
            cols.append(2.0 * phi[:, a].real)
            im_idx.append((len(cols), a))
            cols.append(-2.0 * phi[:, a].imag)
    table = np.stack(cols, axis=1) if cols else np.zeros((n, 0))
    return np.ascontiguousarray(table), re_idx, im_idx


def symmetry_defect(lam, z):
    """runtime.py:55-63."""
    part = partner_map(lam)
    d = 0.0
    for a in range(z.size):
        b = part[a]
        if b == a:
            d = max(d, abs(z[a].imag))
        elif b > a:
            d = max(d, abs(z[b] - np.conj(z[a])))
    return d


def decode(phi, lam, z):
    """runtime.py:66-99 — table GEMV when z is conjugate-symmetric, else Re(phi z)."""
    z = np.asarray(z, dtype=np.complex128).ravel()
    scale = max(float(np.abs(z).max()) if z.size else 0.0, 1e-300)
    if symmetry_defect(lam, z) <= 1e-9 * scale:
        table, re_idx, im_idx = decode_columns(phi, lam)
        c = np.empty(table.shape[1])
        for k, a in re_idx:
            c[k] = z[a].real
        for k, a in im_idx:
            c[k] = z[a].imag
        return table @ c
    return (phi @ z).real


def encode(phi, u):
    """runtime.py:47-52."""
    return pinv_svd(phi) @ np.asarray(u).ravel()


def step_k(lam, z, k):
    """runtime.py:108-124 (without the overflow guard)."""
    return lam ** k * z


def eval_continuous(lam, dt, z, t):
    """runtime.py:127-142."""
    om = np.log(lam) / dt
    return np.exp(om * t) * z


def step_forced(lam, dt, z, reduced_b=(), q=(), pinv_phi=None, f=None):
    """runtime.py:164-200."""
    out = lam * z
    for Bm, qi in zip(reduced_b, q):
        out = out + (Bm @ np.asarray(qi).ravel()) * dt
    if f is not None:
        out = out + (pinv_phi @ f) * dt
    return out


# --------------------------------------------------------------------------
# CholeskyQR2 restatement of sketch_svd (the algorithm the GPU runs).
# Used by tests to separate "algorithm change" from "kernel error".
# --------------------------------------------------------------------------

def cholqr2(Y):
    """Q = Y R^-1 twice (CholeskyQR2); returns Q, R."""
    G = Y.T @ Y
    R1 = np.linalg.cholesky(G).T
    Q1 = np.linalg.solve(R1.T, Y.T).T
    G2 = Q1.T @ Q1
    R2 = np.linalg.cholesky(G2).T
    Q = np.linalg.solve(R2.T, Q1.T).T
    return Q, R2 @ R1


def sketch_svd_cholqr2(M, r, p, q, omega):
    M = np.asarray(M, dtype=np.float64)
    Q = cholqr2(M @ omega)[0]
    for _ in range(q):
        W = np.linalg.qr(M.T @ Q)[0]
        Q = cholqr2(M @ W)[0]
    B = Q.T @ M
    Ub, s, Vh = np.linalg.svd(B, full_matrices=False)
    U, V = canonicalize_columns((Q @ Ub)[:, :r], Vh[:r].T)
    return U, s[:r].copy(), V


# --------------------------------------------------------------------------
# Control-augmented DMDc — PARITY UNPINNED (no reference implementation:
# the reference's DMDc is fit_control with known B, dmd.py:471-491; joint
# identification is a declared non-goal). Restates Proctor
# et al. 2016 as cited by PAPER.md:420.
# --------------------------------------------------------------------------

def dmdc_fit(states, controls, p_rank, r, seed, p=10, q=1):
    """Augmented DMDc: SVD of Omega=[X; Upsilon] at rank p_rank, output basis
    from an SVD of X' at rank r; returns (A~, B~, lam, phi, Uhat)."""
    states = np.asarray(states, dtype=np.float64)
    X, Xp = states[:, :-1], states[:, 1:]
    Ups = np.asarray(controls, dtype=np.float64)          # ell x T
    n = X.shape[0]
    Om = np.vstack([X, Ups])
    Ut, St, Vt = sketch_svd(Om, p_rank, min(p, Om.shape[1] - p_rank), q, seed)
    Uh, Sh, Vh = sketch_svd(Xp, r, min(p, Xp.shape[1] - r), q, None if seed is None else seed + 1)
    U1, U2 = Ut[:n], Ut[n:]
    core = Xp @ (Vt / St)                                  # n x p_rank
    A = Uh.T @ core @ (U1.T @ Uh)
    Bt = Uh.T @ core @ U2.T
    lam, W = eig_checked(A)
    phi = core @ (U1.T @ Uh) @ W
    lam, phi = order_and_pair(lam, phi)
    return dict(A=A, B=Bt, lam=lam, phi=phi, Uhat=Uh, sigma_aug=St)


def dmdc_reduced_b(fit, dt):
    """Modal control matrix pinv(phi) @ U_hat @ B~ / dt, so that
    runtime.step_forced's `reduced_b q dt` (runtime.py:188) adds B u."""
    return pinv_svd(fit["phi"]) @ (fit["Uhat"] @ fit["B"]) / dt


def controlled_system(n, pairs, ell, m, seed, noise=0.0):
    """x_{j+1} = A x_j + B u_j with A = Psi Ablk Psi^+ (rank 2*pairs, known
    eigenvalues rho e^{+-i theta}) and B = ell random fields; returns
    (states n x m, controls ell x (m-1), true eigenvalues, B)."""
    rng = np.random.default_rng(seed)
    Psi = np.linalg.qr(rng.standard_normal((n, 2 * pairs)))[0]
    rho = rng.uniform(0.9, 0.999, pairs)
    th = rng.uniform(0.05, 1.0, pairs)
    Ab = np.zeros((2 * pairs, 2 * pairs))
    eigs = []
    for i in range(pairs):
        c, s = np.cos(th[i]), np.sin(th[i])
        Ab[2 * i:2 * i + 2, 2 * i:2 * i + 2] = rho[i] * np.array([[c, -s], [s, c]])
        eigs += [rho[i] * np.exp(1j * th[i]), rho[i] * np.exp(-1j * th[i])]
    Bf = rng.standard_normal((n, ell)) / np.sqrt(n)
    U = rng.standard_normal((ell, m - 1))
    X = np.empty((n, m))
    X[:, 0] = Psi @ rng.standard_normal(2 * pairs)
    for j in range(m - 1):
        X[:, j + 1] = Psi @ (Ab @ (Psi.T @ X[:, j])) + Bf @ U[:, j]
    if noise:
        X = X + noise * rng.standard_normal(X.shape)
    return X, U, np.asarray(eigs), Bf


# --------------------------------------------------------------------------
# §8(f) rows 2-3: MAC grids, serving frames, spectral editing, guided
# upscaling (grid.py, solver.py, server.py, editing.py, upres.py)
# --------------------------------------------------------------------------

def mac_sizes(nx, ny):
    """grid.py:67-82 — (n_u, n_v)."""
    return (nx + 1) * ny, nx * (ny + 1)


def build_downsample(nx, ny, f):
    """grid.py:195-236 — face-averaging restriction (scipy CSR, entry order t = 0..f-1)."""
    import scipy.sparse as sp
    nxl, nyl = nx // f, ny // f
    n_u, _ = mac_sizes(nx, ny)
    nl_u, nl_v = mac_sizes(nxl, nyl)
    rows, cols, vals = [], [], []
    jl, il = np.meshgrid(np.arange(nyl), np.arange(nxl + 1), indexing="ij")
    low = (jl * (nxl + 1) + il).ravel()
    for t in range(f):
        rows.append(low)
        cols.append(((jl * f + t) * (nx + 1) + il * f).ravel())
        vals.append(np.full(low.size, 1.0 / f))
    jl, il = np.meshgrid(np.arange(nyl + 1), np.arange(nxl), indexing="ij")
    low = (nl_u + jl * nxl + il).ravel()
    for t in range(f):
        rows.append(low)
        cols.append((n_u + (jl * f) * nx + il * f + t).ravel())
        vals.append(np.full(low.size, 1.0 / f))
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(nl_u + nl_v, sum(mac_sizes(nx, ny))))


def build_inject(nx, ny, f):
    """upres.py:21-50 — nearest-face prolongation (scipy CSR, ones)."""
    import scipy.sparse as sp
    nxl, nyl = nx // f, ny // f
    n_u, _ = mac_sizes(nx, ny)
    nl_u, nl_v = mac_sizes(nxl, nyl)
    jh, ih = np.meshgrid(np.arange(ny), np.arange(nx + 1), indexing="ij")
    r1 = (jh * (nx + 1) + ih).ravel()
    c1 = ((jh // f) * (nxl + 1) + np.minimum((ih + f // 2) // f, nxl)).ravel()
    jh, ih = np.meshgrid(np.arange(ny + 1), np.arange(nx), indexing="ij")
    r2 = (n_u + jh * nx + ih).ravel()
    c2 = (nl_u + np.minimum((jh + f // 2) // f, nyl) * nxl + ih // f).ravel()
    rows = np.concatenate([r1, r2])
    return sp.csr_matrix((np.ones(rows.size), (rows, np.concatenate([c1, c2]))),
                         shape=(sum(mac_sizes(nx, ny)), nl_u + nl_v))


def center_planes(flat, nx, ny, field):
    """server.py:205-214 — cell-centred velocity planes or speed."""
    n_u, _ = mac_sizes(nx, ny)
    u = flat[:n_u].reshape(ny, nx + 1)
    v = flat[n_u:].reshape(ny + 1, nx)
    uc = 0.5 * (u[:, :-1] + u[:, 1:])
    vc = 0.5 * (v[:-1, :] + v[1:, :])
    if field == "velocity":
        return np.stack([uc, vc])
    return np.sqrt(uc * uc + vc * vc)[None, :, :]


def encode_planes(planes, fmt):
    """server.py:288-302 — 12-byte header + f32 / u8 planes."""
    channels, ny, nx = planes.shape
    header = np.asarray([nx, ny, channels], dtype="<u4").tobytes()
    if fmt == "bin":
        return header + planes.astype("<f4").tobytes()
    lo, hi = planes.min(), planes.max()
    span = hi - lo
    if span <= 0:
        data = np.zeros(planes.shape, dtype=np.uint8)
    else:
        data = np.clip((planes - lo) / span * 255.0, 0, 255).astype(np.uint8)
    return header + data.tobytes()


def bilinear(f, col, row):
    """solver.py:79-101 (values only)."""
    nr, nc = f.shape
    col = np.clip(col, 0.0, nc - 1.0)
    row = np.clip(row, 0.0, nr - 1.0)
    i0 = np.minimum(col.astype(np.int64), nc - 2)
    j0 = np.minimum(row.astype(np.int64), nr - 2)
    tx = col - i0
    ty = row - j0
    return (f[j0, i0] * (1 - tx) * (1 - ty) + f[j0, i0 + 1] * tx * (1 - ty)
            + f[j0 + 1, i0] * (1 - tx) * ty + f[j0 + 1, i0 + 1] * tx * ty)


def advect_density(flat, nx, ny, h, q, dt):
    """solver.py:133-150 (maccormack=False, cell centres) via 104-108, 111-121."""
    n_u, _ = mac_sizes(nx, ny)
    u = flat[:n_u].reshape(ny, nx + 1)
    v = flat[n_u:].reshape(ny + 1, nx)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    X, Y = (i + 0.5) * h, (j + 0.5) * h
    up = bilinear(u, X / h, Y / h - 0.5)
    vp = bilinear(v, X / h - 0.5, Y / h)
    return bilinear(q, (X - dt * up) / h - 0.5, (Y - dt * vp) / h - 0.5)


def apply_edit(phi, lam, dt, weights, growth, freq):
    """editing.py:130-149 — (new phi, new lam)."""
    part = partner_map(lam)
    om = np.log(lam) / dt
    new_lam = np.exp((growth * om.real + 1j * freq * om.imag) * dt)
    new_phi = phi * weights[None, :]
    for a in range(lam.size):
        b = part[a]
        if b > a:
            new_lam[b] = np.conj(new_lam[a])
            new_phi[:, b] = np.conj(new_phi[:, a])
    return new_phi, new_lam


def constrained_project(nx, ny, f, H, L):
    """upres.py:142-169 — x = H + A^T (A A^T)^-1 (L - A H) with SuperLU."""
    import scipy.sparse.linalg as spla
    A = build_downsample(nx, ny, f)
    lu = spla.splu((A @ A.T).tocsc())
    return H + A.T @ lu.solve(L - A @ H)


def upres_step(phi, lam, z, L, nx, ny, f, split):
    """upres.py:110-130 — (new z, decoded field); split already effective."""
    P = encode(phi, build_inject(nx, ny, f) @ L)
    zn = np.concatenate([P[:split], (lam * z)[split:]])
    return zn, decode(phi, lam, zn)


# --------------------------------------------------------------------------
# §8(f) row 4: solver pieces (solver.py) used to check the device kernels
# --------------------------------------------------------------------------

def _bilinear_ex(f, col, row):
    """solver.py:79-101 with extrema."""
    nr, nc = f.shape
    col = np.clip(col, 0.0, nc - 1.0)
    row = np.clip(row, 0.0, nr - 1.0)
    i0 = np.minimum(col.astype(np.int64), nc - 2)
    j0 = np.minimum(row.astype(np.int64), nr - 2)
    tx = col - i0
    ty = row - j0
    f00, f10, f01, f11 = f[j0, i0], f[j0, i0 + 1], f[j0 + 1, i0], f[j0 + 1, i0 + 1]
    val = f00 * (1 - tx) * (1 - ty) + f10 * tx * (1 - ty) + f01 * (1 - tx) * ty + f11 * tx * ty
    lo = np.minimum(np.minimum(f00, f10), np.minimum(f01, f11))
    hi = np.maximum(np.maximum(f00, f10), np.maximum(f01, f11))
    return val, lo, hi


def advect_array(u, v, q, which, h, dt, maccormack=True):
    """solver.py:111-150 — transport of one component array (u faces, v faces or 'c')."""
    ny, nxp = u.shape
    nx = nxp - 1
    if which == "u":
        j, i = np.meshgrid(np.arange(ny), np.arange(nx + 1), indexing="ij")
        X, Y = i * h, (j + 0.5) * h
        samp = lambda f, x, y: _bilinear_ex(f, x / h, y / h - 0.5)            # noqa: E731
    elif which == "v":
        j, i = np.meshgrid(np.arange(ny + 1), np.arange(nx), indexing="ij")
        X, Y = (i + 0.5) * h, j * h
        samp = lambda f, x, y: _bilinear_ex(f, x / h - 0.5, y / h)            # noqa: E731
    else:
        j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        X, Y = (i + 0.5) * h, (j + 0.5) * h
        samp = lambda f, x, y: _bilinear_ex(f, x / h - 0.5, y / h - 0.5)      # noqa: E731
    up = bilinear(u, X / h, Y / h - 0.5)
    vp = bilinear(v, X / h - 0.5, Y / h)
    q_hat, lo, hi = samp(q, X - dt * up, Y - dt * vp)
    if not maccormack:
        return q_hat
    q_back = samp(q_hat, X + dt * up, Y + dt * vp)[0]
    return np.clip(q_hat + 0.5 * (q - q_back), lo, hi)


def apply_poisson(p, nx, ny, h, solid=None, boundary="open"):
    """solver.py:229-258 — negative masked Laplacian."""
    fluid = ~(np.zeros((ny, nx), dtype=bool) if solid is None else solid)
    cx = np.zeros((ny, nx + 1))
    cy = np.zeros((ny + 1, nx))
    cx[:, 1:-1] = (fluid[:, :-1] & fluid[:, 1:]).astype(np.float64)
    cy[1:-1, :] = (fluid[:-1, :] & fluid[1:, :]).astype(np.float64)
    if boundary == "open":
        cy[-1, :] = fluid[-1, :].astype(np.float64)
    out = np.zeros_like(p)
    fe = cx[:, 1:-1] * (p[:, 1:] - p[:, :-1])
    out[:, :-1] += fe
    out[:, 1:] -= fe
    fn = cy[1:-1, :] * (p[1:, :] - p[:-1, :])
    out[:-1, :] += fn
    out[1:, :] -= fn
    out[-1, :] -= cy[-1, :] * p[-1, :]
    return -out / (h * h)
