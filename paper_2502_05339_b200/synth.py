"""Seeded synthetic snapshot matrices for BASELINE.json configs 0-4.

The reference measures on no public dataset for this path; BASELINE.json
specifies generator recipes instead, and these functions implement them
(DESIGN.md §"Synthetic inputs" records the exact recipe):

    column j = Re(sum_i phi_i lambda_i^j b_i) + sigma_n * N(0, 1)
    lambda_i = exp((s_i + i w_i) dt), s_i ~ U(-0.2, 0), w_i ~ U(0.1, pi), dt = 0.1
    b_i ~ CN(0, 1)

* 2D (config 0): 64x64 periodic grid x 2 components; per mode and component
  a sum of 4 plane sinusoids a_s sin(2pi(kx x + ky y)/G + th_s), integer
  wavenumbers in [1, 8], a_s ~ CN(0, 1).
* 3D (configs 1-4): N^3 grid x 3 components; per mode and component one
  separable sinusoid a sin(2pi kx x/N + thx) sin(2pi ky y/N + thy)
  sin(2pi kz z/N + thz), wavenumbers in [1, 16], a ~ CN(0, 1).

Row order is component-major: row = c N^d + (z N + y) N + x.

Noise is counter-based (splitmix64 of (seed, row, col) -> Box-Muller) so the
device generator (`fdmd_synth_separable3d`) and the host generator below
produce the same noise for the same (seed, row, col) regardless of sharding.
Parameters (eigenvalues, amplitudes, sinusoid tables) are tiny and drawn on
the host with numpy's default_rng.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DT = 0.1

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & _M64
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
    return z ^ (z >> np.uint64(31))


def noise_key(seed: int) -> int:
    with np.errstate(over="ignore"):
        return int(_splitmix(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


def counter_normal(seed: int, rows: np.ndarray, cols: np.ndarray, ncols_total: int) -> np.ndarray:
    """N(0,1) samples for (row, col) pairs (broadcast), independent of layout."""
    key = np.uint64(noise_key(seed))
    with np.errstate(over="ignore"):
        ctr = (np.asarray(rows, dtype=np.uint64) * np.uint64(ncols_total)
               + np.asarray(cols, dtype=np.uint64))
        a = _splitmix((key + np.uint64(2) * ctr) & _M64)
        b = _splitmix((key + np.uint64(2) * ctr + np.uint64(1)) & _M64)
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)
    u2 = ((b >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


@dataclass
class SynthParams:
    """Everything needed to (re)generate a snapshot matrix."""

    dim: int                 # 2 or 3
    grid: int                # G (2D) or N (3D)
    comps: int               # velocity components
    modes: int               # K complex modes
    m: int                   # snapshots
    noise: float
    seed: int
    lam: np.ndarray          # K complex
    b: np.ndarray            # K complex
    # 3D: per (mode, comp): amp (complex), k (3 ints), th (3)
    # 2D: per (mode, comp, s<4): amp, k (2 ints), th
    amp: np.ndarray
    kvec: np.ndarray
    theta: np.ndarray
    dtype: type = np.float32
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.comps * self.grid ** self.dim

    def coef(self) -> np.ndarray:
        """K x m complex: lambda_i^j b_i."""
        j = np.arange(self.m)
        return self.lam[:, None] ** j[None, :] * self.b[:, None]

    def sep_tables(self):
        """3D only: sin tables S[d][i, c, x] and A[i, c, j] = Re(amp_ic coef_ij)."""
        assert self.dim == 3
        x = np.arange(self.grid)
        tabs = []
        for d in range(3):
            arg = 2.0 * np.pi * self.kvec[:, :, d, None] * x[None, None, :] / self.grid \
                + self.theta[:, :, d, None]
            tabs.append(np.sin(arg))
        A = np.real(self.amp[:, :, None] * self.coef()[:, None, :])
        return tabs[0], tabs[1], tabs[2], A


def draw_params(dim, grid, comps, modes, m, noise, seed, kmax, dtype=np.float32) -> SynthParams:
    rng = np.random.default_rng(seed)
    s = rng.uniform(-0.2, 0.0, modes)
    w = rng.uniform(0.1, np.pi, modes)
    lam = np.exp((s + 1j * w) * DT)
    b = (rng.standard_normal(modes) + 1j * rng.standard_normal(modes)) / np.sqrt(2.0)
    if dim == 3:
        amp = (rng.standard_normal((modes, comps)) + 1j * rng.standard_normal((modes, comps))) / np.sqrt(2.0)
        kvec = rng.integers(1, kmax + 1, size=(modes, comps, 3))
        theta = rng.uniform(0.0, 2.0 * np.pi, size=(modes, comps, 3))
    else:
        amp = (rng.standard_normal((modes, comps, 4)) + 1j * rng.standard_normal((modes, comps, 4))) / np.sqrt(2.0)
        kvec = rng.integers(1, kmax + 1, size=(modes, comps, 4, 2))
        theta = rng.uniform(0.0, 2.0 * np.pi, size=(modes, comps, 4))
    return SynthParams(dim, grid, comps, modes, m, noise, seed, lam, b, amp, kvec, theta, dtype)


# BASELINE.json configs (sizes in the JSON; `scale_grid` lets tests shrink the
# grid while keeping modes/m/rank/spectrum).
CONFIGS = {
    0: dict(dim=2, grid=64, comps=2, modes=10, m=101, noise=1e-3, kmax=8, dtype=np.float64,
            r=20, p=10, q=2),
    1: dict(dim=3, grid=128, comps=3, modes=75, m=201, noise=1e-3, kmax=16, dtype=np.float32,
            r=150, p=10, q=1),
    3: dict(dim=3, grid=256, comps=3, modes=100, m=201, noise=1e-3, kmax=16, dtype=np.float32,
            r=200, p=10, q=1),
}


def config_params(cfg: int, seed: int = 0, grid=None) -> SynthParams:
    c = dict(CONFIGS[cfg])
    g = c["grid"] if grid is None else grid
    p = draw_params(c["dim"], g, c["comps"], c["modes"], c["m"], c["noise"], seed, c["kmax"], c["dtype"])
    p.meta = dict(config=cfg, r=c["r"], p=c["p"], q=c["q"])
    return p


def generate_host(p: SynthParams, row0: int = 0, rows=None) -> np.ndarray:
    """Rows [row0, row0+rows) of the n x m snapshot matrix, computed in fp64
    on the host and cast to p.dtype."""
    n = p.n
    rows = n - row0 if rows is None else rows
    idx = np.arange(row0, row0 + rows)
    cells = p.grid ** p.dim
    c = idx // cells
    rem = idx % cells
    coef = p.coef()
    out = np.empty((rows, p.m), dtype=np.float64)
    if p.dim == 3:
        sx, sy, sz, A = p.sep_tables()
        x = rem % p.grid
        y = (rem // p.grid) % p.grid
        z = rem // (p.grid * p.grid)
        for cc in range(p.comps):
            sel = c == cc
            if not sel.any():
                continue
            S = sx[:, cc, x[sel]] * sy[:, cc, y[sel]] * sz[:, cc, z[sel]]   # K x rows
            out[sel] = S.T @ A[:, cc, :]
    else:
        x = rem % p.grid
        y = rem // p.grid
        for cc in range(p.comps):
            sel = c == cc
            if not sel.any():
                continue
            phi = np.zeros((p.modes, int(sel.sum())), dtype=np.complex128)
            for s in range(4):
                arg = 2.0 * np.pi * (p.kvec[:, cc, s, 0, None] * x[None, sel]
                                     + p.kvec[:, cc, s, 1, None] * y[None, sel]) / p.grid \
                    + p.theta[:, cc, s, None]
                phi += p.amp[:, cc, s, None] * np.sin(arg)
            out[sel] = np.real(phi.T @ coef)
    if p.noise:
        out += p.noise * counter_normal(p.seed, idx[:, None], np.arange(p.m)[None, :], p.m)
    return out.astype(p.dtype)


# ---------------------------------------------------------------------------
# Config 2 (DMDc): X_{j+1} = A X_j + B u_j, A = config 1's rank-150 generator
# ---------------------------------------------------------------------------
def _sin_tables(kvec, theta, N):
    """S[d][i, c, x] = sin(2 pi k_icd x / N + th_icd)."""
    x = np.arange(N)
    return [np.sin(2.0 * np.pi * kvec[:, :, d, None] * x[None, None, :] / N + theta[:, :, d, None])
            for d in range(3)]


@dataclass
class ControlledParams:
    """BASELINE config 2: the 3D mode fields of config 1 (75 complex modes,
    rank 150) as the generator A, plus ell seeded smooth control fields B.

    A = F M F^+ (F = the 150 real mode fields Re f_i, Im f_i, f_i = amp_ic s_ic
    per component c; M advances each mode by lambda_i) and B = F F^+ G: the
    smooth random fields G (separable sinusoids, wavenumbers 1..4) projected
    onto A's range, so the controlled states stay in A's 150-dim invariant
    subspace and [X; Upsilon] has rank 150 + ell = 158 — the r = 158 BASELINE
    fits at. In mode coordinates x = Re(sum_i f_i z_i):
        z_{j+1} = lambda * z_j + P u_j,   P = the z-coordinates of F^+ G,
    from z_0 = b; every column is a separable-field superposition generated
    by the same kernel as configs 1/3/4."""

    base: SynthParams        # config-1 modes (grid, comps, K = 75, m, lambda, b, amp, kvec, theta)
    ell: int
    g_amp: np.ndarray        # ell x comps real
    g_kvec: np.ndarray       # ell x comps x 3 (wavenumbers in [1, 4]: smooth)
    g_theta: np.ndarray      # ell x comps x 3
    P: np.ndarray            # K x ell complex: z-coordinates of F^+ g_k

    @property
    def n(self):
        return self.base.n

    @property
    def m(self):
        return self.base.m

    def controls(self, seed, steps=None) -> np.ndarray:
        """ell x steps control sequence u_j ~ N(0, 1), seeded."""
        steps = self.m - 1 if steps is None else steps
        return np.random.default_rng(seed).standard_normal((self.ell, steps))

    def trajectory(self, u: np.ndarray, z0=None) -> np.ndarray:
        """Mode coordinates z_j, j = 0..len(u) (K x (s+1) complex)."""
        K, s = self.base.modes, u.shape[1]
        z = np.empty((K, s + 1), dtype=np.complex128)
        z[:, 0] = self.base.b if z0 is None else z0
        for j in range(s):
            z[:, j + 1] = self.base.lam * z[:, j] + self.P @ u[:, j]
        return z

    def sep_tables(self, u: np.ndarray, z0=None):
        """(sx, sy, sz, A) for the separable generator: one column per state
        of the trajectory driven by u."""
        b = self.base
        z = self.trajectory(u, z0)
        sx, sy, sz = _sin_tables(b.kvec, b.theta, b.grid)
        return sx, sy, sz, np.real(b.amp[:, :, None] * z[:, None, :])

    def true_operator_eigs(self) -> np.ndarray:
        """The nonzero spectrum of A: config 1's lambda and their conjugates."""
        return np.concatenate([self.base.lam, np.conj(self.base.lam)])


def _field_gram(kA, thA, aA, kB, thB, aB, N):
    """<f_a, f_b> over the N^3 x comps grid for separable fields
    f(x) = amp_c prod_d sin(2 pi k_cd x_d / N + th_cd) (amplitudes broadcast
    per component): sums over x factor into three 1-D sums per component."""
    x = np.arange(N)
    G = np.zeros((kA.shape[0], kB.shape[0]), dtype=np.result_type(aA, aB, np.float64))
    for c in range(kA.shape[1]):
        prod = np.ones((kA.shape[0], kB.shape[0]))
        for d in range(3):
            sa = np.sin(2.0 * np.pi * kA[:, c, d, None] * x[None, :] / N + thA[:, c, d, None])
            sb = np.sin(2.0 * np.pi * kB[:, c, d, None] * x[None, :] / N + thB[:, c, d, None])
            prod *= sa @ sb.T
        G += aA[:, c, None] * aB[None, :, c] * prod
    return G


def config2_params(seed: int = 2, grid=None, ell: int = 8) -> ControlledParams:
    base = config_params(1, seed=seed, grid=grid)
    rng = np.random.default_rng(seed + 1000)
    N, C = base.grid, base.comps
    g_amp = rng.standard_normal((ell, C))
    g_kvec = rng.integers(1, 5, size=(ell, C, 3))
    g_theta = rng.uniform(0.0, 2.0 * np.pi, size=(ell, C, 3))
    # real mode fields R_i = Re(amp_i) s_i, I_i = Im(amp_i) s_i; x = sum R_i Re z_i - I_i Im z_i
    kF = np.concatenate([base.kvec, base.kvec])
    thF = np.concatenate([base.theta, base.theta])
    aF = np.concatenate([base.amp.real, base.amp.imag])
    FtF = _field_gram(kF, thF, aF, kF, thF, aF, N)
    FtG = _field_gram(kF, thF, aF, g_kvec, g_theta, g_amp, N)
    beta = np.linalg.solve(FtF, FtG)                      # 2K x ell: g_k's projection on [R | I]
    K = base.modes
    P = beta[:K] - 1j * beta[K:]
    p = ControlledParams(base, ell, g_amp, g_kvec, g_theta, P)
    return p


def generate_host_tables(tables, n: int, comps: int, grid: int, row0: int = 0, rows=None,
                         dtype=np.float32) -> np.ndarray:
    """Rows of sum_i sx[i,c,x] sy[i,c,y] sz[i,c,z] A[i,c,j] (row = c N^3 + (z N + y) N + x),
    fp64 on the host, cast to dtype (the device generator's formula, no noise)."""
    sx, sy, sz, A = tables
    rows = n - row0 if rows is None else rows
    idx = np.arange(row0, row0 + rows)
    cells = grid ** 3
    c = idx // cells
    rem = idx % cells
    x, y, z = rem % grid, (rem // grid) % grid, rem // (grid * grid)
    out = np.empty((rows, A.shape[2]), dtype=np.float64)
    for cc in range(comps):
        sel = c == cc
        if sel.any():
            S = sx[:, cc, x[sel]] * sy[:, cc, y[sel]] * sz[:, cc, z[sel]]
            out[sel] = S.T @ A[:, cc, :]
    return out.astype(dtype)
