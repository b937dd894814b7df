// MAC-grid (2-D staggered) kernels for interactive serving and guided
// upscaling — SURVEY.md §8(f) rows 2-3:
//   mac_decode_kernel      decode -> cell-centred velocity / speed planes
//                          (server.py:205-214: decode, unflatten, centring, speed)
//   mac_advect_kernel      semi-Lagrangian transport of a cell-centred scalar
//                          through a decoded state (solver.py:133-150, maccormack=False,
//                          as called by server.py:232 and runtime.py:259)
//   mac_inject_kernel      nearest-face prolongation (upres.py:21-50)
//   mac_project_kernel     guide-consistency projection x = H + A^T (A A^T)^-1 (L - A H)
//                          for the face-averaging downsample A (upres.py:154-169,
//                          grid.py:195-236): A A^T is diagonal, so it is a stencil
//
// State layout (grid.py:1-18): u block ny x (nx+1) row-major, then v block
// (ny+1) x nx row-major. Arithmetic mirrors the reference's numpy expression
// order with explicit round-to-nearest intrinsics (no FMA contraction), so
// results depend on the inputs' rounding only.
#pragma once
#include "fdmd_kernels.cuh"

namespace fdmd {

constexpr int MAC_VELOCITY = 0;
constexpr int MAC_SPEED = 1;

// One CTA per tile of MAC_TY x MAC_TX cells: the faces the tile needs
// (u rows j0..j0+TY-1 x cols i0..i0+TX, v rows j0..j0+TY x cols i0..i0+TX-1)
// are decoded into shared memory (consecutive threads take consecutive faces
// of a row, so every table load is a coalesced 256-B warp access; the k loop
// keeps 8 independent loads in flight per thread), then centred. Halo
// overhead: 1/TX of the u faces and 1/TY of the v faces are decoded twice.
constexpr int MAC_TX = 128;
constexpr int MAC_TY = 8;

template <typename T>
__global__ void __launch_bounds__(256) mac_decode_kernel(const T* __restrict__ D, int64_t ldd, int ncol,
                                                         const double* __restrict__ coef, int nx, int ny,
                                                         int field, double* __restrict__ out) {
  extern __shared__ __align__(16) double msm[];
  double* cs = msm;                                  // ncol (padded to even)
  double* us = cs + ((ncol + 1) & ~1);               // TY x (TX+1)
  double* vs = us + MAC_TY * (MAC_TX + 1);           // (TY+1) x TX
  for (int k = threadIdx.x; k < ncol; k += blockDim.x) cs[k] = coef[k];
  __syncthreads();
  const int i0 = blockIdx.x * MAC_TX, j0 = blockIdx.y * MAC_TY;
  const int cols = min(MAC_TX, nx - i0), rows = min(MAC_TY, ny - j0);
  const int64_t n_u = (int64_t)(nx + 1) * ny;
  const int uw = cols + 1;
  const int nu_loc = rows * uw, nv_loc = (rows + 1) * cols;
  for (int e = threadIdx.x; e < nu_loc + nv_loc; e += blockDim.x) {
    int64_t idx;
    int slot;
    if (e < nu_loc) {
      const int jj = e / uw, ii = e - jj * uw;
      idx = (int64_t)(j0 + jj) * (nx + 1) + i0 + ii;
      slot = jj * (MAC_TX + 1) + ii;
    } else {
      const int ev = e - nu_loc, jj = ev / cols, ii = ev - jj * cols;
      idx = n_u + (int64_t)(j0 + jj) * nx + i0 + ii;
      slot = MAC_TY * (MAC_TX + 1) + jj * MAC_TX + ii;
    }
    const T* d = D + idx;
    double a0 = 0.0, a1 = 0.0;
    int k = 0;
    for (; k + 8 <= ncol; k += 8) {
      T x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = __ldcs(d + (int64_t)(k + u) * ldd);
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        a0 = fma((double)x[u], cs[k + u], a0);
        a1 = fma((double)x[u + 1], cs[k + u + 1], a1);
      }
    }
    for (; k < ncol; ++k) a0 = fma((double)__ldcs(d + (int64_t)k * ldd), cs[k], a0);
    msm[((ncol + 1) & ~1) + slot] = a0 + a1;
  }
  __syncthreads();
  const int64_t plane = (int64_t)nx * ny;
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    const int jj = e / cols, ii = e - jj * cols;
    // 0.5 * (u[:, :-1] + u[:, 1:]), 0.5 * (v[:-1, :] + v[1:, :])
    const double uc = __dmul_rn(0.5, __dadd_rn(us[jj * (MAC_TX + 1) + ii], us[jj * (MAC_TX + 1) + ii + 1]));
    const double vc = __dmul_rn(0.5, __dadd_rn(vs[jj * MAC_TX + ii], vs[(jj + 1) * MAC_TX + ii]));
    const int64_t o = (int64_t)(j0 + jj) * nx + i0 + ii;
    if (field == MAC_VELOCITY) {
      out[o] = uc;
      out[plane + o] = vc;
    } else {
      out[o] = __dsqrt_rn(__dadd_rn(__dmul_rn(uc, uc), __dmul_rn(vc, vc)));
    }
  }
}

// Clamped bilinear sample of a row-major nr x nc array at fractional
// (col, row) — solver.py:_bilinear, same clip / floor / weight order.
template <typename T>
__device__ __forceinline__ double mac_bilinear(const T* __restrict__ f, int nr, int nc, double col, double row) {
  col = fmin(fmax(col, 0.0), (double)nc - 1.0);
  row = fmin(fmax(row, 0.0), (double)nr - 1.0);
  const int i0 = min((int)col, nc - 2);
  const int j0 = min((int)row, nr - 2);
  const double tx = __dsub_rn(col, (double)i0);
  const double ty = __dsub_rn(row, (double)j0);
  const double f00 = (double)f[(int64_t)j0 * nc + i0], f10 = (double)f[(int64_t)j0 * nc + i0 + 1];
  const double f01 = (double)f[(int64_t)(j0 + 1) * nc + i0], f11 = (double)f[(int64_t)(j0 + 1) * nc + i0 + 1];
  const double sx = __dsub_rn(1.0, tx), sy = __dsub_rn(1.0, ty);
  double v = __dmul_rn(__dmul_rn(f00, sx), sy);
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(f10, tx), sy));
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(f01, sx), ty));
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(f11, tx), ty));
  return v;
}

// q_out[j][i] = q sampled at the cell centre traced back by dt through the
// velocity of `vel` (flat MAC state).
template <typename T>
__global__ void mac_advect_kernel(const T* __restrict__ vel, int nx, int ny, double h, double dt,
                                  const double* __restrict__ q, double* __restrict__ q_out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * ny) return;
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  const T* u = vel;
  const T* v = vel + (int64_t)(nx + 1) * ny;
  const double X = __dmul_rn((double)i + 0.5, h), Y = __dmul_rn((double)j + 0.5, h);
  const double up = mac_bilinear(u, ny, nx + 1, __ddiv_rn(X, h), __dsub_rn(__ddiv_rn(Y, h), 0.5));
  const double vp = mac_bilinear(v, ny + 1, nx, __dsub_rn(__ddiv_rn(X, h), 0.5), __ddiv_rn(Y, h));
  const double xb = __dsub_rn(X, __dmul_rn(dt, up));
  const double yb = __dsub_rn(Y, __dmul_rn(dt, vp));
  q_out[e] = mac_bilinear(q, ny, nx, __dsub_rn(__ddiv_rn(xb, h), 0.5), __dsub_rn(__ddiv_rn(yb, h), 0.5));
}

// fine[i] = low[inject(i)]: u face (jh, ih) copies low u face
// (jh / f, min((ih + f/2) / f, nxl)); v face (jh, ih) copies low v face
// (min((jh + f/2) / f, nyl), ih / f).
__global__ void mac_inject_kernel(const double* __restrict__ low, int nxh, int nyh, int f, int nv,
                                  int64_t ld_low, int64_t ld_fine, double* __restrict__ fine) {
  const int64_t nuh = (int64_t)(nxh + 1) * nyh, nh = nuh + (int64_t)nxh * (nyh + 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nh) return;
  const int nxl = nxh / f, nyl = nyh / f;
  const int64_t nul = (int64_t)(nxl + 1) * nyl;
  int64_t src;
  if (e < nuh) {
    const int jh = (int)(e / (nxh + 1)), ih = (int)(e - (int64_t)jh * (nxh + 1));
    src = (int64_t)(jh / f) * (nxl + 1) + min((ih + f / 2) / f, nxl);
  } else {
    const int64_t ev = e - nuh;
    const int jh = (int)(ev / nxh), ih = (int)(ev - (int64_t)jh * nxh);
    src = nul + (int64_t)min((jh + f / 2) / f, nyl) * nxl + ih / f;
  }
  for (int v = 0; v < nv; ++v) fine[v * ld_fine + e] = low[v * ld_low + src];
}

// x = H + A^T (A A^T)^-1 (L - A H). Low face l averages fine faces
// g_l(0..f-1) (weights w = 1/f, A A^T = diag(gram)); a covered fine face
// recomputes its group's gap in the reference's entry order, an uncovered
// face is copied.
__global__ void mac_project_kernel(const double* __restrict__ H, const double* __restrict__ L, int nxh, int nyh,
                                   int f, double w, double gram, double* __restrict__ x) {
  const int64_t nuh = (int64_t)(nxh + 1) * nyh, nh = nuh + (int64_t)nxh * (nyh + 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nh) return;
  const int nxl = nxh / f;
  const int64_t nul = (int64_t)(nxl + 1) * (nyh / f);
  int64_t base, stride, l;
  bool covered;
  if (e < nuh) {   // group: (jl f + t)(nxh+1) + il f
    const int jh = (int)(e / (nxh + 1)), ih = (int)(e - (int64_t)jh * (nxh + 1));
    covered = (ih % f) == 0;
    const int jl = jh / f, il = ih / f;
    base = (int64_t)(jl * f) * (nxh + 1) + (int64_t)il * f;
    stride = nxh + 1;
    l = (int64_t)jl * (nxl + 1) + il;
  } else {         // group: nuh + (jl f) nxh + il f + t
    const int64_t ev = e - nuh;
    const int jh = (int)(ev / nxh), ih = (int)(ev - (int64_t)jh * nxh);
    covered = (jh % f) == 0;
    const int jl = jh / f, il = ih / f;
    base = nuh + (int64_t)(jl * f) * nxh + (int64_t)il * f;
    stride = 1;
    l = nul + (int64_t)jl * nxl + il;
  }
  const double he = H[e];
  if (!covered) {
    x[e] = he;
    return;
  }
  double s = 0.0;
  for (int t = 0; t < f; ++t) s = __dadd_rn(s, __dmul_rn(w, H[base + t * stride]));
  const double y = __ddiv_rn(__dsub_rn(L[l], s), gram);
  x[e] = __dadd_rn(he, __dmul_rn(w, y));
}

}  // namespace fdmd
