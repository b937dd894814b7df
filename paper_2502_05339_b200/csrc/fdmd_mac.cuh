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

// One CTA per TJ cell rows: the faces those rows need (u rows j0..j0+TJ-1,
// v rows j0..j0+TJ) are decoded into shared memory once (HBM-coalesced over
// the column-major table, one face per thread per pass), then centred.
template <typename T>
__global__ void __launch_bounds__(256) mac_decode_kernel(const T* __restrict__ D, int64_t ldd, int ncol,
                                                         const double* __restrict__ coef, int nx, int ny, int TJ,
                                                         int field, double* __restrict__ out) {
  extern __shared__ __align__(16) double msm[];
  double* cs = msm;                          // ncol
  double* us = cs + ((ncol + 1) & ~1);       // TJ x (nx+1)
  double* vs = us + (int64_t)TJ * (nx + 1);  // (TJ+1) x nx
  for (int k = threadIdx.x; k < ncol; k += blockDim.x) cs[k] = coef[k];
  __syncthreads();
  const int j0 = blockIdx.x * TJ;
  const int rows = min(TJ, ny - j0);
  const int64_t n_u = (int64_t)(nx + 1) * ny;
  const int nu_loc = rows * (nx + 1), nv_loc = (rows + 1) * nx;
  for (int e = threadIdx.x; e < nu_loc + nv_loc; e += blockDim.x) {
    const int64_t idx = e < nu_loc ? (int64_t)j0 * (nx + 1) + e : n_u + (int64_t)j0 * nx + (e - nu_loc);
    double acc = 0.0;
    const T* d = D + idx;
#pragma unroll 4
    for (int k = 0; k < ncol; ++k) acc = fma((double)d[(int64_t)k * ldd], cs[k], acc);
    if (e < nu_loc) us[e] = acc;
    else vs[e - nu_loc] = acc;
  }
  __syncthreads();
  const int64_t plane = (int64_t)nx * ny;
  for (int e = threadIdx.x; e < rows * nx; e += blockDim.x) {
    const int jj = e / nx, i = e - jj * nx;
    // 0.5 * (u[:, :-1] + u[:, 1:]), 0.5 * (v[:-1, :] + v[1:, :])
    const double uc = __dmul_rn(0.5, __dadd_rn(us[jj * (nx + 1) + i], us[jj * (nx + 1) + i + 1]));
    const double vc = __dmul_rn(0.5, __dadd_rn(vs[jj * nx + i], vs[(jj + 1) * nx + i]));
    const int64_t o = (int64_t)(j0 + jj) * nx + i;
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
