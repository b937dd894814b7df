// 2-D smoke solver on the device (reference solver.py, SURVEY.md §8(f) row 4:
// data generation for the fit). One step = sources, MacCormack advection of
// velocity / density / temperature, buoyancy, vorticity confinement, masked
// CG pressure projection (solver.py:337-355).
//
// Layout: the flat MAC state (u block ny x (nx+1), then v block (ny+1) x nx,
// grid.py:1-18); cell arrays ny x nx; all f64. Element arithmetic follows the
// reference's numpy expression order with round-to-nearest intrinsics (no
// FMA contraction); reductions (CG dot products, means) are fixed-order
// two-stage sums, so they differ from BLAS at rounding level only.
#pragma once
#include "fdmd_mac.cuh"

namespace fdmd {

// -------------------------------------------------------------- face masks --
// grid.py:face_masks: walls (u at i = 0, nx; v at j = 0, and j = ny when
// closed) and faces adjoining a solid cell.
__device__ __forceinline__ bool sol_solid(const unsigned char* solid, int nx, int j, int i) {
  return solid != nullptr && solid[(int64_t)j * nx + i] != 0;
}
__device__ __forceinline__ bool sol_u_blocked(const unsigned char* solid, int nx, int j, int i) {
  return i == 0 || i == nx || (i < nx && sol_solid(solid, nx, j, i)) || (i > 0 && sol_solid(solid, nx, j, i - 1));
}
__device__ __forceinline__ bool sol_v_blocked(const unsigned char* solid, int nx, int ny, int closed, int j, int i) {
  return j == 0 || (closed && j == ny) || (j < ny && sol_solid(solid, nx, j, i)) ||
         (j > 0 && sol_solid(solid, nx, j - 1, i));
}

__global__ void sol_mask_kernel(double* __restrict__ vel, int nx, int ny, const unsigned char* __restrict__ solid,
                                int closed) {
  const int64_t nu = (int64_t)(nx + 1) * ny, n = nu + (int64_t)nx * (ny + 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  bool blk;
  if (e < nu) {
    const int j = (int)(e / (nx + 1)), i = (int)(e - (int64_t)j * (nx + 1));
    blk = sol_u_blocked(solid, nx, j, i);
  } else {
    const int64_t ev = e - nu;
    const int j = (int)(ev / nx), i = (int)(ev - (int64_t)j * nx);
    blk = sol_v_blocked(solid, nx, ny, closed, j, i);
  }
  if (blk) vel[e] = 0.0;
}

// --------------------------------------------------------------- advection --
// Clamped bilinear sample with the four corner extrema (solver.py:79-101).
__device__ __forceinline__ double sol_bilinear_ex(const double* __restrict__ f, int nr, int nc, double col, double row,
                                                  double* lo, double* hi) {
  col = fmin(fmax(col, 0.0), (double)nc - 1.0);
  row = fmin(fmax(row, 0.0), (double)nr - 1.0);
  const int i0 = min((int)col, nc - 2);
  const int j0 = min((int)row, nr - 2);
  const double tx = __dsub_rn(col, (double)i0), ty = __dsub_rn(row, (double)j0);
  const double f00 = f[(int64_t)j0 * nc + i0], f10 = f[(int64_t)j0 * nc + i0 + 1];
  const double f01 = f[(int64_t)(j0 + 1) * nc + i0], f11 = f[(int64_t)(j0 + 1) * nc + i0 + 1];
  const double sx = __dsub_rn(1.0, tx), sy = __dsub_rn(1.0, ty);
  double v = __dmul_rn(__dmul_rn(f00, sx), sy);
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(f10, tx), sy));
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(f01, sx), ty));
  v = __dadd_rn(v, __dmul_rn(__dmul_rn(f11, tx), ty));
  if (lo) {
    *lo = fmin(fmin(f00, f10), fmin(f01, f11));
    *hi = fmax(fmax(f00, f10), fmax(f01, f11));
  }
  return v;
}

// component geometry: WHICH 0 = u faces, 1 = v faces, 2 = cell centres
struct SolComp {
  int nr, nc;           // array shape
  double ox, oy;        // position offsets in cells: x = (i + ox) h, y = (j + oy) h
  double sx, sy;        // sampler offsets: col = x / h - sx, row = y / h - sy
};
__device__ __forceinline__ SolComp sol_comp(int which, int nx, int ny) {
  if (which == 0) return {ny, nx + 1, 0.0, 0.5, 0.0, 0.5};
  if (which == 1) return {ny + 1, nx, 0.5, 0.0, 0.5, 0.0};
  return {ny, nx, 0.5, 0.5, 0.5, 0.5};
}

// velocity at the element's position (solver.py:104-108) -> (up, vp), position (X, Y)
__device__ __forceinline__ void sol_trace(const double* __restrict__ vel, int nx, int ny, double h, const SolComp& c,
                                          int j, int i, double& X, double& Y, double& up, double& vp) {
  const double* u = vel;
  const double* v = vel + (int64_t)(nx + 1) * ny;
  X = c.ox == 0.0 ? __dmul_rn((double)i, h) : __dmul_rn((double)i + 0.5, h);
  Y = c.oy == 0.0 ? __dmul_rn((double)j, h) : __dmul_rn((double)j + 0.5, h);
  up = mac_bilinear(u, ny, nx + 1, __ddiv_rn(X, h), __dsub_rn(__ddiv_rn(Y, h), 0.5));
  vp = mac_bilinear(v, ny + 1, nx, __dsub_rn(__ddiv_rn(X, h), 0.5), __ddiv_rn(Y, h));
}
__device__ __forceinline__ double sol_col(const SolComp& c, double x, double h) {
  return c.sx == 0.0 ? __ddiv_rn(x, h) : __dsub_rn(__ddiv_rn(x, h), 0.5);
}
__device__ __forceinline__ double sol_row(const SolComp& c, double y, double h) {
  return c.sy == 0.0 ? __ddiv_rn(y, h) : __dsub_rn(__ddiv_rn(y, h), 0.5);
}

// predictor: q_hat (and the sample extrema) at the backward-traced position
__global__ void sol_advect_pred_kernel(const double* __restrict__ vel, const double* __restrict__ q, int which, int nx,
                                       int ny, double h, double dt, double* __restrict__ qhat,
                                       double* __restrict__ lo, double* __restrict__ hi) {
  const SolComp c = sol_comp(which, nx, ny);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)c.nr * c.nc) return;
  const int j = (int)(e / c.nc), i = (int)(e - (int64_t)j * c.nc);
  double X, Y, up, vp;
  sol_trace(vel, nx, ny, h, c, j, i, X, Y, up, vp);
  const double xb = __dsub_rn(X, __dmul_rn(dt, up)), yb = __dsub_rn(Y, __dmul_rn(dt, vp));
  double l, u;
  qhat[e] = sol_bilinear_ex(q, c.nr, c.nc, sol_col(c, xb, h), sol_row(c, yb, h), lo ? &l : nullptr, &u);
  if (lo) {
    lo[e] = l;
    hi[e] = u;
  }
}

// corrector: fold half the round-trip error back in, clamp to the extrema
__global__ void sol_advect_corr_kernel(const double* __restrict__ vel, const double* __restrict__ q,
                                       const double* __restrict__ qhat, const double* __restrict__ lo,
                                       const double* __restrict__ hi, int which, int nx, int ny, double h, double dt,
                                       double* __restrict__ out) {
  const SolComp c = sol_comp(which, nx, ny);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)c.nr * c.nc) return;
  const int j = (int)(e / c.nc), i = (int)(e - (int64_t)j * c.nc);
  double X, Y, up, vp;
  sol_trace(vel, nx, ny, h, c, j, i, X, Y, up, vp);
  const double xf = __dadd_rn(X, __dmul_rn(dt, up)), yf = __dadd_rn(Y, __dmul_rn(dt, vp));
  const double qb = sol_bilinear_ex(qhat, c.nr, c.nc, sol_col(c, xf, h), sol_row(c, yf, h), nullptr, nullptr);
  const double qn = __dadd_rn(qhat[e], __dmul_rn(0.5, __dsub_rn(q[e], qb)));
  out[e] = fmin(fmax(qn, lo[e]), hi[e]);
}

// ------------------------------------------------------------ source terms --
// solver.py:_emit: disk source adds rate * dt to density and temperature
__global__ void sol_emit_kernel(double* __restrict__ dens, double* __restrict__ temp, int nx, int ny, double h,
                                double cx, double cy, double r2, double dadd, double tadd) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * ny) return;
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  const double x = __dsub_rn(__dmul_rn((double)i + 0.5, h), cx), y = __dsub_rn(__dmul_rn((double)j + 0.5, h), cy);
  if (__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)) <= r2) {
    dens[e] = __dadd_rn(dens[e], dadd);
    temp[e] = __dadd_rn(temp[e], tadd);
  }
}

// solver.py:181-194: v += dt * avg_faces(-alpha rho + beta T)
__global__ void sol_buoyancy_kernel(double* __restrict__ vel, const double* __restrict__ dens,
                                    const double* __restrict__ temp, int nx, int ny, double nalpha, double beta,
                                    double dt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)(ny + 1) * nx) return;
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  auto buoy = [&](int jj) {
    const int64_t c = (int64_t)jj * nx + i;
    return __dadd_rn(__dmul_rn(nalpha, dens[c]), __dmul_rn(beta, temp[c]));
  };
  double fv;
  if (j == 0) fv = buoy(0);
  else if (j == ny) fv = buoy(ny - 1);
  else fv = __dmul_rn(0.5, __dadd_rn(buoy(j - 1), buoy(j)));
  double* v = vel + (int64_t)(nx + 1) * ny;
  v[e] = __dadd_rn(v[e], __dmul_rn(dt, fv));
}

// --------------------------------------------------- vorticity confinement --
// np.gradient with uniform spacing: central (f[k+1] - f[k-1]) / (2h) inside,
// one-sided (f[1] - f[0]) / h at the ends.
template <typename F>
__device__ __forceinline__ double sol_grad(F f, int k, int len, double h) {
  if (k == 0) return __ddiv_rn(__dsub_rn(f(1), f(0)), h);
  if (k == len - 1) return __ddiv_rn(__dsub_rn(f(len - 1), f(len - 2)), h);
  return __ddiv_rn(__dsub_rn(f(k + 1), f(k - 1)), __dmul_rn(2.0, h));
}

__global__ void sol_omega_kernel(const double* __restrict__ vel, int nx, int ny, double h, double* __restrict__ omega) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * ny) return;
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  const double* u = vel;
  const double* v = vel + (int64_t)(nx + 1) * ny;
  auto vc = [&](int ii) {
    return __dmul_rn(0.5, __dadd_rn(v[(int64_t)j * nx + ii], v[(int64_t)(j + 1) * nx + ii]));
  };
  auto uc = [&](int jj) {
    return __dmul_rn(0.5, __dadd_rn(u[(int64_t)jj * (nx + 1) + i], u[(int64_t)jj * (nx + 1) + i + 1]));
  };
  omega[e] = __dsub_rn(sol_grad(vc, i, nx, h), sol_grad(uc, j, ny, h));
}

__global__ void sol_confine_force_kernel(const double* __restrict__ omega, int nx, int ny, double h, double epsh,
                                         double* __restrict__ fx, double* __restrict__ fy) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * ny) return;
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  auto magx = [&](int ii) { return fabs(omega[(int64_t)j * nx + ii]); };
  auto magy = [&](int jj) { return fabs(omega[(int64_t)jj * nx + i]); };
  const double gx = sol_grad(magx, i, nx, h), gy = sol_grad(magy, j, ny, h);
  const double norm = __dadd_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy))), 1e-20);
  const double nxv = __ddiv_rn(gx, norm), nyv = __ddiv_rn(gy, norm);
  const double w = omega[e];
  fx[e] = __dmul_rn(epsh, __dmul_rn(nyv, w));
  fy[e] = __dmul_rn(epsh, __dmul_rn(-nxv, w));
}

__global__ void sol_confine_apply_kernel(double* __restrict__ vel, const double* __restrict__ fx,
                                         const double* __restrict__ fy, int nx, int ny, double dth) {
  const int64_t nu = (int64_t)(nx + 1) * ny, n = nu + (int64_t)nx * (ny + 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  if (e < nu) {
    const int j = (int)(e / (nx + 1)), i = (int)(e - (int64_t)j * (nx + 1));
    if (i == 0 || i == nx) return;
    const double f = __dadd_rn(fx[(int64_t)j * nx + i - 1], fx[(int64_t)j * nx + i]);
    vel[e] = __dadd_rn(vel[e], __dmul_rn(dth, f));
  } else {
    const int64_t ev = e - nu;
    const int j = (int)(ev / nx), i = (int)(ev - (int64_t)j * nx);
    if (j == 0 || j == ny) return;
    const double f = __dadd_rn(fy[(int64_t)(j - 1) * nx + i], fy[(int64_t)j * nx + i]);
    vel[e] = __dadd_rn(vel[e], __dmul_rn(dth, f));
  }
}

// ------------------------------------------------------- pressure projection --
// Poisson connection coefficients (solver.py:_face_coefficients)
__device__ __forceinline__ double sol_cx(const unsigned char* solid, int nx, int j, int i) {   // face i in 1..nx-1
  return (!sol_solid(solid, nx, j, i - 1) && !sol_solid(solid, nx, j, i)) ? 1.0 : 0.0;
}
__device__ __forceinline__ double sol_cy(const unsigned char* solid, int nx, int ny, int open, int j, int i) {
  if (j == ny) return (open && !sol_solid(solid, nx, ny - 1, i)) ? 1.0 : 0.0;   // top Dirichlet face
  return (!sol_solid(solid, nx, j - 1, i) && !sol_solid(solid, nx, j, i)) ? 1.0 : 0.0;   // j in 1..ny-1
}

// b = -div(vel) on fluid cells (0 on solids), minus `mean` on fluid cells
__global__ void sol_rhs_kernel(const double* __restrict__ vel, int nx, int ny, double h,
                               const unsigned char* __restrict__ solid, double* __restrict__ b) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * ny) return;
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  if (sol_solid(solid, nx, j, i)) {
    b[e] = 0.0;
    return;
  }
  const double* u = vel;
  const double* v = vel + (int64_t)(nx + 1) * ny;
  const int64_t uo = (int64_t)j * (nx + 1) + i;
  double d = __dsub_rn(u[uo + 1], u[uo]);
  d = __dadd_rn(d, v[(int64_t)(j + 1) * nx + i]);
  d = __dsub_rn(d, v[(int64_t)j * nx + i]);
  b[e] = -__ddiv_rn(d, h);
}

__global__ void sol_sub_mean_kernel(double* __restrict__ b, int nx, int ny, const unsigned char* __restrict__ solid,
                                    const double* __restrict__ sum, double nfluid) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * ny) return;
  if (solid && solid[e]) return;
  b[e] = __dsub_rn(b[e], __ddiv_rn(*sum, nfluid));
}

// out = A p (negative masked Laplacian / h^2, solver.py:_apply_poisson)
__global__ void sol_poisson_kernel(const double* __restrict__ p, int nx, int ny, double h2,
                                   const unsigned char* __restrict__ solid, int open, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)nx * ny) return;
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  const double pc = p[e];
  double o = 0.0;
  if (i < nx - 1) o = __dadd_rn(o, __dmul_rn(sol_cx(solid, nx, j, i + 1), __dsub_rn(p[e + 1], pc)));
  if (i > 0) o = __dsub_rn(o, __dmul_rn(sol_cx(solid, nx, j, i), __dsub_rn(pc, p[e - 1])));
  if (j < ny - 1) o = __dadd_rn(o, __dmul_rn(sol_cy(solid, nx, ny, open, j + 1, i), __dsub_rn(p[e + nx], pc)));
  if (j > 0) o = __dsub_rn(o, __dmul_rn(sol_cy(solid, nx, ny, open, j, i), __dsub_rn(pc, p[e - nx])));
  if (j == ny - 1) o = __dsub_rn(o, __dmul_rn(sol_cy(solid, nx, ny, open, ny, i), pc));
  out[e] = __ddiv_rn(-o, h2);
}

// fixed-order two-stage reductions: op 0 = sum a*b, 1 = max |a|, 2 = sum a over fluid cells
__global__ void sol_reduce_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                  const unsigned char* __restrict__ solid, int64_t n, int op,
                                  double* __restrict__ part) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    if (op == 0) acc = __dadd_rn(acc, __dmul_rn(a[e], b[e]));
    else if (op == 1) acc = fmax(acc, fabs(a[e]));
    else if (!(solid && solid[e])) acc = __dadd_rn(acc, a[e]);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      red[threadIdx.x] = op == 1 ? fmax(red[threadIdx.x], red[threadIdx.x + s])
                                 : __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void sol_reduce_final_kernel(const double* __restrict__ part, int nparts, int op, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (int k = 0; k < nparts; ++k) acc = op == 1 ? fmax(acc, part[k]) : __dadd_rn(acc, part[k]);
  *out = acc;
}

// CG updates: p += alpha d, r -= alpha Ad  |  d = r + beta d
__global__ void sol_cg_step_kernel(double* __restrict__ p, double* __restrict__ r, const double* __restrict__ d,
                                   const double* __restrict__ Ad, double alpha, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  p[e] = __dadd_rn(p[e], __dmul_rn(alpha, d[e]));
  r[e] = __dsub_rn(r[e], __dmul_rn(alpha, Ad[e]));
}
__global__ void sol_cg_dir_kernel(double* __restrict__ d, const double* __restrict__ r, double beta, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  d[e] = __dadd_rn(r[e], __dmul_rn(beta, d[e]));
}

// velocity -= cx grad p (solver.py:_project tail)
__global__ void sol_pressure_apply_kernel(double* __restrict__ vel, const double* __restrict__ p, int nx, int ny,
                                          double h, const unsigned char* __restrict__ solid, int open) {
  const int64_t nu = (int64_t)(nx + 1) * ny, n = nu + (int64_t)nx * (ny + 1);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  if (e < nu) {
    const int j = (int)(e / (nx + 1)), i = (int)(e - (int64_t)j * (nx + 1));
    if (i == 0 || i == nx) return;
    const int64_t c = (int64_t)j * nx + i;
    vel[e] = __dsub_rn(vel[e], __ddiv_rn(__dmul_rn(sol_cx(solid, nx, j, i), __dsub_rn(p[c], p[c - 1])), h));
  } else {
    const int64_t ev = e - nu;
    const int j = (int)(ev / nx), i = (int)(ev - (int64_t)j * nx);
    if (j == 0) return;
    if (j == ny) {
      vel[e] = __dadd_rn(vel[e], __ddiv_rn(__dmul_rn(sol_cy(solid, nx, ny, open, ny, i), p[(int64_t)(ny - 1) * nx + i]), h));
      return;
    }
    const int64_t c = (int64_t)j * nx + i;
    vel[e] = __dsub_rn(vel[e], __ddiv_rn(__dmul_rn(sol_cy(solid, nx, ny, open, j, i), __dsub_rn(p[c], p[c - nx])), h));
  }
}

}  // namespace fdmd

namespace fdmd {

// ---------------------------------------------- single-CTA CG (small grids) --
// The whole conjugate-gradient solve of solver.py:_project (same iteration,
// break conditions and tolerance) in ONE 1024-thread CTA: vectors stay in
// L2/L1, reductions are fixed-order block tree sums, and the host reads the
// status once per solve instead of two scalars per iteration. Used for grids
// up to SOL_CG1_MAX_CELLS cells (the reference scenes: 64 x 128 .. 128 x 256).
constexpr int SOL_CG1_THREADS = 1024;
constexpr int64_t SOL_CG1_MAX_CELLS = 1 << 17;

__device__ __forceinline__ double sol_block_reduce(double v, int op, double* red) {
  // op 0: sum, 1: max
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = SOL_CG1_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      red[threadIdx.x] = op ? fmax(red[threadIdx.x], red[threadIdx.x + s]) : __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  const double out = red[0];
  __syncthreads();
  return out;
}

__device__ __forceinline__ double sol_poisson_at(const double* __restrict__ p, int nx, int ny, double h2,
                                                 const unsigned char* __restrict__ solid, int open, int64_t e) {
  const int j = (int)(e / nx), i = (int)(e - (int64_t)j * nx);
  const double pc = p[e];
  double o = 0.0;
  if (i < nx - 1) o = __dadd_rn(o, __dmul_rn(sol_cx(solid, nx, j, i + 1), __dsub_rn(p[e + 1], pc)));
  if (i > 0) o = __dsub_rn(o, __dmul_rn(sol_cx(solid, nx, j, i), __dsub_rn(pc, p[e - 1])));
  if (j < ny - 1) o = __dadd_rn(o, __dmul_rn(sol_cy(solid, nx, ny, open, j + 1, i), __dsub_rn(p[e + nx], pc)));
  if (j > 0) o = __dsub_rn(o, __dmul_rn(sol_cy(solid, nx, ny, open, j, i), __dsub_rn(pc, p[e - nx])));
  if (j == ny - 1) o = __dsub_rn(o, __dmul_rn(sol_cy(solid, nx, ny, open, ny, i), pc));
  return __ddiv_rn(-o, h2);
}

// status[0] = final max|r|, status[1] = iterations, status[2] = 1 if the loop
// ran out without a break (solver.py's for/else), status[3] = bnorm
__global__ void __launch_bounds__(SOL_CG1_THREADS, 1)
sol_cg_single_kernel(const double* __restrict__ b, double* __restrict__ p, double* __restrict__ r,
                     double* __restrict__ d, double* __restrict__ Ad, int nx, int ny, double h2,
                     const unsigned char* __restrict__ solid, int open, double cg_tol, int max_iters,
                     double* __restrict__ status) {
  __shared__ double red[SOL_CG1_THREADS];
  const int64_t n = (int64_t)nx * ny;
  const int t = threadIdx.x;
  double m = 0.0;
  for (int64_t e = t; e < n; e += SOL_CG1_THREADS) m = fmax(m, fabs(b[e]));
  const double bnorm = sol_block_reduce(m, 1, red);
  if (bnorm == 0.0) {
    if (t == 0) { status[0] = 0.0; status[1] = 0; status[2] = 0; status[3] = 0.0; }
    return;
  }
  const double tol_abs = cg_tol * bnorm;
  m = 0.0;
  for (int64_t e = t; e < n; e += SOL_CG1_THREADS) {
    const double re = __dsub_rn(b[e], sol_poisson_at(p, nx, ny, h2, solid, open, e));
    r[e] = re;
    m = fmax(m, fabs(re));
  }
  double rmax = sol_block_reduce(m, 1, red);
  int iters = 0, ran_out = 0;
  if (rmax > tol_abs) {
    double acc = 0.0;
    for (int64_t e = t; e < n; e += SOL_CG1_THREADS) {
      const double re = r[e];
      d[e] = re;
      acc = __dadd_rn(acc, __dmul_rn(re, re));
    }
    double rs = sol_block_reduce(acc, 0, red);   // also orders the d writes before A d
    ran_out = 1;
    for (iters = 1; iters <= max_iters; ++iters) {
      acc = 0.0;
      for (int64_t e = t; e < n; e += SOL_CG1_THREADS) {
        const double a = sol_poisson_at(d, nx, ny, h2, solid, open, e);
        Ad[e] = a;
        acc = __dadd_rn(acc, __dmul_rn(d[e], a));
      }
      const double dAd = sol_block_reduce(acc, 0, red);
      if (dAd <= 0.0) { ran_out = 0; break; }
      const double alpha = rs / dAd;
      m = 0.0;
      acc = 0.0;
      for (int64_t e = t; e < n; e += SOL_CG1_THREADS) {
        p[e] = __dadd_rn(p[e], __dmul_rn(alpha, d[e]));
        const double re = __dsub_rn(r[e], __dmul_rn(alpha, Ad[e]));
        r[e] = re;
        m = fmax(m, fabs(re));
        acc = __dadd_rn(acc, __dmul_rn(re, re));
      }
      rmax = sol_block_reduce(m, 1, red);
      if (rmax <= tol_abs) { ran_out = 0; break; }
      const double rs_new = sol_block_reduce(acc, 0, red);
      const double beta = rs_new / rs;
      for (int64_t e = t; e < n; e += SOL_CG1_THREADS) d[e] = __dadd_rn(r[e], __dmul_rn(beta, d[e]));
      rs = rs_new;
      __syncthreads();
    }
    if (ran_out) iters = max_iters;
  }
  if (t == 0) {
    status[0] = rmax;
    status[1] = (double)iters;
    status[2] = (double)ran_out;
    status[3] = bnorm;
  }
}

}  // namespace fdmd
