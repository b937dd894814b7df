// HBM-streaming and small helper kernels: decode/reconstruct, column-major dot,
// table apply, residual, synthetic generator, DMMA probe. Included by fdmd_kernels.cu.
#pragma once
#include "fdmd_kernels.cuh"

namespace fdmd {

// ===========================================================================
// Decode / reconstruct: out[f][i] = sum_k D[k][i] * coef[k][f]
// D is the column-major (mode-major) real table r x n (ld = ldd), coef r x B
// row-major, out frame-major B x n (ld = ldo). HBM-streaming; each thread
// owns RPT consecutive rows (vector load) and FB frames.
// ===========================================================================
template <typename T, int RPT> struct Vec;
template <> struct Vec<float, 4> { using type = float4; };
template <> struct Vec<float, 2> { using type = float2; };
template <> struct Vec<float, 1> { using type = float; };
template <> struct Vec<double, 2> { using type = double2; };
template <> struct Vec<double, 1> { using type = double; };

template <typename T, int RPT>
__device__ __forceinline__ void vload(const T* p, T (&v)[RPT]) {
  using V = typename Vec<T, RPT>::type;
  V x;
  asm volatile("" ::: "memory");
  x = __ldcs(reinterpret_cast<const V*>(p));
  const T* xs = reinterpret_cast<const T*>(&x);
#pragma unroll
  for (int q = 0; q < RPT; ++q) v[q] = xs[q];
}

template <typename T, int RPT, int FB>
__global__ void __launch_bounds__(256) decode_kernel(const T* __restrict__ D, int64_t ldd,
                                                     const T* __restrict__ coef, int ldcoef,
                                                     T* __restrict__ out, int64_t ldo, int64_t n,
                                                     int r, int B, int f0) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T* cs = reinterpret_cast<T*>(smem_raw);  // r x FB
  for (int e = threadIdx.x; e < r * FB; e += blockDim.x) {
    const int k = e / FB, f = e % FB;
    cs[e] = (f0 + f < B) ? coef[(int64_t)k * ldcoef + f0 + f] : T(0);
  }
  __syncthreads();
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * RPT;
  if (i0 >= n) return;
  T acc[FB][RPT];
#pragma unroll
  for (int f = 0; f < FB; ++f)
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[f][q] = T(0);
  const bool full = (i0 + RPT <= n) && ((ldd % RPT) == 0);
  if (full) {
    int k = 0;
    constexpr int U = (FB <= 2) ? 8 : (FB <= 8 ? 4 : 2);
    for (; k + U <= r; k += U) {
      T d[U][RPT];
#pragma unroll
      for (int u = 0; u < U; ++u) vload<T, RPT>(D + (int64_t)(k + u) * ldd + i0, d[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int f = 0; f < FB; ++f) {
          const T c = cs[(k + u) * FB + f];
#pragma unroll
          for (int q = 0; q < RPT; ++q) acc[f][q] = fma(d[u][q], c, acc[f][q]);
        }
    }
    for (; k < r; ++k) {
      T d[RPT];
      vload<T, RPT>(D + (int64_t)k * ldd + i0, d);
#pragma unroll
      for (int f = 0; f < FB; ++f)
#pragma unroll
        for (int q = 0; q < RPT; ++q) acc[f][q] = fma(d[q], cs[k * FB + f], acc[f][q]);
    }
  } else {
    for (int k = 0; k < r; ++k) {
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        if (i0 + q < n) {
          const T d = D[(int64_t)k * ldd + i0 + q];
#pragma unroll
          for (int f = 0; f < FB; ++f) acc[f][q] = fma(d, cs[k * FB + f], acc[f][q]);
        }
      }
    }
  }
#pragma unroll
  for (int f = 0; f < FB; ++f) {
    if (f0 + f >= B) break;
    T* o = out + (int64_t)(f0 + f) * ldo + i0;
    if (full && (ldo % RPT) == 0) {
      using V = typename Vec<T, RPT>::type;
      V v;
      T* vs = reinterpret_cast<T*>(&v);
#pragma unroll
      for (int q = 0; q < RPT; ++q) vs[q] = acc[f][q];
      __stcs(reinterpret_cast<V*>(o), v);
    } else {
#pragma unroll
      for (int q = 0; q < RPT; ++q)
        if (i0 + q < n) o[q] = acc[f][q];
    }
  }
}

// ===========================================================================
// Column-major dot products: y[k][v] = sum_i D[k][i] * U[v][i]   (D^T u for
// encode / pinv / control projection). Partials per split, fixed order.
// ===========================================================================
template <typename TD, typename TU, int NV>
__global__ void __launch_bounds__(256) colmajor_dot_kernel(const TD* __restrict__ D, int64_t ldd,
                                                           const TU* __restrict__ U, int64_t ldu,
                                                           int64_t n, int r, int64_t rows_per_split,
                                                           double* __restrict__ part) {
  const int k = blockIdx.x;
  const int64_t rbeg = (int64_t)blockIdx.y * rows_per_split;
  const int64_t rend = min(n, rbeg + rows_per_split);
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  for (int64_t i = rbeg + threadIdx.x; i < rend; i += blockDim.x) {
    const double d = (double)D[(int64_t)k * ldd + i];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = fma(d, (double)U[(int64_t)v * ldu + i], acc[v]);
  }
  __shared__ double red[NV][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double s = acc[v];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) red[v][w] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += red[threadIdx.x][q];
    part[((int64_t)blockIdx.y * r + k) * NV + threadIdx.x] = s;
  }
}

// ===========================================================================
// Row-major transposed dot: part[split][k] = sum_{i in split} A[i*lda+k] v[i*ldv]
// (y = A^T v over the rows; v may be a column of A itself, e.g. the last
// snapshot: the border X^T s_m of the snapshot Gram). One thread per column,
// a CTA walks its row range: each row is one coalesced read of the CTA's
// columns; v[i] is a broadcast load. HBM-bound (A read once).
// ===========================================================================
template <typename TA>
__global__ void __launch_bounds__(256) tall_tdot_kernel(const TA* __restrict__ A, int64_t lda,
                                                        const TA* __restrict__ v, int64_t ldv, int64_t n, int K,
                                                        int64_t rps, double* __restrict__ part) {
  const int64_t r0 = (int64_t)blockIdx.x * rps;
  const int64_t r1 = min(n, r0 + rps);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t i = r0;
    for (; i + 4 <= r1; i += 4) {   // four independent chains: loads stay in flight
      a0 += (double)__ldcs(A + i * lda + k) * (double)v[i * ldv];
      a1 += (double)__ldcs(A + (i + 1) * lda + k) * (double)v[(i + 1) * ldv];
      a2 += (double)__ldcs(A + (i + 2) * lda + k) * (double)v[(i + 2) * ldv];
      a3 += (double)__ldcs(A + (i + 3) * lda + k) * (double)v[(i + 3) * ldv];
    }
    for (; i < r1; ++i) a0 += (double)A[i * lda + k] * (double)v[i * ldv];
    part[(int64_t)blockIdx.x * K + k] = (a0 + a1) + (a2 + a3);
  }
}

__global__ void axpy_kernel(const double* __restrict__ x, double beta, double* __restrict__ y, int len) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < len) y[e] = beta * y[e] + x[e];
}

// y[e * ldy] = beta * y[e * ldy] + x[e] (a column of a row-major matrix; beta = 0 overwrites)
__global__ void strided_axpby_kernel(const double* __restrict__ x, double beta, double* __restrict__ y, int64_t ldy,
                                     int len) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < len) y[e * ldy] = (beta == 0.0) ? x[e] : beta * y[e * ldy] + x[e];
}

__global__ void split_sum_kernel(const double* __restrict__ part, int splits, int len,
                                 double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= len) return;
  double s = 0.0;
  for (int p = 0; p < splits; ++p) s += part[(int64_t)p * len + e];
  out[e] = s;
}

// ===========================================================================
// Table apply: D[j][i] = alpha_j * R[2u_j][i] + beta_j * R[2u_j+1][i]
// R: raw mode columns, column-major (2U x n, ld = ldr); D column-major.
// ===========================================================================
template <typename TR, typename TD>
__global__ void table_apply_kernel(const TR* __restrict__ R, int64_t ldr, const int* __restrict__ src,
                                   const double* __restrict__ alpha, const double* __restrict__ beta,
                                   TD* __restrict__ D, int64_t ldd, int64_t n, int ncols) {
  const int j = blockIdx.y;
  if (j >= ncols) return;
  const int u = src[j];
  const double a = alpha[j], b = beta[j];
  const TR* re = R + (int64_t)(2 * u) * ldr;
  const TR* im = R + (int64_t)(2 * u + 1) * ldr;
  TD* d = D + (int64_t)j * ldd;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    d[i] = (TD)(a * (double)re[i] + b * (double)im[i]);
  }
}

// In-place variant: the table overwrites the raw buffer (column j of the
// output lands in raw column j). Each block stages ITS rows of all `nraw`
// raw columns in shared memory before writing, so no block reads a value
// another block has overwritten. Saves a second n x r buffer (40 GB at
// config 3) and one HBM allocation per fit.
template <typename T>
__global__ void __launch_bounds__(256) table_apply_inplace_kernel(T* __restrict__ R, int64_t ldr, int nraw,
                                                                  const int* __restrict__ src,
                                                                  const double* __restrict__ alpha,
                                                                  const double* __restrict__ beta, int ncols,
                                                                  int64_t n, int rows_per_block) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T* s = reinterpret_cast<T*>(smem_raw);  // nraw x rows_per_block
  for (int64_t r0 = (int64_t)blockIdx.x * rows_per_block; r0 < n; r0 += (int64_t)gridDim.x * rows_per_block) {
    const int64_t left = n - r0;
    const int rows = left < rows_per_block ? (int)left : rows_per_block;
    // stage with cp.async: all loads in flight at once (a load->st.shared
    // loop serialises on each load's latency; measured 0.67 TB/s)
    constexpr int V = 16 / sizeof(T);
    const bool vec = (rows == rows_per_block) && ((ldr * (int64_t)sizeof(T)) % 16 == 0) &&
                     ((reinterpret_cast<uintptr_t>(R) & 15) == 0) && ((r0 % V) == 0);
    if (vec) {
      const int vpr = rows_per_block / V;
      for (int e = threadIdx.x; e < nraw * vpr; e += blockDim.x) {
        const int c = e / vpr, iv = (e % vpr) * V;
        cp_async16(s + c * rows_per_block + iv, R + (int64_t)c * ldr + r0 + iv, 16);
      }
    } else {
      for (int e = threadIdx.x; e < nraw * rows_per_block; e += blockDim.x) {
        const int c = e / rows_per_block, i = e % rows_per_block;
        if (i < rows) cp_async_small<sizeof(T)>(s + e, R + (int64_t)c * ldr + r0 + i, (int)sizeof(T));
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int e = threadIdx.x; e < ncols * rows_per_block; e += blockDim.x) {
      const int j = e / rows_per_block, i = e % rows_per_block;
      if (i < rows) {
        const int u = src[j];
        const double v = alpha[j] * (double)s[(2 * u) * rows_per_block + i] +
                         beta[j] * (double)s[(2 * u + 1) * rows_per_block + i];
        R[(int64_t)j * ldr + r0 + i] = (T)v;
      }
    }
    __syncthreads();
  }
}

// ===========================================================================
// Residual: part[b] = (sum_i ||S[i, 1:T+1] - D[:, i]^T F||^2, sum_i ||S[i, 1:T+1]||^2)
// per block, used for the exact_dmd one-step residual diagnostic
// (dmd.py:269-272). One thread per row; F (r x T) in smem.
// ===========================================================================
template <typename TS, typename TD>
__global__ void __launch_bounds__(256) residual_kernel(const TS* __restrict__ S, int64_t lds,
                                                       const TD* __restrict__ D, int64_t ldd,
                                                       const double* __restrict__ F, int ldf, int r, int T,
                                                       int jbase, int64_t n, double* __restrict__ part) {
  extern __shared__ double Fs[];  // r x T (chunk of columns [jbase, jbase+T))
  for (int e = threadIdx.x; e < r * T; e += blockDim.x) Fs[e] = F[(int64_t)(e / T) * ldf + e % T];
  __syncthreads();
  double local = 0.0, xnorm = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int j0 = 0; j0 < T; j0 += 16) {
      double rec[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) rec[q] = 0.0;
      for (int k = 0; k < r; ++k) {
        const double d = (double)D[(int64_t)k * ldd + i];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (j0 + q < T) rec[q] = fma(d, Fs[k * T + j0 + q], rec[q]);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (j0 + q < T) {
          const double x = (double)S[i * lds + 1 + jbase + j0 + q];
          const double e = x - rec[q];
          local = fma(e, e, local);
          xnorm = fma(x, x, xnorm);
        }
    }
  }
  __shared__ double red[2][8];
  for (int off = 16; off > 0; off >>= 1) {
    local += __shfl_down_sync(0xffffffffu, local, off);
    xnorm += __shfl_down_sync(0xffffffffu, xnorm, off);
  }
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = local; red[1][threadIdx.x >> 5] = xnorm; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int q = 0; q < 8; ++q) { s0 += red[0][q]; s1 += red[1][q]; }
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

// ===========================================================================
// Synthetic 3D separable generator (synth.py): rows [row0, row0+rows) of
//   X[row][j] = sum_i sx[i,c,x] sy[i,c,y] sz[i,c,z] A[i,c,j] + noise*N(seed,row,j)
// tables: sx/sy/sz [K][C][N] fp64, A [K][C][m] fp64; out row-major (ldo).
// ===========================================================================
__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double counter_normal(uint64_t key, uint64_t ctr) {
  const uint64_t a = splitmix(key + 2ull * ctr);
  const uint64_t b = splitmix(key + 2ull * ctr + 1ull);
  const double u1 = ((double)(a >> 11) + 0.5) * 0x1.0p-53;
  const double u2 = ((double)(b >> 11) + 0.5) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

template <typename TO>
__global__ void __launch_bounds__(256) synth3d_kernel(const double* __restrict__ sx,
                                                      const double* __restrict__ sy,
                                                      const double* __restrict__ sz,
                                                      const double* __restrict__ Am, int K, int C,
                                                      int N, int m, double noise, uint64_t key,
                                                      int64_t row0, int64_t rows,
                                                      TO* __restrict__ out, int64_t ldo) {
  const int64_t cells = (int64_t)N * N * N;
  const int jb = blockIdx.y * 8;  // 8 snapshot columns per thread
  for (int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lr < rows;
       lr += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = row0 + lr;
    const int c = (int)(row / cells);
    const int64_t rem = row % cells;
    const int x = (int)(rem % N), y = (int)((rem / N) % N), z = (int)(rem / ((int64_t)N * N));
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int i = 0; i < K; ++i) {
      const int64_t base = ((int64_t)i * C + c) * N;
      const double s = sx[base + x] * sy[base + y] * sz[base + z];
      const double* a = Am + ((int64_t)i * C + c) * m + jb;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (jb + q < m) acc[q] = fma(s, a[q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = jb + q;
      if (j < m) {
        double v = acc[q];
        if (noise != 0.0) v += noise * counter_normal(key, (uint64_t)row * (uint64_t)m + (uint64_t)j);
        out[lr * ldo + j] = (TO)v;
      }
    }
  }
}

// ===========================================================================
// FP64 tensor-pipe (DMMA) throughput probe: the roofline denominator for the
// fit contractions (MEASURED_PEAKS.json carries no FP64 figure).
// ===========================================================================
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

}  // namespace fdmd
