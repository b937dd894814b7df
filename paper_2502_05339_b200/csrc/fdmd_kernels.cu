// B200 (sm_100a) kernels for the DMD hot path. See fdmd_kernels.cuh.
#include "fdmd_kernels.cuh"

#include <cfloat>
#include <cstdio>

namespace fdmd {

// ===========================================================================
// tall_gemm: C[n x N] = A[n x K] * B[K x N], FP64 DMMA, fp32/fp64 A and C.
//
// CTA = 8 warps (2 along M x 4 along N); warp tile 32 x 8*NF; CTA tile
// 64 x 32*NF; K streamed in chunks of 16 with register double buffering.
// Persistent over row tiles (grid-stride), so the pair-statistics epilogue
// keeps one partial per CTA. A is converted to fp64 on its way into smem,
// which is stored k-major (As[k][m]) with a row stride = 8 mod 16 doubles so
// the fragment reads (4 k-rows x 8 contiguous m) hit distinct banks.
// ===========================================================================
namespace tg {
constexpr int BM = 64;
constexpr int BK = 16;
constexpr int LDA_S = BM + 8;  // 72 doubles
constexpr int THREADS = 256;
}  // namespace tg

template <int NF> struct TGSmem {
  static constexpr int BN = 32 * NF;
  static constexpr int LDB_S = BN + 8;
  double As[2][tg::BK][tg::LDA_S];
  double Bs[2][tg::BK][LDB_S];
  double red[2][4][8 * NF / 2][3];  // cross-warp (wm) stats exchange
};

template <typename TA, int A_LAYOUT>
struct ATileLoader {
  // Each thread owns 4 elements of the 64 x 16 chunk.
  double v[4];
  __device__ __forceinline__ void load(const TA* __restrict__ A, int64_t lda, int64_t n, int K,
                                       int64_t row0, int k0, int tid, bool vec_ok) {
    if (A_LAYOUT == LAYOUT_ROW) {
      const int i = tid >> 2, j = (tid & 3) * 4;
      const int64_t row = row0 + i;
      const int k = k0 + j;
      if (row < n && vec_ok && k + 3 < K) {
        const TA* p = A + row * lda + k;
        if (sizeof(TA) == 4) {
          float4 f = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
          double2 a = __ldg(reinterpret_cast<const double2*>(p));
          double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
          v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          v[q] = (row < n && k + q < K) ? to_f64(__ldg(A + row * lda + k + q)) : 0.0;
      }
    } else {
      const int k = k0 + (tid >> 4);
      const int i = (tid & 15) * 4;
      const int64_t row = row0 + i;
      if (k < K && vec_ok && row + 3 < n) {
        const TA* p = A + (int64_t)k * lda + row;
        if (sizeof(TA) == 4) {
          float4 f = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
          double2 a = __ldg(reinterpret_cast<const double2*>(p));
          double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
          v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          v[q] = (k < K && row + q < n) ? to_f64(__ldg(A + (int64_t)k * lda + row + q)) : 0.0;
      }
    }
  }
  __device__ __forceinline__ void store(double (*As)[tg::LDA_S], int tid) {
    if (A_LAYOUT == LAYOUT_ROW) {
      const int i = tid >> 2, j = (tid & 3) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) As[j + q][i] = v[q];
    } else {
      const int k = tid >> 4, i = (tid & 15) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) As[k][i + q] = v[q];
    }
  }
};

template <int NF>
struct BTileLoader {
  static constexpr int BN = 32 * NF;
  static constexpr int PER = (tg::BK * BN) / tg::THREADS;  // = 2*NF
  double v[PER];
  __device__ __forceinline__ void load(const double* __restrict__ B, int64_t ldb, int K, int N,
                                       int k0, int n0, int tid) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * tg::THREADS;
      const int kk = e / BN, jj = e % BN;
      const int k = k0 + kk, j = n0 + jj;
      v[q] = (k < K && j < N) ? __ldg(B + (int64_t)k * ldb + j) : 0.0;
    }
  }
  template <int LDB_S>
  __device__ __forceinline__ void store(double (*Bs)[LDB_S], int tid) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + q * tg::THREADS;
      Bs[e / BN][e % BN] = v[q];
    }
  }
};

template <typename TA, int A_LAYOUT, int NF, typename TC, int C_LAYOUT, bool STATS>
__global__ void __launch_bounds__(tg::THREADS, 1) tall_gemm_kernel(TallGemmArgs args) {
  using S = TGSmem<NF>;
  constexpr int BN = S::BN;
  constexpr int LDB_S = S::LDB_S;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const TA* __restrict__ A = static_cast<const TA*>(args.A);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int n0 = blockIdx.y * BN;
  const int64_t ntiles = (args.n + tg::BM - 1) / tg::BM;
  const int nk = (args.K + tg::BK - 1) / tg::BK;
  const bool vec_ok =
      ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
      ((args.lda * (int64_t)sizeof(TA)) % 16 == 0);

  // per-thread stats: NF frags, each frag's lane covers unit (col 2t,2t+1)
  double st_sum[NF], st_max[NF];
  int64_t st_idx[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) { st_sum[f] = 0.0; st_max[f] = -1.0; st_idx[f] = INT64_MAX; }

  ATileLoader<TA, A_LAYOUT> la;
  BTileLoader<NF> lb;

  int64_t tile = blockIdx.x;
  if (tile < ntiles) {
    la.load(A, args.lda, args.n, args.K, tile * tg::BM, 0, tid, vec_ok);
    lb.load(args.B, args.ldb, args.K, args.N, 0, n0, tid);
  }
  int buf = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t row0 = tile * tg::BM;
    double acc[4][NF][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[mi][f][0] = acc[mi][f][1] = 0.0;

    for (int kc = 0; kc < nk; ++kc) {
      la.store(sm.As[buf], tid);
      lb.template store<LDB_S>(sm.Bs[buf], tid);
      __syncthreads();
      // prefetch the next chunk (or the next tile's first chunk)
      if (kc + 1 < nk) {
        la.load(A, args.lda, args.n, args.K, row0, (kc + 1) * tg::BK, tid, vec_ok);
        lb.load(args.B, args.ldb, args.K, args.N, (kc + 1) * tg::BK, n0, tid);
      } else if (tile + gridDim.x < ntiles) {
        la.load(A, args.lda, args.n, args.K, (tile + gridDim.x) * tg::BM, 0, tid, vec_ok);
        lb.load(args.B, args.ldb, args.K, args.N, 0, n0, tid);
      }
#pragma unroll
      for (int ks = 0; ks < tg::BK / 4; ++ks) {
        double a[4], b[NF];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = sm.As[buf][ks * 4 + t][wm * 32 + mi * 8 + g];
#pragma unroll
        for (int f = 0; f < NF; ++f) b[f] = sm.Bs[buf][ks * 4 + t][wn * 8 * NF + f * 8 + g];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int f = 0; f < NF; ++f) dmma884(acc[mi][f], a[mi], b[f]);
      }
      buf ^= 1;
    }

    // epilogue: store C (+ pair statistics)
    TC* __restrict__ C = static_cast<TC*>(args.C);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int64_t row = row0 + wm * 32 + mi * 8 + g;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int col = n0 + wn * 8 * NF + f * 8 + 2 * t;
        if (row < args.n) {
          if (C != nullptr) {
            if (C_LAYOUT == LAYOUT_ROW) {
              TC* p = C + row * args.ldc + col;
              if (col < args.N) p[0] = (TC)acc[mi][f][0];
              if (col + 1 < args.N) p[1] = (TC)acc[mi][f][1];
            } else {
              if (col < args.N) C[(int64_t)col * args.ldc + row] = (TC)acc[mi][f][0];
              if (col + 1 < args.N) C[(int64_t)(col + 1) * args.ldc + row] = (TC)acc[mi][f][1];
            }
          }
          if (STATS) {
            const double v = acc[mi][f][0] * acc[mi][f][0] + acc[mi][f][1] * acc[mi][f][1];
            st_sum[f] += v;
            if (v > st_max[f]) { st_max[f] = v; st_idx[f] = row + args.row_offset; }
          }
        }
      }
    }
  }

  if (STATS) {
    // reduce over the 8 g-lanes sharing t (fixed butterfly order)
#pragma unroll
    for (int f = 0; f < NF; ++f) {
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, st_sum[f], off);
        const double om = __shfl_xor_sync(0xffffffffu, st_max[f], off);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, st_idx[f], off);
        st_sum[f] += os;
        if (om > st_max[f] || (om == st_max[f] && oi < st_idx[f])) { st_max[f] = om; st_idx[f] = oi; }
      }
    }
    // combine the two wm warps through smem: unit index within warp's N slice
    if (g == 0) {
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int u = f * 4 + t;  // unit within this warp's 8*NF columns
        sm.red[wm][wn][u][0] = st_sum[f];
        sm.red[wm][wn][u][1] = st_max[f];
        sm.red[wm][wn][u][2] = __longlong_as_double((long long)st_idx[f]);
      }
    }
    __syncthreads();
    const int units_cta = BN / 2;
    for (int e = tid; e < units_cta; e += tg::THREADS) {
      const int wn_ = e / (4 * NF), u = e % (4 * NF);
      double s0 = sm.red[0][wn_][u][0], m0 = sm.red[0][wn_][u][1];
      long long i0 = __double_as_longlong(sm.red[0][wn_][u][2]);
      const double s1 = sm.red[1][wn_][u][0], m1 = sm.red[1][wn_][u][1];
      const long long i1 = __double_as_longlong(sm.red[1][wn_][u][2]);
      s0 += s1;
      if (m1 > m0 || (m1 == m0 && i1 < i0)) { m0 = m1; i0 = i1; }
      const int gunit = (n0 >> 1) + e;
      if (2 * gunit < args.N) {
        double* out = args.pair_stats + ((int64_t)blockIdx.x * (args.N / 2) + gunit) * 3;
        out[0] = s0; out[1] = m0; out[2] = __longlong_as_double(i0);
      }
    }
  }
}

// pair_stats partials [P][U][3] -> [U][3] in fixed order (argmax ties -> lowest row)
__global__ void pair_stats_reduce_kernel(const double* __restrict__ part, int P, int U,
                                         double* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= U) return;
  double s = 0.0, m = -1.0;
  long long idx = LLONG_MAX;
  for (int p = 0; p < P; ++p) {
    const double* q = part + ((int64_t)p * U + u) * 3;
    s += q[0];
    const long long qi = __double_as_longlong(q[2]);
    if (q[1] > m || (q[1] == m && qi < idx)) { m = q[1]; idx = qi; }
  }
  out[u * 3 + 0] = s;
  out[u * 3 + 1] = m;
  out[u * 3 + 2] = (double)idx;
}

// ===========================================================================
// tall_gram: partial[split] = A[rows]^T B[rows], 64x64 output tiles, FP64 DMMA.
// Rows are the MMA k-dimension, streamed in chunks of 16 with register
// double-buffering. smem is row-major (As[row][col]), stride 72 doubles.
// ===========================================================================
namespace gr {
constexpr int T = 64;   // output tile (both dims)
constexpr int BR = 16;  // rows per chunk
constexpr int LD = T + 8;
constexpr int THREADS = 256;
}  // namespace gr

template <typename TA, int LAYOUT>
struct GramLoader {
  double v[4];
  // chunk: rows [r0, r0+16) x cols [c0, c0+64) -> v holds 4 elements
  __device__ __forceinline__ void load(const TA* __restrict__ A, int64_t lda, int64_t rend, int K,
                                       int64_t r0, int c0, int tid, bool vec_ok) {
    if (LAYOUT == LAYOUT_ROW) {
      const int rr = tid >> 4, cc = (tid & 15) * 4;
      const int64_t row = r0 + rr;
      const int col = c0 + cc;
      if (row < rend && vec_ok && col + 3 < K) {
        const TA* p = A + row * lda + col;
        if (sizeof(TA) == 4) {
          float4 f = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
          double2 a = __ldg(reinterpret_cast<const double2*>(p));
          double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
          v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          v[q] = (row < rend && col + q < K) ? to_f64(__ldg(A + row * lda + col + q)) : 0.0;
      }
    } else {
      const int cc = tid >> 2, rr = (tid & 3) * 4;
      const int col = c0 + cc;
      const int64_t row = r0 + rr;
      if (col < K && vec_ok && row + 3 < rend) {
        const TA* p = A + (int64_t)col * lda + row;
        if (sizeof(TA) == 4) {
          float4 f = __ldg(reinterpret_cast<const float4*>(p));
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
          double2 a = __ldg(reinterpret_cast<const double2*>(p));
          double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
          v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          v[q] = (col < K && row + q < rend) ? to_f64(__ldg(A + (int64_t)col * lda + row + q)) : 0.0;
      }
    }
  }
  __device__ __forceinline__ void store(double (*As)[gr::LD], int tid) {
    if (LAYOUT == LAYOUT_ROW) {
      const int rr = tid >> 4, cc = (tid & 15) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) As[rr][cc + q] = v[q];
    } else {
      const int cc = tid >> 2, rr = (tid & 3) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) As[rr + q][cc] = v[q];
    }
  }
};

template <typename TA, int LA, typename TB, int LB>
__global__ void __launch_bounds__(gr::THREADS, 2) tall_gram_kernel(TallGramArgs args) {
  __shared__ __align__(16) double As[2][gr::BR][gr::LD];
  __shared__ __align__(16) double Bs[2][gr::BR][gr::LD];
  const TA* __restrict__ A = static_cast<const TA*>(args.A);
  const TB* __restrict__ B = static_cast<const TB*>(args.B);

  // map blockIdx.x -> (ti, tj)
  int ti, tj;
  {
    int x = blockIdx.x;
    if (args.symmetric) {
      // upper-triangular enumeration: row ti has (tiles_j - ti) tiles
      ti = 0;
      int rowlen = args.tiles_j;
      while (x >= rowlen) { x -= rowlen; ++ti; --rowlen; }
      tj = ti + x;
    } else {
      ti = x / args.tiles_j;
      tj = x % args.tiles_j;
    }
  }
  const int c0a = ti * gr::T, c0b = tj * gr::T;
  const int64_t rbeg = (int64_t)blockIdx.y * args.rows_per_split;
  const int64_t rend = min(args.n, rbeg + args.rows_per_split);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const bool vec_a = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((args.lda * (int64_t)sizeof(TA)) % 16 == 0);
  const bool vec_b = ((reinterpret_cast<uintptr_t>(B) & 15) == 0) && ((args.ldb * (int64_t)sizeof(TB)) % 16 == 0);

  double acc[4][2][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int f = 0; f < 2; ++f) acc[mi][f][0] = acc[mi][f][1] = 0.0;

  GramLoader<TA, LA> la;
  GramLoader<TB, LB> lb;
  const int64_t nchunks = rend > rbeg ? (rend - rbeg + gr::BR - 1) / gr::BR : 0;
  if (nchunks > 0) {
    la.load(A, args.lda, rend, args.K1, rbeg, c0a, tid, vec_a);
    lb.load(B, args.ldb, rend, args.K2, rbeg, c0b, tid, vec_b);
  }
  int buf = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    la.store(As[buf], tid);
    lb.store(Bs[buf], tid);
    __syncthreads();
    if (c + 1 < nchunks) {
      const int64_t r0 = rbeg + (c + 1) * gr::BR;
      la.load(A, args.lda, rend, args.K1, r0, c0a, tid, vec_a);
      lb.load(B, args.ldb, rend, args.K2, r0, c0b, tid, vec_b);
    }
#pragma unroll
    for (int ks = 0; ks < gr::BR / 4; ++ks) {
      double a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[buf][ks * 4 + t][wm * 32 + mi * 8 + g];
#pragma unroll
      for (int f = 0; f < 2; ++f) b[f] = Bs[buf][ks * 4 + t][wn * 16 + f * 8 + g];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int f = 0; f < 2; ++f) dmma884(acc[mi][f], a[mi], b[f]);
    }
    buf ^= 1;
  }
  // write partial tile
  double* W = args.W + (int64_t)blockIdx.y * args.K1p * args.K2p;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = c0a + wm * 32 + mi * 8 + g;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int j = c0b + wn * 16 + f * 8 + 2 * t;
      double2 v = make_double2(acc[mi][f][0], acc[mi][f][1]);
      *reinterpret_cast<double2*>(W + (int64_t)i * args.K2p + j) = v;
    }
  }
}

// out[i][j] = beta*out[i][j] + sum_s W[s][i][j]  (fixed order); symmetric mirrors upper
__global__ void gram_reduce_kernel(const double* __restrict__ W, int splits, int K1, int K2, int K1p,
                                   int K2p, int symmetric, double* __restrict__ out, int64_t ldo,
                                   double beta) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (i >= K1 || j >= K2) return;
  int si = i, sj = j;
  if (symmetric && (i / gr::T) > (j / gr::T)) { si = j; sj = i; }
  double s = 0.0;
  for (int p = 0; p < splits; ++p) s += W[((int64_t)p * K1p + si) * K2p + sj];
  double* o = out + (int64_t)i * ldo + j;
  *o = (beta == 0.0) ? s : beta * (*o) + s;
}

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
  extern __shared__ __align__(16) unsigned char smem_raw[];
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
