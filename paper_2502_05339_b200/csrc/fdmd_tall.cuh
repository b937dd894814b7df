// FP64 DMMA contractions for the tall-skinny products of the fit.
// Included by fdmd_kernels.cu.
//
// Shared-memory layout rule (both kernels): a DMMA m8n8k4 fragment read is
// 4 rows (t = lane&3) x 8 consecutive doubles (g = lane>>2), executed as two
// half-warp phases of 4 rows x 4 doubles (32 B each). A row stride of 4 mod 16
// doubles (32 B mod 128 B) puts the four rows of a phase on disjoint bank
// groups, so every fragment read is the minimum 2 wavefronts. (The first
// version used 8 mod 16 and measured 2x excess wavefronts in ncu.)
//
// Fragments that are entirely outside the valid output (padding to the tile
// size), entirely below the diagonal of a symmetric Gram, or entirely zero
// because the small operand is upper triangular (CholeskyQR's R^-1) are
// skipped with warp-uniform branches, so the DMMA pipe only executes useful
// work; the counted flops are the algorithmic ones of SURVEY.md §8d.
#pragma once
#include "fdmd_kernels.cuh"

namespace fdmd {

// ===========================================================================
// tall_gemm: C[n x N] = A[n x K] * B[K x N]
// CTA = 8 warps (2 along M x 4 along N); warp tile 32 x 8*NF; CTA tile
// 64 x 32*NF; K streamed in chunks of 16, register double buffering;
// persistent over row tiles (grid-stride) so the pair-statistics epilogue
// keeps one partial per CTA.
// ===========================================================================
namespace tg {
constexpr int BM = 64;
constexpr int BK = 16;
constexpr int LDAR = BK + 4;   // row-major A staging: As[m][k], 20 doubles
constexpr int LDAC = BM + 4;   // k-major A staging:   As[k][m], 68 doubles
constexpr int THREADS = 256;
}  // namespace tg

template <int A_LAYOUT> struct ASmem;
template <> struct ASmem<LAYOUT_ROW> { double a[tg::BM][tg::LDAR]; };
template <> struct ASmem<LAYOUT_COL> { double a[tg::BK][tg::LDAC]; };

template <int NF, int A_LAYOUT> struct TGSmem {
  static constexpr int BN = 32 * NF;
  static constexpr int LDB_S = BN + 4;
  ASmem<A_LAYOUT> As[2];
  double Bs[2][tg::BK][LDB_S];
  double red[2][4][8 * NF / 2][3];  // cross-warp (wm) stats exchange
};

template <typename TA>
__device__ __forceinline__ void load4(const TA* p, double (&v)[4]) {
  if (sizeof(TA) == 4) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}

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
        load4(A + row * lda + k, v);
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
        load4(A + (int64_t)k * lda + row, v);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          v[q] = (k < K && row + q < n) ? to_f64(__ldg(A + (int64_t)k * lda + row + q)) : 0.0;
      }
    }
  }
  __device__ __forceinline__ void store(ASmem<A_LAYOUT>& s, int tid) {
    if (A_LAYOUT == LAYOUT_ROW) {
      const int i = tid >> 2, j = (tid & 3) * 4;
      double2* p = reinterpret_cast<double2*>(&s.a[i][j]);
      p[0] = make_double2(v[0], v[1]);
      p[1] = make_double2(v[2], v[3]);
    } else {
      const int k = tid >> 4, i = (tid & 15) * 4;
      double2* p = reinterpret_cast<double2*>(&s.a[k][i]);
      p[0] = make_double2(v[0], v[1]);
      p[1] = make_double2(v[2], v[3]);
    }
  }
};

template <int A_LAYOUT>
__device__ __forceinline__ double afrag(const ASmem<A_LAYOUT>& s, int m, int k) {
  if (A_LAYOUT == LAYOUT_ROW) return s.a[m][k];
  return s.a[k][m];
}

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
  using S = TGSmem<NF, A_LAYOUT>;
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
  // first output column of each of this warp's fragments; warp-uniform validity
  const int wcol0 = n0 + wn * 8 * NF;
  const bool upper = args.b_upper != 0;

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
      if (kc + 1 < nk) {
        la.load(A, args.lda, args.n, args.K, row0, (kc + 1) * tg::BK, tid, vec_ok);
        lb.load(args.B, args.ldb, args.K, args.N, (kc + 1) * tg::BK, n0, tid);
      } else if (tile + gridDim.x < ntiles) {
        la.load(A, args.lda, args.n, args.K, (tile + gridDim.x) * tg::BM, 0, tid, vec_ok);
        lb.load(args.B, args.ldb, args.K, args.N, 0, n0, tid);
      }
#pragma unroll
      for (int ks = 0; ks < tg::BK / 4; ++ks) {
        const int kb = kc * tg::BK + ks * 4;  // first k of this step (warp-uniform)
        if (kb >= args.K) break;
        double a[4], b[NF];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = afrag<A_LAYOUT>(sm.As[buf], wm * 32 + mi * 8 + g, ks * 4 + t);
#pragma unroll
        for (int f = 0; f < NF; ++f) b[f] = sm.Bs[buf][ks * 4 + t][wn * 8 * NF + f * 8 + g];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const int c0 = wcol0 + f * 8;
          if (c0 >= args.N) continue;                 // padded columns
          if (upper && kb > c0 + 7) continue;         // B[k][c] = 0 for k > c
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) dmma884(acc[mi][f], a[mi], b[f]);
        }
      }
      buf ^= 1;
    }

    TC* __restrict__ C = static_cast<TC*>(args.C);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int64_t row = row0 + wm * 32 + mi * 8 + g;
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int col = wcol0 + f * 8 + 2 * t;
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
    if (g == 0) {
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int u = f * 4 + t;
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
// tall_gram: partial[split] = A[rows]^T B[rows], 64x64 output tiles.
// Rows are the MMA k-dimension, streamed in chunks of 16 with register
// double-buffering; smem row-major As[row][col] with stride 68 doubles.
// ===========================================================================
namespace gr {
constexpr int T = 64;   // output tile (both dims)
constexpr int BR = 16;  // rows per chunk
constexpr int LD = T + 4;
constexpr int THREADS = 256;
}  // namespace gr

template <typename TA, int LAYOUT>
struct GramLoader {
  double v[4];
  __device__ __forceinline__ void load(const TA* __restrict__ A, int64_t lda, int64_t rend, int K,
                                       int64_t r0, int c0, int tid, bool vec_ok) {
    if (LAYOUT == LAYOUT_ROW) {
      const int rr = tid >> 4, cc = (tid & 15) * 4;
      const int64_t row = r0 + rr;
      const int col = c0 + cc;
      if (row < rend && vec_ok && col + 3 < K) {
        load4(A + row * lda + col, v);
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
        load4(A + (int64_t)col * lda + row, v);
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
      double2* p = reinterpret_cast<double2*>(&As[rr][cc]);
      p[0] = make_double2(v[0], v[1]);
      p[1] = make_double2(v[2], v[3]);
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

  int ti, tj;
  {
    int x = blockIdx.x;
    if (args.symmetric) {
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

  // warp-uniform fragment validity: in range, and (symmetric) on/above the diagonal
  bool live[4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int r = c0a + wm * 32 + mi * 8, c = c0b + wn * 16 + f * 8;
      live[mi][f] = r < args.K1 && c < args.K2 && !(args.symmetric && r > c);
    }

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
        for (int f = 0; f < 2; ++f)
          if (live[mi][f]) dmma884(acc[mi][f], a[mi], b[f]);
    }
    buf ^= 1;
  }
  double* W = args.W + (int64_t)blockIdx.y * args.K1p * args.K2p;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = c0a + wm * 32 + mi * 8 + g;
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const int j = c0b + wn * 16 + f * 8 + 2 * t;
      *reinterpret_cast<double2*>(W + (int64_t)i * args.K2p + j) = make_double2(acc[mi][f][0], acc[mi][f][1]);
    }
  }
}

// out[i][j] = beta*out[i][j] + sum_s W[s][i][j] (fixed order). Symmetric Grams
// compute 8x8 blocks on/above the diagonal only; the rest is mirrored.
__global__ void gram_reduce_kernel(const double* __restrict__ W, int splits, int K1, int K2, int K1p,
                                   int K2p, int symmetric, double* __restrict__ out, int64_t ldo,
                                   double beta) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (i >= K1 || j >= K2) return;
  int si = i, sj = j;
  if (symmetric && (i >> 3) > (j >> 3)) { si = j; sj = i; }
  double s = 0.0;
  for (int p = 0; p < splits; ++p) s += W[((int64_t)p * K1p + si) * K2p + sj];
  double* o = out + (int64_t)i * ldo + j;
  *o = (beta == 0.0) ? s : beta * (*o) + s;
}

}  // namespace fdmd
