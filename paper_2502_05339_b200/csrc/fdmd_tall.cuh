// FP64 DMMA contractions for the tall-skinny products of the fit.
// Included by fdmd_kernels.cu.
//
// Pipeline: a 4-stage cp.async ring streams raw (fp32 or fp64) operand tiles
// into shared memory; fragments are converted to fp64 at read time, so no
// register ever waits on HBM at a prefetch point and the loads run three
// chunks ahead of the DMMA work. Tails are zero-filled by cp.async (src-size),
// never read from padding.
//
// Shared-memory layout rule: every DMMA m8n8k4 fragment read (4 k x 8 m
// elements per warp) must hit distinct bank groups. With raw-type staging the
// required row stride depends on the element size and on which index is
// contiguous; each stage type below states its stride. Fragments entirely in
// padding, below the diagonal of a symmetric Gram, or zero because the small
// operand is upper triangular (CholeskyQR's R^-1) are skipped with warp-
// uniform branches, so the DMMA pipe executes only algorithmic work.
#pragma once
#include "fdmd_kernels.cuh"

namespace fdmd {

// ------------------------------------------------------------- cp.async ----
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ int clamp_valid(int64_t rem, int V) {
  return rem <= 0 ? 0 : (rem < V ? (int)rem : V);
}

// Copy `vlen` consecutive elements starting at gmem (of which `valid` are in
// bounds) into smem; vectorised (16 B) when `vec`, element-wise otherwise.
template <typename T>
__device__ __forceinline__ void cp_vec(T* smem, const T* gmem, int valid, bool vec, const T* safe) {
  constexpr int V = 16 / sizeof(T);
  if (vec) {
    cp_async16(smem, valid > 0 ? gmem : safe, valid > 0 ? valid * (int)sizeof(T) : 0);
  } else {
#pragma unroll
    for (int q = 0; q < V; ++q)
      cp_async_small<sizeof(T)>(smem + q, q < valid ? gmem + q : safe, q < valid ? (int)sizeof(T) : 0);
  }
}

// ===========================================================================
// tall_gemm: C[n x N] = A[n x K] * B[K x N]
// CTA = 8 warps (2 along M x 4 along N); warp tile 32 x 8*NF; CTA tile
// 64 x 32*NF; K in chunks of 16; persistent over row tiles (grid-stride) with
// one flat (tile, chunk) pipeline, so loads run ahead across tile boundaries
// and the pair-statistics epilogue keeps one partial per CTA.
// ===========================================================================
namespace tg {
constexpr int BM = 64;
constexpr int BK = 16;
constexpr int STAGES = 4;
constexpr int THREADS = 256;
}  // namespace tg

// A stage. ROW: a[m][k], stride 20 elements (fp32: 80 B = 16 mod 128 -> the 8
// rows x 16 B of a fragment read are distinct; fp64: 160 B = 32 mod 128 -> each
// half-warp's 4 rows x 32 B are distinct). COL: a[k][m], stride 72 floats
// (288 B) or 68 doubles (544 B), both 32 mod 128 B.
template <typename TA, int AL> struct AStage;
template <typename TA> struct AStage<TA, LAYOUT_ROW> {
  static constexpr int LD = 20;
  TA a[tg::BM][LD];
  __device__ __forceinline__ double frag(int m, int k) const { return (double)a[m][k]; }
};
template <typename TA> struct AStage<TA, LAYOUT_COL> {
  static constexpr int LD = sizeof(TA) == 4 ? 72 : 68;
  TA a[tg::BK][LD];
  __device__ __forceinline__ double frag(int m, int k) const { return (double)a[k][m]; }
};

template <typename TA, int AL, int NF> struct TGSmem {
  static constexpr int BN = 32 * NF;
  static constexpr int LDB = BN + 4;  // 4 mod 16 doubles
  AStage<TA, AL> As[tg::STAGES];
  double Bs[tg::STAGES][tg::BK][LDB];
  double red[2][4][8 * NF / 2][3];    // cross-warp (wm) statistics exchange
};

template <typename TA, int AL>
__device__ __forceinline__ void tg_load_a(AStage<TA, AL>& st, const TA* __restrict__ A, int64_t lda, int64_t n,
                                          int K, int64_t row0, int k0, int tid, bool vec) {
  constexpr int V = 16 / sizeof(TA);
  if (AL == LAYOUT_ROW) {
    constexpr int VPR = tg::BK / V;                 // vectors per row
    constexpr int PER = tg::BM * VPR / tg::THREADS;  // 1 (fp32) or 2 (fp64)
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = tid + p * tg::THREADS;
      const int i = e / VPR, kv = (e % VPR) * V;
      const int64_t row = row0 + i;
      const int k = k0 + kv;
      const int valid = row < n ? max(0, min(V, K - k)) : 0;
      cp_vec<TA>(&st.a[i][kv], A + row * lda + k, valid, vec, A);
    }
  } else {
    constexpr int VPR = tg::BM / V;
    constexpr int PER = tg::BK * VPR / tg::THREADS;
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = tid + p * tg::THREADS;
      const int kk = e / VPR, iv = (e % VPR) * V;
      const int k = k0 + kk;
      const int64_t row = row0 + iv;
      const int valid = k < K ? clamp_valid(n - row, V) : 0;
      cp_vec<TA>(&st.a[kk][iv], A + (int64_t)k * lda + row, valid, vec, A);
    }
  }
}

template <int NF, int LDB>
__device__ __forceinline__ void tg_load_b(double (*Bs)[LDB], const double* __restrict__ B, int64_t ldb, int K,
                                          int N, int k0, int n0, int tid, bool vec) {
  constexpr int BN = 32 * NF;
  constexpr int VPR = BN / 2;
  constexpr int PER = tg::BK * VPR / tg::THREADS;    // = NF
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int e = tid + p * tg::THREADS;
    const int kk = e / VPR, jv = (e % VPR) * 2;
    const int k = k0 + kk, j = n0 + jv;
    const int valid = k < K ? max(0, min(2, N - j)) : 0;
    cp_vec<double>(&Bs[kk][jv], B + (int64_t)k * ldb + j, valid, vec, B);
  }
}

template <typename TA, int A_LAYOUT, int NF, typename TC, int C_LAYOUT, bool STATS>
__global__ void __launch_bounds__(tg::THREADS, (NF <= 4) ? 2 : 1) tall_gemm_kernel(TallGemmArgs args) {
  using S = TGSmem<TA, A_LAYOUT, NF>;
  constexpr int BN = S::BN;
  constexpr int LDB = S::LDB;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);

  const TA* __restrict__ A = static_cast<const TA*>(args.A);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int n0 = blockIdx.y * BN;
  const int64_t ntiles = (args.n + tg::BM - 1) / tg::BM;
  const int nk = (args.K + tg::BK - 1) / tg::BK;
  const bool vec_a = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && ((args.lda * (int64_t)sizeof(TA)) % 16 == 0);
  const bool vec_b = ((reinterpret_cast<uintptr_t>(args.B) & 15) == 0) && ((args.ldb * 8) % 16 == 0);
  const int wcol0 = n0 + wn * 8 * NF;

  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total = my_tiles * nk;

  // Producer-side position (row tile, k chunk, ring stage), advanced
  // incrementally: no 64-bit division on the critical path.
  int64_t p_it = 0, p_tile = blockIdx.x;
  int p_kc = 0, p_s = 0;
  auto issue = [&]() {
    if (p_it < total && !(args.debug & 1)) {
      tg_load_a<TA, A_LAYOUT>(sm.As[p_s], A, args.lda, args.n, args.K, p_tile * tg::BM, p_kc * tg::BK, tid, vec_a);
      tg_load_b<NF, LDB>(sm.Bs[p_s], args.B, args.ldb, args.K, args.N, p_kc * tg::BK, n0, tid, vec_b);
    }
    cp_async_commit();
    ++p_it;
    p_s = (p_s + 1 == tg::STAGES) ? 0 : p_s + 1;
    if (++p_kc == nk) { p_kc = 0; p_tile += gridDim.x; }
  };

  double st_sum[NF], st_max[NF];
  int64_t st_idx[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) { st_sum[f] = 0.0; st_max[f] = -1.0; st_idx[f] = INT64_MAX; }

#pragma unroll
  for (int s = 0; s < tg::STAGES - 1; ++s) issue();

  double acc[4][NF][2];
  int kc = 0, s = 0;
  int64_t tile = blockIdx.x;
  for (int64_t it = 0; it < total; ++it) {
    cp_async_wait<tg::STAGES - 2>();
    __syncthreads();
    issue();
    if (kc == 0) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[mi][f][0] = acc[mi][f][1] = 0.0;
    }
#pragma unroll
    for (int ks = 0; ks < tg::BK / 4; ++ks) {
      // branch-free: tails are zero-filled by cp.async, so padded k-steps and
      // columns contribute exact zeros (a branch around mma.sync costs a
      // WARPSYNC/BSSY pair per fragment, measured ~2x slower)
      double a[4], b[NF];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sm.As[s].frag(wm * 32 + mi * 8 + g, ks * 4 + t);
#pragma unroll
      for (int f = 0; f < NF; ++f) b[f] = sm.Bs[s][ks * 4 + t][wn * 8 * NF + f * 8 + g];
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) dmma884(acc[mi][f], a[mi], b[f]);
    }
    if (kc == nk - 1) {
      const int64_t row0 = tile * tg::BM;
      TC* __restrict__ C = static_cast<TC*>(args.C);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int64_t row = row0 + wm * 32 + mi * 8 + g;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const int col = wcol0 + f * 8 + 2 * t;
          if (row < args.n) {
            if (C != nullptr && !(args.debug & 2)) {
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
    s = (s + 1 == tg::STAGES) ? 0 : s + 1;
    if (++kc == nk) { kc = 0; tile += gridDim.x; }
  }
  cp_async_wait<0>();

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
// tall_gram: partial[split] = A[rows]^T B[rows], 64x64 output tiles; rows are
// the MMA k-dimension, 16 per chunk, 4-stage cp.async ring.
// ===========================================================================
namespace gr {
constexpr int T = 64;   // output tile (both dims)
constexpr int BR = 16;  // rows per chunk
constexpr int STAGES = 4;
constexpr int THREADS = 256;
}  // namespace gr

// Operand stage. ROW (global row-major): s[row][col], stride 72 floats / 68
// doubles (32 mod 128 B: a fragment's 4 rows x 8 cols are distinct). COL
// (global column-major): s[col][row], stride 20 elements (fp32 80 B = 16 mod
// 128: 8 cols x 16 B distinct; fp64 160 B = 32 mod 128 per half-warp).
template <typename T, int L> struct GStage;
template <typename T> struct GStage<T, LAYOUT_ROW> {
  static constexpr int LD = sizeof(T) == 4 ? 72 : 68;
  T s[gr::BR][LD];
  __device__ __forceinline__ double frag(int col, int row) const { return (double)s[row][col]; }
};
template <typename T> struct GStage<T, LAYOUT_COL> {
  static constexpr int LD = 20;
  T s[gr::T][LD];
  __device__ __forceinline__ double frag(int col, int row) const { return (double)s[col][row]; }
};

template <typename T, int L>
__device__ __forceinline__ void gr_load(GStage<T, L>& st, const T* __restrict__ A, int64_t lda, int64_t rend,
                                        int K, int64_t r0, int c0, int tid, bool vec) {
  constexpr int V = 16 / sizeof(T);
  if (L == LAYOUT_ROW) {
    constexpr int VPR = gr::T / V;
    constexpr int PER = gr::BR * VPR / gr::THREADS;
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = tid + p * gr::THREADS;
      const int rr = e / VPR, cv = (e % VPR) * V;
      const int64_t row = r0 + rr;
      const int col = c0 + cv;
      const int valid = row < rend ? max(0, min(V, K - col)) : 0;
      cp_vec<T>(&st.s[rr][cv], A + row * lda + col, valid, vec, A);
    }
  } else {
    constexpr int VPR = gr::BR / V;
    constexpr int PER = gr::T * VPR / gr::THREADS;
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int e = tid + p * gr::THREADS;
      const int cc = e / VPR, rv = (e % VPR) * V;
      const int col = c0 + cc;
      const int64_t row = r0 + rv;
      const int valid = col < K ? clamp_valid(rend - row, V) : 0;
      cp_vec<T>(&st.s[cc][rv], A + (int64_t)col * lda + row, valid, vec, A);
    }
  }
}

template <typename TA, int LA, typename TB, int LB> struct GramSmem {
  GStage<TA, LA> a[gr::STAGES];
  GStage<TB, LB> b[gr::STAGES];
};

template <typename TA, int LA, typename TB, int LB>
__global__ void __launch_bounds__(gr::THREADS, 2) tall_gram_kernel(TallGramArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<GramSmem<TA, LA, TB, LB>*>(smem_raw);
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

  const int64_t nchunks = rend > rbeg ? (rend - rbeg + gr::BR - 1) / gr::BR : 0;
  auto issue = [&](int64_t c) {
    if (c < nchunks) {
      const int s = (int)(c % gr::STAGES);
      const int64_t r0 = rbeg + c * gr::BR;
      gr_load<TA, LA>(sm.a[s], A, args.lda, rend, args.K1, r0, c0a, tid, vec_a);
      gr_load<TB, LB>(sm.b[s], B, args.ldb, rend, args.K2, r0, c0b, tid, vec_b);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < gr::STAGES - 1; ++s) issue(s);
  for (int64_t c = 0; c < nchunks; ++c) {
    cp_async_wait<gr::STAGES - 2>();
    __syncthreads();
    issue(c + gr::STAGES - 1);
    const int s = (int)(c % gr::STAGES);
#pragma unroll
    for (int ks = 0; ks < gr::BR / 4; ++ks) {
      double a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sm.a[s].frag(wm * 32 + mi * 8 + g, ks * 4 + t);
#pragma unroll
      for (int f = 0; f < 2; ++f) b[f] = sm.b[s].frag(wn * 16 + f * 8 + g, ks * 4 + t);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int f = 0; f < 2; ++f)
          if (live[mi][f]) dmma884(acc[mi][f], a[mi], b[f]);
    }
  }
  cp_async_wait<0>();
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
// transposed: the partials hold (B^T A) (W[s][j][i], row length K2p).
__global__ void gram_reduce_kernel(const double* __restrict__ W, int splits, int K1, int K2, int K1p,
                                   int K2p, int symmetric, double* __restrict__ out, int64_t ldo,
                                   double beta, int transposed = 0) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y;
  if (i >= K1 || j >= K2) return;
  int si = i, sj = j;
  if (symmetric && (i >> 3) > (j >> 3)) { si = j; sj = i; }
  if (transposed) { const int x = si; si = sj; sj = x; }
  double s = 0.0;
  for (int p = 0; p < splits; ++p) s += W[((int64_t)p * K1p + si) * K2p + sj];
  double* o = out + (int64_t)i * ldo + j;
  *o = (beta == 0.0) ? s : beta * (*o) + s;
}

}  // namespace fdmd
