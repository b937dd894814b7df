// Warp-specialised tall_gemm: one producer warp feeds a STAGES-deep ring with
// TMA (A: 2-D tensor tiles, zero-filled out of bounds) and bulk copies (B: one
// 1-D copy per k-row into padded smem rows); 8 consumer warps wait on full
// mbarriers, run LDS + DMMA only, and release stages through empty mbarriers.
// Included by fdmd_kernels.cu after fdmd_tall.cuh (shares tg::, dmma884).
#pragma once
#include <cuda.h>

#include "fdmd_tall.cuh"

namespace fdmd {

namespace tt {
constexpr int BM = 64;
constexpr int BK = 16;
constexpr int STAGES = 4;
constexpr int CONSUMERS = 256;          // 8 warps, 2 (M) x 4 (N)
constexpr int THREADS = CONSUMERS + 32;  // + producer warp
}  // namespace tt

// ---------------------------------------------------------------- mbarrier --
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n"
               ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity));
}

// ---------------------------------------------------------------- TMA / bulk --
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <typename TA, int AL, int NF> struct TTSmem {
  static constexpr int BN = 32 * NF;
  static constexpr int LDB = BN + 4;                     // padded B rows (4 mod 16 doubles)
  // A as written by TMA (dense box): ROW -> a[m][k] (BM x BK), COL -> a[k][m] (BK x BM)
  TA A[tt::STAGES][tt::BM * tt::BK];
  double B[tt::STAGES][tt::BK][LDB];
  double red[2][4][8 * NF / 2][3];
  uint64_t full[tt::STAGES];
  uint64_t empty[tt::STAGES];
};

struct TTArgs {
  TallGemmArgs g;
  const double* Bp;   // padded small operand, Kp x ldbp (Kp multiple of BK, ldbp >= gridDim.y*BN)
  int64_t ldbp;
};

template <typename TA, int A_LAYOUT, int NF, typename TC, int C_LAYOUT, bool STATS>
__global__ void __launch_bounds__(tt::THREADS, 1)
tall_gemm_tma_kernel(const __grid_constant__ CUtensorMap amap, const TTArgs ta) {
  using S = TTSmem<TA, A_LAYOUT, NF>;
  constexpr int BN = S::BN;
  constexpr int LDB = S::LDB;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  const TallGemmArgs& args = ta.g;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.y * BN;
  const int64_t ntiles = (args.n + tt::BM - 1) / tt::BM;
  const int nk = (args.K + tt::BK - 1) / tt::BK;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total = my_tiles * nk;

  if (tid == 0) {
    for (int s = 0; s < tt::STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], tt::CONSUMERS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == tt::CONSUMERS / 32) {
    // ============================ producer ============================
    if (lane == 0) {
      constexpr unsigned A_BYTES = tt::BM * tt::BK * sizeof(TA);
      constexpr unsigned B_ROW = BN * sizeof(double);
      int s = 0, kc = 0;
      unsigned phase = 0;
      int64_t tile = blockIdx.x;
      for (int64_t it = 0; it < total; ++it) {
        mbar_wait(&sm.empty[s], phase ^ 1);
        mbar_expect_tx(&sm.full[s], A_BYTES + tt::BK * B_ROW);
        const int k0 = kc * tt::BK;
        if (A_LAYOUT == LAYOUT_ROW)
          tma_load_2d(sm.A[s], &amap, k0, (int)(tile * tt::BM), &sm.full[s]);
        else
          tma_load_2d(sm.A[s], &amap, (int)(tile * tt::BM), k0, &sm.full[s]);
#pragma unroll 4
        for (int kk = 0; kk < tt::BK; ++kk)
          bulk_load(&sm.B[s][kk][0], ta.Bp + (int64_t)(k0 + kk) * ta.ldbp + n0, B_ROW, &sm.full[s]);
        if (++s == tt::STAGES) { s = 0; phase ^= 1; }
        if (++kc == nk) { kc = 0; tile += gridDim.x; }
      }
    }
    return;
  }

  // ============================ consumers ============================
  // SM sub-partition = warp & 3; pairing column block wn with 3 - wn on each
  // sub-partition balances the DMMA work when B is upper triangular.
  const int wm = warp >> 2, wn = (wm == 0) ? (warp & 3) : 3 - (warp & 3);
  const int g = lane >> 2, t = lane & 3;
  const int wcol0 = n0 + wn * 8 * NF;
  // upper-triangular B (B[k][j] = 0 for k > j): k-chunks past this warp's last
  // column contribute nothing and are skipped (still consumed from the ring)
  const int kc_last = args.b_upper ? (wcol0 + 8 * NF - 1) / tt::BK : INT32_MAX;
  double st_sum[NF], st_max[NF];
  int64_t st_idx[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) { st_sum[f] = 0.0; st_max[f] = -1.0; st_idx[f] = INT64_MAX; }

  double acc[4][NF][2];
  int s = 0, kc = 0;
  unsigned phase = 0;
  int64_t tile = blockIdx.x;
  for (int64_t it = 0; it < total; ++it) {
    if (kc == 0) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[mi][f][0] = acc[mi][f][1] = 0.0;
    }
    mbar_wait(&sm.full[s], phase);
    const TA* As = sm.A[s];
    if (kc <= kc_last) {
#pragma unroll
    for (int ks = 0; ks < tt::BK / 4; ++ks) {
      double a[4], b[NF];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int m = wm * 32 + mi * 8 + g, k = ks * 4 + t;
        a[mi] = (double)(A_LAYOUT == LAYOUT_ROW ? As[m * tt::BK + k] : As[k * tt::BM + m]);
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) b[f] = sm.B[s][ks * 4 + t][wn * 8 * NF + f * 8 + g];
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) dmma884(acc[mi][f], a[mi], b[f]);
    }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    if (kc == nk - 1) {
      const int64_t row0 = tile * tt::BM;
      TC* __restrict__ C = static_cast<TC*>(args.C);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int64_t row = row0 + wm * 32 + mi * 8 + g;
        if (row < args.n) {
#pragma unroll
          for (int f = 0; f < NF; ++f) {
            const int col = wcol0 + f * 8 + 2 * t;
            if (C != nullptr && !(args.debug & 2)) {
              if (C_LAYOUT == LAYOUT_ROW) {
                TC* p = C + row * args.ldc + col;
                if (sizeof(TC) == 8 && col + 1 < args.N && ((args.ldc & 1) == 0)) {
                  *reinterpret_cast<double2*>(p) = make_double2(acc[mi][f][0], acc[mi][f][1]);
                } else {
                  if (col < args.N) p[0] = (TC)acc[mi][f][0];
                  if (col + 1 < args.N) p[1] = (TC)acc[mi][f][1];
                }
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
    if (++s == tt::STAGES) { s = 0; phase ^= 1; }
    if (++kc == nk) { kc = 0; tile += gridDim.x; }
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
    // consumers only (the producer warp has exited): named barrier 1
    asm volatile("bar.sync 1, %0;\n" ::"n"(tt::CONSUMERS));
    const int units_cta = BN / 2;
    for (int e = tid; e < units_cta; e += tt::CONSUMERS) {
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

}  // namespace fdmd
