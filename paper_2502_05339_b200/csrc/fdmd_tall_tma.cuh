// TMA-fed tall_gemm: a STAGES-deep ring of (64-row A tile, 16 k) chunks filled
// by TMA (A: 2-D tensor tiles, zero-filled out of bounds) and bulk copies (B:
// one 1-D copy per k-row into padded smem rows); 8 warps wait on full
// mbarriers, run LDS + DMMA, and release stages through empty mbarriers.
// Lane 0 of warp 0 refills each stage once all 8 warps released it — no
// dedicated producer warp: a 9th warp puts 3 warps on one SM sub-partition
// and caps registers at 168 (the 7-block accumulator tile spilled).
// Included by fdmd_kernels.cu after fdmd_tall.cuh (shares tg::, dmma884).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include "fdmd_tall.cuh"

namespace fdmd {

namespace tt {
constexpr int BM = 64;
constexpr int BK = 16;
constexpr int STAGES = 4;
constexpr int CONSUMERS = 256;          // 8 warps (2 warpgroups), 2 (M) x 4 (N)
constexpr int THREADS = CONSUMERS + 128; // + producer warpgroup (one lane issues; setmaxnreg moves its
                                         //   registers to the consumers: 232 each instead of 168)
constexpr int REG_CONSUMER = 232;   // 2 x 232 + 40 = 3 x 168 (the launch allocation)
constexpr int REG_PRODUCER = 40;
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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <typename TA, int AL, int NF> struct TTSmem {
  static constexpr int BN = 32 * NF;
  // B rows padded to 4 mod 16 doubles: 64-bit loads are served per half-warp
  // (lanes g = 0..3 or 4..7, t = 0..3); rows t then start 8 banks apart and a
  // half-warp's 16 doubles cover all 32 banks once (no conflict)
  static constexpr int LDB = BN + 4;
  // A as written by TMA with a swizzle (tt_a_offset): ROW -> [m][k] rows of
  // BK elements (64-B / 128-B swizzle for f32 / f64); COL -> 128-B boxes of
  // m, one 128-B row per k, 128-B swizzle. Both read conflict-free (f32 COL: 2-way).
  alignas(1024) TA A[tt::STAGES][tt::BM * tt::BK];
  double B[tt::STAGES][tt::BK][LDB];
  double red[2][4][8 * NF / 2][3];
  uint64_t full[tt::STAGES];
  uint64_t empty[tt::STAGES];
};

// byte offset of A(m, k) inside a stage (see TTSmem)
template <typename TA, int AL> __device__ __forceinline__ int tt_a_offset(int m, int k) {
  if (AL == LAYOUT_ROW) {
    if (sizeof(TA) == 8) return m * 128 + (((k >> 1) ^ (m & 7)) << 4) + (k & 1) * 8;
    return m * 64 + (((k >> 2) ^ ((m >> 1) & 3)) << 4) + (k & 3) * 4;
  }
  if (sizeof(TA) == 8) return (m >> 4) * (tt::BK * 128) + k * 128 + ((((m & 15) >> 1) ^ (k & 7)) << 4) + (m & 1) * 8;
  return (m >> 5) * (tt::BK * 128) + k * 128 + ((((m & 31) >> 2) ^ (k & 7)) << 4) + (m & 3) * 4;
}

struct TTArgs {
  TallGemmArgs g;
  const double* Bp;   // padded small operand, Kp x ldbp (Kp multiple of BK, ldbp >= gridDim.y*BN)
  int64_t ldbp;
  int wblk[4];        // 8-column blocks per warp column group (NF or NF-1; sum covers N)
};

template <typename S, int A_LAYOUT> struct TTFeed {
  const CUtensorMap* amap;
  const CUtensorMap* bmap;   // padded B: one {LDB, 16} box per chunk lands as the padded smem rows
  const double* Bp;
  int64_t ldbp;
  int n0;
  __device__ __forceinline__ void issue(S& sm, int s, int64_t tile, int kc) const {
    constexpr unsigned A_BYTES = tt::BM * tt::BK * sizeof(sm.A[0][0]);
    constexpr unsigned B_ROW = S::LDB * sizeof(double);
    mbar_expect_tx(&sm.full[s], A_BYTES + tt::BK * B_ROW);
    const int k0 = kc * tt::BK;
    if (A_LAYOUT == LAYOUT_ROW) {
      tma_load_2d(sm.A[s], amap, k0, (int)(tile * tt::BM), &sm.full[s]);
    } else {
      constexpr int MB = 128 / (int)sizeof(sm.A[0][0]);        // m per 128-B box row
#pragma unroll
      for (int j = 0; j < tt::BM / MB; ++j)
        tma_load_2d(reinterpret_cast<unsigned char*>(sm.A[s]) + j * tt::BK * 128, amap,
                    (int)(tile * tt::BM) + j * MB, k0, &sm.full[s]);
    }
    tma_load_2d(&sm.B[s][0][0], bmap, n0, k0, &sm.full[s]);
  }
};

// One consumer warp: rows wm*32..+32 of each 64-row tile, NFW 8-col blocks
// starting at column wcol0 (NFW = NF, or NF - 1 when N is not a multiple of 32*NF:
// e.g. N = 200 -> 7,6,6,6 blocks instead of 4 x 7 with 24 padding columns).
template <typename S, typename TA, int A_LAYOUT, int NFW, typename TC, int C_LAYOUT, bool STATS>
__device__ __forceinline__ void tt_consume(S& sm, const TallGemmArgs& args, const TTFeed<S, A_LAYOUT>& fd,
                                           bool feeder, int64_t total, int nk, int wm, int wn, int wcol0,
                                           int bcol0, int lane) {
  const int g = lane >> 2, t = lane & 3;
  // feeder: coordinates of the next chunk to load (item it + STAGES)
  int64_t p_tile = blockIdx.x + (int64_t)(tt::STAGES / nk) * gridDim.x;
  int p_kc = tt::STAGES % nk;
  // upper-triangular B (B[k][j] = 0 for k > j): k-chunks past this warp's last
  // column contribute nothing and are skipped (still consumed from the ring)
  const int kc_last = args.b_upper ? (wcol0 + 8 * NFW - 1) / tt::BK : INT32_MAX;
  const int ks_tail = (args.K - (nk - 1) * tt::BK + 3) / 4;
  double st_sum[NFW], st_max[NFW];
  int64_t st_idx[NFW];
#pragma unroll
  for (int f = 0; f < NFW; ++f) { st_sum[f] = 0.0; st_max[f] = -1.0; st_idx[f] = INT64_MAX; }

  double acc[4][NFW][2];
  int s = 0, kc = 0;
  unsigned phase = 0;
  int64_t tile = blockIdx.x;
  for (int64_t it = 0; it < total; ++it) {
    if (kc == 0) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int f = 0; f < NFW; ++f) acc[mi][f][0] = acc[mi][f][1] = 0.0;
    }
    mbar_wait(&sm.full[s], phase);
    const unsigned char* As = reinterpret_cast<const unsigned char*>(sm.A[s]);
    if (kc <= kc_last) {
      // the last k-chunk only runs the k-steps that hold columns < K (K = 200:
      // 12.5 chunks, the zero half of chunk 13 is skipped)
      const int ksn = (kc == nk - 1) ? ks_tail : tt::BK / 4;
#pragma unroll
      for (int ks = 0; ks < tt::BK / 4; ++ks) {
        if (ks >= ksn) break;
        double a[4], b[NFW];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int m = wm * 32 + mi * 8 + g, k = ks * 4 + t;
          a[mi] = (double)*reinterpret_cast<const TA*>(As + tt_a_offset<TA, A_LAYOUT>(m, k));
        }
#pragma unroll
        for (int f = 0; f < NFW; ++f) b[f] = sm.B[s][ks * 4 + t][bcol0 + f * 8 + g];
#pragma unroll
        for (int f = 0; f < NFW; ++f)
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) dmma884(acc[mi][f], a[mi], b[f]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    if (feeder && it + tt::STAGES < total) {
      if (lane == 0) {
        mbar_wait(&sm.empty[s], phase);
        fd.issue(sm, s, p_tile, p_kc);
      }
      if (++p_kc == nk) { p_kc = 0; p_tile += gridDim.x; }
    }
    if (kc == nk - 1) {
      const int64_t row0 = tile * tt::BM;
      TC* __restrict__ C = static_cast<TC*>(args.C);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int64_t row = row0 + wm * 32 + mi * 8 + g;
        if (row < args.n) {
#pragma unroll
          for (int f = 0; f < NFW; ++f) {
            const int col = wcol0 + f * 8 + 2 * t;
            if (C_LAYOUT == LAYOUT_PLANES) {
              // fp16 hi/lo planes of C * cscale (split_rows_kernel's split),
              // zero in the padding columns N <= col < ldc
              if (!(args.debug & 2) && col < args.ldc) {
                // one f64 -> f32 conversion per value (XU pipe), then the split in
                // fp32 like the tcgen05 plane epilogue: 24 bits carry the 22-bit
                // hi + lo pair; cscale is a power of two (exact). The all-f64 split
                // (4 XU conversions + 2 FP64-pipe ops per value) idled the DMMA pipe
                // ~9% per tile (ncu r02: tensor 84%, XU 12%)
                const float x0 = col < args.N ? (float)acc[mi][f][0] * (float)args.cscale : 0.f;
                const float x1 = col + 1 < args.N ? (float)acc[mi][f][1] * (float)args.cscale : 0.f;
                const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
                const __half l0 = __float2half_rn(x0 - __half2float(h0));
                const __half l1 = __float2half_rn(x1 - __half2float(h1));
                const int64_t o = row * args.ldc + col;
                *reinterpret_cast<__half2*>(static_cast<__half*>(args.C) + o) = __halves2half2(h0, h1);
                *reinterpret_cast<__half2*>(static_cast<__half*>(args.C2) + o) = __halves2half2(l0, l1);
              }
            } else if (C != nullptr && !(args.debug & 2)) {
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
    for (int f = 0; f < NFW; ++f) {
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
      for (int f = 0; f < NFW; ++f) {
        const int u = f * 4 + t;
        sm.red[wm][wn][u][0] = st_sum[f];
        sm.red[wm][wn][u][1] = st_max[f];
        sm.red[wm][wn][u][2] = __longlong_as_double((long long)st_idx[f]);
      }
    }
  }
}

template <typename TA, int A_LAYOUT, int NF, typename TC, int C_LAYOUT, bool STATS>
__global__ void __launch_bounds__(tt::THREADS, 1)
tall_gemm_tma_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                     const TTArgs ta) {
  using S = TTSmem<TA, A_LAYOUT, NF>;
  constexpr int BN = S::BN;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align by offsetting the __shared__ array (keeps LDS addressing)
  S& sm = *reinterpret_cast<S*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
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

  const TTFeed<S, A_LAYOUT> fd{&amap, &bmap, ta.Bp, ta.ldbp, n0};
  if (warp >= tt::CONSUMERS / 32) {
    // ============================ producer ============================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(tt::REG_PRODUCER));
    if (warp == tt::CONSUMERS / 32 && lane == 0) {
      int s = 0, kc = 0;
      unsigned phase = 0;
      int64_t tile = blockIdx.x;
      for (int64_t it = 0; it < total; ++it) {
        mbar_wait(&sm.empty[s], phase ^ 1);
        fd.issue(sm, s, tile, kc);
        if (++s == tt::STAGES) { s = 0; phase ^= 1; }
        if (++kc == nk) { kc = 0; tile += gridDim.x; }
      }
    }
    return;
  }
  const bool feeder = false;
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(tt::REG_CONSUMER));

  // ============================ consumers ============================
  // SM sub-partition = warp & 3; pairing column group wn with 3 - wn on each
  // sub-partition balances the DMMA work when B is upper triangular or the
  // groups have unequal widths.
  const int wm = warp >> 2, wn = (wm == 0) ? (warp & 3) : 3 - (warp & 3);
  // prefix sums of the group widths without dynamic indexing (no local memory)
  const int w0 = ta.wblk[0], w1 = ta.wblk[1], w2 = ta.wblk[2], w3 = ta.wblk[3];
  const int b1 = w0, b2 = w0 + w1, b3 = w0 + w1 + w2, b4 = b3 + w3;
  const int my_blk = wn == 0 ? w0 : wn == 1 ? w1 : wn == 2 ? w2 : w3;
  const int bcol0 = 8 * (wn == 0 ? 0 : wn == 1 ? b1 : wn == 2 ? b2 : b3);
  const int wcol0 = n0 + bcol0;
  if (my_blk == NF)
    tt_consume<S, TA, A_LAYOUT, NF, TC, C_LAYOUT, STATS>(sm, args, fd, feeder, total, nk, wm, wn, wcol0, bcol0,
                                                         lane);
  else
    tt_consume<S, TA, A_LAYOUT, (NF > 1 ? NF - 1 : 1), TC, C_LAYOUT, STATS>(sm, args, fd, feeder, total, nk, wm,
                                                                            wn, wcol0, bcol0, lane);

  if (STATS) {
    asm volatile("bar.sync 1, %0;\n" ::"n"(tt::CONSUMERS));   // consumers only (producer exited)
    const int units_cta = 4 * b4;
    for (int e = tid; e < units_cta; e += tt::CONSUMERS) {
      const int wn_ = (e >= 4 * b1) + (e >= 4 * b2) + (e >= 4 * b3);
      const int u = e - 4 * (wn_ == 0 ? 0 : wn_ == 1 ? b1 : wn_ == 2 ? b2 : b3);
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
