// tcgen05 reconstruction on CTA PAIRS (cta_group::2): frames[f][i] =
// sum_k U[i][k] C[k][f], same FP16 2-way split as fdmd_tc_decode.cuh.
//
// Why pairs: the single-CTA kernel keeps all 128 frames' coefficients
// resident (128 KB) and streams the basis through a 3-stage ring; every
// 128-row basis tile (128 KB of hi/lo planes) then yields only 128 frames,
// and the ring's 96 KB in flight caps the rate (ncu: MMA warp waiting on
// afull, tensor pipe ~45%). A pair issues M = 256 (128 rows per CTA), N = 256
// frames, with each CTA holding HALF the coefficients (128 frames): same smem
// per CTA, but every basis byte an SM ingests now produces twice the frames.
//
// Protocol (cluster = 2 CTAs along x, rank 0 = leader):
//   * both CTAs TMA their own 128 basis rows and their 128-frame coefficient
//     half into local smem, signalling the LEADER's full barriers
//     (.cta_group::2 TMA with the leader's mbarrier address from mapa);
//   * the leader's elected thread issues tcgen05.mma.cta_group::2 and commits
//     with .multicast::cluster to both CTAs' empty / accumulator-full barriers;
//   * each CTA's 8 epilogue warps drain their own TMEM half (128 rows x 256
//     frames) and arrive on the leader's accumulator-empty barrier (count 16);
//   * TMEM (512 columns = 2 accumulators x 256) is allocated / freed by one
//     warp in each CTA with cta_group::2.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include "fdmd_tc_decode.cuh"

namespace fdmd {

namespace tc2 {
constexpr int BM = 128;           // basis rows per CTA (pair tile: 256)
constexpr int BN = 256;           // frames per pair tile
constexpr int BNH = 128;          // coefficient rows held per CTA
constexpr int BKC = 64;
constexpr int MAXKC = 4;          // r <= 256
constexpr int AST = 3;
#ifndef FDMD_TC2_EPI
#define FDMD_TC2_EPI 16
#endif
constexpr int EPI = FDMD_TC2_EPI;   // epilogue warps (4 per TMEM lane quadrant)
constexpr int THREADS = 64 + 32 * EPI;
constexpr int A_CHUNK_BYTES = BM * BKC * 2;    // 16 KB per plane
constexpr int B_CHUNK_BYTES = BNH * BKC * 2;   // 16 KB per plane
}  // namespace tc2

// TMAO (TMA-store epilogue): each of the 4 epilogue parts stages 16 frames x
// 128 rows (8 KB) and writes them with ONE 2-D TMA store — 512 contiguous
// bytes per frame per CTA tile. Register stores from the TMEM lane layout
// (lane = row) write 128 B per frame per warp instruction, which HBM absorbs
// at 4.5 TB/s against 6.0-6.3 TB/s for 512-B runs (tools/write_pattern.cu,
// profiles/r02_write_pattern.txt). The staging space comes from a 2-deep
// basis ring (3 before): at 256 frames per basis tile a pair SM needs ~15 GB/s
// of basis, covered by 64 KB in flight.
constexpr int TMAO_FR = 8;                       // frames per staged chunk (2 buffers per part)
// TMAO: 0 register stores, 1 staged + TMA store, 2 staged + 16-byte register
// stores (each warp instruction writes 512 contiguous bytes of one frame)
template <int AST_, int TMAO>
struct TC2SmemT {
  __half A[AST_][2][tc2::BM * tc2::BKC];
  __half B[tc2::MAXKC][2][tc2::BNH * tc2::BKC];
  alignas(128) float stage[TMAO ? tc2::EPI / 4 : 1][2][TMAO ? TMAO_FR * tc2::BM : 1];
  alignas(16) float fs[tc2::BN];
  uint64_t afull[AST_], aempty[AST_];
  uint64_t bfull;
  uint64_t tfull[2], tempty[2];
  uint32_t tmem_base;
};
using TC2Smem = TC2SmemT<tc2::AST, 0>;

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
               ::"l"(map), "r"(x), "r"(y), "r"(smem_u32(src)) : "memory");
}

__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// TMA tile into local smem, completion signalled on a (possibly peer) barrier
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* map, int x, int y, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void umma2_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  // relaxed: only the (already waited) TMEM reads must precede the arrive, not the
  // epilogue's global stores (a release would MEMBAR on every store of the tile)
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

template <bool PLANES, int TMAO, int AST_, bool STATS = false>
__global__ void __launch_bounds__(tc2::THREADS, 1)
tc_decode2_kernel(const __grid_constant__ CUtensorMap amap_h, const __grid_constant__ CUtensorMap amap_l,
                  const __grid_constant__ CUtensorMap bmap_h, const __grid_constant__ CUtensorMap bmap_l,
                  const __grid_constant__ CUtensorMap omap, const TCArgs args) {
  using SM = TC2SmemT<AST_, TMAO>;
  constexpr uint32_t TCOLS = 2 * tc2::BN;   // 512: two 256-column accumulators
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int nkc = (args.r + tc2::BKC - 1) / tc2::BKC;
  const int ksteps_last = ((args.r - (nkc - 1) * tc2::BKC) + 15) / 16;
  const int64_t ptiles = (args.n + 2 * tc2::BM - 1) / (2 * tc2::BM);
  // frame tiles interleave with the row pairs along x (CTA 2 (gy p + y) + rank):
  // the gy pairs reading the same basis rows get adjacent CTA ids, hence SMs on
  // the same die, so the second frame tile's basis reads hit the same L2
  // (grid (npairs, gy) placed the two frame tiles on different dies: 1.8x
  // basis DRAM reads at 512 frames)
  const int gy = (args.nf + tc2::BN - 1) / tc2::BN;
  const int64_t pid = blockIdx.x >> 1;
  const int64_t pair = pid / gy, npairs = (gridDim.x >> 1) / gy;
  const int64_t my_tiles = pair < ptiles ? (ptiles - pair + npairs - 1) / npairs : 0;
  const int f0 = (int)(pid % gy) * tc2::BN;

  for (int f = threadIdx.x; f < tc2::BN; f += blockDim.x)
    sm.fs[f] = (f0 + f < args.nf) ? args.fscale[f0 + f] : 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < AST_; ++s) { mbar_init(&sm.afull[s], 1); mbar_init(&sm.aempty[s], 1); }
    mbar_init(&sm.bfull, 1);
    for (int a = 0; a < 2; ++a) { mbar_init(&sm.tfull[a], 1); mbar_init(&sm.tempty[a], 2 * tc2::EPI); }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n"
                 ::"r"(smem_u32(&sm.tmem_base)), "n"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // coefficient half: frames f0 + rank * 128 .. +127, every K chunk
      const uint32_t bfull_l = mapa_u32(&sm.bfull, 0);
      if (leader) mbar_expect_tx(&sm.bfull, (uint32_t)(2 * nkc * 2 * tc2::B_CHUNK_BYTES));
      for (int c = 0; c < nkc; ++c) {
        tma_load_2d_cg2(sm.B[c][0], &bmap_h, c * tc2::BKC, f0 + (int)rank * tc2::BNH, bfull_l);
        tma_load_2d_cg2(sm.B[c][1], &bmap_l, c * tc2::BKC, f0 + (int)rank * tc2::BNH, bfull_l);
      }
      int sa = 0;
      uint32_t pa = 0;
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int row0 = (int)((pair + t * npairs) * (2 * tc2::BM) + rank * tc2::BM);
        for (int c = 0; c < nkc; ++c) {
          mbar_wait(&sm.aempty[sa], pa ^ 1);                          // leader's MMAs released it
          if (leader) mbar_expect_tx(&sm.afull[sa], 2 * 2 * tc2::A_CHUNK_BYTES);   // both CTAs' planes
          const uint32_t afull_l = mapa_u32(&sm.afull[sa], 0);
          tma_load_2d_cg2(sm.A[sa][0], &amap_h, c * tc2::BKC, row0, afull_l);
          tma_load_2d_cg2(sm.A[sa][1], &amap_l, c * tc2::BKC, row0, afull_l);
          if (++sa == AST_) { sa = 0; pa ^= 1; }
        }
      }
      // tail: the leader's last releases of this CTA's ring have landed
      for (int s = 0; s < AST_; ++s) {
        mbar_wait(&sm.aempty[sa], pa ^ 1);
        if (++sa == AST_) { sa = 0; pa ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // kind::f16, fp16 x fp16 -> fp32, K-major A and B, M = 256, N = 256
      const uint32_t idesc = (1u << 4) | ((uint32_t)(tc2::BN >> 3) << 17) | ((uint32_t)((2 * tc2::BM) >> 4) << 24);
      int sa = 0;
      uint32_t pa = 0;
      mbar_wait(&sm.bfull, 0);
      for (int64_t t = 0; t < my_tiles; ++t) {
        const int acc = (int)(t & 1);
        mbar_wait(&sm.tempty[acc], (uint32_t)(((t >> 1) & 1) ^ 1));   // both CTAs' epilogues drained it
        tc_fence_after();
        const uint32_t d = tmem + acc * tc2::BN;
        uint32_t first = 1;
        for (int c = 0; c < nkc; ++c) {
          mbar_wait(&sm.afull[sa], pa);
          tc_fence_after();
          const int ksteps = (c == nkc - 1) ? ksteps_last : tc2::BKC / 16;
          const uint64_t ah = umma_desc_sw128(sm.A[sa][0]), al = umma_desc_sw128(sm.A[sa][1]);
          const uint64_t bh = umma_desc_sw128(sm.B[c][0]), bl = umma_desc_sw128(sm.B[c][1]);
          for (int k = 0; k < ksteps; ++k) {
            const uint64_t adv = (uint64_t)((k * 32) >> 4);
            umma2_f16(d, ah + adv, bh + adv, idesc, first ? 0u : 1u);
            umma2_f16(d, ah + adv, bl + adv, idesc, 1u);
            umma2_f16(d, al + adv, bh + adv, idesc, 1u);
            first = 0;
          }
          umma2_commit_mc(&sm.aempty[sa]);          // both CTAs may refill this stage
          if (++sa == AST_) { sa = 0; pa ^= 1; }
        }
        umma2_commit_mc(&sm.tfull[acc]);            // both CTAs' TMEM halves ready
      }
      // every peer epilogue arrival on our tempty has landed before teardown
      for (int64_t t = my_tiles; t < my_tiles + 2; ++t)
        mbar_wait(&sm.tempty[t & 1], (uint32_t)(((t >> 1) & 1) ^ 1));
    }
  } else {
    const int q = warp & 3;
    constexpr int SPLIT = tc2::EPI / 4;
    const int part = (warp - 2) / 4;
    const int c_lo = part * (tc2::BN / SPLIT), c_hi = c_lo + tc2::BN / SPLIT;
    const uint32_t tempty_l[2] = {mapa_u32(&sm.tempty[0], 0), mapa_u32(&sm.tempty[1], 0)};
    int buf = 0;   // staging buffer parity: alternates over ALL chunks (also across tiles)
    // STATS: lane L owns column pair L of the warp's 64 columns (the (Re, Im) columns
    // of one mode): running max of re^2 + im^2 over the warp's rows and the first
    // row attaining it (tiles arrive in increasing row order; strict > keeps the first)
    float st_best = -1.f;
    double st_sum0 = 0.0, st_sum1 = 0.0;   // sums: pairs lane / 2 and 16 + lane / 2
    long long st_row = 0;
    for (int64_t t = 0; t < my_tiles; ++t) {
      const int acc = (int)(t & 1);
      mbar_wait(&sm.tfull[acc], (uint32_t)((t >> 1) & 1));
      tc_fence_after();
      const int64_t row = (pair + t * npairs) * (2 * tc2::BM) + rank * tc2::BM + q * 32 + lane;
      if constexpr (TMAO && !PLANES) {
        const int64_t row0 = row - q * 32 - lane;              // first row of this CTA's tile half
#pragma unroll 1
        for (int cb = c_lo; cb < c_hi; cb += 2 * TMAO_FR) {
          if (f0 + cb >= args.nf) break;                       // uniform over the part's 4 warps
          float v[2 * TMAO_FR];
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * tc2::BN + cb), v);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (f0 + cb + h * TMAO_FR >= args.nf) break;
            float* stg = sm.stage[part][buf];
#pragma unroll
            for (int j = 0; j < TMAO_FR; ++j)
              stg[j * tc2::BM + q * 32 + lane] = v[h * TMAO_FR + j] * sm.fs[cb + h * TMAO_FR + j];
            if constexpr (TMAO == 2) {
              // staged chunk -> global with 16-byte stores: warp q writes frames q, q + 4
              // of the chunk, lane = 4 consecutive rows, so one instruction covers 512
              // contiguous bytes of one frame (HBM absorbs 512-B runs at 6.0-6.3 TB/s
              // against 4.5 for the 128-B runs of the lane = row layout). One barrier
              // per chunk: the other buffer is rewritten only after every warp of the
              // part passed the next barrier, i.e. finished reading this one.
              asm volatile("bar.sync %0, 128;\n" ::"r"(1 + part) : "memory");
#pragma unroll
              for (int jj = 0; jj < TMAO_FR / 4; ++jj) {
                const int j = q + 4 * jj;
                const int fr = f0 + cb + h * TMAO_FR + j;
                const int64_t r4 = row0 + 4 * lane;
                if (fr < args.nf && r4 < args.n) {
                  const float4 w = *reinterpret_cast<const float4*>(stg + j * tc2::BM + 4 * lane);
                  float* o = args.out + (int64_t)fr * args.ldo + r4;
                  if (r4 + 3 < args.n) {
                    __stcs(reinterpret_cast<float4*>(o), w);
                  } else {
                    o[0] = w.x;
                    if (r4 + 1 < args.n) o[1] = w.y;
                    if (r4 + 2 < args.n) o[2] = w.z;
                  }
                }
              }
              buf ^= 1;
              continue;
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("bar.sync %0, 128;\n" ::"r"(1 + part) : "memory");
            if (q == 0 && lane == 0) {
              tma_store_2d(&omap, stg, (int)row0, f0 + cb + h * TMAO_FR);   // rows >= n / frames >= nf clipped
              asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
              // the OTHER buffer (the store before this one) is free for the next chunk
              asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            }
            asm volatile("bar.sync %0, 128;\n" ::"r"(1 + part) : "memory");
            buf ^= 1;
          }
        }
      } else {
#pragma unroll 1
      for (int cb = c_lo; cb < c_hi; cb += 32) {
        if (f0 + cb >= args.nf) break;
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * tc2::BN + cb), v);
        if constexpr (PLANES) {
          // planes: lane = row (q * 32 + lane), 32 consecutive columns. The hi / lo
          // halves are packed into half2 registers and transposed across the warp
          // with shuffles so every store instruction writes 8 rows x 64 contiguous
          // bytes (one uint4 per lane) instead of 32 rows' scattered 16-B pieces.
          const int c0 = f0 + cb;
          uint32_t hp[16], lp[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int j = 2 * u;
            const float x0 = (c0 + j < args.nf ? v[j] * sm.fs[cb + j] : 0.f) * args.pscale;
            const float x1 = (c0 + j + 1 < args.nf ? v[j + 1] * sm.fs[cb + j + 1] : 0.f) * args.pscale;
            const __half a0 = __float2half_rn(x0), a1 = __float2half_rn(x1);
            const __half2 h = __halves2half2(a0, a1);
            const __half2 l = __halves2half2(__float2half_rn(x0 - __half2float(a0)), __float2half_rn(x1 - __half2float(a1)));
            hp[u] = *reinterpret_cast<const uint32_t*>(&h);
            lp[u] = *reinterpret_cast<const uint32_t*>(&l);
          }
          const int64_t rowbase = row - lane;
          const int cq = lane & 3;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int src = 8 * k + (lane >> 2);
            uint4 oh, ol;
            uint32_t* ohp = reinterpret_cast<uint32_t*>(&oh);
            uint32_t* olp = reinterpret_cast<uint32_t*>(&ol);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint32_t hc[4], lc[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                hc[c] = __shfl_sync(0xffffffffu, hp[4 * c + j], src);
                lc[c] = __shfl_sync(0xffffffffu, lp[4 * c + j], src);
              }
              ohp[j] = cq == 0 ? hc[0] : cq == 1 ? hc[1] : cq == 2 ? hc[2] : hc[3];
              olp[j] = cq == 0 ? lc[0] : cq == 1 ? lc[1] : cq == 2 ? lc[2] : lc[3];
            }
            const int64_t r_out = rowbase + src;
            const int col = c0 + 8 * cq;
            if (r_out < args.n && col < args.ldp) {
              *reinterpret_cast<uint4*>(args.ph + r_out * args.ldp + col) = oh;
              *reinterpret_cast<uint4*>(args.pl + r_out * args.ldp + col) = ol;
            }
          }
          continue;
        }
        if constexpr (STATS) {
          const bool live = row < args.n;
          float wf[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            // |phi|^2 of the stored f32 values, evaluated in f32 (f64 here made the
            // epilogue XU / FP64-pipe bound: 26 ms against 16 ms for the plain
            // product). Magnitudes within 2^-23 of each other may order differently
            // than in f64 — below the resolution of the f32 table itself.
            const float x0 = v[2 * u] * sm.fs[cb + 2 * u], x1 = v[2 * u + 1] * sm.fs[cb + 2 * u + 1];
            const float w = live ? __fmaf_rn(x0, x0, x1 * x1) : 0.f;
            // w >= 0: its bits order like unsigned integers (one redux.sync)
            const unsigned mb = __float_as_uint(w);
            const unsigned mx = __reduce_max_sync(0xffffffffu, mb);
            const unsigned who = __ballot_sync(0xffffffffu, live && mb == mx);
            if (lane == ((cb - c_lo) >> 1) + u && who != 0u) {
              const float m = __uint_as_float(mx);   // a NaN wins once and stays (reported downstream)
              if (m > st_best || m != m) { st_best = m; st_row = (long long)(row - lane) + (__ffs(who) - 1); }
            }
            wf[u] = w;
          }
          // sum over the warp's 32 rows of all 16 pairs at once (transposing butterfly:
          // 16 shuffles): lanes 2p, 2p + 1 end up with pair p's total. f32 is enough
          // for a 32-row partial (it only feeds the f64 running sum of the norm)
#pragma unroll
          for (int b = 4; b >= 1; --b) {
            const int half = 1 << (b - 1);
            const bool up = (lane >> b) & 1;
#pragma unroll
            for (int j = 0; j < half; ++j) {
              const float send = up ? wf[j] : wf[j + half], keep = up ? wf[j + half] : wf[j];
              wf[j] = keep + __shfl_xor_sync(0xffffffffu, send, 1 << b);
            }
          }
          const float tot = wf[0] + __shfl_xor_sync(0xffffffffu, wf[0], 1);
          if (cb == c_lo) st_sum0 += (double)tot; else st_sum1 += (double)tot;
        }
        if (row < args.n) {
          float* o = args.out + (int64_t)(f0 + cb) * args.ldo + row;
          const int jn = min(32, args.nf - (f0 + cb));
          const float4* fs4 = reinterpret_cast<const float4*>(sm.fs + cb);
          if (jn == 32) {
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
              const float4 s = fs4[j4];
              __stcs(o, v[4 * j4] * s.x); o += args.ldo;
              __stcs(o, v[4 * j4 + 1] * s.y); o += args.ldo;
              __stcs(o, v[4 * j4 + 2] * s.z); o += args.ldo;
              __stcs(o, v[4 * j4 + 3] * s.w); o += args.ldo;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < jn) { __stcs(o, v[j] * sm.fs[cb + j]); o += args.ldo; }
          }
        }
      }
      }  // register-store / plane epilogue
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_l[acc]);
    }
    if constexpr (STATS && !PLANES && TMAO == 0) {
      const size_t slot = ((size_t)blockIdx.x * tc2::EPI + (warp - 2)) * 32 + lane;
      args.st_max[slot] = (double)st_best;
      args.st_idx[slot] = st_row;
      if ((lane & 1) == 0) {
        args.st_sum[slot - lane + (lane >> 1)] = st_sum0;
        args.st_sum[slot - lane + 16 + (lane >> 1)] = st_sum1;
      }
    }
  }
  if constexpr (TMAO == 1 && !PLANES)
    if (warp >= 2) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");   // stores complete
  __syncwarp();
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TCOLS));
  }
}

// Combine the fused statistics of tc_decode2_kernel<.., STATS>: column pair u
// (columns 2u, 2u + 1) lives in frame tile ft = 2u / 256, epilogue part
// (2u % 256) / 64, lane ((2u % 64) / 2); candidates are the 4 quadrant warps of
// that part in every CTA of the tile (CTA x: pid = x >> 1, tile pid % gy).
// st[u] = {sum, max, first row attaining it + row_offset} (ties: lowest row).
__global__ void tc2_pair_stats_final_kernel(const double* __restrict__ st_max, const long long* __restrict__ st_idx,
                                            const double* __restrict__ st_sum, int nctas, int gy, int units,
                                            long long row_offset, double* __restrict__ st) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= units) return;
  const int f = 2 * u, ft = f / tc2::BN, part = (f % tc2::BN) / (tc2::BN / (tc2::EPI / 4)), lane = (f % 64) >> 1;
  double best = -1.0, sum = 0.0;
  long long row = 0;
  for (int x = 0; x < nctas; ++x) {
    if (((x >> 1) % gy) != ft) continue;
    for (int q = 0; q < 4; ++q) {
      const size_t slot = ((size_t)x * tc2::EPI + part * 4 + q) * 32 + lane;
      sum += st_sum[slot];                                   // fixed order: deterministic
      const double m = st_max[slot];
      const long long r = st_idx[slot];
      if (best != best) continue;   // NaN seen: keep it
      if (m != m || m > best || (m == best && r < row)) { best = m; row = r; }
    }
  }
  st[3 * u] = sum;
  st[3 * u + 1] = best;
  st[3 * u + 2] = (double)(row + row_offset);
}

}  // namespace fdmd
