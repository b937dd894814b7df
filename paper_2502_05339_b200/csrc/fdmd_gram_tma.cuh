// Warp-specialised tall_gram: partial[split] = A[rows]^T B[rows] for one
// 64 x (32*NFB) output tile (row-major operands). With NFB = 7 a CTA covers
// the whole 200-224 wide K2 range, so each reduction row is fetched from L2
// by 4 CTAs instead of 16 (64x64 tiles measured 2-2.5x DRAM re-reads and a
// consumer-side wait on every chunk).
//
// A producer lane streams 16-row chunks of both operands as TMA boxes of
// 128-byte rows with SWIZZLE_128B (one box per 128 B of columns); 8 consumer
// warps (2 x 4, warp tile 32 x 8*NFB) run LDS + DMMA and release stages via
// mbarriers.
//
// Conflict-free fragment reads under the 128-B swizzle: a DMMA fragment reads
// 4 reduction rows (t) x 8 columns (g). In a swizzled box the 16-B chunk c of
// row r lives at chunk c ^ (r % 8); rows r and r+1 would collide, so k-step ks
// uses the rows {b, b+2, b+4, b+6} (b = 8*(ks/2) + ks%2) instead of 4
// consecutive rows. A Gram A^T B is invariant under a common permutation of
// its rows, so this is free; every row of a chunk is used exactly once.
// Warps whose block is padding or strictly below the diagonal of a symmetric
// Gram skip their DMMAs (warp-uniform, outside the k-loop); whole CTA tiles
// below the diagonal exit at once.
#pragma once
#include <cuda.h>

#include "fdmd_tall_tma.cuh"

namespace fdmd {

namespace tgs {
constexpr int TM = 64;
constexpr int BR = 16;
constexpr int STAGES = 4;
constexpr int CONSUMERS = 256;
constexpr int THREADS = CONSUMERS + 32;
constexpr int BOX_BYTES = BR * 128;   // 16 rows x 128 B
}  // namespace tgs

template <typename TX, int COLS> struct SwOperand {
  static constexpr int W = 128 / sizeof(TX);        // elements per swizzled row
  static constexpr int NBOX = COLS / W;
  static constexpr int BYTES = NBOX * tgs::BOX_BYTES;
  __device__ __forceinline__ static int offset(int row, int col) {
    const int box = col / W;
    const int cb = (col % W) * (int)sizeof(TX);
    return box * tgs::BOX_BYTES + row * 128 + ((((cb >> 4) ^ (row & 7))) << 4) + (cb & 15);
  }
};

template <typename TA, typename TB, int NFB> struct TGSSmem {
  alignas(1024) unsigned char a[tgs::STAGES][SwOperand<TA, tgs::TM>::BYTES];
  alignas(1024) unsigned char b[tgs::STAGES][SwOperand<TB, 32 * NFB>::BYTES];
  uint64_t full[tgs::STAGES];
  uint64_t empty[tgs::STAGES];
};

template <typename TA, typename TB, int NFB>
__global__ void __launch_bounds__(tgs::THREADS, (NFB <= 2) ? 2 : 1)
tall_gram_sw_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                    const TallGramArgs args) {
  constexpr int TN = 32 * NFB;
  using SA = SwOperand<TA, tgs::TM>;
  using SB = SwOperand<TB, TN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TGSSmem<TA, TB, NFB>& sm =
      *reinterpret_cast<TGSSmem<TA, TB, NFB>*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));

  int ti, tj;
  if (args.symmetric && TN == tgs::TM) {   // square tiles: enumerate the upper triangle only
    int x = blockIdx.x;
    ti = 0;
    int rowlen = args.tiles_j;
    while (x >= rowlen) { x -= rowlen; ++ti; --rowlen; }
    tj = ti + x;
  } else {
    ti = blockIdx.x / args.tiles_j;
    tj = blockIdx.x % args.tiles_j;
  }
  const int c0a = ti * tgs::TM, c0b = tj * TN;
  if (args.symmetric && c0a > c0b + TN - 1) return;   // tile strictly below the diagonal: mirrored
  const int64_t rbeg = (int64_t)blockIdx.y * args.rows_per_split;
  const int64_t rend = min(args.n, rbeg + args.rows_per_split);
  const int64_t nchunks = rend > rbeg ? (rend - rbeg + tgs::BR - 1) / tgs::BR : 0;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < tgs::STAGES; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], tgs::CONSUMERS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == tgs::CONSUMERS / 32) {
    if (lane == 0) {
      // boxes entirely past K are skipped (their smem is never read by live fragments)
      const int nba = min(SA::NBOX, (args.K1 - c0a + SA::W - 1) / SA::W);
      const int nbb = min(SB::NBOX, (args.K2 - c0b + SB::W - 1) / SB::W);
      const unsigned bytes = (unsigned)((nba + nbb) * tgs::BOX_BYTES);
      int s = 0;
      unsigned ph = 0;
      for (int64_t c = 0; c < nchunks; ++c) {
        mbar_wait(&sm.empty[s], ph ^ 1);
        mbar_expect_tx(&sm.full[s], bytes);
        const int r0 = (int)(rbeg + c * tgs::BR);
        for (int j = 0; j < nba; ++j)
          tma_load_2d(sm.a[s] + j * tgs::BOX_BYTES, &amap, c0a + j * SA::W, r0, &sm.full[s]);
        for (int j = 0; j < nbb; ++j)
          tma_load_2d(sm.b[s] + j * tgs::BOX_BYTES, &bmap, c0b + j * SB::W, r0, &sm.full[s]);
        if (++s == tgs::STAGES) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int rw = c0a + wm * 32, cw = c0b + wn * 8 * NFB;
  // live: any in-range column of this warp block, and not strictly below the diagonal
  const bool live = rw < args.K1 && cw < args.K2 && !(args.symmetric && rw >= cw + 8 * NFB);

  // swizzled byte offsets of this thread's fragments, fixed for the whole kernel
  int offa[tgs::BR / 4][4], offb[tgs::BR / 4][NFB];
#pragma unroll
  for (int ks = 0; ks < tgs::BR / 4; ++ks) {
    const int row = (ks >> 1) * 8 + (ks & 1) + 2 * t;     // permuted reduction rows
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) offa[ks][mi] = SA::offset(row, wm * 32 + mi * 8 + g);
#pragma unroll
    for (int f = 0; f < NFB; ++f) offb[ks][f] = SB::offset(row, wn * 8 * NFB + f * 8 + g);
  }

  double acc[4][NFB][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int f = 0; f < NFB; ++f) acc[mi][f][0] = acc[mi][f][1] = 0.0;

  int s = 0;
  unsigned ph = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    mbar_wait(&sm.full[s], ph);
    if (live) {
      const unsigned char* pa = sm.a[s];
      const unsigned char* pb = sm.b[s];
#pragma unroll
      for (int ks = 0; ks < tgs::BR / 4; ++ks) {
        double a[4], b[NFB];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = (double)*reinterpret_cast<const TA*>(pa + offa[ks][mi]);
#pragma unroll
        for (int f = 0; f < NFB; ++f) b[f] = (double)*reinterpret_cast<const TB*>(pb + offb[ks][f]);
#pragma unroll
        for (int f = 0; f < NFB; ++f)
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) dmma884(acc[mi][f], a[mi], b[f]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[s]);
    if (++s == tgs::STAGES) { s = 0; ph ^= 1; }
  }
  double* W = args.W + (int64_t)blockIdx.y * args.K1p * args.K2p;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int i = c0a + wm * 32 + mi * 8 + g;
#pragma unroll
    for (int f = 0; f < NFB; ++f) {
      const int j = c0b + wn * 8 * NFB + f * 8 + 2 * t;
      *reinterpret_cast<double2*>(W + (int64_t)i * args.K2p + j) = make_double2(acc[mi][f][0], acc[mi][f][1]);
    }
  }
}

}  // namespace fdmd
