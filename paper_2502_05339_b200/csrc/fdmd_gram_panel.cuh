// Panel tall_gram: partial[split] = A[rows]^T B[rows] where ONE CTA covers the
// whole K1 x K2 output (or a 1/P share of it) for its row range, so every
// reduction row is streamed into shared memory once per CTA partition and no
// DMMA is spent on tile padding.
//
// Why (ncu, r01): with 64 x 64 / 64 x 224 CTA tiles the 200 x 200 Grams of the
// fit executed 1.4x (general) and 2x (symmetric: the 10 upper tiles of a 4 x 4
// grid are 64-row squares) the algorithmic DMMA work. Here the output is cut
// into warp tiles of WR x WC 8x8 blocks (5 x 7 general, 5 x 5 symmetric, where
// the diagonal tiles skip their lower blocks at compile time); the host packs
// warp tiles into partitions of 8 consumer warps, balancing the DMMA count per
// SM sub-partition (warps w and w+4 share one: w & 3).
//
// Data movement is the SW128 scheme of fdmd_gram_tma.cuh: 16-row chunks of
// both operands arrive as 128-byte-row TMA boxes; k-step ks reads the permuted
// rows {b, b+2, b+4, b+6} (b = 8*(ks/2) + ks%2) so the fragment loads are
// bank-conflict free. A symmetric Gram loads one operand. There is no
// dedicated producer warp: a 9th warp would put 3 warps on one sub-partition
// and cap registers at 168 (spills with a 5 x 7 accumulator tile). Lane 0 of
// warp 0 — placed on the most lightly loaded sub-partition by the host —
// refills each stage after all 8 warps released it.
#pragma once
#include <cuda.h>

#include "fdmd_gram_tma.cuh"

namespace fdmd {

namespace tgp {
constexpr int BR = 16;
#ifndef FDMD_GRAM_STAGES
#define FDMD_GRAM_STAGES 4
#endif
constexpr int STAGES = FDMD_GRAM_STAGES;
constexpr int THREADS = 256;            // 8 warps = 2 per SM sub-partition -> up to 255 regs
constexpr int MAXP = 8;                 // partitions (x 8 warp tiles) per launch
constexpr int BOX_BYTES = BR * 128;
}  // namespace tgp

struct PanelTile {
  short i0, j0;   // first 8x8 block row / column of the warp tile
  // 0 idle, 1 full WR x WC, 2 diagonal (symmetric: blocks ii <= jj only),
  // 3 diagonal + its 5 border blocks (ii, jb) (bordered symmetric Gram),
  // 4 / 5: full 5 x 3 / 5 x 4 (two adjacent 5 x 5 tiles of a symmetric Gram cut
  // into 3 + 4 + 3 block columns so that every sub-partition carries 40-45
  // blocks instead of 25 + 25 next to 25 + 15; host: panel_plan)
  short kind;
  short pad;
};

struct TallGramPanelArgs {
  TallGramArgs g;
  int nba, nbb;                               // 128-B boxes per chunk row (A, B; nbb = 0 when symmetric)
  int lda_boxes, ldb_boxes;                   // boxes actually loaded (those holding columns < K)
  int a_full, b_full, a_tail, b_tail;         // full 128-B blocks (one 3-D TMA) + ragged block (2-D TMA)
  int jb;                                     // bordered symmetric Gram: block column of the border (K / 8)
  PanelTile tile[tgp::MAXP * 8];
};

template <typename TX> __device__ __forceinline__ int panel_offset(int row, int col) {
  constexpr int W = 128 / sizeof(TX);
  const int box = col / W;
  const int cb = (col % W) * (int)sizeof(TX);
  return box * tgp::BOX_BYTES + row * 128 + ((((cb >> 4) ^ (row & 7))) << 4) + (cb & 15);
}

// ---- cluster sharing of the row stream (CL > 1) ----------------------------
// The P output partitions of one row split run as ONE cluster of CL = P CTAs:
// every 128-B box of a stage is loaded ONCE per cluster — CTA k issues the
// boxes b with b % CL == k as 2-D TMA multicasts into the same smem offset of
// all CL CTAs — so DRAM / L2 traffic is the operands once per split instead of
// once per partition (r01 ncu: 2-3x the algorithmic bytes). A stage is
// refilled only after every warp of every CTA released it: each warp arrives
// on the empty barrier of all CL CTAs (count 8 * CL).
__device__ __forceinline__ void gp_tma_2d_mc(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;\n"
      ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask) : "memory");
}
__device__ __forceinline__ void gp_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(bar)), "r"(rank));
  // relaxed: the warp's fragment loads of the stage have been consumed by its
  // DMMAs (register dependences) before the arrive; a release would fence
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void gp_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

struct PanelFeed {
  int cl = 1, rank = 0;                        // cluster size / this CTA's rank in it
  const CUtensorMap* amap;
  const CUtensorMap* bmap;
  const CUtensorMap* atmap;
  const CUtensorMap* btmap;
  int afull, bfull, atail, btail;
  unsigned char* a_sm;
  unsigned char* b_sm;
  int a_stage, b_stage, la, lb, wa, wb;
  unsigned bytes;
  int64_t rbeg, nchunks;
  __device__ __forceinline__ void issue(int64_t c, int s, uint64_t* full) const {
    mbar_expect_tx(&full[s], bytes);
    const int r0 = (int)(rbeg + c * tgp::BR);
    if (cl > 1) {
      // box b of the stage (A boxes, then B boxes) is issued by CTA b % cl for the
      // whole cluster; every box is a 2-D {W, 16} tile (zero fill past K)
      const uint16_t mask = (uint16_t)((1u << cl) - 1);
      const int na = la, nb = lb;
      for (int b = rank; b < na + nb; b += cl) {
        if (b < na)
          gp_tma_2d_mc(a_sm + s * a_stage + b * tgp::BOX_BYTES, atmap, b * wa, r0, &full[s], mask);
        else
          gp_tma_2d_mc(b_sm + s * b_stage + (b - na) * tgp::BOX_BYTES, btmap, (b - na) * wb, r0, &full[s], mask);
      }
      return;
    }
    // one 3-D TMA per operand for its full 128-B column blocks (they land as
    // consecutive 16-row x 128-B SW128 boxes, the layout panel_offset reads)
    // + one 2-D TMA for a ragged last block (zero-filled past K)
    if (afull > 0) tma_load_3d(a_sm + s * a_stage, amap, 0, r0, 0, &full[s]);
    if (atail) tma_load_2d(a_sm + s * a_stage + afull * tgp::BOX_BYTES, atmap, afull * wa, r0, &full[s]);
    if (bfull > 0) tma_load_3d(b_sm + s * b_stage, bmap, 0, r0, 0, &full[s]);
    if (btail) tma_load_2d(b_sm + s * b_stage + bfull * tgp::BOX_BYTES, btmap, bfull * wb, r0, &full[s]);
  }
};

// Release stage s of chunk c; the feeding lane then waits for all 8 warps to
// release it and loads chunk c + STAGES into it.
__device__ __forceinline__ void panel_release(const PanelFeed& fd, bool feeder, int lane, int64_t c, int s,
                                              unsigned ph, uint64_t* full, uint64_t* empty) {
  __syncwarp();
  if (lane == 0) {
    if (fd.cl > 1) {
      mbar_arrive(&empty[s]);
      for (int k = 1; k < fd.cl; ++k) gp_arrive_remote(&empty[s], (uint32_t)((fd.rank + k) % fd.cl));
    } else {
      mbar_arrive(&empty[s]);
    }
  }
  if (feeder && lane == 0 && c + tgp::STAGES < fd.nchunks) {
    mbar_wait(&empty[s], ph);
    fd.issue(c + tgp::STAGES, s, full);
  }
}

template <typename TA, typename TB, int WR, int WC, bool DIAG, bool BORDER = false>
__device__ __forceinline__ void panel_consume(const PanelFeed& fd, bool feeder, const unsigned char* b_base,
                                              int b_stage_bytes, uint64_t* full, uint64_t* empty, int i0, int j0,
                                              int lane, double* __restrict__ W, int K2p, int jb = 0) {
  const int g = lane >> 2, t = lane & 3;
  // byte offsets of this lane's fragments for the two row parities of a k-step.
  // Column 8 ii + c lands in box (c + 8 ii) / W at a swizzled position that
  // repeats every W / 8 blocks (a whole box further on), so only W / 8 base
  // offsets per operand and parity live in registers; the rest are immediate
  // +BOX_BYTES displacements of the unrolled loads (5 x 9 tiles: 12 instead of
  // 28 offset registers next to 90 accumulators).
  constexpr int PA = 128 / (int)sizeof(TA) / 8, PB = 128 / (int)sizeof(TB) / 8;
  constexpr int NA = PA < WR ? PA : WR, NB = PB < WC ? PB : WC;
  int offa[NA][2], offb[NB][2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int row = p + 2 * t;
#pragma unroll
    for (int ii = 0; ii < NA; ++ii) offa[ii][p] = panel_offset<TA>(row, 8 * (i0 + ii) + g);
#pragma unroll
    for (int jj = 0; jj < NB; ++jj) offb[jj][p] = panel_offset<TB>(row, 8 * (j0 + jj) + g);
  }
  // border blocks (ii, jb): the extra column block of a bordered symmetric Gram
  int offbd[2] = {0, 0};
  double accb[BORDER ? WR : 1][2];
  if (BORDER) {
#pragma unroll
    for (int p = 0; p < 2; ++p) offbd[p] = panel_offset<TB>(p + 2 * t, 8 * jb + g);
#pragma unroll
    for (int ii = 0; ii < WR; ++ii) accb[ii][0] = accb[ii][1] = 0.0;
  }
  double acc[WR][WC][2];
#pragma unroll
  for (int ii = 0; ii < WR; ++ii)
#pragma unroll
    for (int jj = 0; jj < WC; ++jj) acc[ii][jj][0] = acc[ii][jj][1] = 0.0;

  int s = 0;
  unsigned ph = 0;
  for (int64_t c = 0; c < fd.nchunks; ++c) {
    mbar_wait(&full[s], ph);
    const unsigned char* pa = fd.a_sm + s * fd.a_stage;
    const unsigned char* pb = b_base + s * b_stage_bytes;
#pragma unroll
    for (int ks = 0; ks < tgp::BR / 4; ++ks) {
      const int p = ks & 1, hi = (ks >> 1) * 1024;   // rows +8 -> +1024 B, same swizzle key
      double a[WR], b[WC];
#pragma unroll
      for (int ii = 0; ii < WR; ++ii)
        a[ii] = (double)*reinterpret_cast<const TA*>(pa + offa[ii % NA][p] + (ii / NA) * tgp::BOX_BYTES + hi);
#pragma unroll
      for (int jj = 0; jj < WC; ++jj)
        b[jj] = (double)*reinterpret_cast<const TB*>(pb + offb[jj % NB][p] + (jj / NB) * tgp::BOX_BYTES + hi);
#pragma unroll
      for (int ii = 0; ii < WR; ++ii)
#pragma unroll
        for (int jj = 0; jj < WC; ++jj)
          if (!DIAG || ii <= jj) dmma884(acc[ii][jj], a[ii], b[jj]);
      if (BORDER) {
        const double bd = (double)*reinterpret_cast<const TB*>(pb + offbd[p] + hi);
#pragma unroll
        for (int ii = 0; ii < WR; ++ii) dmma884(accb[ii], a[ii], bd);
      }
    }
    panel_release(fd, feeder, lane, c, s, ph, full, empty);
    if (++s == tgp::STAGES) { s = 0; ph ^= 1; }
  }
#pragma unroll
  for (int ii = 0; ii < WR; ++ii) {
    const int i = 8 * (i0 + ii) + g;
#pragma unroll
    for (int jj = 0; jj < WC; ++jj) {
      if (DIAG && ii > jj) continue;
      const int j = 8 * (j0 + jj) + 2 * t;
      *reinterpret_cast<double2*>(W + (int64_t)i * K2p + j) = make_double2(acc[ii][jj][0], acc[ii][jj][1]);
    }
    if (BORDER)
      *reinterpret_cast<double2*>(W + (int64_t)i * K2p + 8 * jb + 2 * t) = make_double2(accb[ii][0], accb[ii][1]);
  }
}

template <typename TA, typename TB, int WR, int WC, bool SYM, int CL>
__global__ void __launch_bounds__(tgp::THREADS, 1)
tall_gram_panel_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                       const __grid_constant__ CUtensorMap atmap, const __grid_constant__ CUtensorMap btmap,
                       const __grid_constant__ TallGramPanelArgs pa) {
  const TallGramArgs& args = pa.g;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align by offsetting the __shared__ array itself (keeps the shared window:
  // LDS, not generic LD, for every fragment load)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  PanelFeed fd;
  fd.amap = &amap;
  fd.bmap = &bmap;
  fd.atmap = &atmap;
  fd.btmap = &btmap;
  fd.afull = pa.a_full;
  fd.bfull = pa.b_full;
  fd.atail = pa.a_tail;
  fd.btail = pa.b_tail;
  fd.a_stage = pa.nba * tgp::BOX_BYTES;
  fd.b_stage = pa.nbb * tgp::BOX_BYTES;
  fd.a_sm = base;
  fd.b_sm = base + tgp::STAGES * fd.a_stage;
  fd.la = pa.lda_boxes;
  fd.lb = pa.ldb_boxes;
  fd.wa = 128 / sizeof(TA);
  fd.wb = 128 / sizeof(TB);
  // boxes wholly past K are never loaded: their smem only feeds padding outputs
  fd.bytes = (unsigned)((pa.lda_boxes + pa.ldb_boxes) * tgp::BOX_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(fd.b_sm + tgp::STAGES * fd.b_stage);
  uint64_t* empty = full + tgp::STAGES;

  const int part = blockIdx.x;
  fd.cl = CL;
  fd.rank = CL > 1 ? (int)(blockIdx.x % CL) : 0;   // cluster dims (CL, 1, 1): rank = x % CL
  fd.rbeg = (int64_t)blockIdx.y * args.rows_per_split;
  const int64_t rend = min(args.n, fd.rbeg + args.rows_per_split);
  fd.nchunks = rend > fd.rbeg ? (rend - fd.rbeg + tgp::BR - 1) / tgp::BR : 0;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const bool feeder = warp == 0;

  if (tid == 0) {
    for (int s = 0; s < tgp::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL * tgp::THREADS / 32);
    }
    mbar_fence_init();
  }
  if (CL > 1)
    gp_cluster_sync();   // every CTA's barriers initialised before any multicast / remote arrive
  else
    __syncthreads();
  if (tid == 0)
    for (int s = 0; s < tgp::STAGES && s < fd.nchunks; ++s) fd.issue(s, s, full);

  const PanelTile tl = pa.tile[part * 8 + warp];
  double* W = args.W + (int64_t)blockIdx.y * args.K1p * args.K2p;
  const unsigned char* bb = SYM ? fd.a_sm : fd.b_sm;
  const int bst = SYM ? fd.a_stage : fd.b_stage;
  bool done = true;
  if (tl.kind == 1) {
    panel_consume<TA, TB, WR, WC, false>(fd, feeder, bb, bst, full, empty, tl.i0, tl.j0, lane, W, args.K2p);
  } else if (SYM && tl.kind == 2) {
    panel_consume<TA, TB, WR, WC, true>(fd, feeder, bb, bst, full, empty, tl.i0, tl.j0, lane, W, args.K2p);
  } else {
    done = false;
    if constexpr (SYM && CL == 1) {   // bordered / rebalanced symmetric plans (host: panel_plan)
      done = true;
      if (tl.kind == 3)
        panel_consume<TA, TB, WR, WC, true, true>(fd, feeder, bb, bst, full, empty, tl.i0, tl.j0, lane, W,
                                                  args.K2p, pa.jb);
      else if (tl.kind == 4)
        panel_consume<TA, TB, WR, 3, false>(fd, feeder, bb, bst, full, empty, tl.i0, tl.j0, lane, W, args.K2p);
      else if (tl.kind == 5)
        panel_consume<TA, TB, WR, 4, false>(fd, feeder, bb, bst, full, empty, tl.i0, tl.j0, lane, W, args.K2p);
      else
        done = false;
    }
  }
  if (!done) {   // idle slot: keep the ring moving
    int s = 0;
    unsigned ph = 0;
    for (int64_t c = 0; c < fd.nchunks; ++c) {
      mbar_wait(&full[s], ph);
      panel_release(fd, feeder, lane, c, s, ph, full, empty);
      if (++s == tgp::STAGES) { s = 0; ph ^= 1; }
    }
  }
  if (CL > 1) gp_cluster_sync();   // no peer may still arrive on / multicast into an exited CTA
}

}  // namespace fdmd
