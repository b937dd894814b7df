// extern "C" boundary of libfdmd.so (declared in include/fdmd.h).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cusolverDn.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>
#include <algorithm>

#include "../../include/fdmd.h"
#include "fdmd_kernels.cuh"

// kernels live in fdmd_kernels.cu (same translation unit, see build)
#include "fdmd_kernels.cu"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) return fail(FDMD_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

#define LAUNCH_CHECK(name)                                                                  \
  do {                                                                                      \
    cudaError_t _e = cudaGetLastError();                                                    \
    if (_e != cudaSuccess) return fail(FDMD_ERR_CUDA, "%s launch: %s", name, cudaGetErrorString(_e)); \
  } while (0)

int sm_count_cached() {
  static thread_local int dev_cached = -1, sms = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    dev_cached = dev;
  }
  return sms > 0 ? sms : 148;
}

inline size_t dsize(int dt) { return dt == FDMD_F32 ? 4 : 8; }

// ------------------------------- tall_gemm --------------------------------
template <int NF> constexpr int bn_of() { return 32 * NF; }

int pick_nf(int N) {
  static const int forced = [] {
    const char* e = getenv("FDMD_TG_NF");  // tuning override: 1, 2, 4 or 7
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2 || forced == 4 || forced == 7) return forced;
  if (N <= 32) return 1;
  if (N <= 64) return 2;
  if (N <= 128) return 4;
  return 7;
}

int64_t tg_tiles(int64_t n) { return (n + fdmd::tg::BM - 1) / fdmd::tg::BM; }

// Stream-ordered scratch (padded B, solver workspaces) comes from the device's
// default memory pool with an unbounded release threshold, so repeated calls
// reuse the same pages instead of unmapping/remapping them at every sync.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static thread_local int tuned = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (tuned != dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    tuned = dev;
  }
  return cudaMallocAsync(p, bytes, s);
}

// ---- TMA / warp-specialised variant (default; FDMD_TG_IMPL=cpasync selects the ring kernel)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

bool tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("FDMD_TG_IMPL");
    return !(e && strcmp(e, "cpasync") == 0);
  }();
  return on;
}

template <typename TA, int AL, int NF, typename TC, int CL, bool ST>
int launch_tg_tma(const fdmd::TallGemmArgs& a, cudaStream_t s, int& grid_x, bool& used) {
  used = false;
  auto encode = tensor_map_encoder();
  const size_t elt = sizeof(TA);
  if (!tma_enabled() || !encode || (reinterpret_cast<uintptr_t>(a.A) & 15) || ((a.lda * elt) % 16) != 0 ||
      a.n >= (int64_t)INT32_MAX)
    return FDMD_OK;
  CUtensorMap map;
  cuuint64_t dims[2], strides[1];
  cuuint32_t box[2], estr[2] = {1, 1};
  // swizzled boxes (layout in fdmd_tall_tma.cuh: TTSmem / tt_a_offset)
  CUtensorMapSwizzle swz;
  if (AL == fdmd::LAYOUT_ROW) {
    dims[0] = (cuuint64_t)a.K; dims[1] = (cuuint64_t)a.n; box[0] = fdmd::tt::BK; box[1] = fdmd::tt::BM;
    swz = elt == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  } else {
    dims[0] = (cuuint64_t)a.n; dims[1] = (cuuint64_t)a.K; box[0] = (cuuint32_t)(128 / elt); box[1] = fdmd::tt::BK;
    swz = CU_TENSOR_MAP_SWIZZLE_128B;
  }
  strides[0] = (cuuint64_t)(a.lda * elt);
  CUresult r = encode(&map, elt == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                      const_cast<void*>(a.A), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return FDMD_OK;  // unsupported shape: ring kernel
  constexpr int BN = 32 * NF;
  const int gy = (a.N + BN - 1) / BN;
  const int Kp = (a.K + fdmd::tt::BK - 1) / fdmd::tt::BK * fdmd::tt::BK;
  const int64_t ldbp = (int64_t)gy * BN;
  double* Bp = nullptr;
  CUDA_TRY(scratch_alloc((void**)&Bp, sizeof(double) * Kp * ldbp, s));
  CUDA_TRY(cudaMemsetAsync(Bp, 0, sizeof(double) * Kp * ldbp, s));
  CUDA_TRY(cudaMemcpy2DAsync(Bp, ldbp * sizeof(double), a.B, a.ldb * sizeof(double), a.N * sizeof(double), a.K,
                             cudaMemcpyDeviceToDevice, s));
  // B as one TMA box per chunk: {BN + 4 columns (the smem row padding), 16 k}
  CUtensorMap bmap;
  {
    constexpr int LDB = fdmd::TTSmem<TA, AL, NF>::LDB;
    cuuint64_t bd[2] = {(cuuint64_t)ldbp, (cuuint64_t)Kp};
    cuuint64_t bs[1] = {(cuuint64_t)(ldbp * sizeof(double))};
    cuuint32_t bb[2] = {(cuuint32_t)LDB, (cuuint32_t)fdmd::tt::BK};
    cuuint32_t be[2] = {1, 1};
    if (encode(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, Bp, bd, bs, bb, be, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      cudaFreeAsync(Bp, s);
      return FDMD_OK;   // fall back to the ring kernel (used stays false)
    }
  }
  fdmd::TTArgs ta{a, Bp, ldbp, {NF, NF, NF, NF}};
  const int nb = (a.N + 7) / 8;
  if (gy == 1 && NF > 1 && nb >= 4 * (NF - 1) && nb < 4 * NF)   // e.g. N = 200: 7,6,6,6 blocks
    for (int q = 0; q < 4; ++q) ta.wblk[q] = nb / 4 + (q < nb % 4 ? 1 : 0);
  auto kern = fdmd::tall_gemm_tma_kernel<TA, AL, NF, TC, CL, ST>;
  const int smem = (int)sizeof(fdmd::TTSmem<TA, AL, NF>) + 1024;   // + alignment slack
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = dev;
  }
  const int64_t ntiles = (a.n + fdmd::tt::BM - 1) / fdmd::tt::BM;
  grid_x = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, std::max(1, sm_count_cached() - a.reserve_sms)));
  dim3 grid(grid_x, gy);
  kern<<<grid, fdmd::tt::THREADS, smem, s>>>(map, bmap, ta);
  LAUNCH_CHECK("tall_gemm_tma");
  CUDA_TRY(cudaFreeAsync(Bp, s));
  used = true;
  return FDMD_OK;
}

template <typename TA, int AL, int NF, typename TC, int CL, bool ST>
int launch_tg(const fdmd::TallGemmArgs& a, cudaStream_t s, int& grid_x) {
  bool used = false;
  int rc = launch_tg_tma<TA, AL, NF, TC, CL, ST>(a, s, grid_x, used);
  if (rc != FDMD_OK || used) return rc;
  auto kern = fdmd::tall_gemm_kernel<TA, AL, NF, TC, CL, ST>;
  const int smem = (int)sizeof(fdmd::TGSmem<TA, AL, NF>);
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = dev;
  }
  dim3 grid(grid_x, (a.N + 32 * NF - 1) / (32 * NF));
  kern<<<grid, fdmd::tg::THREADS, smem, s>>>(a);
  LAUNCH_CHECK("tall_gemm");
  return FDMD_OK;
}

template <typename TA, int AL, int NF>
int dispatch_tg_c(const fdmd::TallGemmArgs& a, int c_dtype, int c_layout, bool stats, cudaStream_t s,
                  int& grid_x) {
  if (c_layout == FDMD_ROW) {
    if (stats) return fail(FDMD_ERR_INVALID, "pair_stats requires column-major C (or C == NULL)");
    if (c_dtype == FDMD_F64) return launch_tg<TA, AL, NF, double, fdmd::LAYOUT_ROW, false>(a, s, grid_x);
    return launch_tg<TA, AL, NF, float, fdmd::LAYOUT_ROW, false>(a, s, grid_x);
  }
  if (c_dtype == FDMD_F64)
    return stats ? launch_tg<TA, AL, NF, double, fdmd::LAYOUT_COL, true>(a, s, grid_x)
                 : launch_tg<TA, AL, NF, double, fdmd::LAYOUT_COL, false>(a, s, grid_x);
  return stats ? launch_tg<TA, AL, NF, float, fdmd::LAYOUT_COL, true>(a, s, grid_x)
               : launch_tg<TA, AL, NF, float, fdmd::LAYOUT_COL, false>(a, s, grid_x);
}

template <typename TA, int AL>
int dispatch_tg_nf(const fdmd::TallGemmArgs& a, int c_dtype, int c_layout, bool stats, cudaStream_t s,
                   int& grid_x) {
  switch (pick_nf(a.N)) {
    case 1: return dispatch_tg_c<TA, AL, 1>(a, c_dtype, c_layout, stats, s, grid_x);
    case 2: return dispatch_tg_c<TA, AL, 2>(a, c_dtype, c_layout, stats, s, grid_x);
    case 4: return dispatch_tg_c<TA, AL, 4>(a, c_dtype, c_layout, stats, s, grid_x);
    default: return dispatch_tg_c<TA, AL, 7>(a, c_dtype, c_layout, stats, s, grid_x);
  }
}

int tg_grid_x(int64_t n) {
  const int64_t tiles = tg_tiles(n);
  const int64_t want = (int64_t)sm_count_cached() * 2;
  return (int)std::max<int64_t>(1, std::min(tiles, want));
}

// ------------------------------- tall_gram --------------------------------
struct GramPlan {
  int ti, tj, tiles, splits;
  int64_t rows_per_split;
  int K1p, K2p;
};

// sw = warp-specialised TMA kernel (64 x TN tiles, full tile grid with
// early exit below the diagonal); otherwise the cp.async ring kernel (64 x 64
// tiles, triangular enumeration when symmetric).
GramPlan gram_plan(int64_t n, int K1, int K2, int symmetric, bool sw = false, int TN = 64) {
  GramPlan p;
  p.ti = (K1 + fdmd::gr::T - 1) / fdmd::gr::T;
  p.tj = (K2 + TN - 1) / TN;
  p.tiles = (symmetric && TN == fdmd::gr::T) ? p.ti * (p.ti + 1) / 2 : p.ti * p.tj;
  p.K1p = p.ti * fdmd::gr::T;
  p.K2p = p.tj * TN;
  const int64_t target = (int64_t)sm_count_cached() * (sw ? (TN > 64 ? 2 : 4) : 4);
  const int64_t max_splits = std::max<int64_t>(1, (n + 255) / 256);
  int64_t splits = std::max<int64_t>(1, target / p.tiles);
  splits = std::min(splits, max_splits);
  p.rows_per_split = ((n + splits - 1) / splits + 15) / 16 * 16;
  if (p.rows_per_split == 0) p.rows_per_split = 16;
  p.splits = (int)std::max<int64_t>(1, (n + p.rows_per_split - 1) / p.rows_per_split);
  return p;
}

bool gram_sw_eligible(const void* A, int a_dtype, int a_layout, int64_t lda, const void* B, int b_dtype,
                      int b_layout, int64_t ldb, int64_t n) {
  return a_layout == FDMD_ROW && b_layout == FDMD_ROW && tma_enabled() && tensor_map_encoder() &&
         !(reinterpret_cast<uintptr_t>(A) & 15) && !(reinterpret_cast<uintptr_t>(B) & 15) &&
         (lda * (int64_t)dsize(a_dtype)) % 16 == 0 && (ldb * (int64_t)dsize(b_dtype)) % 16 == 0 &&
         n < (int64_t)INT32_MAX;
}

template <typename TA, typename TB, int NFB>
int launch_gram_sw(const fdmd::TallGramArgs& a, int tiles, int splits, cudaStream_t s) {
  {
    auto kt = fdmd::tall_gram_sw_kernel<TA, TB, NFB>;
    const int smt = (int)sizeof(fdmd::TGSSmem<TA, TB, NFB>) + 1024;
    CUtensorMap maps[2];
    const void* ptr[2] = {a.A, a.B};
    const int64_t ld[2] = {a.lda, a.ldb};
    const int kdim[2] = {a.K1, a.K2};
    const size_t elt[2] = {sizeof(TA), sizeof(TB)};
    bool ok = true;
    for (int i = 0; i < 2 && ok; ++i) {
      cuuint64_t dims[2] = {(cuuint64_t)kdim[i], (cuuint64_t)a.n};
      cuuint64_t strides[1] = {(cuuint64_t)(ld[i] * elt[i])};
      cuuint32_t box[2] = {(cuuint32_t)(128 / elt[i]), (cuuint32_t)fdmd::tgs::BR};
      cuuint32_t estr[2] = {1, 1};
      ok = tensor_map_encoder()(&maps[i], elt[i] == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                                2, const_cast<void*>(ptr[i]), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (!ok) return fail(FDMD_ERR_CUDA, "tall_gram: tensor map encode failed");
    static thread_local int conf_t = -1;
    int dv = 0;
    cudaGetDevice(&dv);
    if (conf_t != dv) {
      CUDA_TRY(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, smt));
      conf_t = dv;
    }
    kt<<<dim3(tiles, splits), fdmd::tgs::THREADS, smt, s>>>(maps[0], maps[1], a);
    LAUNCH_CHECK("tall_gram_sw");
    return FDMD_OK;
  }
}

// ---- panel Gram (fdmd_gram_panel.cuh): whole output per CTA partition -----
struct PanelPlan {
  bool ok = false;
  bool transposed = false;   // run as B^T A (better tiling), reduce transposes back
  int cost = 0;              // sum over partitions of the busiest sub-partition (8x8 blocks)
  int WR = 5, WC = 7, P = 0, splits = 0, K1p = 0, K2p = 0, nba = 0, nbb = 0;
  int cl = 1;                // cluster size (the P partitions of a split share one row stream)
  int border = 0, jb = 0;    // bordered symmetric Gram: extra column K (block column jb when K % 8 == 0)
  int cuts = 0;              // pairs of adjacent full tiles re-cut into 3 + 4 + 3 block columns
  int64_t rows_per_split = 0;
  size_t smem = 0;
  fdmd::PanelTile tile[fdmd::tgp::MAXP * 8];
};

bool panel_enabled() {
  static const bool on = [] {
    const char* e = getenv("FDMD_GRAM_IMPL");
    return !(e && strcmp(e, "tile") == 0);
  }();
  return on;
}

// Opt-in (FDMD_GRAM_CLUSTER=1): the cluster-shared row stream brings DRAM
// traffic down to the algorithmic bytes (ncu: 41 / 80.5 / 121.6 GB for the
// three fit Grams, from 82 / 161 / 257) but ties the partitions of a split to
// one pace — the lighter partition's SM can no longer move on to its next
// CTA — and GPC packing leaves SMs idle for 3-CTA clusters: 72 -> 88 ms
// (X^T X), 150 -> 197 ms (Q^T S) at config-3 size (tools/gram_sweep.py).
bool gram_cluster_enabled() {
  static const bool on = [] {
    const char* e = getenv("FDMD_GRAM_CLUSTER");
    return e && strcmp(e, "1") == 0;
  }();
  return on;
}

// co-resident clusters of `cl` panel-Gram CTAs (cudaOccupancyMaxActiveClusters;
// cached per device, cluster size and smem footprint)
int gram_cluster_capacity(int cl, size_t smem);

// Warp tiles of WR x WC 8x8 blocks cover the (upper, if symmetric) block grid;
// they are packed into partitions of 8 consumer warps so that the DMMA count
// per SM sub-partition (warps w, w+4) is balanced: tiles sorted by weight, the
// k-th heaviest sharing a sub-partition with the k-th lightest, sub-partitions
// grouped into partitions by load (cost = sum over partitions of the busiest
// sub-partition = SM time per 16-row chunk).
//
// Symmetric Grams (r02): 10 full (25 blocks) + 5 diagonal (15) tiles of a
// 200 x 200 Gram leave two sub-partitions with 25 + 25 next to 25 + 15 (cost
// 90 for 325 blocks). `cuts` pairs of horizontally adjacent full tiles are
// re-cut into 3 + 4 + 3 block columns (15 + 20 + 15 blocks, kinds 4 / 5), one
// more warp tile per cut: one cut gives 7 x 40 + 45 (cost 85). border = 1
// (bordered Gram: C = [A^T A | A^T a_K], A with K + 1 columns): when K is a
// multiple of 8 the border column block jb = K / 8 is attached to the diagonal
// tiles (kind 3: 15 + 5 blocks; with one cut 6 x 45 + 2 x 40, cost 90 for 350
// blocks — the separate HBM-bound X^T s_m pass is gone); otherwise column K
// lies inside the last block columns of the tile grid and only has to be
// loaded. The number of cuts is the one with the cheapest schedule.
PanelPlan panel_plan(int64_t n, int K1, int K2, int symmetric, size_t ea, size_t eb, int wc = 7, int border = 0,
                     int cuts = -1) {
  PanelPlan p;
  p.WC = wc;
  if (symmetric) { p.WR = 5; p.WC = 5; }
  const int MB = (K1 + 7) / 8, NB = (K2 + 7) / 8;
  const int TI = (MB + p.WR - 1) / p.WR, TJ = (NB + p.WC - 1) / p.WC;
  // the border needs its own block column only when column K starts a block the
  // tile grid does not cover (K % 8 == 0 and the block count a multiple of WR);
  // otherwise it lies inside the last (possibly padding) block columns of the grid
  const bool bcol = symmetric && border && K1 % 8 == 0 && K1 / 8 >= TJ * p.WC;
  if (border && (!symmetric || gram_cluster_enabled())) return p;
  if (symmetric && cuts < 0) {
    // cheapest schedule over the number of cuts (ties: fewer partitions, fewer cuts)
    PanelPlan best;
    const int max_cuts = gram_cluster_enabled() ? 0 : 4;
    for (int c = 0; c <= max_cuts; ++c) {
      PanelPlan q = panel_plan(n, K1, K2, symmetric, ea, eb, wc, border, c);
      if (!q.ok || q.cuts != c) break;
      if (!best.ok || q.cost < best.cost || (q.cost == best.cost && q.P < best.P)) best = q;
    }
    return best;
  }
  struct T { short i0, j0, kind; int w; };
  std::vector<T> ts;
  int ncut = 0;
  for (int I = 0; I < TI; ++I)
    for (int J = 0; J < TJ; ++J) {
      if (symmetric && J < I) continue;
      const bool diag = symmetric && I == J;
      if (symmetric && !diag && ncut < cuts && J + 1 < TJ) {
        // (I, J) and (I, J + 1) as 3 + 4 + 3 block columns
        const short i0 = (short)(I * p.WR), j0 = (short)(J * p.WC);
        ts.push_back({i0, j0, 4, p.WR * 3});
        ts.push_back({i0, (short)(j0 + 3), 5, p.WR * 4});
        ts.push_back({i0, (short)(j0 + 7), 4, p.WR * 3});
        ++ncut;
        ++J;
        continue;
      }
      const int w = diag ? p.WR * (p.WR + 1) / 2 + (bcol ? p.WR : 0) : p.WR * p.WC;
      ts.push_back({(short)(I * p.WR), (short)(J * p.WC), (short)(diag ? (bcol ? 3 : 2) : 1), w});
    }
  p.cuts = ncut;
  p.border = border;
  p.jb = bcol ? K1 / 8 : 0;
  const int ntile = (int)ts.size();
  p.P = (ntile + 7) / 8;
  if (p.P > fdmd::tgp::MAXP) return p;
  p.K1p = TI * p.WR * 8;
  p.K2p = std::max(TJ * p.WC * 8, bcol ? 8 * (p.jb + 1) : 0);
  p.nba = (int)((std::max(p.K1p, bcol ? 8 * (p.jb + 1) : 0) * ea + 127) / 128);
  p.nbb = symmetric ? 0 : (int)((p.K2p * eb + 127) / 128);
  p.smem = (size_t)fdmd::tgp::STAGES * (p.nba + p.nbb) * fdmd::tgp::BOX_BYTES + 2 * fdmd::tgp::STAGES * 8 + 1024;
  if (p.smem > 227 * 1024) return p;
  std::stable_sort(ts.begin(), ts.end(), [](const T& x, const T& y) { return x.w > y.w; });
  const int nbins = p.P * 4;                       // (partition, sub-partition)
  std::vector<int> load(nbins, 0);
  std::vector<std::vector<const T*>> bin(nbins);
  // bins in order of their heavy tile; bin k also takes tile 2 * nbins - 1 - k
  // (the k-th lightest, idle slots counted as weight 0)
  for (int k = 0; k < nbins; ++k) {
    if (k < ntile) { bin[k].push_back(&ts[k]); load[k] += ts[k].w; }
    const int o = 2 * nbins - 1 - k;
    if (o < ntile && o >= nbins) { bin[k].push_back(&ts[o]); load[k] += ts[o].w; }
  }
  // partitions = groups of 4 bins by decreasing load
  std::vector<int> ord(nbins);
  for (int k = 0; k < nbins; ++k) ord[k] = k;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return load[x] > load[y]; });
  {
    std::vector<int> l2(nbins);
    std::vector<std::vector<const T*>> b2(nbins);
    for (int k = 0; k < nbins; ++k) { l2[k] = load[ord[k]]; b2[k] = bin[ord[k]]; }
    load.swap(l2);
    bin.swap(b2);
  }
  for (int part = 0; part < p.P; ++part) {
    int mx = 0;
    for (int sub = 0; sub < 4; ++sub) mx = std::max(mx, load[part * 4 + sub]);
    p.cost += mx;
  }
  // warp 0 also feeds the ring (it waits for the slowest warp every chunk):
  // give it the lightest sub-partition of its CTA, and the idle slot if any
  for (auto& e : p.tile) e = fdmd::PanelTile{0, 0, 0, 0};
  for (int part = 0; part < p.P; ++part) {
    int order[4] = {0, 1, 2, 3};
    std::stable_sort(order, order + 4, [&](int x, int y) { return load[part * 4 + x] < load[part * 4 + y]; });
    for (int sub = 0; sub < 4; ++sub) {
      auto& bl = bin[part * 4 + order[sub]];
      std::stable_sort(bl.begin(), bl.end(), [](const T* x, const T* y) { return x->w < y->w; });
      const int off = (int)(2 - bl.size());       // idle first (warp sub), then lightest
      for (size_t q = 0; q < bl.size(); ++q) {
        const int warp = sub + 4 * (off + (int)q);
        p.tile[part * 8 + warp] = fdmd::PanelTile{bl[q]->i0, bl[q]->j0, bl[q]->kind, 0};
      }
    }
  }
  // row splits: 2 waves of one CTA per SM, chunk-aligned (16 rows). With
  // clusters (P in 2..4) a wave is the number of co-resident P-CTA clusters
  // (GPC-limited, e.g. 45 clusters of 3 = 135 SMs), so 2 waves never leave a
  // straggler cluster. FDMD_GRAM_SPLITS overrides the split count
  // (tools/gram_sweep.py); FDMD_GRAM_CLUSTER=1 enables the clusters.
  const int64_t max_splits = std::max<int64_t>(1, (n + 15) / 16);
  p.cl = (p.P >= 2 && p.P <= 4 && gram_cluster_enabled()) ? p.P : 1;
  int64_t splits = std::max<int64_t>(1, ((int64_t)sm_count_cached() * 2 + p.P - 1) / p.P);
  if (p.cl > 1) {
    const int per_wave = gram_cluster_capacity(p.cl, p.smem);
    if (per_wave > 0)
      splits = 2 * (int64_t)per_wave;
    else
      p.cl = 1;
  }
  if (const char* e = getenv("FDMD_GRAM_SPLITS")) {
    const int64_t v = atoll(e);
    if (v > 0) splits = v;
  }
  splits = std::min(splits, max_splits);
  p.rows_per_split = ((n + splits - 1) / splits + 15) / 16 * 16;
  if (p.rows_per_split == 0) p.rows_per_split = 16;
  p.splits = (int)std::max<int64_t>(1, (n + p.rows_per_split - 1) / p.rows_per_split);
  p.ok = true;
  return p;
}

// orientation and warp-tile width with the cheapest schedule: cost = sum over
// partitions of the busiest sub-partition = SM time per 16-row chunk. 5 x 9
// tiles (90 accumulators per lane) cover a 200 x 201 projection in 2
// partitions of 15 tiles (0.90 of the DMMA work per SM-time) where 5 x 7
// needs 3 partitions of 20 (0.77); ties keep fewer partitions (DRAM reads).
PanelPlan panel_plan_best(int64_t n, int K1, int K2, int symmetric, size_t ea, size_t eb) {
  PanelPlan p = panel_plan(n, K1, K2, symmetric, ea, eb);
  if (symmetric) return p;
  static const int wide = [] {
    const char* e = getenv("FDMD_GRAM_WC");   // 7 or 9 forces the tile width (tools/gram_sweep.py)
    return e ? atoi(e) : 0;
  }();
  auto better = [](const PanelPlan& a, const PanelPlan& b) {   // a better than b?
    if (!a.ok) return false;
    if (!b.ok) return true;
    return a.cost < b.cost || (a.cost == b.cost && a.P < b.P);
  };
  PanelPlan best;
  for (int wc : {7, 9}) {
    if (wide && wc != wide) continue;
    PanelPlan q = panel_plan(n, K1, K2, 0, ea, eb, wc);
    if (better(q, best)) best = q;
    PanelPlan t = panel_plan(n, K2, K1, 0, eb, ea, wc);
    t.transposed = true;
    if (better(t, best)) best = t;
  }
  return best.ok ? best : p;
}

int gram_cluster_capacity(int cl, size_t smem) {
  static thread_local std::unordered_map<long long, int> cache;
  int dv = 0;
  cudaGetDevice(&dv);
  const long long key = ((long long)dv << 40) | ((long long)cl << 32) | (long long)smem;
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cl, 64);
  cfg.blockDim = dim3(fdmd::tgp::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int num = 0;
  cudaError_t e = cudaErrorInvalidValue;
  auto probe = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    return cudaOccupancyMaxActiveClusters(&num, kern, &cfg);
  };
  if (cl == 2) e = probe(fdmd::tall_gram_panel_kernel<double, double, 5, 7, false, 2>);
  if (cl == 3) e = probe(fdmd::tall_gram_panel_kernel<double, double, 5, 7, false, 3>);
  if (cl == 4) e = probe(fdmd::tall_gram_panel_kernel<double, double, 5, 7, false, 4>);
  if (e != cudaSuccess) {
    cudaGetLastError();
    num = 0;
  }
  cache[key] = num;
  return num;
}

template <typename TA, typename TB, int WR, int WC, bool SYM, int CL>
int launch_gram_panel_cl(const fdmd::TallGramArgs& a, const PanelPlan& pl, cudaStream_t s);

template <typename TA, typename TB, int WR, int WC, bool SYM>
int launch_gram_panel(const fdmd::TallGramArgs& a, const PanelPlan& pl, cudaStream_t s) {
  switch (pl.cl) {
    case 2: return launch_gram_panel_cl<TA, TB, WR, WC, SYM, 2>(a, pl, s);
    case 3: return launch_gram_panel_cl<TA, TB, WR, WC, SYM, 3>(a, pl, s);
    case 4: return launch_gram_panel_cl<TA, TB, WR, WC, SYM, 4>(a, pl, s);
    default: return launch_gram_panel_cl<TA, TB, WR, WC, SYM, 1>(a, pl, s);
  }
}

template <typename TA, typename TB, int WR, int WC, bool SYM, int CL>
int launch_gram_panel_cl(const fdmd::TallGramArgs& a, const PanelPlan& pl, cudaStream_t s) {
  auto kt = fdmd::tall_gram_panel_kernel<TA, TB, WR, WC, SYM, CL>;
  CUtensorMap maps[2], tmaps[2];
  const void* ptr[2] = {a.A, a.B};
  const int64_t ld[2] = {a.lda, a.ldb};
  const int kdim[2] = {a.K1 + (SYM && pl.border ? 1 : 0), a.K2};   // bordered: column K is loaded too
  const size_t elt[2] = {sizeof(TA), sizeof(TB)};
  int nfull[2] = {0, 0}, tail[2] = {0, 0};
  // Full 128-B column blocks of a row-major n x K operand are one 3-D box
  // ({W elements, 16 rows, full blocks} over dims {W, n, K / W} with strides
  // {ld, W}): they land as consecutive 16-row x 128-B SW128 boxes, the layout
  // panel_offset reads. A ragged last block (K % W != 0) is a 2-D box with
  // zero fill past K (a 3-D box would read the next row's columns, and past
  // the allocation on the last row).
  for (int i = 0; i < (SYM ? 1 : 2); ++i) {
    const int W = 128 / (int)elt[i];
    const int loaded = i == 0 ? std::min(pl.nba, (kdim[0] + W - 1) / W) : std::min(pl.nbb, (kdim[1] + W - 1) / W);
    const int full = std::min(loaded, kdim[i] / W);
    nfull[i] = full;
    tail[i] = loaded > full ? 1 : 0;
    const bool need_2d = tail[i] || CL > 1;   // clusters load every box as a 2-D {W, 16} tile
    const auto dt = elt[i] == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    if (full > 0) {
      cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)a.n, (cuuint64_t)(kdim[i] / W)};
      cuuint64_t strides[2] = {(cuuint64_t)(ld[i] * elt[i]), (cuuint64_t)(W * elt[i])};
      cuuint32_t box[3] = {(cuuint32_t)W, (cuuint32_t)fdmd::tgp::BR, (cuuint32_t)full};
      cuuint32_t estr[3] = {1, 1, 1};
      if (tensor_map_encoder()(&maps[i], dt, 3, const_cast<void*>(ptr[i]), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(FDMD_ERR_CUDA, "tall_gram: tensor map encode failed");
    }
    if (need_2d) {
      cuuint64_t dims[2] = {(cuuint64_t)kdim[i], (cuuint64_t)a.n};
      cuuint64_t strides[1] = {(cuuint64_t)(ld[i] * elt[i])};
      cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)fdmd::tgp::BR};
      cuuint32_t estr[2] = {1, 1};
      if (tensor_map_encoder()(&tmaps[i], dt, 2, const_cast<void*>(ptr[i]), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(FDMD_ERR_CUDA, "tall_gram: tensor map encode failed");
    }
  }
  if (SYM) { maps[1] = maps[0]; tmaps[1] = tmaps[0]; }
  fdmd::TallGramPanelArgs pa{};
  pa.g = a;
  pa.g.K1p = pl.K1p;
  pa.g.K2p = pl.K2p;
  pa.g.rows_per_split = pl.rows_per_split;
  pa.nba = pl.nba;
  pa.nbb = pl.nbb;
  pa.lda_boxes = nfull[0] + tail[0];
  pa.ldb_boxes = SYM ? 0 : nfull[1] + tail[1];
  pa.a_full = nfull[0];
  pa.b_full = SYM ? 0 : nfull[1];
  pa.a_tail = tail[0];
  pa.b_tail = SYM ? 0 : tail[1];
  pa.jb = pl.jb;
  for (int i = 0; i < fdmd::tgp::MAXP * 8; ++i) pa.tile[i] = pl.tile[i];
  static thread_local int conf_t = -1;
  static thread_local size_t conf_smem = 0;
  int dv = 0;
  cudaGetDevice(&dv);
  if (conf_t != dv || conf_smem < pl.smem) {
    CUDA_TRY(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    conf_t = dv;
    conf_smem = 227 * 1024;
  }
  if (CL == 1) {
    kt<<<dim3(pl.P, pl.splits), fdmd::tgp::THREADS, pl.smem, s>>>(maps[0], maps[1], tmaps[0], tmaps[1], pa);
  } else {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(pl.P, pl.splits);
    cfg.blockDim = dim3(fdmd::tgp::THREADS);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, kt, maps[0], maps[1], tmaps[0], tmaps[1], pa));
  }
  LAUNCH_CHECK("tall_gram_panel");
  return FDMD_OK;
}

template <typename TA, int LA, typename TB, int LB>
int launch_gram(const fdmd::TallGramArgs& a, int tiles, int splits, cudaStream_t s) {
  auto kern = fdmd::tall_gram_kernel<TA, LA, TB, LB>;
  const int smem = (int)sizeof(fdmd::GramSmem<TA, LA, TB, LB>);
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = dev;
  }
  dim3 grid(tiles, splits);
  kern<<<grid, fdmd::gr::THREADS, smem, s>>>(a);
  LAUNCH_CHECK("tall_gram");
  return FDMD_OK;
}

template <typename TA, int LA>
int dispatch_gram_b(const fdmd::TallGramArgs& a, int b_dtype, int b_layout, int tiles, int splits,
                    cudaStream_t s) {
  if (b_dtype == FDMD_F32)
    return b_layout == FDMD_ROW ? launch_gram<TA, LA, float, fdmd::LAYOUT_ROW>(a, tiles, splits, s)
                                : launch_gram<TA, LA, float, fdmd::LAYOUT_COL>(a, tiles, splits, s);
  return b_layout == FDMD_ROW ? launch_gram<TA, LA, double, fdmd::LAYOUT_ROW>(a, tiles, splits, s)
                              : launch_gram<TA, LA, double, fdmd::LAYOUT_COL>(a, tiles, splits, s);
}

// ------------------------------- cuSOLVER ---------------------------------
struct SolverCtx {
  cusolverDnHandle_t h = nullptr;
  cusolverDnParams_t p = nullptr;
};

SolverCtx* solver_ctx() {
  static thread_local std::unordered_map<int, SolverCtx> ctxs;
  int dev = 0;
  cudaGetDevice(&dev);
  auto& c = ctxs[dev];
  if (!c.h) {
    if (cusolverDnCreate(&c.h) != CUSOLVER_STATUS_SUCCESS) return nullptr;
    if (cusolverDnCreateParams(&c.p) != CUSOLVER_STATUS_SUCCESS) return nullptr;
  }
  return &c;
}

template <int BN, int AST, int BST, int MC>
int launch_tc_decode_mc(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch,
                        const void* cl, int ldk, int nf, const float* fscale, float* out, int64_t ldo,
                        void* stream) {
  auto encode = tensor_map_encoder();
  if (!encode) return fail(FDMD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap maps[4];
  const void* ptrs[4] = {uh, ul, ch, cl};
  for (int i = 0; i < 4; ++i) {
    const bool a = i < 2;
    cuuint64_t dims[2] = {(cuuint64_t)r, (cuuint64_t)(a ? n : nf)};
    cuuint64_t strides[1] = {(cuuint64_t)((a ? ldu : ldk) * 2)};
    // A: each cluster CTA loads a 128/MC-row slice and multicasts it
    cuuint32_t box[2] = {(cuuint32_t)fdmd::tc::BKC, (cuuint32_t)(a ? fdmd::tc::BM / MC : BN)};
    cuuint32_t estr[2] = {1, 1};
    CUresult res = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptrs[i]), dims, strides,
                          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return fail(FDMD_ERR_CUDA, "tc_decode: tensor map encode failed (%d)", (int)res);
  }
  auto kern = fdmd::tc_decode_kernel<BN, AST, BST, MC>;
  const int smem = (int)sizeof(fdmd::TCSmem<BN, AST, BST>) + 1024;
  static thread_local int configured = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured != dev) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = dev;
  }
  fdmd::TCArgs ta{out, ldo, n, r, nf, fscale};
  const int64_t mtiles = (n + fdmd::tc::BM - 1) / fdmd::tc::BM;
  const int ny = (nf + BN - 1) / BN;
  const int gy = (ny + MC - 1) / MC * MC;          // whole clusters (tail CTAs of a cluster only compute)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(fdmd::tc::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  int gx;
  if (MC == 1) {
    gx = (int)std::max<int64_t>(1, std::min<int64_t>(mtiles, std::max(1, sm_count_cached() / ny)));
    cfg.numAttrs = 0;
  } else {
    // persistent: every cluster co-resident (clusters are packed per GPC, so
    // fewer than sm_count / MC may fit)
    static thread_local int max_clusters[9] = {0};
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = MC;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (max_clusters[MC] <= 0) {
      cfg.gridDim = dim3(1, MC);
      int nc = 0;
      CUDA_TRY(cudaOccupancyMaxActiveClusters(&nc, (void*)kern, &cfg));
      max_clusters[MC] = std::max(1, nc);
    }
    const int rows_of_clusters = gy / MC;
    gx = (int)std::max<int64_t>(1, std::min<int64_t>(mtiles, std::max(1, max_clusters[MC] / rows_of_clusters)));
  }
  cfg.gridDim = dim3(gx, MC == 1 ? ny : gy);
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], ta));
  LAUNCH_CHECK("tc_decode");
  return FDMD_OK;
}

// CTA-pair variant (cta_group::2, M = 256 rows x N = 256 frames per pair tile)
int launch_tc_decode_pair(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch,
                          const void* cl, int ldk, int nf, const float* fscale, float* out, int64_t ldo,
                          void* stream, int reserve_pairs = 0, void* ph = nullptr, void* pl = nullptr,
                          int64_t ldp = 0, float pscale = 1.f, double* st = nullptr, int64_t row_offset = 0) {
  auto encode = tensor_map_encoder();
  if (!encode) return fail(FDMD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap maps[4];
  const void* ptrs[4] = {uh, ul, ch, cl};
  for (int i = 0; i < 4; ++i) {
    const bool a = i < 2;
    cuuint64_t dims[2] = {(cuuint64_t)r, (cuuint64_t)(a ? n : nf)};
    cuuint64_t strides[1] = {(cuuint64_t)((a ? ldu : ldk) * 2)};
    cuuint32_t box[2] = {(cuuint32_t)fdmd::tc2::BKC, (cuuint32_t)(a ? fdmd::tc2::BM : fdmd::tc2::BNH)};
    cuuint32_t estr[2] = {1, 1};
    CUresult res = encode(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptrs[i]), dims, strides,
                          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return fail(FDMD_ERR_CUDA, "tc_decode2: tensor map encode failed (%d)", (int)res);
  }
  // the plane-output epilogue is a separate instantiation: sharing one body
  // pushed the frame path over the 113-register budget of 576 threads (spills).
  // FDMD_TC2_TMAO=1: frames go out through TMA stores of 16-frame x 128-row
  // staged chunks (2-deep basis ring) when the output rows are 16-byte aligned.
  // Measured at n = 50.3M: B = 256 18.2 ms vs 16.7 ms with register stores,
  // B = 512 equal (33.4 ms) — off by default.
  // FDMD_TC2_TMAO=2: the same staging, written out with 16-byte register stores
  // (512 contiguous bytes of one frame per warp instruction).
  static const int tmao_mode = [] { const char* e = getenv("FDMD_TC2_TMAO"); return e ? atoi(e) : 0; }();
  const bool aligned = !ph && (ldo * 4) % 16 == 0 && ((uintptr_t)out % 16) == 0;
  // st != nullptr: the frame epilogue also keeps per column pair the max |phi|^2 and the
  // first row attaining it (the modes product: no separate statistics pass over the table)
  const int tmao = !st && aligned && (tmao_mode == 1 || tmao_mode == 2) ? tmao_mode : 0;
  if (st && ph) return fail(FDMD_ERR_INVALID, "tc_decode2: statistics need the frame output");
  auto kern = ph ? fdmd::tc_decode2_kernel<true, 0, fdmd::tc2::AST>
                 : (st ? fdmd::tc_decode2_kernel<false, 0, fdmd::tc2::AST, true>
                    : tmao == 1 ? fdmd::tc_decode2_kernel<false, 1, 2>
                    : tmao == 2 ? fdmd::tc_decode2_kernel<false, 2, 2>
                                : fdmd::tc_decode2_kernel<false, 0, fdmd::tc2::AST>);
  const int smem = (int)(tmao ? sizeof(fdmd::TC2SmemT<2, 1>) : sizeof(fdmd::TC2Smem)) + 1024;
  static thread_local int configured[5] = {-1, -1, -1, -1, -1};
  static thread_local int max_clusters[5] = {0, 0, 0, 0, 0};
  const int kv = ph ? 1 : (st ? 4 : (tmao ? 1 + tmao : 0));
  CUtensorMap omap;
  memset(&omap, 0, sizeof(omap));
  if (tmao == 1) {
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)nf};
    cuuint64_t strides[1] = {(cuuint64_t)(ldo * 4)};
    cuuint32_t box[2] = {(cuuint32_t)fdmd::tc2::BM, (cuuint32_t)fdmd::TMAO_FR};
    cuuint32_t estr[2] = {1, 1};
    CUresult res = encode(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, out, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) return fail(FDMD_ERR_CUDA, "tc_decode2: output tensor map encode failed (%d)", (int)res);
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(fdmd::tc2::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  if (configured[kv] != dev) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cfg.gridDim = dim3(2, 1);
    int nc = 0;
    CUDA_TRY(cudaOccupancyMaxActiveClusters(&nc, (void*)kern, &cfg));
    max_clusters[kv] = std::max(1, nc);
    configured[kv] = dev;
  }
  fdmd::TCArgs ta{out, ldo, n, r, nf, fscale};
  ta.ph = static_cast<__half*>(ph);
  ta.pl = static_cast<__half*>(pl);
  ta.ldp = ldp;
  ta.pscale = pscale;
  const int64_t ptiles = (n + 2 * fdmd::tc2::BM - 1) / (2 * fdmd::tc2::BM);
  const int gy = (nf + fdmd::tc2::BN - 1) / fdmd::tc2::BN;
  const int64_t npairs =
      std::max<int64_t>(1, std::min<int64_t>(ptiles, std::max(1, max_clusters[kv] / gy - reserve_pairs)));
  cfg.gridDim = dim3((unsigned)(2 * npairs * gy), 1);
  const int nctas = (int)(2 * npairs * gy);
  void* stbuf = nullptr;
  if (st) {
    const size_t slots = (size_t)nctas * fdmd::tc2::EPI * 32;
    CUDA_TRY(scratch_alloc(&stbuf, slots * (sizeof(long long) + 2 * sizeof(double)), (cudaStream_t)stream));
    ta.st_idx = static_cast<long long*>(stbuf);
    ta.st_max = reinterpret_cast<double*>(ta.st_idx + slots);
    ta.st_sum = ta.st_max + slots;
  }
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], omap, ta));
  LAUNCH_CHECK("tc_decode2");
  if (st) {
    const int units = nf / 2;
    fdmd::tc2_pair_stats_final_kernel<<<(units + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
        ta.st_max, ta.st_idx, ta.st_sum, nctas, gy, units, (long long)row_offset, st);
    LAUNCH_CHECK("tc2_pair_stats_final");
    cudaFreeAsync(stbuf, (cudaStream_t)stream);
  }
  return FDMD_OK;
}

}  // namespace

extern "C" {

int fdmd_version(void) { return 1; }

const char* fdmd_last_error(void) { return g_err.c_str(); }

int fdmd_device_info(int device, int* sm_count, int* cc_major, int* cc_minor) {
  CUDA_TRY(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  CUDA_TRY(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  CUDA_TRY(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return FDMD_OK;
}

size_t fdmd_tall_gemm_workspace(int64_t n, int N) {
  (void)n;
  const int gx = tg_grid_x(n);
  return (size_t)gx * (size_t)((N + 1) / 2) * 3 * sizeof(double) + 256;
}

int fdmd_tall_gemm(const void* A, int a_dtype, int a_layout, int64_t lda, const double* B, int64_t ldb,
                   void* C, int c_dtype, int c_layout, int64_t ldc, int64_t n, int K, int N, int flags,
                   double* pair_stats, int64_t row_offset, void* workspace, size_t workspace_bytes,
                   void* stream) {
  if (n < 0 || K < 0 || N < 0) return fail(FDMD_ERR_INVALID, "negative size");
  if (!A || !B) return fail(FDMD_ERR_INVALID, "null operand");
  if (a_dtype != FDMD_F32 && a_dtype != FDMD_F64) return fail(FDMD_ERR_INVALID, "bad a_dtype");
  if (c_dtype != FDMD_F32 && c_dtype != FDMD_F64) return fail(FDMD_ERR_INVALID, "bad c_dtype");
  if (pair_stats && (N % 2)) return fail(FDMD_ERR_INVALID, "pair_stats needs even N");
  if (a_layout == FDMD_ROW && lda < K) return fail(FDMD_ERR_INVALID, "lda < K");
  if (a_layout == FDMD_COL && lda < n) return fail(FDMD_ERR_INVALID, "lda < n");
  if (ldb < N) return fail(FDMD_ERR_INVALID, "ldb < N");
  if (C && c_layout == FDMD_ROW && ldc < N) return fail(FDMD_ERR_INVALID, "ldc < N");
  if (C && c_layout == FDMD_COL && ldc < n) return fail(FDMD_ERR_INVALID, "ldc < n");
  if (n == 0 || N == 0) return FDMD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int gx = tg_grid_x(n);
  fdmd::TallGemmArgs a{};
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb; a.C = C; a.ldc = ldc;
  a.n = n; a.K = K; a.N = N; a.row_offset = row_offset;
  a.b_upper = (flags & FDMD_B_UPPER) ? 1 : 0;
  a.reserve_sms = (flags & FDMD_SHARE_SMS) ? 8 : 0;
  static const int dbg = [] { const char* e = getenv("FDMD_TG_DEBUG"); return e ? atoi(e) : 0; }();
  a.debug = dbg;
  const bool stats = pair_stats != nullptr;
  if (stats) {
    const size_t need = (size_t)gx * (size_t)(N / 2) * 3 * sizeof(double);
    if (!workspace || workspace_bytes < need)
      return fail(FDMD_ERR_WORKSPACE, "tall_gemm workspace %zu < %zu", workspace_bytes, need);
    a.pair_stats = static_cast<double*>(workspace);
  }
  if (!C) c_layout = FDMD_COL;  // stats-only pass: no stores
  int rc;
  if (a_dtype == FDMD_F32)
    rc = a_layout == FDMD_ROW ? dispatch_tg_nf<float, fdmd::LAYOUT_ROW>(a, c_dtype, c_layout, stats, s, gx)
                              : dispatch_tg_nf<float, fdmd::LAYOUT_COL>(a, c_dtype, c_layout, stats, s, gx);
  else
    rc = a_layout == FDMD_ROW ? dispatch_tg_nf<double, fdmd::LAYOUT_ROW>(a, c_dtype, c_layout, stats, s, gx)
                              : dispatch_tg_nf<double, fdmd::LAYOUT_COL>(a, c_dtype, c_layout, stats, s, gx);
  if (rc != FDMD_OK) return rc;
  if (stats) {
    const int U = N / 2;
    fdmd::pair_stats_reduce_kernel<<<(U + 127) / 128, 128, 0, s>>>(a.pair_stats, gx, U, pair_stats);
    LAUNCH_CHECK("pair_stats_reduce");
  }
  return FDMD_OK;
}

int fdmd_tall_gemm_planes(const void* A, int a_dtype, int64_t lda, const double* B, int64_t ldb, void* uh, void* ul,
                          int64_t ldu, double scale, int64_t n, int K, int N, int flags, void* stream) {
  if (n < 0 || K <= 0 || N <= 0) return fail(FDMD_ERR_INVALID, "tall_gemm_planes: bad sizes");
  if (!A || !B || !uh || !ul) return fail(FDMD_ERR_INVALID, "tall_gemm_planes: null operand");
  if (a_dtype != FDMD_F32 && a_dtype != FDMD_F64) return fail(FDMD_ERR_INVALID, "tall_gemm_planes: bad a_dtype");
  if (lda < K || ldb < N) return fail(FDMD_ERR_INVALID, "tall_gemm_planes: lda < K or ldb < N");
  if (ldu < N || ldu % 8 || ldu > 256 || ldu > (N + 7) / 8 * 8)
    return fail(FDMD_ERR_INVALID, "tall_gemm_planes: ldu must be round_up(N, 8) <= 256");
  if (n == 0) return FDMD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int gx = tg_grid_x(n);
  fdmd::TallGemmArgs a{};
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb; a.C = uh; a.C2 = ul; a.ldc = ldu; a.cscale = scale;
  a.n = n; a.K = K; a.N = N;
  a.reserve_sms = (flags & FDMD_SHARE_SMS) ? 8 : 0;
  bool used = false;
  int rc;
  const int nf = pick_nf(N);
#define TGP(TA, NFV) launch_tg_tma<TA, fdmd::LAYOUT_ROW, NFV, __half, fdmd::LAYOUT_PLANES, false>(a, s, gx, used)
  if (a_dtype == FDMD_F32)
    rc = nf == 1 ? TGP(float, 1) : nf == 2 ? TGP(float, 2) : nf == 4 ? TGP(float, 4) : TGP(float, 7);
  else
    rc = nf == 1 ? TGP(double, 1) : nf == 2 ? TGP(double, 2) : nf == 4 ? TGP(double, 4) : TGP(double, 7);
#undef TGP
  if (rc != FDMD_OK) return rc;
  if (!used) return fail(FDMD_ERR_INVALID, "tall_gemm_planes: A not TMA-eligible (16-B aligned rows needed)");
  return FDMD_OK;
}

size_t fdmd_tall_gram_workspace(int64_t n, int K1, int K2) {
  // large enough for either plan (a symmetric Gram has fewer tiles -> more splits)
  size_t need = 0;
  for (int sym = 0; sym < 2; ++sym) {
    for (int v = 0; v < 3; ++v) {
      const bool sw = v > 0;
      const int TN = v == 2 ? 224 : 64;
      GramPlan q = gram_plan(n, K1, K2, sym, sw, TN);
      need = std::max(need, (size_t)q.splits * q.K1p * q.K2p * sizeof(double));
    }
    for (int ea = 4; ea <= 8; ea += 4)
      for (int eb = 4; eb <= 8; eb += 4) {
        PanelPlan q = panel_plan_best(n, K1, K2, sym, ea, eb);
        if (q.ok) need = std::max(need, (size_t)q.splits * q.K1p * q.K2p * sizeof(double));
      }
  }
  return need + 256;
}

int fdmd_tall_gram(const void* A, int a_dtype, int a_layout, int64_t lda, const void* B, int b_dtype,
                   int b_layout, int64_t ldb, double* C, int64_t ldc, double beta, int64_t n, int K1,
                   int K2, int symmetric, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || K1 <= 0 || K2 <= 0) return fail(FDMD_ERR_INVALID, "bad sizes n=%lld K1=%d K2=%d", (long long)n, K1, K2);
  if (!A || !B || !C) return fail(FDMD_ERR_INVALID, "null operand");
  if (symmetric && (K1 != K2 || A != B)) return fail(FDMD_ERR_INVALID, "symmetric needs A==B, K1==K2");
  if (ldc < K2) return fail(FDMD_ERR_INVALID, "ldc < K2");
  if ((a_layout == FDMD_ROW && lda < K1) || (a_layout == FDMD_COL && lda < n))
    return fail(FDMD_ERR_INVALID, "bad lda");
  if ((b_layout == FDMD_ROW && ldb < K2) || (b_layout == FDMD_COL && ldb < n))
    return fail(FDMD_ERR_INVALID, "bad ldb");
  cudaStream_t s = (cudaStream_t)stream;
  const bool sw = gram_sw_eligible(A, a_dtype, a_layout, lda, B, b_dtype, b_layout, ldb, n);
  if (sw && panel_enabled() && n > 0) {
    PanelPlan pl = panel_plan_best(n, K1, K2, symmetric, dsize(a_dtype), dsize(b_dtype));
    if (pl.ok && !(symmetric && a_dtype != b_dtype)) {
      const size_t need = (size_t)pl.splits * pl.K1p * pl.K2p * sizeof(double);
      if (!workspace || workspace_bytes < need)
        return fail(FDMD_ERR_WORKSPACE, "tall_gram workspace %zu < %zu", workspace_bytes, need);
      fdmd::TallGramArgs a{};
      const bool tr = pl.transposed;
      a.A = tr ? B : A; a.lda = tr ? ldb : lda; a.B = tr ? A : B; a.ldb = tr ? lda : ldb;
      a.W = static_cast<double*>(workspace);
      a.n = n; a.K1 = tr ? K2 : K1; a.K2 = tr ? K1 : K2; a.symmetric = symmetric;
      const int da = tr ? b_dtype : a_dtype, db = tr ? a_dtype : b_dtype;
      int rc;
      if (symmetric)
        rc = da == FDMD_F32 ? launch_gram_panel<float, float, 5, 5, true>(a, pl, s)
                            : launch_gram_panel<double, double, 5, 5, true>(a, pl, s);
      else if (pl.WC == 9 && da == FDMD_F32)
        rc = db == FDMD_F32 ? launch_gram_panel<float, float, 5, 9, false>(a, pl, s)
                            : launch_gram_panel<float, double, 5, 9, false>(a, pl, s);
      else if (pl.WC == 9)
        rc = db == FDMD_F32 ? launch_gram_panel<double, float, 5, 9, false>(a, pl, s)
                            : launch_gram_panel<double, double, 5, 9, false>(a, pl, s);
      else if (da == FDMD_F32)
        rc = db == FDMD_F32 ? launch_gram_panel<float, float, 5, 7, false>(a, pl, s)
                            : launch_gram_panel<float, double, 5, 7, false>(a, pl, s);
      else
        rc = db == FDMD_F32 ? launch_gram_panel<double, float, 5, 7, false>(a, pl, s)
                            : launch_gram_panel<double, double, 5, 7, false>(a, pl, s);
      if (rc != FDMD_OK) return rc;
      dim3 grid((K2 + 127) / 128, K1);
      fdmd::gram_reduce_kernel<<<grid, 128, 0, s>>>(a.W, pl.splits, K1, K2, pl.K1p, pl.K2p, symmetric, C, ldc, beta,
                                                    tr ? 1 : 0);
      LAUNCH_CHECK("gram_reduce");
      return FDMD_OK;
    }
  }
  // wide tiles for general products; 64x64 for symmetric Grams (a 64 x 224 stripe
  // of a triangle leaves the lower stripes nearly idle: measured 9.8 vs 16 TF/s)
  const int nfb = (K2 > 64 && !symmetric) ? 7 : 2;
  GramPlan p = gram_plan(n, K1, K2, symmetric, sw, sw ? 32 * nfb : fdmd::gr::T);
  const size_t need = (size_t)p.splits * p.K1p * p.K2p * sizeof(double);
  if (!workspace || workspace_bytes < need)
    return fail(FDMD_ERR_WORKSPACE, "tall_gram workspace %zu < %zu", workspace_bytes, need);
  fdmd::TallGramArgs a{};
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb; a.W = static_cast<double*>(workspace);
  a.n = n; a.K1 = K1; a.K2 = K2; a.K1p = p.K1p; a.K2p = p.K2p; a.tiles_j = p.tj;
  a.symmetric = symmetric; a.rows_per_split = p.rows_per_split;
  int rc;
  if (sw) {
#define GSW(TA, TB) (nfb == 7 ? launch_gram_sw<TA, TB, 7>(a, p.tiles, p.splits, s) : launch_gram_sw<TA, TB, 2>(a, p.tiles, p.splits, s))
    if (a_dtype == FDMD_F32) rc = b_dtype == FDMD_F32 ? GSW(float, float) : GSW(float, double);
    else rc = b_dtype == FDMD_F32 ? GSW(double, float) : GSW(double, double);
#undef GSW
  } else if (a_dtype == FDMD_F32)
    rc = a_layout == FDMD_ROW ? dispatch_gram_b<float, fdmd::LAYOUT_ROW>(a, b_dtype, b_layout, p.tiles, p.splits, s)
                              : dispatch_gram_b<float, fdmd::LAYOUT_COL>(a, b_dtype, b_layout, p.tiles, p.splits, s);
  else
    rc = a_layout == FDMD_ROW ? dispatch_gram_b<double, fdmd::LAYOUT_ROW>(a, b_dtype, b_layout, p.tiles, p.splits, s)
                              : dispatch_gram_b<double, fdmd::LAYOUT_COL>(a, b_dtype, b_layout, p.tiles, p.splits, s);
  if (rc != FDMD_OK) return rc;
  dim3 grid((K2 + 127) / 128, K1);
  fdmd::gram_reduce_kernel<<<grid, 128, 0, s>>>(a.W, p.splits, K1, K2, p.K1p, p.K2p, symmetric, C, ldc, beta);
  LAUNCH_CHECK("gram_reduce");
  return FDMD_OK;
}

int fdmd_decode(const void* D, int dtype, int64_t ldd, const void* coef, int ldcoef, void* out, int64_t ldo,
                int64_t n, int r, int B, void* stream) {
  if (n < 0 || r < 0 || B < 0) return fail(FDMD_ERR_INVALID, "negative size");
  if (!D || !coef || !out) return fail(FDMD_ERR_INVALID, "null operand");
  if (ldd < n || ldo < n || ldcoef < B) return fail(FDMD_ERR_INVALID, "bad leading dimension");
  if (n == 0 || B == 0) return FDMD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // frame groups: <=2 -> (4 rows, FB), <=8 -> (4, 8), <=16 -> (2,16), else 32 per pass (1 row)
  for (int f0 = 0; f0 < B; ) {
    const int left = B - f0;
    int rpt, fb;
    if (left <= 1) { rpt = 4; fb = 1; }
    else if (left <= 2) { rpt = 4; fb = 2; }
    else if (left <= 4) { rpt = 4; fb = 4; }
    else if (left <= 8) { rpt = 4; fb = 8; }
    else if (left <= 16) { rpt = 2; fb = 16; }
    else { rpt = (dtype == FDMD_F32) ? 2 : 1; fb = 32; }
    if (dtype == FDMD_F64 && rpt == 4) rpt = 2;
    const int threads = 256;
    const int64_t nthreads = (n + rpt - 1) / rpt;
    const int64_t blocks = (nthreads + threads - 1) / threads;
    const size_t smem = (size_t)r * fb * dsize(dtype);
    if (smem > 200 * 1024) return fail(FDMD_ERR_INVALID, "rank too large for decode smem");
#define DEC(T, RPT, FB)                                                                          \
  do {                                                                                          \
    auto k = fdmd::decode_kernel<T, RPT, FB>;                                                    \
    if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k<<<(unsigned)blocks, threads, smem, s>>>((const T*)D, ldd, (const T*)coef, ldcoef, (T*)out, ldo, n, r, B, f0); \
  } while (0)
    if (dtype == FDMD_F32) {
      if (fb == 1) DEC(float, 4, 1);
      else if (fb == 2) DEC(float, 4, 2);
      else if (fb == 4) DEC(float, 4, 4);
      else if (fb == 8) DEC(float, 4, 8);
      else if (fb == 16) DEC(float, 2, 16);
      else DEC(float, 2, 32);
    } else {
      if (fb == 1) DEC(double, 2, 1);
      else if (fb == 2) DEC(double, 2, 2);
      else if (fb == 4) DEC(double, 2, 4);
      else if (fb == 8) DEC(double, 2, 8);
      else if (fb == 16) DEC(double, 2, 16);
      else DEC(double, 1, 32);
    }
#undef DEC
    LAUNCH_CHECK("decode");
    f0 += fb;
  }
  return FDMD_OK;
}

static int64_t cd_rows_per_split(int64_t n, int r) {
  const int64_t target = (int64_t)sm_count_cached() * 8;
  int64_t splits = std::max<int64_t>(1, target / std::max(1, r));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, (n + 4095) / 4096));
  return (n + splits - 1) / splits;
}

size_t fdmd_colmajor_dot_workspace(int64_t n, int r, int nv) {
  const int64_t rps = cd_rows_per_split(n, r);
  const int64_t splits = (n + rps - 1) / std::max<int64_t>(rps, 1);
  return (size_t)std::max<int64_t>(splits, 1) * r * nv * sizeof(double) + 256;
}

int fdmd_colmajor_dot(const void* D, int d_dtype, int64_t ldd, const void* U, int u_dtype, int64_t ldu,
                      int64_t n, int r, int nv, double* y, void* workspace, size_t workspace_bytes,
                      void* stream) {
  if (n <= 0 || r <= 0 || nv <= 0 || nv > 8) return fail(FDMD_ERR_INVALID, "bad sizes (nv must be 1..8)");
  if (!D || !U || !y) return fail(FDMD_ERR_INVALID, "null operand");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rps = cd_rows_per_split(n, r);
  const int splits = (int)((n + rps - 1) / rps);
  const size_t need = (size_t)splits * r * nv * sizeof(double);
  if (!workspace || workspace_bytes < need) return fail(FDMD_ERR_WORKSPACE, "colmajor_dot workspace");
  double* part = static_cast<double*>(workspace);
  dim3 grid(r, splits);
#define CD(TD, TU, NV) fdmd::colmajor_dot_kernel<TD, TU, NV><<<grid, 256, 0, s>>>((const TD*)D, ldd, (const TU*)U, ldu, n, r, rps, part)
#define CDV(TD, TU)                                                         \
  switch (nv) {                                                             \
    case 1: CD(TD, TU, 1); break; case 2: CD(TD, TU, 2); break;             \
    case 3: CD(TD, TU, 3); break; case 4: CD(TD, TU, 4); break;             \
    case 5: CD(TD, TU, 5); break; case 6: CD(TD, TU, 6); break;             \
    case 7: CD(TD, TU, 7); break; default: CD(TD, TU, 8); break;            \
  }
  if (d_dtype == FDMD_F32) { if (u_dtype == FDMD_F32) { CDV(float, float) } else { CDV(float, double) } }
  else { if (u_dtype == FDMD_F32) { CDV(double, float) } else { CDV(double, double) } }
#undef CDV
#undef CD
  LAUNCH_CHECK("colmajor_dot");
  const int len = r * nv;
  fdmd::split_sum_kernel<<<(len + 127) / 128, 128, 0, s>>>(part, splits, len, y);
  LAUNCH_CHECK("split_sum");
  return FDMD_OK;
}

static int64_t tdot_splits(int64_t n) {
  return std::max<int64_t>(1, std::min<int64_t>((n + 1023) / 1024, (int64_t)sm_count_cached() * 8));
}

size_t fdmd_tall_tdot_workspace(int64_t n, int K) {
  return (size_t)tdot_splits(n) * std::max(K, 1) * sizeof(double) + 256;
}

int fdmd_tall_tdot(const void* A, int dtype, int64_t lda, const void* v, int64_t ldv, int64_t n, int K, double* y,
                   double beta, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || K <= 0 || lda < K || ldv < 1) return fail(FDMD_ERR_INVALID, "tall_tdot: bad sizes");
  if (!A || !v || !y) return fail(FDMD_ERR_INVALID, "tall_tdot: null operand");
  if (dtype != FDMD_F32 && dtype != FDMD_F64) return fail(FDMD_ERR_INVALID, "tall_tdot: bad dtype");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t splits = tdot_splits(n);
  if (!workspace || workspace_bytes < (size_t)splits * K * sizeof(double))
    return fail(FDMD_ERR_WORKSPACE, "tall_tdot workspace");
  double* part = static_cast<double*>(workspace);
  const int64_t rps = (n + splits - 1) / splits;
  if (dtype == FDMD_F32)
    fdmd::tall_tdot_kernel<float><<<(unsigned)splits, 256, 0, s>>>((const float*)A, lda, (const float*)v, ldv, n, K,
                                                                     rps, part);
  else
    fdmd::tall_tdot_kernel<double><<<(unsigned)splits, 256, 0, s>>>((const double*)A, lda, (const double*)v, ldv, n,
                                                                      K, rps, part);
  LAUNCH_CHECK("tall_tdot");
  if (beta == 0.0) {
    fdmd::split_sum_kernel<<<(K + 127) / 128, 128, 0, s>>>(part, (int)splits, K, y);
  } else {   // y += sum (streamed accumulation): sum into the tail of the workspace first
    fdmd::split_sum_kernel<<<(K + 127) / 128, 128, 0, s>>>(part, (int)splits, K, part);
    fdmd::axpy_kernel<<<(K + 127) / 128, 128, 0, s>>>(part, beta, y, K);
  }
  LAUNCH_CHECK("tall_tdot_reduce");
  return FDMD_OK;
}

// ---- bordered symmetric Gram: C (K x (K + 1)) = [A^T A | A^T a_K] ----------
// One pass over the rows of a row-major A with K + 1 columns: the snapshot
// Gram X^T X and the border X^T s_m of S^T S (S = [X | s_m]) that the
// projection from the snapshot Gram needs (linalg.sketch_factors). The panel
// kernel carries the border as 5 extra 8x8 blocks per diagonal warp tile
// (kind 3); operands the panel path cannot take fall back to the symmetric
// Gram + fdmd_tall_tdot.
static PanelPlan bordered_plan(const void* A, int dtype, int64_t lda, int64_t n, int K) {
  PanelPlan none;
  if (!panel_enabled() || n <= 0) return none;
  if (!gram_sw_eligible(A, dtype, FDMD_ROW, lda, A, dtype, FDMD_ROW, lda, n)) return none;
  return panel_plan(n, K, K, 1, dsize(dtype), dsize(dtype), 7, 1);
}

// Host-side introspection of the panel-Gram schedule (tests, DESIGN numbers):
// info = {ok, P, cost, cuts, splits, K1p, K2p, jb, blocks}; tiles (optional, up to
// 4 * max_tiles ints) = {i0, j0, kind, slot} per non-idle warp tile, slot =
// 8 * partition + warp. No device work.
int fdmd_gram_plan_info(int64_t n, int K, int symmetric, int border, int elt_bytes, int* info, int* tiles,
                        int max_tiles) {
  if (!info || K <= 0 || (elt_bytes != 4 && elt_bytes != 8)) return fail(FDMD_ERR_INVALID, "gram_plan_info: bad args");
  PanelPlan pl = symmetric ? panel_plan(n, K, K, 1, (size_t)elt_bytes, (size_t)elt_bytes, 7, border)
                           : panel_plan_best(n, K, K, 0, (size_t)elt_bytes, (size_t)elt_bytes);
  int blocks = 0, nt = 0;
  for (int i = 0; i < fdmd::tgp::MAXP * 8 && pl.ok; ++i) {
    const fdmd::PanelTile& t = pl.tile[i];
    if (t.kind == 0) continue;
    const int w = t.kind == 1 ? pl.WR * pl.WC : t.kind == 2 ? pl.WR * (pl.WR + 1) / 2
                  : t.kind == 3 ? pl.WR * (pl.WR + 1) / 2 + pl.WR : t.kind == 4 ? pl.WR * 3 : pl.WR * 4;
    blocks += w;
    if (tiles && nt < max_tiles) {
      tiles[4 * nt + 0] = t.i0; tiles[4 * nt + 1] = t.j0; tiles[4 * nt + 2] = t.kind; tiles[4 * nt + 3] = i;
    }
    ++nt;
  }
  const int v[9] = {pl.ok ? 1 : 0, pl.P, pl.cost, pl.cuts, pl.splits, pl.K1p, pl.K2p, pl.jb, blocks};
  for (int i = 0; i < 9; ++i) info[i] = v[i];
  return nt;
}

size_t fdmd_tall_gram_bordered_workspace(int64_t n, int K) {
  size_t need = std::max(fdmd_tall_gram_workspace(n, K, K), fdmd_tall_tdot_workspace(n, K));
  for (size_t ea = 4; ea <= 8; ea += 4) {
    PanelPlan q = panel_plan(n, K, K, 1, ea, ea, 7, 1);
    if (q.ok) need = std::max(need, (size_t)q.splits * q.K1p * q.K2p * sizeof(double) + 256);
  }
  return need;
}

int fdmd_tall_gram_bordered(const void* A, int dtype, int64_t lda, double* C, int64_t ldc, double beta, int64_t n,
                            int K, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || K <= 0) return fail(FDMD_ERR_INVALID, "tall_gram_bordered: bad sizes n=%lld K=%d", (long long)n, K);
  if (!A || !C) return fail(FDMD_ERR_INVALID, "tall_gram_bordered: null operand");
  if (dtype != FDMD_F32 && dtype != FDMD_F64) return fail(FDMD_ERR_INVALID, "tall_gram_bordered: bad dtype");
  if (lda < K + 1 || ldc < K + 1) return fail(FDMD_ERR_INVALID, "tall_gram_bordered: lda / ldc < K + 1");
  cudaStream_t s = (cudaStream_t)stream;
  PanelPlan pl = bordered_plan(A, dtype, lda, n, K);
  if (pl.ok) {
    const size_t need = (size_t)pl.splits * pl.K1p * pl.K2p * sizeof(double);
    if (!workspace || workspace_bytes < need)
      return fail(FDMD_ERR_WORKSPACE, "tall_gram_bordered workspace %zu < %zu", workspace_bytes, need);
    fdmd::TallGramArgs a{};
    a.A = A; a.lda = lda; a.B = A; a.ldb = lda;
    a.W = static_cast<double*>(workspace);
    a.n = n; a.K1 = K; a.K2 = K; a.symmetric = 1;
    const int rc = dtype == FDMD_F32 ? launch_gram_panel<float, float, 5, 5, true>(a, pl, s)
                                     : launch_gram_panel<double, double, 5, 5, true>(a, pl, s);
    if (rc != FDMD_OK) return rc;
    // the mirror rule of the reduce is per 8x8 block, so column K (its own block
    // column, or inside the last one) is read where the kernel wrote it
    dim3 grid((K + 1 + 127) / 128, K);
    fdmd::gram_reduce_kernel<<<grid, 128, 0, s>>>(a.W, pl.splits, K, K + 1, pl.K1p, pl.K2p, 1, C, ldc, beta, 0);
    LAUNCH_CHECK("gram_reduce");
    return FDMD_OK;
  }
  int rc = fdmd_tall_gram(A, dtype, FDMD_ROW, lda, A, dtype, FDMD_ROW, lda, C, ldc, beta, n, K, K, 1, workspace,
                          workspace_bytes, stream);
  if (rc != FDMD_OK) return rc;
  const int64_t splits = tdot_splits(n);
  if (workspace_bytes < (size_t)splits * K * sizeof(double)) return fail(FDMD_ERR_WORKSPACE, "tall_gram_bordered workspace");
  const char* v = static_cast<const char*>(A) + (size_t)K * dsize(dtype);
  double* part = static_cast<double*>(workspace);
  const int64_t rps = (n + splits - 1) / splits;
  if (dtype == FDMD_F32)
    fdmd::tall_tdot_kernel<float><<<(unsigned)splits, 256, 0, s>>>((const float*)A, lda, (const float*)v, lda, n, K,
                                                                     rps, part);
  else
    fdmd::tall_tdot_kernel<double><<<(unsigned)splits, 256, 0, s>>>((const double*)A, lda, (const double*)v, lda, n,
                                                                      K, rps, part);
  LAUNCH_CHECK("tall_tdot");
  fdmd::split_sum_kernel<<<(K + 127) / 128, 128, 0, s>>>(part, (int)splits, K, part);
  fdmd::strided_axpby_kernel<<<(K + 127) / 128, 128, 0, s>>>(part, beta, C + K, ldc, K);
  LAUNCH_CHECK("tall_tdot_reduce");
  return FDMD_OK;
}


int fdmd_table_apply(const void* R, int r_dtype, int64_t ldr, const int* src, const double* alpha,
                     const double* beta, void* D, int d_dtype, int64_t ldd, int64_t n, int ncols,
                     void* stream) {
  if (n < 0 || ncols < 0) return fail(FDMD_ERR_INVALID, "negative size");
  if (n == 0 || ncols == 0) return FDMD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t per = std::min<int64_t>((n + 255) / 256, std::max<int64_t>(1, sm_count_cached() * 8 / std::max(ncols, 1)));
  dim3 grid((unsigned)std::max<int64_t>(per, 1), ncols);
#define TA_(TR, TD) fdmd::table_apply_kernel<TR, TD><<<grid, 256, 0, s>>>((const TR*)R, ldr, src, alpha, beta, (TD*)D, ldd, n, ncols)
  if (r_dtype == FDMD_F32) { if (d_dtype == FDMD_F32) TA_(float, float); else TA_(float, double); }
  else { if (d_dtype == FDMD_F32) TA_(double, float); else TA_(double, double); }
#undef TA_
  LAUNCH_CHECK("table_apply");
  return FDMD_OK;
}

static int residual_chunk(int r, int T) {
  const int maxcols = (int)((200 * 1024) / ((size_t)r * sizeof(double)));
  return std::max(1, std::min(T, maxcols));
}

int fdmd_table_apply_inplace(void* R, int dtype, int64_t ldr, int nraw, const int* src, const double* alpha,
                             const double* beta, int ncols, int64_t n, void* stream) {
  if (n < 0 || ncols < 0 || nraw <= 0 || ncols > nraw) return fail(FDMD_ERR_INVALID, "table_apply_inplace: bad sizes");
  if (n == 0 || ncols == 0) return FDMD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t elt = dsize(dtype);
  int rpb = 128;  // rows per block: keep ~4 blocks resident per SM
  while (rpb > 8 && (size_t)nraw * rpb * elt > 56 * 1024) rpb /= 2;
  const size_t smem = (size_t)nraw * rpb * elt;
  if (smem > 200 * 1024) return fail(FDMD_ERR_INVALID, "table_apply_inplace: too many raw columns");
  const int64_t tiles = (n + rpb - 1) / rpb;
  const int blocks = (int)std::min<int64_t>(tiles, (int64_t)sm_count_cached() * 8);
#define TAI(T)                                                                                        \
  do {                                                                                                \
    auto k = fdmd::table_apply_inplace_kernel<T>;                                                     \
    CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));       \
    k<<<blocks, 256, smem, s>>>((T*)R, ldr, nraw, src, alpha, beta, ncols, n, rpb);                  \
  } while (0)
  if (dtype == FDMD_F32) TAI(float); else TAI(double);
#undef TAI
  LAUNCH_CHECK("table_apply_inplace");
  return FDMD_OK;
}

size_t fdmd_residual_workspace(int64_t n) {
  (void)n;
  // up to 64 column chunks x blocks x 2 partial sums
  return (size_t)64 * sm_count_cached() * 4 * 2 * sizeof(double) + 256;
}

int fdmd_residual(const void* S, int s_dtype, int64_t lds, const void* D, int d_dtype, int64_t ldd,
                  const double* F, int r, int T, int64_t n, double* out, void* workspace,
                  size_t workspace_bytes, void* stream) {
  if (n < 0 || r <= 0 || T <= 0) return fail(FDMD_ERR_INVALID, "bad sizes");
  const int Tc = residual_chunk(r, T);
  const int nch = (T + Tc - 1) / Tc;
  if (nch > 64 || (size_t)r * sizeof(double) > 200 * 1024) return fail(FDMD_ERR_INVALID, "residual: r too large");
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = sm_count_cached() * 4;
  if (!workspace || workspace_bytes < (size_t)nch * blocks * 2 * sizeof(double))
    return fail(FDMD_ERR_WORKSPACE, "residual workspace");
  double* part = static_cast<double*>(workspace);
  for (int c = 0; c < nch; ++c) {
    const int j0 = c * Tc, tc = std::min(Tc, T - j0);
    const size_t smem = (size_t)r * tc * sizeof(double);
#define RS(TS, TD)                                                                                   \
  do {                                                                                               \
    auto k = fdmd::residual_kernel<TS, TD>;                                                          \
    CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));      \
    k<<<blocks, 256, smem, s>>>((const TS*)S, lds, (const TD*)D, ldd, F + j0, T, r, tc, j0, n,       \
                                part + (size_t)c * blocks * 2);                                      \
  } while (0)
    if (s_dtype == FDMD_F32) { if (d_dtype == FDMD_F32) RS(float, float); else RS(float, double); }
    else { if (d_dtype == FDMD_F32) RS(double, float); else RS(double, double); }
#undef RS
    LAUNCH_CHECK("residual");
  }
  fdmd::split_sum_kernel<<<1, 32, 0, s>>>(part, nch * blocks, 2, out);
  LAUNCH_CHECK("residual_sum");
  return FDMD_OK;
}

int fdmd_geev(int n, double* A, double* w_host, double* vr_host, void* stream) {
  if (n <= 0 || !A || !w_host) return fail(FDMD_ERR_INVALID, "geev: bad arguments");
  const cusolverEigMode_t jobvr = vr_host ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
  SolverCtx* c = solver_ctx();
  if (!c) return fail(FDMD_ERR_SOLVER, "cusolverDnCreate failed");
  cudaStream_t s = (cudaStream_t)stream;
  if (cusolverDnSetStream(c->h, s) != CUSOLVER_STATUS_SUCCESS) return fail(FDMD_ERR_SOLVER, "set stream");
  double* W = nullptr;  // complex n
  double* VR = nullptr;
  int* info = nullptr;
  CUDA_TRY(scratch_alloc((void**)&W, sizeof(double) * 2 * n, s));
  if (vr_host) CUDA_TRY(scratch_alloc((void**)&VR, sizeof(double) * n * n, s));
  CUDA_TRY(scratch_alloc((void**)&info, sizeof(int), s));
  size_t dws = 0, hws = 0;
  cusolverStatus_t st = cusolverDnXgeev_bufferSize(c->h, c->p, CUSOLVER_EIG_MODE_NOVECTOR, jobvr,
                                                   n, CUDA_R_64F, A, n, CUDA_C_64F, W, CUDA_R_64F, nullptr, n,
                                                   CUDA_R_64F, VR, n, CUDA_R_64F, &dws, &hws);
  if (st != CUSOLVER_STATUS_SUCCESS) return fail(FDMD_ERR_SOLVER, "Xgeev_bufferSize status %d", (int)st);
  void* dbuf = nullptr;
  CUDA_TRY(scratch_alloc(&dbuf, dws > 0 ? dws : 1, s));
  std::vector<char> hbuf(hws > 0 ? hws : 1);
  st = cusolverDnXgeev(c->h, c->p, CUSOLVER_EIG_MODE_NOVECTOR, jobvr, n, CUDA_R_64F, A, n,
                       CUDA_C_64F, W, CUDA_R_64F, nullptr, n, CUDA_R_64F, VR, n, CUDA_R_64F, dbuf, dws,
                       hbuf.data(), hws, info);
  if (st != CUSOLVER_STATUS_SUCCESS) return fail(FDMD_ERR_SOLVER, "Xgeev status %d", (int)st);
  int info_h = 0;
  CUDA_TRY(cudaMemcpyAsync(&info_h, info, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(w_host, W, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, s));
  if (vr_host) CUDA_TRY(cudaMemcpyAsync(vr_host, VR, sizeof(double) * n * n, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  cudaFreeAsync(W, s);
  if (VR) cudaFreeAsync(VR, s);
  cudaFreeAsync(info, s);
  cudaFreeAsync(dbuf, s);
  if (info_h != 0) return fail(FDMD_ERR_SOLVER, "Xgeev info %d", info_h);
  return FDMD_OK;
}

// Thin SVD of the fit's small row-major B (l x T, l <= T, f64, device): B = Ub diag(s) Vh.
// cuSOLVER gesvdp (polar decomposition + symmetric eigensolver; 5.8 ms at 200 x 200 where
// the one-sided Jacobi gesvdj torch calls takes 13-15 ms, tools/svdp_probe.cu). The
// row-major B is the column-major T x l matrix B^T = Um diag(s) Vm^T, so Vh is Um's
// buffer as it stands (l x T row-major) and Ub^T is Vm's buffer. Stream-ordered: no
// host synchronisation; *info_dev (device int) receives cuSOLVER's info. B is destroyed.
int fdmd_svd_small(double* B, int64_t ldb, int l, int T, double* ubt, double* s_out, double* vh, int* info_dev,
                   void* stream) {
  if (!B || !ubt || !s_out || !vh || !info_dev || l <= 0 || T < l || ldb < T)
    return fail(FDMD_ERR_INVALID, "svd_small: bad arguments (needs l <= T <= ldb)");
  SolverCtx* c = solver_ctx();
  if (!c) return fail(FDMD_ERR_SOLVER, "cusolverDnCreate failed");
  cudaStream_t s = (cudaStream_t)stream;
  if (cusolverDnSetStream(c->h, s) != CUSOLVER_STATUS_SUCCESS) return fail(FDMD_ERR_SOLVER, "set stream");
  size_t dws = 0, hws = 0;
  cusolverStatus_t st = cusolverDnXgesvdp_bufferSize(c->h, c->p, CUSOLVER_EIG_MODE_VECTOR, 1, T, l, CUDA_R_64F, B,
                                                     ldb, CUDA_R_64F, s_out, CUDA_R_64F, vh, T, CUDA_R_64F, ubt, l,
                                                     CUDA_R_64F, &dws, &hws);
  if (st != CUSOLVER_STATUS_SUCCESS) return fail(FDMD_ERR_SOLVER, "Xgesvdp_bufferSize status %d", (int)st);
  void* dbuf = nullptr;
  CUDA_TRY(scratch_alloc(&dbuf, dws > 0 ? dws : 1, s));
  std::vector<char> hbuf(hws > 0 ? hws : 1);
  double h_err = 0.0;
  st = cusolverDnXgesvdp(c->h, c->p, CUSOLVER_EIG_MODE_VECTOR, 1, T, l, CUDA_R_64F, B, ldb, CUDA_R_64F, s_out,
                         CUDA_R_64F, vh, T, CUDA_R_64F, ubt, l, CUDA_R_64F, dbuf, dws, hbuf.data(), hws, info_dev,
                         &h_err);
  cudaFreeAsync(dbuf, s);
  if (st != CUSOLVER_STATUS_SUCCESS) return fail(FDMD_ERR_SOLVER, "Xgesvdp status %d", (int)st);
  return FDMD_OK;
}

int fdmd_split_basis(const float* D, int64_t ldd, int64_t n, int r, float scale, void* uh, void* ul, int64_t ldu,
                     void* stream) {
  if (!D || !uh || !ul || n <= 0 || r <= 0 || ldu < r || ldd < n || ldu % 8 || ldu > 256)
    return fail(FDMD_ERR_INVALID, "split_basis: bad arguments (ldu must be a multiple of 8, <= 256)");
  const size_t smem = (size_t)ldu * (fdmd::SPLIT_ROWS + 1) * sizeof(float);
  auto k = fdmd::split_basis_kernel;
  if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)((n + fdmd::SPLIT_ROWS - 1) / fdmd::SPLIT_ROWS), 256, smem, (cudaStream_t)stream>>>(
      D, ldd, n, r, scale, (__half*)uh, (__half*)ul, ldu);
  LAUNCH_CHECK("split_basis");
  return FDMD_OK;
}

int fdmd_split_rows_f64(const double* A, int64_t lda, int64_t n, int K, double scale, void* uh, void* ul,
                        int64_t ldu, void* stream) {
  if (!A || !uh || !ul || n <= 0 || K <= 0 || ldu < K || lda < K || ldu % 8 || ldu > 256)
    return fail(FDMD_ERR_INVALID, "split_rows_f64: bad arguments (ldu must be a multiple of 8, <= 256)");
  const int64_t items = n * (ldu / 8);
  fdmd::split_rows_kernel<double><<<(unsigned)((items + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      A, lda, n, K, scale, (__half*)uh, (__half*)ul, ldu);
  LAUNCH_CHECK("split_rows_f64");
  return FDMD_OK;
}

int fdmd_split_rows(const void* A, int dtype, int64_t lda, int64_t n, int K, double scale, void* uh, void* ul,
                    int64_t ldu, void* stream) {
  if (dtype == FDMD_F64) return fdmd_split_rows_f64((const double*)A, lda, n, K, scale, uh, ul, ldu, stream);
  if (dtype != FDMD_F32) return fail(FDMD_ERR_INVALID, "split_rows: bad dtype");
  if (!A || !uh || !ul || n <= 0 || K <= 0 || ldu < K || lda < K || ldu % 8 || ldu > 256)
    return fail(FDMD_ERR_INVALID, "split_rows: bad arguments (ldu must be a multiple of 8, <= 256)");
  const int64_t items = n * (ldu / 8);
  fdmd::split_rows_kernel<float><<<(unsigned)((items + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const float*)A, lda, n, K, scale, (__half*)uh, (__half*)ul, ldu);
  LAUNCH_CHECK("split_rows");
  return FDMD_OK;
}

size_t fdmd_pair_stats_workspace(int64_t n, int units) {
  const int64_t splits = std::max<int64_t>(1, std::min<int64_t>((n + 65535) / 65536, 4 * sm_count_cached() / std::max(1, units) + 1));
  return (size_t)splits * units * 3 * sizeof(double) + 256;
}

int fdmd_pair_stats(const float* raw, int64_t ld, int64_t n, int units, int64_t row_offset, double* out,
                    void* workspace, size_t workspace_bytes, void* stream) {
  if (!raw || !out || n <= 0 || units <= 0 || ld < n) return fail(FDMD_ERR_INVALID, "pair_stats: bad arguments");
  const int64_t splits = std::max<int64_t>(1, std::min<int64_t>((n + 65535) / 65536, 4 * sm_count_cached() / std::max(1, units) + 1));
  if (!workspace || workspace_bytes < (size_t)splits * units * 3 * sizeof(double))
    return fail(FDMD_ERR_WORKSPACE, "pair_stats workspace");
  const int64_t rps = (n + splits - 1) / splits;
  cudaStream_t s = (cudaStream_t)stream;
  fdmd::pair_stats_kernel<<<dim3(units, (unsigned)splits), 256, 0, s>>>(raw, ld, n, units, rps, (double*)workspace);
  fdmd::pair_stats_final_kernel<<<(units + 127) / 128, 128, 0, s>>>((const double*)workspace, (int)splits, units,
                                                                   row_offset, out);
  LAUNCH_CHECK("pair_stats");
  return FDMD_OK;
}

int fdmd_split_coef(const float* coef, int ldc, int r, int nf, float su_inv, void* ch, void* cl, int ldk,
                    float* fscale, void* stream) {
  if (!coef || !ch || !cl || !fscale || r <= 0 || nf <= 0 || ldk < r || ldc < nf)
    return fail(FDMD_ERR_INVALID, "split_coef: bad arguments");
  fdmd::split_coef_kernel<<<nf, 128, 0, (cudaStream_t)stream>>>(coef, ldc, r, nf, su_inv, (__half*)ch, (__half*)cl, ldk, fscale);
  LAUNCH_CHECK("split_coef");
  return FDMD_OK;
}

int fdmd_tc_decode(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch, const void* cl,
                   int ldk, int nf, const float* fscale, float* out, int64_t ldo, void* stream) {
  return fdmd_tc_decode_ex(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, 0, stream);
}

int fdmd_tc_decode_ex(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch, const void* cl,
                      int ldk, int nf, const float* fscale, float* out, int64_t ldo, int flags, void* stream) {
  if (!uh || !ul || !ch || !cl || !fscale || !out || n <= 0 || r <= 0 || nf <= 0 || r > fdmd::tc::BKC * fdmd::tc::MAXKC)
    return fail(FDMD_ERR_INVALID, "tc_decode: bad arguments (r must be <= %d)", fdmd::tc::BKC * fdmd::tc::MAXKC);
  if ((ldu * 2) % 16 || (ldk * 2) % 16 || ldu < r || ldk < r || ldo < n || n >= (int64_t)UINT32_MAX)
    return fail(FDMD_ERR_INVALID, "tc_decode: leading dimensions must be multiples of 8 halves");
  // N = 128 frames per CTA column with the coefficients resident in smem and a
  // 3-deep ring of U chunks (96 KB of HBM reads in flight per SM). Measured at
  // n = 50.3M, r = 200: B = 32 at 5.8 TB/s (0.88 of HBM; 2-deep ring: 4.5);
  // streaming the coefficients from L2 per chunk (to allow N = 256) cost more
  // in L2/TMA traffic than it saved in U re-reads (3.0-3.3 TB/s).
  // Batches over 128 frames run as clusters of MC CTAs along the frame axis
  // sharing every basis chunk through TMA multicast (basis read once per
  // MC * 128 frames).
  const int ny = (nf + 127) / 128;
  // > 128 frames: CTA pairs (cta_group::2, 256 frames per pair tile; B = 256
  // at n = 50.3M: 16.5 ms vs 21.3 ms for MC = 2 clusters); FDMD_TC_IMPL=mc
  // selects the multicast clusters instead
  static const int pair_on = [] { const char* e = getenv("FDMD_TC_IMPL"); return e ? (strcmp(e, "mc") == 0 ? 0 : 1) : 1; }();
  if (ny > 1 && pair_on)   // FDMD_SHARE_SMS: leave 4 SM pairs to a concurrent stream
    return launch_tc_decode_pair(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, stream,
                                 (flags & FDMD_SHARE_SMS) ? 4 : 0);
  static const int mc_cap = [] { const char* e = getenv("FDMD_TC_MAX_CLUSTER"); return e ? atoi(e) : 8; }();
  if (ny == 1 || mc_cap <= 1)
    return launch_tc_decode_mc<128, 3, 0, 1>(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, stream);
  if (ny == 2 || mc_cap < 4)
    return launch_tc_decode_mc<128, 3, 0, 2>(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, stream);
  if (ny <= 4 || mc_cap < 8)
    return launch_tc_decode_mc<128, 3, 0, 4>(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, stream);
  return launch_tc_decode_mc<128, 3, 0, 8>(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, stream);
}

// fdmd_tc_decode of a modes product (column pairs (2u, 2u + 1) = (Re, Im) of mode u) with the
// normalisation / phase-pivot statistics of _order_and_pair fused into the frame epilogue:
// st[u] = {sum_i |phi_u[i]|^2, max_i |phi_u[i]|^2, first row attaining it + row_offset}. *fused = 1 when
// the CTA-pair kernel ran (nf > 128) and filled st; 0 = frames only (run fdmd_pair_stats).
int fdmd_tc_decode_pairstats(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch,
                             const void* cl, int ldk, int nf, const float* fscale, float* out, int64_t ldo,
                             int64_t row_offset, double* st, int* fused, void* stream) {
  if (!st || !fused || nf % 2) return fail(FDMD_ERR_INVALID, "tc_decode_pairstats: bad arguments (nf even)");
  *fused = 0;
  static const int pair_on = [] { const char* e = getenv("FDMD_TC_IMPL"); return e ? (strcmp(e, "mc") == 0 ? 0 : 1) : 1; }();
  static const int fuse_on = [] { const char* e = getenv("FDMD_TC_STATS"); return e ? atoi(e) : 1; }();
  if (nf <= 128 || !pair_on || !fuse_on)
    return fdmd_tc_decode_ex(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, 0, stream);
  if (!uh || !ul || !ch || !cl || !fscale || !out || n <= 0 || r <= 0 || r > fdmd::tc::BKC * fdmd::tc::MAXKC)
    return fail(FDMD_ERR_INVALID, "tc_decode: bad arguments (r must be <= %d)", fdmd::tc::BKC * fdmd::tc::MAXKC);
  if ((ldu * 2) % 16 || (ldk * 2) % 16 || ldu < r || ldk < r || ldo < n || n >= (int64_t)UINT32_MAX)
    return fail(FDMD_ERR_INVALID, "tc_decode: leading dimensions must be multiples of 8 halves");
  const int rc = launch_tc_decode_pair(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, out, ldo, stream, 0, nullptr, nullptr,
                                       0, 1.f, st, row_offset);
  if (rc == FDMD_OK) *fused = 1;
  return rc;
}

int fdmd_tc_decode_planes(const void* uh, const void* ul, int64_t ldu, int64_t n, int r, const void* ch,
                          const void* cl, int ldk, int nf, const float* fscale, void* out_h, void* out_l,
                          int64_t ldp, float pscale, int flags, void* stream) {
  if (!uh || !ul || !ch || !cl || !fscale || !out_h || !out_l || n <= 0 || r <= 0 || nf <= 0 ||
      r > fdmd::tc::BKC * fdmd::tc::MAXKC || nf > fdmd::tc2::BN)
    return fail(FDMD_ERR_INVALID, "tc_decode_planes: bad arguments (r <= %d, nf <= %d)",
                fdmd::tc::BKC * fdmd::tc::MAXKC, fdmd::tc2::BN);
  if ((ldu * 2) % 16 || (ldk * 2) % 16 || ldu < r || ldk < r || ldp % 8 || ldp < nf || n >= (int64_t)UINT32_MAX)
    return fail(FDMD_ERR_INVALID, "tc_decode_planes: leading dimensions must be multiples of 8 halves, ldp >= nf");
  // one 256-column tile; the unused out pointer/ld keep the kernel's frame path inert
  return launch_tc_decode_pair(uh, ul, ldu, n, r, ch, cl, ldk, nf, fscale, static_cast<float*>(out_h), n, stream,
                               (flags & FDMD_SHARE_SMS) ? 4 : 0, out_h, out_l, ldp, pscale);
}

int fdmd_mac_decode(const void* D, int dtype, int64_t ldd, int ncol, const double* coef, int nx, int ny,
                    int field, double* out, void* stream) {
  if (!D || !coef || !out || ncol <= 0 || nx < 2 || ny < 2) return fail(FDMD_ERR_INVALID, "mac_decode: bad arguments");
  if (field != FDMD_MAC_VELOCITY && field != FDMD_MAC_SPEED) return fail(FDMD_ERR_INVALID, "mac_decode: bad field");
  const int64_t n = (int64_t)(nx + 1) * ny + (int64_t)nx * (ny + 1);
  if (ldd < n) return fail(FDMD_ERR_INVALID, "mac_decode: ldd < n_state");
  const size_t smem = (size_t)(((ncol + 1) & ~1) + fdmd::MAC_TY * (fdmd::MAC_TX + 1) +
                                (fdmd::MAC_TY + 1) * fdmd::MAC_TX) * sizeof(double);
  if (smem > 200 * 1024) return fail(FDMD_ERR_INVALID, "mac_decode: too many table columns");
  const dim3 grid((nx + fdmd::MAC_TX - 1) / fdmd::MAC_TX, (ny + fdmd::MAC_TY - 1) / fdmd::MAC_TY);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == FDMD_F32) {
    auto k = fdmd::mac_decode_kernel<float>;
    if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, s>>>((const float*)D, ldd, ncol, coef, nx, ny, field, out);
  } else {
    auto k = fdmd::mac_decode_kernel<double>;
    if (smem > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, 256, smem, s>>>((const double*)D, ldd, ncol, coef, nx, ny, field, out);
  }
  LAUNCH_CHECK("mac_decode");
  return FDMD_OK;
}

int fdmd_mac_advect(const void* vel, int dtype, int nx, int ny, double h, double dt, const double* q, double* q_out,
                    void* stream) {
  if (!vel || !q || !q_out || nx < 2 || ny < 2 || !(h > 0)) return fail(FDMD_ERR_INVALID, "mac_advect: bad arguments");
  if (q == q_out) return fail(FDMD_ERR_INVALID, "mac_advect: q_out must not alias q");
  const int64_t cells = (int64_t)nx * ny;
  const int blocks = (int)((cells + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == FDMD_F32)
    fdmd::mac_advect_kernel<float><<<blocks, 256, 0, s>>>((const float*)vel, nx, ny, h, dt, q, q_out);
  else
    fdmd::mac_advect_kernel<double><<<blocks, 256, 0, s>>>((const double*)vel, nx, ny, h, dt, q, q_out);
  LAUNCH_CHECK("mac_advect");
  return FDMD_OK;
}

int fdmd_mac_inject(const double* low, int nx_high, int ny_high, int factor, int nv, int64_t ld_low,
                    int64_t ld_fine, double* fine, void* stream) {
  if (!low || !fine || factor < 2 || nx_high % factor || ny_high % factor || nv < 1)
    return fail(FDMD_ERR_INVALID, "mac_inject: bad arguments");
  const int64_t nh = (int64_t)(nx_high + 1) * ny_high + (int64_t)nx_high * (ny_high + 1);
  const int nxl = nx_high / factor, nyl = ny_high / factor;
  const int64_t nl = (int64_t)(nxl + 1) * nyl + (int64_t)nxl * (nyl + 1);
  if (ld_low < nl || ld_fine < nh) return fail(FDMD_ERR_INVALID, "mac_inject: bad leading dimension");
  fdmd::mac_inject_kernel<<<(unsigned)((nh + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      low, nx_high, ny_high, factor, nv, ld_low, ld_fine, fine);
  LAUNCH_CHECK("mac_inject");
  return FDMD_OK;
}

int fdmd_mac_project(const double* H, const double* L, int nx_high, int ny_high, int factor, double gram_diag,
                     double* x, void* stream) {
  if (!H || !L || !x || factor < 2 || nx_high % factor || ny_high % factor || !(gram_diag > 0))
    return fail(FDMD_ERR_INVALID, "mac_project: bad arguments");
  if (x == H) return fail(FDMD_ERR_INVALID, "mac_project: x must not alias H");
  const int64_t nh = (int64_t)(nx_high + 1) * ny_high + (int64_t)nx_high * (ny_high + 1);
  fdmd::mac_project_kernel<<<(unsigned)((nh + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      H, L, nx_high, ny_high, factor, 1.0 / factor, gram_diag, x);
  LAUNCH_CHECK("mac_project");
  return FDMD_OK;
}

// ---- 2-D smoke solver (fdmd_solver.cuh) ------------------------------------
static inline unsigned sol_blocks(int64_t n) { return (unsigned)((n + 255) / 256); }
static inline int64_t sol_nstate(int nx, int ny) { return (int64_t)(nx + 1) * ny + (int64_t)nx * (ny + 1); }
#define SOL_CHECK_GRID() \
  if (nx < 2 || ny < 2) return fail(FDMD_ERR_INVALID, "solver: grid must be at least 2x2")

int fdmd_sol_mask(double* vel, int nx, int ny, const unsigned char* solid, int closed, void* stream) {
  SOL_CHECK_GRID();
  const int64_t n = sol_nstate(nx, ny);
  fdmd::sol_mask_kernel<<<sol_blocks(n), 256, 0, (cudaStream_t)stream>>>(vel, nx, ny, solid, closed);
  LAUNCH_CHECK("sol_mask");
  return FDMD_OK;
}

int fdmd_sol_advect(const double* vel, const double* q, int which, int nx, int ny, double h, double dt,
                    int maccormack, double* scratch, double* out, void* stream) {
  SOL_CHECK_GRID();
  if (which < 0 || which > 2 || !vel || !q || !out || !scratch) return fail(FDMD_ERR_INVALID, "sol_advect: bad arguments");
  if (out == q) return fail(FDMD_ERR_INVALID, "sol_advect: out must not alias q");
  const int64_t len = which == 0 ? (int64_t)(nx + 1) * ny : which == 1 ? (int64_t)nx * (ny + 1) : (int64_t)nx * ny;
  cudaStream_t s = (cudaStream_t)stream;
  if (!maccormack) {
    fdmd::sol_advect_pred_kernel<<<sol_blocks(len), 256, 0, s>>>(vel, q, which, nx, ny, h, dt, out, nullptr, nullptr);
  } else {
    double* qhat = scratch;
    double* lo = scratch + len;
    double* hi = scratch + 2 * len;
    fdmd::sol_advect_pred_kernel<<<sol_blocks(len), 256, 0, s>>>(vel, q, which, nx, ny, h, dt, qhat, lo, hi);
    fdmd::sol_advect_corr_kernel<<<sol_blocks(len), 256, 0, s>>>(vel, q, qhat, lo, hi, which, nx, ny, h, dt, out);
  }
  LAUNCH_CHECK("sol_advect");
  return FDMD_OK;
}

int fdmd_sol_emit(double* dens, double* temp, int nx, int ny, double h, double cx, double cy, double r2, double dadd,
                  double tadd, void* stream) {
  SOL_CHECK_GRID();
  fdmd::sol_emit_kernel<<<sol_blocks((int64_t)nx * ny), 256, 0, (cudaStream_t)stream>>>(dens, temp, nx, ny, h, cx, cy,
                                                                                        r2, dadd, tadd);
  LAUNCH_CHECK("sol_emit");
  return FDMD_OK;
}

int fdmd_sol_buoyancy(double* vel, const double* dens, const double* temp, int nx, int ny, double alpha, double beta,
                      double dt, void* stream) {
  SOL_CHECK_GRID();
  fdmd::sol_buoyancy_kernel<<<sol_blocks((int64_t)(ny + 1) * nx), 256, 0, (cudaStream_t)stream>>>(
      vel, dens, temp, nx, ny, -alpha, beta, dt);
  LAUNCH_CHECK("sol_buoyancy");
  return FDMD_OK;
}

int fdmd_sol_vorticity(double* vel, int nx, int ny, double h, double eps, double dt, double* scratch, void* stream) {
  SOL_CHECK_GRID();
  const int64_t cells = (int64_t)nx * ny;
  cudaStream_t s = (cudaStream_t)stream;
  double* omega = scratch;
  double* fx = scratch + cells;
  double* fy = scratch + 2 * cells;
  fdmd::sol_omega_kernel<<<sol_blocks(cells), 256, 0, s>>>(vel, nx, ny, h, omega);
  fdmd::sol_confine_force_kernel<<<sol_blocks(cells), 256, 0, s>>>(omega, nx, ny, h, eps * h, fx, fy);
  fdmd::sol_confine_apply_kernel<<<sol_blocks(sol_nstate(nx, ny)), 256, 0, s>>>(vel, fx, fy, nx, ny, dt * 0.5);
  LAUNCH_CHECK("sol_vorticity");
  return FDMD_OK;
}

int fdmd_sol_reduce(const double* a, const double* b, const unsigned char* solid, int64_t n, int op, double* part,
                    double* out, void* stream) {
  if (!a || !out || !part || n <= 0 || op < 0 || op > 2 || (op == 0 && !b))
    return fail(FDMD_ERR_INVALID, "sol_reduce: bad arguments");
  const int blocks = (int)std::min<int64_t>(FDMD_SOL_REDUCE_BLOCKS, (n + 255) / 256);
  cudaStream_t s = (cudaStream_t)stream;
  fdmd::sol_reduce_kernel<<<blocks, 256, 0, s>>>(a, b, solid, n, op, part);
  fdmd::sol_reduce_final_kernel<<<1, 32, 0, s>>>(part, blocks, op, out);
  LAUNCH_CHECK("sol_reduce");
  return FDMD_OK;
}

int fdmd_sol_rhs(const double* vel, int nx, int ny, double h, const unsigned char* solid, int closed, double nfluid,
                 double* b, double* part, double* sum, void* stream) {
  SOL_CHECK_GRID();
  const int64_t cells = (int64_t)nx * ny;
  cudaStream_t s = (cudaStream_t)stream;
  fdmd::sol_rhs_kernel<<<sol_blocks(cells), 256, 0, s>>>(vel, nx, ny, h, solid, b);
  if (closed) {
    int rc = fdmd_sol_reduce(b, nullptr, solid, cells, 2, part, sum, stream);
    if (rc) return rc;
    fdmd::sol_sub_mean_kernel<<<sol_blocks(cells), 256, 0, s>>>(b, nx, ny, solid, sum, nfluid);
  }
  LAUNCH_CHECK("sol_rhs");
  return FDMD_OK;
}

int fdmd_sol_poisson(const double* p, int nx, int ny, double h2, const unsigned char* solid, int open, double* out,
                     void* stream) {
  SOL_CHECK_GRID();
  fdmd::sol_poisson_kernel<<<sol_blocks((int64_t)nx * ny), 256, 0, (cudaStream_t)stream>>>(p, nx, ny, h2, solid, open,
                                                                                           out);
  LAUNCH_CHECK("sol_poisson");
  return FDMD_OK;
}

int fdmd_sol_cg_step(double* p, double* r, const double* d, const double* Ad, double alpha, int64_t n, void* stream) {
  fdmd::sol_cg_step_kernel<<<sol_blocks(n), 256, 0, (cudaStream_t)stream>>>(p, r, d, Ad, alpha, n);
  LAUNCH_CHECK("sol_cg_step");
  return FDMD_OK;
}

int fdmd_sol_cg_dir(double* d, const double* r, double beta, int64_t n, void* stream) {
  fdmd::sol_cg_dir_kernel<<<sol_blocks(n), 256, 0, (cudaStream_t)stream>>>(d, r, beta, n);
  LAUNCH_CHECK("sol_cg_dir");
  return FDMD_OK;
}

int fdmd_sol_pressure_apply(double* vel, const double* p, int nx, int ny, double h, const unsigned char* solid,
                            int open, void* stream) {
  SOL_CHECK_GRID();
  fdmd::sol_pressure_apply_kernel<<<sol_blocks(sol_nstate(nx, ny)), 256, 0, (cudaStream_t)stream>>>(vel, p, nx, ny, h,
                                                                                                  solid, open);
  LAUNCH_CHECK("sol_pressure_apply");
  return FDMD_OK;
}

int fdmd_sol_cg_single(const double* b, double* p, double* r, double* d, double* Ad, int nx, int ny, double h2,
                       const unsigned char* solid, int open, double cg_tol, int max_iters, double* status,
                       void* stream) {
  SOL_CHECK_GRID();
  if ((int64_t)nx * ny > fdmd::SOL_CG1_MAX_CELLS) return fail(FDMD_ERR_INVALID, "sol_cg_single: grid too large");
  fdmd::sol_cg_single_kernel<<<1, fdmd::SOL_CG1_THREADS, 0, (cudaStream_t)stream>>>(
      b, p, r, d, Ad, nx, ny, h2, solid, open, cg_tol, max_iters, status);
  LAUNCH_CHECK("sol_cg_single");
  return FDMD_OK;
}

int fdmd_dmma_peak(double seconds, double* tflops) {
  if (!tflops || seconds <= 0) return fail(FDMD_ERR_INVALID, "dmma_peak: bad arguments");
  double* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, sizeof(double)));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  const int blocks = sm_count_cached() * 4, threads = 256;
  int iters = 2000;
  float ms = 0.f;
  fdmd::dmma_peak_kernel<<<blocks, threads>>>(d, 100);
  for (int rep = 0; rep < 8; ++rep) {  // grow until one launch lasts ~seconds/4
    CUDA_TRY(cudaEventRecord(e0));
    fdmd::dmma_peak_kernel<<<blocks, threads>>>(d, iters);
    CUDA_TRY(cudaEventRecord(e1));
    CUDA_TRY(cudaEventSynchronize(e1));
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    if (ms >= 250.0 * seconds) break;
    iters = (int)std::min<double>(2e9 / 8, iters * std::max(2.0, 250.0 * seconds / std::max(ms, 0.01f)));
  }
  const double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  LAUNCH_CHECK("dmma_peak");
  return FDMD_OK;
}

int fdmd_copy2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                int kind, void* stream) {
  if (height <= 0 || width <= 0) return FDMD_OK;
  CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                             (cudaMemcpyKind)kind, (cudaStream_t)stream));
  return FDMD_OK;
}

int fdmd_synth3d(const double* sx, const double* sy, const double* sz, const double* Am, int K, int C, int N,
                 int m, double noise, uint64_t key, int64_t row0, int64_t rows, void* out, int out_dtype,
                 int64_t ldo, void* stream) {
  if (K <= 0 || C <= 0 || N <= 0 || m <= 0 || rows < 0 || ldo < m) return fail(FDMD_ERR_INVALID, "synth3d: bad sizes");
  if (rows == 0) return FDMD_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t bx = std::min<int64_t>((rows + 255) / 256, (int64_t)sm_count_cached() * 16);
  dim3 grid((unsigned)bx, (m + 7) / 8);
  if (out_dtype == FDMD_F32)
    fdmd::synth3d_kernel<float><<<grid, 256, 0, s>>>(sx, sy, sz, Am, K, C, N, m, noise, key, row0, rows, (float*)out, ldo);
  else
    fdmd::synth3d_kernel<double><<<grid, 256, 0, s>>>(sx, sy, sz, Am, K, C, N, m, noise, key, row0, rows, (double*)out, ldo);
  LAUNCH_CHECK("synth3d");
  return FDMD_OK;
}

}  // extern "C"

// Internal hooks for the host orchestration unit (fdmd_fit.cpp, compiled
// separately with g++): the thread-local error slot, the stream-ordered scratch
// pool and the per-thread cuSOLVER handle. Not part of include/fdmd.h.
extern "C" {
int fdmdi_set_error(int code, const char* msg) {
  g_err = msg ? msg : "";
  return code;
}
cudaError_t fdmdi_scratch_alloc(void** p, size_t bytes, void* stream) {
  return scratch_alloc(p, bytes, (cudaStream_t)stream);
}
void* fdmdi_solver_handle(void* stream) {
  SolverCtx* c = solver_ctx();
  if (!c || cusolverDnSetStream(c->h, (cudaStream_t)stream) != CUSOLVER_STATUS_SUCCESS) return nullptr;
  return (void*)c->h;
}
}  // extern "C"
