// B200 (sm_100a) kernels for the DMD hot path.
//
// FP64 contractions run on the DMMA pipe (mma.sync m8n8k4 f64 -> SASS
// DMMA.8x8x4): tcgen05 has no f64 kind, and eigenvalue parity with the
// reference needs FP64 (SURVEY.md finding 4).
//
// Two contraction shapes cover every tall product of the fit:
//   * tall_gemm : C[n x N] = A[n x K] * B[K x N]      (A tall, B small)
//                 sketch X*Omega, power X*W, CholQR Y*R^-1, lift Q*Ub, modes S*C
//   * tall_gram : C[K1 x K2] = A[n x K1]^T B[n x K2] (reduction over n)
//                 Gram Y^T Y, X^T Q, Q^T S, D^T D, D^T S
// plus the HBM-streaming reconstruction (decode) and small helpers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fdmd {

enum { LAYOUT_ROW = 0, LAYOUT_COL = 1, LAYOUT_PLANES = 2 };  // PLANES: row-major fp16 hi (C) + lo (C2) of C * cscale
enum { DT_F32 = 0, DT_F64 = 1 };

// ---------------------------------------------------------------------------
// DMMA primitive: c(8x8) += a(8x4) * b(4x8); fragment ownership
//   a: A[m = lane>>2][k = lane&3]     b: B[k = lane&3][n = lane>>2]
//   c: C[m = lane>>2][n = 2*(lane&3) + {0,1}]
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <typename T> __device__ __forceinline__ double to_f64(T v) { return (double)v; }

struct TallGemmArgs {
  const void* A;  int64_t lda;  // A: n x K (ROW: A[i*lda+k]; COL: A[k*lda+i])
  const double* B; int64_t ldb; // B: K x N row-major
  void* C; int64_t ldc;         // C: n x N (ROW: C[i*ldc+j]; COL: C[j*ldc+i])
  int64_t n; int K; int N;
  int b_upper;         // B upper triangular (B[k][c] = 0 for k > c): skip zero blocks
  int reserve_sms;     // persistent grid leaves this many SMs free
  int debug;           // tuning experiments: bit0 no loads, bit1 no stores, bit2 no DMMA
  // epilogue statistics over column pairs (2u, 2u+1) = (Re, Im) of unit u:
  // per CTA: sum_i |c|^2 and (max_i |c|^2, first argmax i)
  double* pair_stats;  // [gridDim.x][N/2][3] or nullptr
  int64_t row_offset;  // global row index of row 0 (for sharded argmax)
  void* C2;            // LAYOUT_PLANES: the lo plane (C holds the hi plane), both ld ldc
  double cscale;       // LAYOUT_PLANES: planes hold C * cscale split as hi + lo
};

struct TallGramArgs {
  const void* A; int64_t lda;   // A: n x K1
  const void* B; int64_t ldb;   // B: n x K2
  double* W;                    // partials [splits][K1p][K2p]
  int64_t n; int K1; int K2; int K1p; int K2p;
  int tiles_j;                  // number of 64-wide tiles along K2
  int symmetric;                // only tiles ti <= tj
  int64_t rows_per_split;
};

}  // namespace fdmd
