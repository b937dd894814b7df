// Do DMMA (mma.sync f64) and DFMA (SIMT FP64) share one pipe on sm_100a?
// Runs each alone, then both at once (split by warp and interleaved within a
// warp), and prints the combined FP64 rate. If the rates add, FP64 work can be
// split between the tensor pipe and the FMA pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// mode 0: DMMA only; 1: DFMA only; 2: even warps DMMA, odd warps DFMA;
// 3: every warp interleaves (8 DMMA + nf DFMA chains per iteration)
template <int MODE>
__global__ void mix(double* out, int iters, int fma_per_dmma) {
  const int warp = threadIdx.x >> 5;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  double x[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-9 + i;
  const bool do_mma = MODE == 0 || MODE == 3 || (MODE == 2 && !(warp & 1));
  const bool do_fma = MODE == 1 || MODE == 3 || (MODE == 2 && (warp & 1));
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
    }
    if (do_fma) {
      for (int r = 0; r < fma_per_dmma; ++r) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 2, iters = 4000;
  const double warps = (double)blocks * threads / 32;
  auto run = [&](auto kern, int nf, const char* name, double mma_warps, double fma_warps) {
    kern<<<blocks, threads>>>(d, 10, nf);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, iters, nf);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fm = 512.0 * 8 * iters * mma_warps;        // DMMA.884 = 512 flop
    const double ff = 2.0 * 16 * nf * iters * 32 * fma_warps;
    printf("%-34s nf=%2d  %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TF/s\n", name, nf, ms, fm / ms / 1e9, ff / ms / 1e9,
           (fm + ff) / ms / 1e9);
  };
  run(mix<0>, 0, "DMMA only", warps, 0);
  for (int nf : {1, 2, 4}) run(mix<1>, nf, "DFMA only", 0, warps);
  for (int nf : {1, 2, 4, 8}) run(mix<2>, nf, "split by warp (even MMA, odd FMA)", warps / 2, warps / 2);
  for (int nf : {1, 2, 4}) run(mix<3>, nf, "interleaved in every warp", warps, warps);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
