// What limits DMMA.8x8x4 throughput in a tiled kernel? Variants:
//  A: MI x NF accumulators, constant fragments (pure issue rate)
//  B: same, fragments re-read from shared memory every k-step (LDS.64)
//  C: as B with the accumulator loop order f-outer (same as fdmd tall_gemm)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int MI, int NF, int MODE>
__global__ void k(double* out, int iters) {
  __shared__ double sA[4][68 * 2];
  __shared__ double sB[4][260];
  for (int i = threadIdx.x; i < 4 * 136; i += blockDim.x) (&sA[0][0])[i] = i * 1e-3;
  for (int i = threadIdx.x; i < 4 * 260; i += blockDim.x) (&sB[0][0])[i] = i * 1e-4;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  double acc[MI][NF][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[i][f][0] = acc[i][f][1] = 0;
  double a[MI], b[NF];
#pragma unroll
  for (int i = 0; i < MI; ++i) a[i] = sA[t][(w & 1) * 32 + i * 8 + g];
#pragma unroll
  for (int f = 0; f < NF; ++f) b[f] = sB[t][(w >> 1) * 8 * NF % 200 + f * 8 + g];
  for (int it = 0; it < iters; ++it) {
    if (MODE >= 1) {
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = sA[t][(w & 1) * 32 + i * 8 + g + (it & 1)];
#pragma unroll
      for (int f = 0; f < NF; ++f) b[f] = sB[t][(w >> 1) * 8 * NF % 200 + f * 8 + g + (it & 1)];
    }
    if (MODE == 3 && (it & 3) == 0) __syncthreads();
    if (MODE == 4 && (it & 3) == 0) {
      // emulate the per-chunk cp.async issue + wait + barrier
      __syncthreads();
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 2;\n" ::);
    }
    if (MODE == 2) {
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int i = 0; i < MI; ++i) dmma(acc[i][f], a[i], b[f]);
    } else {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int f = 0; f < NF; ++f) dmma(acc[i][f], a[i], b[f]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int f = 0; f < NF; ++f) s += acc[i][f][0] + acc[i][f][1];
  if (s == 1234.5) out[0] = s;
}

template <int MI, int NF, int MODE>
void run(const char* name, int threads, int bps) {
  double* d;
  cudaMalloc(&d, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * bps, iters = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MI, NF, MODE><<<blocks, threads>>>(d, 10);
  cudaEventRecord(e0);
  k<MI, NF, MODE><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * MI * NF * (double)iters * blocks * (threads / 32);
  printf("%-28s thr=%3d bps=%d  %6.2f TF/s  (%s)\n", name, threads, bps, fl / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<4, 7, 3>("lds 4x7 + sync/4 steps", 256, 1);
  run<4, 7, 4>("lds 4x7 + sync+cpasync/4", 256, 1);
  run<4, 2, 3>("lds 4x2 + sync/4 steps", 256, 2);
  run<4, 7, 0>("const 4x7", 256, 1);
  run<4, 7, 1>("lds   4x7", 256, 1);
  run<4, 7, 2>("lds   4x7 f-outer", 256, 1);
  run<4, 2, 1>("lds   4x2 (gram tile)", 256, 1);
  run<4, 2, 1>("lds   4x2 (gram tile)", 256, 2);
  run<4, 4, 1>("lds   4x4", 256, 1);
  run<4, 4, 1>("lds   4x4", 256, 2);
  run<8, 4, 1>("lds   8x4", 256, 1);
  run<4, 7, 1>("lds   4x7", 128, 2);
  run<4, 7, 1>("lds   4x7", 512, 1);
  run<2, 2, 1>("lds   2x2", 256, 4);
  return 0;
}
