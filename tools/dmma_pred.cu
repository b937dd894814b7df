// Does predicating DMMA (warp-uniform runtime condition) cost throughput?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* out, int iters, int live_mask) {
  __shared__ double sA[4][136];
  __shared__ double sB[4][260];
  for (int i = threadIdx.x; i < 4 * 136; i += blockDim.x) (&sA[0][0])[i] = i * 1e-3;
  for (int i = threadIdx.x; i < 4 * 260; i += blockDim.x) (&sB[0][0])[i] = i * 1e-4;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  bool live[4][2];
  for (int i = 0; i < 4; ++i) for (int f = 0; f < 2; ++f) live[i][f] = (live_mask >> (i * 2 + f)) & 1;
  double acc[4][2][2];
  for (int i = 0; i < 4; ++i) for (int f = 0; f < 2; ++f) acc[i][f][0] = acc[i][f][1] = 0;
  for (int it = 0; it < iters; ++it) {
    double a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sA[t][(w & 1) * 32 + i * 8 + g + (it & 7)];
#pragma unroll
    for (int f = 0; f < 2; ++f) b[f] = sB[t][(w >> 1) * 16 + f * 8 + g + (it & 7)];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        if (MODE == 0) dmma(acc[i][f], a[i], b[f]);
        else if (live[i][f]) dmma(acc[i][f], a[i], b[f]);
      }
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int f = 0; f < 2; ++f) s += acc[i][f][0] + acc[i][f][1];
  if (s == 1234.5) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) for (int bps = 1; bps <= 2; ++bps) {
    const int iters = 20000; float ms;
    k<0><<<sms, 256>>>(d, 10, 255);
    cudaEventRecord(e0);
    if (mode) k<1><<<sms * bps, 256>>>(d, iters, 255); else k<0><<<sms * bps, 256>>>(d, iters, 255);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 8 * (double)iters * sms * bps * 8;
    printf("%s bps=%d: %.2f TF/s\n", mode ? "predicated" : "plain     ", bps, fl / ms / 1e9);
  }
  return 0;
}
