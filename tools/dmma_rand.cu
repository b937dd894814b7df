// DMMA throughput with random operand bits (power / toggling sensitivity).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ double rnd(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return ((double)(x >> 11) * 0x1.0p-53) * 2.0 - 1.0;
}
template <int RANDOM>
__global__ void k(double* out, int iters) {
  __shared__ double sA[4][136];
  __shared__ double sB[4][260];
  for (int i = threadIdx.x; i < 4 * 136; i += blockDim.x) (&sA[0][0])[i] = RANDOM ? rnd(i + 7 * blockIdx.x) : i * 1e-3;
  for (int i = threadIdx.x; i < 4 * 260; i += blockDim.x) (&sB[0][0])[i] = RANDOM ? rnd(i + 100000 + blockIdx.x) : i * 1e-4;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, w = threadIdx.x >> 5;
  double acc[4][7][2];
  for (int i = 0; i < 4; ++i) for (int f = 0; f < 7; ++f) acc[i][f][0] = acc[i][f][1] = 0;
  for (int it = 0; it < iters; ++it) {
    double a[4], b[7];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = sA[t][(w & 1) * 32 + i * 8 + g + (it & 7)];
#pragma unroll
    for (int f = 0; f < 7; ++f) b[f] = sB[t][(w >> 1) * 56 % 200 + f * 8 + g + (it & 7)];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int f = 0; f < 7; ++f) dmma(acc[i][f], a[i], b[f]);
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int f = 0; f < 7; ++f) s += acc[i][f][0] + acc[i][f][1];
  if (s == 1234.5) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep)
  for (int R = 0; R < 2; ++R) {
    const int iters = 40000; float ms;
    cudaEventRecord(e0);
    if (R) k<1><<<sms, 256>>>(d, iters); else k<0><<<sms, 256>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 256 * 28 * (double)iters * sms * 8;
    printf("random=%d: %.2f TF/s (%.0f ms)\n", R, fl / ms / 1e9, ms);
  }
  return 0;
}
