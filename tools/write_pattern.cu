// HBM write bandwidth for the reconstruction's output pattern, without any
// math: frames are frame-major (out[f * n + i]); a CTA writes tiles of
// 128 rows x 256 frames (512 B per frame row) in the tc_decode2 tile order
// (tile = p + t * P for CTA p of P). Compared with a contiguous fill.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/write_pattern tools/write_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fill(float* out, size_t n4) {
  float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<float4*>(out)[i] = v;
}

// 512 threads: warp w writes rows (w % 4) * 32 + lane of frames [ (w / 4) * 64, +64 )
template <bool STCS>
__global__ void __launch_bounds__(512) tiles(float* out, long n, int nf, long ptiles) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = w & 3, part = w >> 2;
  for (long t = blockIdx.x; t < ptiles; t += gridDim.x) {
    const long row = t * 128 + q * 32 + lane;
    if (row >= n) continue;
    for (int f = part * 64; f < part * 64 + 64 && f < nf; ++f) {
      float* o = out + (long)f * n + row;
      if (STCS) __stcs(o, (float)f); else *o = (float)f;
    }
  }
}

// the tc_decode2 epilogue shape with 16-B stores: warp (q, part) owns rows
// q*32..+31 of frames part*64..+63; per instruction lane l writes rows
// q*32 + 4*(l%8)..+3 of frame f + l/8 (4 frames x 128 B per instruction)
__global__ void __launch_bounds__(512) tiles_v4(float* out, long n, int nf, long ptiles) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = w & 3, part = w >> 2;
  for (long t = blockIdx.x; t < ptiles; t += gridDim.x) {
    const long row = t * 128 + q * 32 + 4 * (lane & 7);
    if (row + 3 >= n) continue;
    for (int f = part * 64 + (lane >> 3); f < part * 64 + 64 && f < nf; f += 4)
      __stcs(reinterpret_cast<float4*>(out + (long)f * n + row), make_float4(1.f, 2.f, 3.f, (float)f));
  }
}

// generalised: tiles of ROWS rows x nf frames; CTA b takes tiles b, b + G, ...
// (cyclic) or a contiguous range of tiles (blocked)
template <int ROWS, bool BLOCKED>
__global__ void __launch_bounds__(512) tiles2(float* out, long n, int nf, long ptiles) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long per = (ptiles + gridDim.x - 1) / gridDim.x;
  const long t0 = BLOCKED ? blockIdx.x * per : blockIdx.x;
  const long t1 = BLOCKED ? min(ptiles, t0 + per) : ptiles;
  const long dt = BLOCKED ? 1 : gridDim.x;
  for (long t = t0; t < t1; t += dt) {
    for (int f = w; f < nf; f += 16) {            // 16 warps: warp w takes frames w, w+16, ...
      float* o = out + (long)f * n + t * ROWS;
      for (int i = lane * 4; i < ROWS; i += 128) {
        const long row = t * ROWS + i;
        if (row + 3 < n) __stcs(reinterpret_cast<float4*>(o + i), make_float4(1.f, 2.f, 3.f, 4.f));
      }
    }
  }
}

template <int ROWS, bool BLOCKED>
void run2(float* out, long n, int nf, int sms, cudaEvent_t e0, cudaEvent_t e1, double bytes) {
  float ms;
  const long ptiles = (n + ROWS - 1) / ROWS;
  tiles2<ROWS, BLOCKED><<<sms, 512>>>(out, n, nf, ptiles);
  cudaEventRecord(e0);
  tiles2<ROWS, BLOCKED><<<sms, 512>>>(out, n, nf, ptiles);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("tiles %4d rows x %d frames %s  %.2f ms  %.0f GB/s\n", ROWS, nf, BLOCKED ? "blocked" : "cyclic ", ms,
         bytes / ms / 1e6);
}

int main() {
  const long n = 50331648;
  const int nf = 256;
  float* out;
  if (cudaMalloc(&out, (size_t)nf * n * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)nf * n * 4;
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0);
    fill<<<sms * 8, 512>>>(out, (size_t)nf * n / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("contiguous fill   %.2f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    const long ptiles = (n + 127) / 128;
    cudaEventRecord(e0);
    tiles<true><<<sms, 512>>>(out, n, nf, ptiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("frame tiles stcs  %.2f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(e0);
    tiles<false><<<sms, 512>>>(out, n, nf, ptiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("frame tiles st    %.2f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
  }
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    const long ptiles = (n + 127) / 128;
    cudaEventRecord(e0);
    tiles_v4<<<sms, 512>>>(out, n, nf, ptiles);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("frame tiles v4 (epilogue shape, 16-B stores)  %.2f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
  }
  run2<128, false>(out, n, nf, sms, e0, e1, bytes);
  run2<256, false>(out, n, nf, sms, e0, e1, bytes);
  run2<512, false>(out, n, nf, sms, e0, e1, bytes);
  run2<1024, false>(out, n, nf, sms, e0, e1, bytes);
  run2<4096, false>(out, n, nf, sms, e0, e1, bytes);
  run2<256, true>(out, n, nf, sms, e0, e1, bytes);
  run2<1024, true>(out, n, nf, sms, e0, e1, bytes);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
