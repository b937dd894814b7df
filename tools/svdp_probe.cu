// Probe: cuSOLVER SVD routines on the fit's small B (l x T fp64): gesvdj (what torch's driver="gesvdj"
// runs), gesvdp (polar decomposition) and gesvd, latency and accuracy against each other.
//   nvcc -O2 -o build/svdp_probe tools/svdp_probe.cu -lcusolver && ./build/svdp_probe [n] [cond]
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { auto e_ = (x); if (e_ != 0) { printf("error %d at line %d\n", (int)e_, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 200;
  const double cond = argc > 2 ? atof(argv[2]) : 1.2e4;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  // B = G1 diag(s) G2 with Gaussian factors (cond ~ cond * few): column-major n x n
  std::vector<double> G1(n * n), G2(n * n), B(n * n, 0.0);
  for (auto& v : G1) v = nd(rng) / std::sqrt((double)n);
  for (auto& v : G2) v = nd(rng) / std::sqrt((double)n);
  for (int k = 0; k < n; ++k) {
    const double s = std::pow(cond, -(double)k / (n - 1));
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) B[i + (size_t)j * n] += G1[i + (size_t)k * n] * s * G2[k + (size_t)j * n];
  }
  cusolverDnHandle_t h;
  CK(cusolverDnCreate(&h));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  CK(cusolverDnSetStream(h, st));
  double *dA, *dA0, *dS, *dU, *dV;
  int* dinfo;
  CK(cudaMalloc(&dA, sizeof(double) * n * n));
  CK(cudaMalloc(&dA0, sizeof(double) * n * n));
  CK(cudaMalloc(&dS, sizeof(double) * n));
  CK(cudaMalloc(&dU, sizeof(double) * n * n));
  CK(cudaMalloc(&dV, sizeof(double) * n * n));
  CK(cudaMalloc(&dinfo, sizeof(int)));
  CK(cudaMemcpy(dA0, B.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice));
  std::vector<double> s_j(n), s_p(n), s_q(n);
  auto timeit = [&](auto fn, const char* name, std::vector<double>& sv) {
    double best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemcpyAsync(dA, dA0, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st);
      cudaStreamSynchronize(st);
      auto t0 = std::chrono::steady_clock::now();
      if (fn() != 0) { printf("%s failed\n", name); return; }
      cudaStreamSynchronize(st);
      best = std::min(best, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    cudaMemcpy(sv.data(), dS, sizeof(double) * n, cudaMemcpyDeviceToHost);
    printf("%-10s n=%d  %.3f ms  s[0]=%.15e s[n-1]=%.15e\n", name, n, best, sv[0], sv[n - 1]);
  };
  // gesvdj
  gesvdjInfo_t jp;
  CK(cusolverDnCreateGesvdjInfo(&jp));
  int lw = 0;
  CK(cusolverDnDgesvdj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, dA, n, dS, dU, n, dV, n, &lw, jp));
  double* dw;
  CK(cudaMalloc(&dw, sizeof(double) * lw));
  timeit([&] { return (int)cusolverDnDgesvdj(h, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, dA, n, dS, dU, n, dV, n, dw, lw, dinfo, jp); },
         "gesvdj", s_j);
  // gesvdp
  cusolverDnParams_t pr;
  CK(cusolverDnCreateParams(&pr));
  size_t wd = 0, wh = 0;
  CK(cusolverDnXgesvdp_bufferSize(h, pr, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_R_64F, dA, n, CUDA_R_64F, dS, CUDA_R_64F,
                                  dU, n, CUDA_R_64F, dV, n, CUDA_R_64F, &wd, &wh));
  void* dwp;
  CK(cudaMalloc(&dwp, wd ? wd : 8));
  std::vector<char> hw(wh ? wh : 8);
  double herr = 0;
  timeit([&] { return (int)cusolverDnXgesvdp(h, pr, CUSOLVER_EIG_MODE_VECTOR, 1, n, n, CUDA_R_64F, dA, n, CUDA_R_64F, dS,
                                            CUDA_R_64F, dU, n, CUDA_R_64F, dV, n, CUDA_R_64F, dwp, wd, hw.data(), wh,
                                            dinfo, &herr); },
         "gesvdp", s_p);
  printf("gesvdp h_err_sigma %.3e  (host workspace %zu B)\n", herr, wh);
  // gesvd (QR iteration)
  int lg = 0;
  CK(cusolverDnDgesvd_bufferSize(h, n, n, &lg));
  double* dg;
  CK(cudaMalloc(&dg, sizeof(double) * lg));
  timeit([&] { return (int)cusolverDnDgesvd(h, 'S', 'S', n, n, dA, n, dS, dU, n, dV, n, dg, lg, nullptr, dinfo); }, "gesvd", s_q);
  double ej = 0, ep = 0;
  for (int i = 0; i < n; ++i) {
    ej = std::max(ej, std::fabs(s_j[i] - s_q[i]) / s_q[i]);
    ep = std::max(ep, std::fabs(s_p[i] - s_q[i]) / s_q[i]);
  }
  printf("max rel sigma diff vs gesvd: gesvdj %.3e  gesvdp %.3e\n", ej, ep);
  return 0;
}
