// fdmd_fit.cpp — host orchestration of the fit / model C ABI:
//
//   fdmd_rsvd                 randomized_svd            (linalg.py:62-90)
//   fdmd_dmd_fit  EXACT       exact_dmd                 (dmd.py:240-274)
//   fdmd_dmd_fit  OPT         optdmd + _varpro_lm       (dmd.py:277-455)
//   fdmd_model_phi_to_host    ReducedModel.phi          (dmd.py:53-77), chunked
//   fdmd_encode               encode = pinv(phi) u      (runtime.py:47-52)
//   fdmd_model_decode         decode = Re(phi z)        (runtime.py:66-99)
//
// for a flowdmd maintainer who binds libfdmd through ctypes without this
// package's Python layer. Every n-sized product runs on
// libfdmd's sm_100a kernels (fdmd_tall_gemm / fdmd_tall_gram / fdmd_decode /
// fdmd_colmajor_dot, FP64 DMMA); the r x r / T x r work (Cholesky factors,
// the QR of Z, the variable-projection LM, the pair plan) is formed on the
// host in fp64 (r, T <= 256: milliseconds), svd(B) and eig(K) on cuSOLVER.
// Compiled with g++ (no device code) and linked into libfdmd.so.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numeric>
#include <set>
#include <vector>

#include "../../include/fdmd.h"
#include "fdmd_internal.h"

using cd = std::complex<double>;

namespace {

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return fdmdi_set_error(code, buf);
}

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess) return fail(FDMD_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)
#define TRY(x)                     \
  do {                             \
    int _rc = (x);                 \
    if (_rc != FDMD_OK) return _rc; \
  } while (0)

inline int64_t round_up(int64_t x, int64_t q) { return (x + q - 1) / q * q; }
inline size_t esize(int dt) { return dt == FDMD_F32 ? 4 : 8; }

// ============================================================================
// small dense host linear algebra (row-major, fp64 / complex128)
// ============================================================================

// upper R with G = R^T R (G symmetric positive definite, l x l); false if not PD
bool chol_upper(const std::vector<double>& G, int l, std::vector<double>& R) {
  R.assign((size_t)l * l, 0.0);
  for (int j = 0; j < l; ++j) {
    double d = G[(size_t)j * l + j];
    for (int k = 0; k < j; ++k) d -= R[(size_t)k * l + j] * R[(size_t)k * l + j];
    if (!(d > 0.0)) return false;
    const double rjj = std::sqrt(d);
    R[(size_t)j * l + j] = rjj;
    for (int i = j + 1; i < l; ++i) {
      double s = G[(size_t)j * l + i];
      for (int k = 0; k < j; ++k) s -= R[(size_t)k * l + j] * R[(size_t)k * l + i];
      R[(size_t)j * l + i] = s / rjj;
    }
  }
  return true;
}

std::vector<double> inv_upper(const std::vector<double>& R, int l) {
  std::vector<double> X((size_t)l * l, 0.0);
  for (int j = 0; j < l; ++j) {  // column j of R^-1: solve R x = e_j
    X[(size_t)j * l + j] = 1.0 / R[(size_t)j * l + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += R[(size_t)i * l + k] * X[(size_t)k * l + j];
      X[(size_t)i * l + j] = -s / R[(size_t)i * l + i];
    }
  }
  return X;
}

std::vector<double> matmul(const std::vector<double>& A, const std::vector<double>& B, int m, int k, int n) {
  std::vector<double> C((size_t)m * n, 0.0);
  for (int i = 0; i < m; ++i)
    for (int p = 0; p < k; ++p) {
      const double a = A[(size_t)i * k + p];
      if (a == 0.0) continue;
      for (int j = 0; j < n; ++j) C[(size_t)i * n + j] += a * B[(size_t)p * n + j];
    }
  return C;
}

std::vector<double> transpose(const std::vector<double>& A, int m, int n) {
  std::vector<double> T((size_t)m * n);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) T[(size_t)j * m + i] = A[(size_t)i * n + j];
  return T;
}

double fro(const std::vector<double>& A) {
  double s2 = 0.0;
  for (double x : A) s2 += x * x;
  return std::sqrt(s2);
}

// thin Householder QR of Z (T x l, T >= l): returns Q (T x l)
std::vector<double> householder_q(std::vector<double> Z, int T, int l) {
  std::vector<std::vector<double>> vs;
  for (int j = 0; j < l; ++j) {
    double nrm = 0.0;
    for (int i = j; i < T; ++i) nrm += Z[(size_t)i * l + j] * Z[(size_t)i * l + j];
    nrm = std::sqrt(nrm);
    std::vector<double> v(T - j);
    for (int i = j; i < T; ++i) v[i - j] = Z[(size_t)i * l + j];
    const double alpha = (v[0] >= 0 ? -nrm : nrm);
    v[0] -= alpha;
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn > 0) {
      for (int c = j; c < l; ++c) {
        double s = 0.0;
        for (int i = j; i < T; ++i) s += v[i - j] * Z[(size_t)i * l + c];
        s = 2.0 * s / vn;
        for (int i = j; i < T; ++i) Z[(size_t)i * l + c] -= s * v[i - j];
      }
    }
    vs.push_back(std::move(v));
  }
  std::vector<double> Q((size_t)T * l, 0.0);
  for (int j = 0; j < l; ++j) Q[(size_t)j * l + j] = 1.0;
  for (int j = l - 1; j >= 0; --j) {
    const std::vector<double>& v = vs[j];
    double vn = 0.0;
    for (double x : v) vn += x * x;
    if (vn == 0) continue;
    for (int c = 0; c < l; ++c) {
      double s = 0.0;
      for (int i = j; i < T; ++i) s += v[i - j] * Q[(size_t)i * l + c];
      s = 2.0 * s / vn;
      for (int i = j; i < T; ++i) Q[(size_t)i * l + c] -= s * v[i - j];
    }
  }
  return Q;
}

// complex matrix, row-major
struct CM {
  int m = 0, n = 0;
  std::vector<cd> a;
  CM() = default;
  CM(int m_, int n_) : m(m_), n(n_), a((size_t)m_ * n_) {}
  cd& operator()(int i, int j) { return a[(size_t)i * n + j]; }
  const cd& operator()(int i, int j) const { return a[(size_t)i * n + j]; }
};

CM cmul(const CM& A, const CM& B) {  // A B
  CM C(A.m, B.n);
  for (int i = 0; i < A.m; ++i)
    for (int p = 0; p < A.n; ++p) {
      const cd x = A(i, p);
      if (x == 0.0) continue;
      const cd* b = &B.a[(size_t)p * B.n];
      cd* c = &C.a[(size_t)i * C.n];
      for (int j = 0; j < B.n; ++j) c[j] += x * b[j];
    }
  return C;
}

CM cmulH(const CM& A, const CM& B) {  // A^H B
  CM C(A.n, B.n);
  for (int p = 0; p < A.m; ++p)
    for (int i = 0; i < A.n; ++i) {
      const cd x = std::conj(A(p, i));
      if (x == 0.0) continue;
      const cd* b = &B.a[(size_t)p * B.n];
      cd* c = &C.a[(size_t)i * C.n];
      for (int j = 0; j < B.n; ++j) c[j] += x * b[j];
    }
  return C;
}

double cfro(const CM& A) {
  double s = 0.0;
  for (const cd& x : A.a) s += std::norm(x);
  return std::sqrt(s);
}

// thin complex Householder QR of A (m x n, m >= n): A = Q R
void cqr(CM A, CM& Q, CM& R) {
  const int m = A.m, n = A.n;
  std::vector<std::vector<cd>> vs(n);
  std::vector<double> vn(n, 0.0);
  for (int j = 0; j < n; ++j) {
    double nrm2 = 0.0;
    for (int i = j; i < m; ++i) nrm2 += std::norm(A(i, j));
    const double nrm = std::sqrt(nrm2);
    std::vector<cd> v(m - j);
    for (int i = j; i < m; ++i) v[i - j] = A(i, j);
    const cd x0 = v[0];
    const double ax0 = std::abs(x0);
    const cd ph = ax0 > 0 ? x0 / ax0 : cd(1.0, 0.0);
    const cd alpha = -ph * nrm;
    v[0] -= alpha;
    double s = 0.0;
    for (const cd& x : v) s += std::norm(x);
    vn[j] = s;
    if (s > 0) {
      for (int c = j; c < n; ++c) {
        cd dot = 0.0;
        for (int i = j; i < m; ++i) dot += std::conj(v[i - j]) * A(i, c);
        dot *= 2.0 / s;
        for (int i = j; i < m; ++i) A(i, c) -= dot * v[i - j];
      }
    }
    vs[j] = std::move(v);
  }
  R = CM(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = i; j < n; ++j) R(i, j) = A(i, j);
  Q = CM(m, n);
  for (int j = 0; j < n; ++j) Q(j, j) = 1.0;
  for (int j = n - 1; j >= 0; --j) {
    if (vn[j] == 0) continue;
    const std::vector<cd>& v = vs[j];
    for (int c = 0; c < n; ++c) {
      cd dot = 0.0;
      for (int i = j; i < m; ++i) dot += std::conj(v[i - j]) * Q(i, c);
      dot *= 2.0 / vn[j];
      for (int i = j; i < m; ++i) Q(i, c) -= dot * v[i - j];
    }
  }
}

// one-sided (Hestenes) Jacobi SVD of A (m x n, m >= n): A = U diag(s) V^H,
// s descending
void csvd(CM A, CM& U, std::vector<double>& s, CM& V) {
  const int m = A.m, n = A.n;
  V = CM(n, n);
  for (int i = 0; i < n; ++i) V(i, i) = 1.0;
  // column-major working copies for cache-friendly column sweeps
  std::vector<std::vector<cd>> col(n, std::vector<cd>(m)), vcol(n, std::vector<cd>(n));
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) col[j][i] = A(i, j);
    vcol[j][j] = 1.0;
  }
  const double eps = 2.220446049250313e-16;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0.0, be = 0.0;
        cd ga = 0.0;
        const cd* ap = col[p].data();
        const cd* aq = col[q].data();
        for (int i = 0; i < m; ++i) {
          al += std::norm(ap[i]);
          be += std::norm(aq[i]);
          ga += std::conj(ap[i]) * aq[i];
        }
        const double g = std::abs(ga);
        if (g == 0.0 || g <= eps * std::sqrt(al * be)) continue;
        rotated = true;
        const cd ph = ga / g;  // a_q' = a_q conj(ph) makes a_p^H a_q' real
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        cd* xp = col[p].data();
        cd* xq = col[q].data();
        for (int i = 0; i < m; ++i) {
          const cd u = xp[i], w = xq[i] * std::conj(ph);
          xp[i] = c * u - sn * w;
          xq[i] = sn * u + c * w;
        }
        cd* vp = vcol[p].data();
        cd* vq = vcol[q].data();
        for (int i = 0; i < n; ++i) {
          const cd u = vp[i], w = vq[i] * std::conj(ph);
          vp[i] = c * u - sn * w;
          vq[i] = sn * u + c * w;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> nr(n);
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int i = 0; i < m; ++i) s2 += std::norm(col[j][i]);
    nr[j] = std::sqrt(s2);
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return nr[a] > nr[b]; });
  U = CM(m, n);
  s.assign(n, 0.0);
  CM Vs(n, n);
  for (int k = 0; k < n; ++k) {
    const int j = ord[k];
    s[k] = nr[j];
    for (int i = 0; i < m; ++i) U(i, k) = nr[j] > 0 ? col[j][i] / nr[j] : cd(0.0);
    for (int i = 0; i < n; ++i) Vs(i, k) = vcol[j][i];
  }
  V = Vs;
}

// inverse of an upper-triangular complex n x n matrix
CM cinv_upper(const CM& R) {
  const int n = R.n;
  CM X(n, n);
  for (int j = 0; j < n; ++j) {
    X(j, j) = 1.0 / R(j, j);
    for (int i = j - 1; i >= 0; --i) {
      cd s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += R(i, k) * X(k, j);
      X(i, j) = -s / R(i, i);
    }
  }
  return X;
}

// min-norm least squares A X = B (numpy lstsq rcond=None -> gelsd cut
// eps * max(M, N) * s_max, linalg.py:136-141); QR fast path when R is
// provably well inside the cut (the same rule as linalg.lstsq_minnorm)
CM lstsq_minnorm(const CM& A, const CM& B) {
  const int M = A.m, N = A.n;
  const double rcond = 2.220446049250313e-16 * std::max(M, N);
  if (M >= N) {
    CM Qa, Ra;
    cqr(A, Qa, Ra);
    bool nonsingular = true;
    for (int i = 0; i < N; ++i)
      if (Ra(i, i) == 0.0) nonsingular = false;
    if (nonsingular) {
      CM Ri = cinv_upper(Ra);
      const double bound = cfro(Ra) * cfro(Ri);
      if (std::isfinite(bound) && bound * rcond < 1e-3) return cmul(Ri, cmulH(Qa, B));
    }
  }
  CM U, V;
  std::vector<double> s;
  if (M >= N) {
    csvd(A, U, s, V);
  } else {  // A^H = U' s V'^H  ->  A = V' s U'^H
    CM Ah(N, M);
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) Ah(j, i) = std::conj(A(i, j));
    CM U2, V2;
    csvd(Ah, U2, s, V2);
    U = V2;
    V = U2;
  }
  const int k = (int)s.size();
  CM UhB = cmulH(U, B);  // k x nrhs
  for (int i = 0; i < k; ++i) {
    const double inv = (s[0] > 0 && s[i] > rcond * s[0]) ? 1.0 / s[i] : 0.0;
    for (int j = 0; j < UhB.n; ++j) UhB(i, j) *= inv;
  }
  return cmul(V, UhB);
}

// LU with partial pivoting; false on an exactly singular pivot (getrf info > 0)
bool csolve(CM A, std::vector<cd>& b) {
  const int n = A.n;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::abs(A(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > best) best = std::abs(A(i, k)), p = i;
    if (best == 0.0) return false;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      std::swap(b[k], b[p]);
    }
    for (int i = k + 1; i < n; ++i) {
      const cd f = A(i, k) / A(k, k);
      if (f == 0.0) continue;
      for (int j = k + 1; j < n; ++j) A(i, j) -= f * A(k, j);
      b[i] -= f * b[k];
    }
  }
  for (int i = n - 1; i >= 0; --i) {
    cd s = b[i];
    for (int j = i + 1; j < n; ++j) s -= A(i, j) * b[j];
    b[i] = s / A(i, i);
  }
  return true;
}

// ============================================================================
// eigenvalue bookkeeping: conjugate_pairs (dmd.py:131-155), the frequency
// order and pair locking of _order_and_pair (dmd.py:158-213)
// ============================================================================
std::vector<int> conjugate_pairs(const std::vector<cd>& lam, double tol = 1e-8) {
  const int r = (int)lam.size();
  double scale = 1.0;
  if (r) {
    scale = 0.0;
    for (const cd& x : lam) scale = std::max(scale, std::abs(x));
    scale = std::max(scale, 1e-300);
  }
  std::vector<int> partner(r, -1);
  for (int i = 0; i < r; ++i) {
    if (partner[i] >= 0) continue;
    if (std::abs(lam[i].imag()) <= tol * scale) {
      partner[i] = i;
      continue;
    }
    int best = -1;
    double bd = 0.0;
    for (int j = 0; j < r; ++j) {
      if (partner[j] >= 0 || j == i) continue;
      const double d = std::abs(lam[j] - std::conj(lam[i]));
      if (best < 0 || d < bd) best = j, bd = d;  // first minimum
    }
    if (best >= 0 && bd <= 10 * tol * scale + tol) {
      partner[i] = best;
      partner[best] = i;
      continue;
    }
    partner[i] = i;
  }
  return partner;
}

struct PairPlan {
  std::vector<cd> lam;                      // final eigenvalues (sorted, locked, real-ified)
  std::vector<int> src;                     // per unit: source eigen-column
  std::vector<std::pair<int, bool>> pos;    // per position: (unit, conjugate?)
  std::set<int> realify;                    // units whose lambda was real-ified (unpaired)
};

PairPlan pair_plan(const std::vector<cd>& lam_raw) {
  const int r = (int)lam_raw.size();
  std::vector<int> partner = conjugate_pairs(lam_raw);
  std::vector<std::pair<int, int>> units;
  std::vector<char> seen(r, 0);
  for (int i = 0; i < r; ++i) {
    if (seen[i]) continue;
    const int j = partner[i];
    seen[i] = seen[j] = 1;
    if (i == j)
      units.push_back({i, -1});
    else
      units.push_back(lam_raw[i].imag() >= lam_raw[j].imag() ? std::make_pair(i, j) : std::make_pair(j, i));
  }
  auto key_less = [&](const std::pair<int, int>& a, const std::pair<int, int>& b) {
    const cd x = lam_raw[a.first], y = lam_raw[b.first];
    const double ax = std::abs(std::atan2(x.imag(), x.real())), ay = std::abs(std::atan2(y.imag(), y.real()));
    if (ax != ay) return ax < ay;
    if (-std::abs(x) != -std::abs(y)) return -std::abs(x) < -std::abs(y);
    return x.real() < y.real();
  };
  std::stable_sort(units.begin(), units.end(), key_less);
  std::vector<int> order;
  for (auto& u : units) {
    order.push_back(u.first);
    if (u.second >= 0) order.push_back(u.second);
  }
  PairPlan p;
  p.lam.resize(r);
  for (int k = 0; k < r; ++k) p.lam[k] = lam_raw[order[k]];
  p.pos.assign(r, {-1, false});
  int k = 0;
  while (k < r) {
    const int u = (int)p.src.size();
    p.src.push_back(order[k]);
    p.pos[k] = {u, false};
    const bool paired = k + 1 < r && p.lam[k].imag() > 0 &&
                        std::abs(p.lam[k + 1] - std::conj(p.lam[k])) <= 1e-6 * std::max(std::abs(p.lam[k]), 1e-300);
    if (paired) {
      p.lam[k + 1] = std::conj(p.lam[k]);
      p.pos[k + 1] = {u, true};
      k += 2;
      continue;
    }
    if (std::abs(p.lam[k].imag()) <= 1e-12 * std::max(std::abs(p.lam[k]), 1e-300)) {
      p.lam[k] = p.lam[k].real();
      p.realify.insert(u);
    }
    k += 1;
  }
  return p;
}

// ============================================================================
// device scratch + the randomized range finder (linalg.py:62-90)
// ============================================================================
struct Dev {
  cudaStream_t s;
  std::vector<void*> ptrs;
  bool trim = false;
  explicit Dev(cudaStream_t st) : s(st) {}
  ~Dev() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
    if (cudaStreamSynchronize(s) == cudaSuccess && trim) {
      // the n x l sketch is a one-off (80 GB at n = 50M, l = 200): hand its pages
      // back instead of keeping them reserved in the pool (release threshold is
      // infinite for the fit's stream-ordered scratch)
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolTrimTo(pool, 0);
    }
  }
  template <typename T> T* alloc(size_t count) {
    void* p = nullptr;
    if (fdmdi_scratch_alloc(&p, std::max<size_t>(count, 1) * sizeof(T), s) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  int up(const void* h, void* d, size_t bytes) {
    CUDA_TRY(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    return FDMD_OK;
  }
  int down(void* h, const void* d, size_t bytes) {
    CUDA_TRY(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FDMD_OK;
  }
};

// the CholeskyQR condition limit of linalg.CHOLQR2_COND_LIMIT (decided on the
// Frobenius bound ||R|| ||R^-1|| >= cond_2(R))
constexpr double RSVD_COND_LIMIT = 3e7;

struct Tall {  // row-major n x k device matrix
  const void* p;
  int dt;
  int64_t ld;
};

// Householder QR of the tall buffer (n x l, row-major, ld ldq) in place on
// cuSOLVER (geqrf + orgqr on a column-major copy made by the tall GEMM): the
// fallback of linalg.cholqr2_deferred when the (shifted) CholeskyQR Gram is not
// positive definite, i.e. a rank-deficient sketch. Leaves fix = identity.
int householder(Dev& d, double* Q, int64_t ldq, int64_t n, int l, std::vector<double>& fix,
                std::vector<double>* R_out = nullptr) {
  cusolverDnHandle_t h = (cusolverDnHandle_t)fdmdi_solver_handle(d.s);
  if (!h) return fail(FDMD_ERR_SOLVER, "cusolverDnCreate failed");
  if (n > INT32_MAX) return fail(FDMD_ERR_SOLVER, "Householder fallback limited to n < 2^31 rows");
  std::vector<double> I((size_t)l * l, 0.0);
  for (int i = 0; i < l; ++i) I[(size_t)i * l + i] = 1.0;
  const int64_t lda = round_up(n, 2);
  double* A = d.alloc<double>((size_t)lda * l);
  double* Id = d.alloc<double>(I.size());
  double* tau = d.alloc<double>(l);
  int* info = d.alloc<int>(1);
  if (!A || !Id || !tau || !info) return fail(FDMD_ERR_CUDA, "householder: device allocation failed");
  TRY(d.up(I.data(), Id, I.size() * sizeof(double)));
  TRY(fdmd_tall_gemm(Q, FDMD_F64, FDMD_ROW, ldq, Id, l, A, FDMD_F64, FDMD_COL, lda, n, l, l, 0, nullptr, 0, nullptr, 0,
                     d.s));
  int lw1 = 0, lw2 = 0;
  if (cusolverDnDgeqrf_bufferSize(h, (int)n, l, A, (int)lda, &lw1) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDorgqr_bufferSize(h, (int)n, l, l, A, (int)lda, tau, &lw2) != CUSOLVER_STATUS_SUCCESS)
    return fail(FDMD_ERR_SOLVER, "householder: bufferSize");
  double* work = d.alloc<double>((size_t)std::max(lw1, lw2));
  if (!work) return fail(FDMD_ERR_CUDA, "householder: device allocation failed");
  if (cusolverDnDgeqrf(h, (int)n, l, A, (int)lda, tau, work, std::max(lw1, lw2), info) != CUSOLVER_STATUS_SUCCESS)
    return fail(FDMD_ERR_SOLVER, "householder: geqrf failed");
  if (R_out) {   // R = upper triangle of the factored block (column-major, ld lda) -> row-major l x l
    std::vector<double> top((size_t)l * l);
    CUDA_TRY(cudaMemcpy2DAsync(top.data(), l * sizeof(double), A, lda * sizeof(double), l * sizeof(double), l,
                               cudaMemcpyDeviceToHost, d.s));
    CUDA_TRY(cudaStreamSynchronize(d.s));
    R_out->assign((size_t)l * l, 0.0);
    for (int j = 0; j < l; ++j)
      for (int i = 0; i <= j; ++i) (*R_out)[(size_t)i * l + j] = top[(size_t)j * l + i];
  }
  if (cusolverDnDorgqr(h, (int)n, l, l, A, (int)lda, tau, work, std::max(lw1, lw2), info) != CUSOLVER_STATUS_SUCCESS)
    return fail(FDMD_ERR_SOLVER, "householder: orgqr failed");
  int ih = 0;
  TRY(d.down(&ih, info, sizeof(int)));
  if (ih != 0) return fail(FDMD_ERR_SOLVER, "householder: info %d", ih);
  TRY(fdmd_tall_gemm(A, FDMD_F64, FDMD_COL, lda, Id, l, Q, FDMD_F64, FDMD_ROW, ldq, n, l, l, 0, nullptr, 0, nullptr, 0,
                     d.s));
  fix.clear();
  return FDMD_OK;
}

struct Sketch {
  double* Q = nullptr;      // device row-major n x l, ld ldq (buffer; Q = buffer @ fix)
  int l = 0;
  int64_t ldq = 0;          // round_up(l, 2): 16-byte rows for the TMA-fed kernels
  std::vector<double> fix;  // l x l (empty = identity)
  std::vector<double> Ub;   // l x l left vectors of B (row-major)
  std::vector<double> s;    // l singular values
  std::vector<double> V;    // T x l right vectors (row-major)
  std::vector<double> QtS;  // l x m = Q^T S over all m columns (fix applied)
};

// The explicit range finder over X = S[:, c0:c0+T] (S: n x m, m >= c0 + T): Y = X Omega
// -> CholeskyQR (one pass while power iterating, CholeskyQR2 at the end, the
// shifted CholeskyQR3 of Fukaya et al. 2020 when the factor is ill-conditioned)
// -> q x {Z = X^T Q -> W = qr(Z) -> Y = X W -> CholeskyQR} -> Q^T S -> svd(Q^T X).
int sketch(Dev& d, const Tall& S, int64_t n, int T, int m, int l, int q, const double* omega_host, Sketch& out,
           int c0 = 0) {
  cudaStream_t s = d.s;
  const int K2max = std::max(m, l);
  const size_t gws = std::max(fdmd_tall_gram_workspace(n, l, l),
                              std::max(fdmd_tall_gram_workspace(n, c0 + T, l), fdmd_tall_gram_workspace(n, l, K2max)));
  const int64_t ldq = round_up(l, 2);
  double* Q = d.alloc<double>((size_t)n * ldq);
  double* Bd = d.alloc<double>((size_t)K2max * 2 * l + 16);
  double* Gd = d.alloc<double>((size_t)K2max * l);
  void* ws = d.alloc<unsigned char>(gws);
  if (!Q || !Bd || !Gd || !ws) return fail(FDMD_ERR_CUDA, "sketch: device allocation failed");
  out.Q = Q;
  out.l = l;
  out.ldq = ldq;
  CUDA_TRY(cudaMemsetAsync(Q, 0, (size_t)n * ldq * sizeof(double), d.s));   // pad column stays zero
  auto gemm = [&](const void* A, int adt, int64_t lda, const std::vector<double>& Bh, int K, int N, int flags) {
    TRY(d.up(Bh.data(), Bd, Bh.size() * sizeof(double)));
    return fdmd_tall_gemm(A, adt, FDMD_ROW, lda, Bd, N, Q, FDMD_F64, FDMD_ROW, ldq, n, K, N, flags, nullptr, 0, nullptr,
                          0, s);
  };
  auto gram = [&](const void* A, int adt, int64_t lda, const void* B, int bdt, int64_t ldb, int K1, int K2, int sym,
                  std::vector<double>& G) {
    TRY(fdmd_tall_gram(A, adt, FDMD_ROW, lda, B, bdt, FDMD_ROW, ldb, Gd, K2, 0.0, n, K1, K2, sym, ws, gws, s));
    G.resize((size_t)K1 * K2);
    return d.down(G.data(), Gd, G.size() * sizeof(double));
  };
  std::vector<double>& fix = out.fix;
  auto cholqr = [&](int passes) -> int {
    std::vector<double> G, R1, R2;
    TRY(gram(Q, FDMD_F64, ldq, Q, FDMD_F64, ldq, l, l, 1, G));
    const bool ok = chol_upper(G, l, R1);
    std::vector<double> R1i;
    double cond = INFINITY;
    if (ok) {
      R1i = inv_upper(R1, l);
      cond = fro(R1) * fro(R1i);
    }
    if (!ok || !(cond <= RSVD_COND_LIMIT)) {
      const double u = 1.1102230246251565e-16;
      const double shift = 11.0 * ((double)n * l + (double)l * (l + 1)) * u * fro(G);
      std::vector<double> Gs = G, R0, R1b;
      for (int i = 0; i < l; ++i) Gs[(size_t)i * l + i] += shift;
      // Householder fallback on Cholesky failure (a rank-deficient sketch), as
      // linalg.cholqr2_deferred: Q orthonormal, no deferred factor
      if (!chol_upper(Gs, l, R0)) return householder(d, Q, ldq, n, l, fix);
      TRY(gemm(Q, FDMD_F64, ldq, inv_upper(R0, l), l, l, FDMD_B_UPPER));
      TRY(gram(Q, FDMD_F64, ldq, Q, FDMD_F64, ldq, l, l, 1, G));
      if (!chol_upper(G, l, R1b)) return householder(d, Q, ldq, n, l, fix);
      TRY(gemm(Q, FDMD_F64, ldq, inv_upper(R1b, l), l, l, FDMD_B_UPPER));
      if (passes == 1) {
        fix.clear();
        return FDMD_OK;
      }
    } else if (passes == 1) {
      fix = R1i;
      return FDMD_OK;
    } else {
      TRY(gemm(Q, FDMD_F64, ldq, R1i, l, l, FDMD_B_UPPER));  // Q <- Y R1^-1
    }
    TRY(gram(Q, FDMD_F64, ldq, Q, FDMD_F64, ldq, l, l, 1, G));
    if (!chol_upper(G, l, R2)) return householder(d, Q, ldq, n, l, fix);
    fix = inv_upper(R2, l);
    return FDMD_OK;
  };
  // a column window c0 > 0 (X' = S[:, 1:]) multiplies S by the small matrix
  // padded with c0 zero rows on top (TMA needs the 16-byte aligned base of S)
  const int Kc = c0 + T;
  auto placed = [&](const std::vector<double>& M) {
    std::vector<double> P((size_t)Kc * l, 0.0);
    std::copy(M.begin(), M.end(), P.begin() + (size_t)c0 * l);
    return P;
  };
  std::vector<double> Om(omega_host, omega_host + (size_t)T * l);
  TRY(gemm(S.p, S.dt, S.ld, placed(Om), Kc, l, 0));  // Y = X Omega
  TRY(cholqr(q == 0 ? 2 : 1));
  for (int it = 0; it < q; ++it) {
    std::vector<double> Zf, Z((size_t)T * l);
    TRY(gram(S.p, S.dt, S.ld, Q, FDMD_F64, ldq, Kc, l, 0, Zf));  // (c0 + T) x l; X^T buffer = its last T rows
    std::copy(Zf.begin() + (size_t)c0 * l, Zf.end(), Z.begin());
    if (!fix.empty()) Z = matmul(Z, fix, T, l, l);
    std::vector<double> W = householder_q(Z, T, l);
    TRY(gemm(S.p, S.dt, S.ld, placed(W), Kc, l, 0));
    TRY(cholqr(it == q - 1 ? 2 : 1));
  }
  // Q^T S (l x m) with Q = buffer fix
  TRY(gram(Q, FDMD_F64, ldq, S.p, S.dt, S.ld, l, m, 0, out.QtS));
  if (!fix.empty()) out.QtS = matmul(transpose(fix, l, l), out.QtS, l, l, m);
  // svd(B), B = Q^T X (l x T) on cuSOLVER gesvd (rows >= cols: factor B^T, T x l)
  cusolverDnHandle_t h = (cusolverDnHandle_t)fdmdi_solver_handle(s);
  if (!h) return fail(FDMD_ERR_SOLVER, "cusolverDnCreate failed");
  std::vector<double> Bt((size_t)T * l);  // column-major T x l = B^T: A[i + j*T] = B[j][i]
  for (int j = 0; j < l; ++j)
    for (int i = 0; i < T; ++i) Bt[i + (size_t)j * T] = out.QtS[(size_t)j * m + c0 + i];
  double* A = d.alloc<double>((size_t)T * l);
  double* Sv = d.alloc<double>(l);
  double* Ua = d.alloc<double>((size_t)T * l);
  double* VTa = d.alloc<double>((size_t)l * l);
  int* info = d.alloc<int>(1);
  if (!A || !Sv || !Ua || !VTa || !info) return fail(FDMD_ERR_CUDA, "sketch: device allocation failed");
  TRY(d.up(Bt.data(), A, Bt.size() * sizeof(double)));
  int lwork = 0;
  if (cusolverDnDgesvd_bufferSize(h, T, l, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return fail(FDMD_ERR_SOLVER, "gesvd_bufferSize");
  double* work = d.alloc<double>((size_t)lwork);
  double* rwork = d.alloc<double>(l);
  if (!work || !rwork) return fail(FDMD_ERR_CUDA, "sketch: device allocation failed");
  if (cusolverDnDgesvd(h, 'S', 'S', T, l, A, T, Sv, Ua, T, VTa, l, work, lwork, rwork, info) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(FDMD_ERR_SOLVER, "gesvd failed");
  int info_h = 0;
  std::vector<double> ua((size_t)T * l), vta((size_t)l * l);
  out.s.resize(l);
  TRY(d.down(&info_h, info, sizeof(int)));
  if (info_h != 0) return fail(FDMD_ERR_SOLVER, "gesvd info %d", info_h);
  TRY(d.down(out.s.data(), Sv, l * sizeof(double)));
  TRY(d.down(ua.data(), Ua, ua.size() * sizeof(double)));
  TRY(d.down(vta.data(), VTa, vta.size() * sizeof(double)));
  // B^T = Ua diag(s) VTa (column-major): left vectors of B Ub[i][k] = VTa(k, i);
  // right vectors V[j][k] = Ua(j, k)
  out.Ub.assign((size_t)l * l, 0.0);
  out.V.assign((size_t)T * l, 0.0);
  for (int i = 0; i < l; ++i)
    for (int k = 0; k < l; ++k) out.Ub[(size_t)i * l + k] = vta[k + (size_t)i * l];
  for (int j = 0; j < T; ++j)
    for (int k = 0; k < l; ++k) out.V[(size_t)j * l + k] = ua[j + (size_t)k * T];
  return FDMD_OK;
}

// l x r matrix fix @ Ub[:, :r] (the lift U = Q_buffer (fix Ub_r), linalg.py:88)
std::vector<double> lift_map(const Sketch& f, int r) {
  const int l = f.l;
  std::vector<double> Ubr((size_t)l * r);
  for (int i = 0; i < l; ++i)
    for (int k = 0; k < r; ++k) Ubr[(size_t)i * r + k] = f.Ub[(size_t)i * l + k];
  return f.fix.empty() ? Ubr : matmul(f.fix, Ubr, l, l, r);
}

}  // namespace

// ============================================================================
// handles
// ============================================================================
struct fdmd_ctx {
  int device = 0;
  std::vector<cudaStream_t> streams;
  std::vector<char> busy;
  std::mutex mu;
  std::condition_variable cv;
};

struct fdmd_mat {
  int device = 0;
  void* p = nullptr;
  int dt = FDMD_F64;
  int64_t n = 0, m = 0, ld = 0;
};

struct fdmd_model {
  int device = 0;
  int64_t n = 0;
  int r = 0, units = 0, dt = FDMD_F64;
  double step_dt = 1.0;
  void* raw = nullptr;            // column-major table: 2*units columns (Re, Im per unit) of n rows, ld ldr
  int64_t ldr = 0;
  std::vector<cd> lam;            // r
  std::vector<double> sigma;      // r
  std::vector<int> unit_of;       // per position a: unit
  std::vector<cd> cre, cim;       // phi[:, a] = cre[a] * raw_re(unit) + cim[a] * raw_im(unit)
  std::vector<double> history;
  int converged = 1;
  std::mutex mu;                  // guards the lazily built pseudo-inverse
  bool have_pinv = false;
  std::vector<cd> pinv;           // r x 2*units: pinv(phi) = pinv @ raw^T (or r x qcols: pinv @ Q^T)
  double* qbuf = nullptr;         // ill-conditioned table: Householder Q (row-major n x ldq) of its columns
  int64_t ldq = 0;
  int qcols = 0;
};

namespace {

struct StreamLease {
  fdmd_ctx* c;
  int idx = -1;
  explicit StreamLease(fdmd_ctx* ctx) : c(ctx) {
    std::unique_lock<std::mutex> lk(c->mu);
    c->cv.wait(lk, [&] {
      for (size_t i = 0; i < c->busy.size(); ++i)
        if (!c->busy[i]) return true;
      return false;
    });
    for (size_t i = 0; i < c->busy.size(); ++i)
      if (!c->busy[i]) {
        c->busy[i] = 1;
        idx = (int)i;
        break;
      }
  }
  ~StreamLease() {
    {
      std::lock_guard<std::mutex> lk(c->mu);
      c->busy[idx] = 0;
    }
    c->cv.notify_one();
  }
  cudaStream_t s() const { return c->streams[idx]; }
};

// The modes pass shared by exact DMD and OptDMD: raw = A @ [0_top; Cs] for
// every computed unit (Re, Im columns) with fused per-unit statistics, then
// the normalisation, phase canonicalisation, pair locking and real-ification
// of _order_and_pair (dmd.py:189-213) folded into per-position coefficients.
int modes_pass(Dev& d, const Tall& A, int64_t n, int K, int top, const CM& Cmap, const PairPlan& plan, int table_dt,
               fdmd_model* model) {
  cudaStream_t s = d.s;
  const int U = (int)plan.src.size();
  const int r = (int)plan.lam.size();
  const int Kc = Cmap.m;
  std::vector<double> Bm((size_t)K * 2 * U, 0.0);
  CM Cs(Kc, U);
  for (int u = 0; u < U; ++u)
    for (int i = 0; i < Kc; ++i) {
      Cs(i, u) = Cmap(i, plan.src[u]);
      Bm[(size_t)(top + i) * 2 * U + 2 * u] = Cs(i, u).real();
      Bm[(size_t)(top + i) * 2 * U + 2 * u + 1] = Cs(i, u).imag();
    }
  const int64_t ldr = round_up(n, 4);
  CUDA_TRY(cudaMalloc(&model->raw, (size_t)ldr * 2 * U * esize(table_dt)));
  model->ldr = ldr;
  model->units = U;
  model->dt = table_dt;
  const size_t wsb = fdmd_tall_gemm_workspace(n, 2 * U);
  double* Bd = d.alloc<double>(Bm.size());
  double* st = d.alloc<double>((size_t)3 * U);
  void* ws = d.alloc<unsigned char>(wsb);
  if (!Bd || !st || !ws) return fail(FDMD_ERR_CUDA, "modes: device allocation failed");
  TRY(d.up(Bm.data(), Bd, Bm.size() * sizeof(double)));
  TRY(fdmd_tall_gemm(A.p, A.dt, FDMD_ROW, A.ld, Bd, 2 * U, model->raw, table_dt, FDMD_COL, ldr, n, K, 2 * U, 0, st, 0,
                     ws, wsb, s));
  std::vector<double> sth((size_t)3 * U);
  TRY(d.down(sth.data(), st, sth.size() * sizeof(double)));
  // pivots: the first largest-|phi| entry of each unit (validated before any read)
  std::vector<cd> sc(U);
  const size_t es = esize(table_dt);
  for (int u = 0; u < U; ++u) {
    const double nrm2 = sth[3 * u], a = sth[3 * u + 2];
    if (!std::isfinite(nrm2) || !std::isfinite(sth[3 * u + 1]) || !std::isfinite(a) || a < 0.0 || a >= (double)n)
      return fail(FDMD_ERR_SOLVER, "modes: non-finite mode statistics");
    const int64_t piv = (int64_t)llround(a);
    double pr = 0, pi = 0;
    if (table_dt == FDMD_F32) {
      float v[2];
      const char* base = (const char*)model->raw;
      CUDA_TRY(cudaMemcpyAsync(&v[0], base + ((size_t)(2 * u) * ldr + piv) * es, es, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaMemcpyAsync(&v[1], base + ((size_t)(2 * u + 1) * ldr + piv) * es, es, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      pr = v[0], pi = v[1];
    } else {
      const double* base = (const double*)model->raw;
      CUDA_TRY(cudaMemcpyAsync(&pr, base + (size_t)(2 * u) * ldr + piv, 8, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaMemcpyAsync(&pi, base + (size_t)(2 * u + 1) * ldr + piv, 8, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    const cd pc(pr, pi);
    const double pab = std::abs(pc);
    const cd phase = pab > 0 ? std::conj(pc) / pab : cd(1.0);
    const double nrm = std::sqrt(nrm2);
    sc[u] = nrm > 0 ? phase / nrm : phase;
  }
  // real-ification of phi for real-ified eigenvalues (dmd.py:208-211):
  // max_i |Im(phi_u s_u)_i| <= 1e-10, measured in one statistics-only pass
  std::set<int> realified;
  std::vector<std::pair<int, std::vector<double>>> check;
  for (int u : plan.realify) {
    std::vector<double> im(Kc);
    bool any = false;
    for (int i = 0; i < Kc; ++i) {
      im[i] = (Cs(i, u) * sc[u]).imag();
      any |= im[i] != 0.0;
    }
    if (!any)
      realified.insert(u);
    else
      check.push_back({u, std::move(im)});
  }
  if (!check.empty()) {
    const int nc = (int)check.size();
    std::vector<double> Bq((size_t)K * 2 * nc, 0.0);
    for (int k = 0; k < nc; ++k)
      for (int i = 0; i < Kc; ++i) Bq[(size_t)(top + i) * 2 * nc + 2 * k] = check[k].second[i];
    const size_t wq = fdmd_tall_gemm_workspace(n, 2 * nc);
    double* Bqd = d.alloc<double>(Bq.size());
    double* stq = d.alloc<double>((size_t)3 * nc);
    void* wsq = d.alloc<unsigned char>(wq);
    if (!Bqd || !stq || !wsq) return fail(FDMD_ERR_CUDA, "modes: device allocation failed");
    TRY(d.up(Bq.data(), Bqd, Bq.size() * sizeof(double)));
    TRY(fdmd_tall_gemm(A.p, A.dt, FDMD_ROW, A.ld, Bqd, 2 * nc, nullptr, FDMD_F64, FDMD_COL, n, n, K, 2 * nc, 0, stq, 0,
                       wsq, wq, s));
    std::vector<double> h((size_t)3 * nc);
    TRY(d.down(h.data(), stq, h.size() * sizeof(double)));
    for (int k = 0; k < nc; ++k)
      if (std::sqrt(h[3 * k + 1]) <= 1e-10) realified.insert(check[k].first);
  }
  model->unit_of.assign(r, 0);
  model->cre.assign(r, 0.0);
  model->cim.assign(r, 0.0);
  for (int a = 0; a < r; ++a) {
    const int u = plan.pos[a].first;
    const bool cj = plan.pos[a].second;
    const cd su = sc[u];
    model->unit_of[a] = u;
    if (realified.count(u)) {  // Re(s (re + i im)) = Re(s) re - Im(s) im
      model->cre[a] = su.real();
      model->cim[a] = -su.imag();
    } else if (!cj) {          // s (re + i im)
      model->cre[a] = su;
      model->cim[a] = cd(0.0, 1.0) * su;
    } else {                   // conj(s (re + i im))
      model->cre[a] = std::conj(su);
      model->cim[a] = cd(0.0, -1.0) * std::conj(su);
    }
  }
  return FDMD_OK;
}

// la._check_eig: unit-norm eigenvectors, residual <= 1e-8 ||M||_F
int eig_checked(Dev& d, const std::vector<double>& K, int r, bool vectors, std::vector<cd>& w, CM& W) {
  std::vector<double> Acm((size_t)r * r);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) Acm[i + (size_t)j * r] = K[(size_t)i * r + j];
  double* Ad = d.alloc<double>(Acm.size());
  if (!Ad) return fail(FDMD_ERR_CUDA, "eig: device allocation failed");
  TRY(d.up(Acm.data(), Ad, Acm.size() * sizeof(double)));
  std::vector<double> wh(2 * (size_t)r), vr(vectors ? (size_t)r * r : 0);
  TRY(fdmd_geev(r, Ad, wh.data(), vectors ? vr.data() : nullptr, d.s));
  w.resize(r);
  for (int j = 0; j < r; ++j) w[j] = cd(wh[2 * j], wh[2 * j + 1]);
  if (!vectors) return FDMD_OK;
  W = CM(r, r);
  for (int j = 0; j < r;) {  // LAPACK packing: a complex pair occupies columns j (Re), j+1 (Im)
    if (w[j].imag() != 0.0 && j + 1 < r) {
      for (int i = 0; i < r; ++i) {
        const double re = vr[i + (size_t)j * r], im = vr[i + (size_t)(j + 1) * r];
        W(i, j) = cd(re, im);
        W(i, j + 1) = cd(re, -im);
      }
      j += 2;
    } else {
      for (int i = 0; i < r; ++i) W(i, j) = vr[i + (size_t)j * r];
      j += 1;
    }
  }
  for (int j = 0; j < r; ++j) {
    double s2 = 0.0;
    for (int i = 0; i < r; ++i) s2 += std::norm(W(i, j));
    const double nr = s2 > 0 ? std::sqrt(s2) : 1.0;
    for (int i = 0; i < r; ++i) W(i, j) /= nr;
  }
  double scale = fro(K), res2 = 0.0;
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      cd acc = 0.0;
      for (int k = 0; k < r; ++k) acc += K[(size_t)i * r + k] * W(k, j);
      res2 += std::norm(acc - W(i, j) * w[j]);
    }
  const double res = std::sqrt(res2);
  if (scale > 0 && res > 1e-8 * scale)
    return fail(FDMD_ERR_SOLVER, "eigendecomposition residual %.3e exceeds 1e-8 * ||M||", res);
  return FDMD_OK;
}

// ---- variable projection (dmd.py:277-363), host complex128 -----------------
struct LMResult {
  std::vector<cd> alpha;
  CM B;
  std::vector<double> history;
  bool converged = false;
};

CM vander(const std::vector<cd>& alpha, int T) {
  CM P(T, (int)alpha.size());
  for (int i = 0; i < T; ++i)
    for (size_t j = 0; j < alpha.size(); ++j) P(i, (int)j) = i == 0 ? cd(1.0) : std::pow(alpha[j], (double)i);
  return P;
}

double min_sep(const std::vector<cd>& a) {
  double m = INFINITY;
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < a.size(); ++j)
      if (i != j) m = std::min(m, std::abs(a[i] - a[j]));
  return m;
}

double objective(const std::vector<cd>& alpha, const CM& D, int T, CM& B, CM& P, CM& R) {
  P = vander(alpha, T);
  B = lstsq_minnorm(P, D);
  CM PB = cmul(P, B);
  R = CM(D.m, D.n);
  for (size_t i = 0; i < D.a.size(); ++i) R.a[i] = D.a[i] - PB.a[i];
  return cfro(R);
}

// returns 1 on collapse (the caller retries with jitter), 0 otherwise
int varpro_lm(const CM& D, const std::vector<cd>& alpha0, int max_iters, LMResult& out) {
  const double init_damping = 1.0, damping_up = 2.0, damping_down = 3.0, rel_tol = 1e-8, collapse_tol = 1e-12;
  const int T = D.m, r = (int)alpha0.size();
  std::vector<cd> alpha = alpha0;
  if (min_sep(alpha) < collapse_tol) return 1;
  CM B, P, R;
  double f = objective(alpha, D, T, B, P, R);
  const double floor = 1e-14 * cfro(D);
  out.history = {f};
  out.converged = false;
  if (max_iters == 0) {
    out.alpha = alpha;
    out.B = B;
    out.converged = true;
    return 0;
  }
  double mu = init_damping;
  for (int it = 0; it < max_iters; ++it) {
    if (f <= floor) {
      out.converged = true;
      break;
    }
    CM Qp, Rp;
    cqr(P, Qp, Rp);
    CM dphi(T, r);
    for (int i = 1; i < T; ++i)
      for (int j = 0; j < r; ++j) dphi(i, j) = (double)i * (i == 1 ? cd(1.0) : std::pow(alpha[j], (double)(i - 1)));
    CM proj = cmul(Qp, cmulH(Qp, dphi));
    CM Wk(T, r);
    for (size_t i = 0; i < Wk.a.size(); ++i) Wk.a[i] = dphi.a[i] - proj.a[i];
    CM WW = cmulH(Wk, Wk);
    CM BBh(r, r);
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < r; ++j) {
        cd acc = 0.0;
        for (int k = 0; k < B.n; ++k) acc += B(i, k) * std::conj(B(j, k));
        BBh(i, j) = acc;
      }
    CM JHJ(r, r);
    for (size_t i = 0; i < JHJ.a.size(); ++i) JHJ.a[i] = WW.a[i] * std::conj(BBh.a[i]);
    // g = diag(Wk^H R B^H): g_j = sum_t conj(Wk[t, j]) (R B^H)[t, j]
    std::vector<cd> g(r, 0.0);
    for (int t = 0; t < T; ++t)
      for (int j = 0; j < r; ++j) {
        cd rb = 0.0;
        for (int k = 0; k < B.n; ++k) rb += R(t, k) * std::conj(B(j, k));
        g[j] += std::conj(Wk(t, j)) * rb;
      }
    CM A = JHJ;
    for (int i = 0; i < r; ++i) A(i, i) += mu;
    std::vector<cd> delta = g;
    if (!csolve(A, delta)) {
      mu *= damping_up;
      continue;
    }
    std::vector<cd> cand(r);
    for (int j = 0; j < r; ++j) cand[j] = alpha[j] + delta[j];
    if (min_sep(cand) < collapse_tol) return 1;
    CM Bn, Pn, Rn;
    const double fn = objective(cand, D, T, Bn, Pn, Rn);
    if (fn < f) {
      const double rel = (f - fn) / std::max(f, 1e-300);
      alpha = cand, f = fn, B = Bn, P = Pn, R = Rn;
      out.history.push_back(f);
      mu /= damping_down;
      if (rel < rel_tol || f <= floor) {
        out.converged = true;
        break;
      }
    } else {
      mu *= damping_up;
    }
  }
  out.alpha = alpha;
  out.B = B;
  return 0;
}

// _symmetrize (dmd.py:439-455)
void symmetrize(std::vector<cd>& alpha, CM& B) {
  std::vector<int> partner = conjugate_pairs(alpha);
  for (int i = 0; i < (int)alpha.size(); ++i) {
    const int j = partner[i];
    if (j > i) {
      const cd a = 0.5 * (alpha[i] + std::conj(alpha[j]));
      alpha[i] = a;
      alpha[j] = std::conj(a);
      for (int k = 0; k < B.n; ++k) {
        const cd row = 0.5 * (B(i, k) + std::conj(B(j, k)));
        B(i, k) = row;
        B(j, k) = std::conj(row);
      }
    } else if (j == i && std::abs(alpha[i].imag()) <= 1e-8 * std::max(std::abs(alpha[i]), 1e-300)) {
      alpha[i] = alpha[i].real();
      for (int k = 0; k < B.n; ++k) B(i, k) = B(i, k).real();
    }
  }
}

void free_model(fdmd_model* m) {
  if (!m) return;
  if (m->raw) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaFree(m->raw);
    if (m->qbuf) cudaFree(m->qbuf);
    cudaSetDevice(prev);
  }
  delete m;
}

// pinv(phi) in raw-table coordinates (r x 2U): from the Hermitian Gram
// phi^H phi = M^H (D^T D) M (one symmetric tall Gram of the raw table); the
// reference's SVD cut sigma > 1e-12 sigma_max (linalg.py:93-104) is applied
// to the Gram's eigenvalues (mu = sigma^2) when the basis is well conditioned.
int ensure_pinv(Dev& d, fdmd_model* m) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->have_pinv) return FDMD_OK;
  const int U = m->units, r = m->r, nc = 2 * U;
  const size_t gws = fdmd_tall_gram_workspace(m->n, nc, nc);
  double* G = d.alloc<double>((size_t)nc * nc);
  void* ws = d.alloc<unsigned char>(gws);
  if (!G || !ws) return fail(FDMD_ERR_CUDA, "pinv: device allocation failed");
  TRY(fdmd_tall_gram(m->raw, m->dt, FDMD_COL, m->ldr, m->raw, m->dt, FDMD_COL, m->ldr, G, nc, 0.0, m->n, nc, nc, 1, ws,
                     gws, d.s));
  std::vector<double> Gh((size_t)nc * nc);
  TRY(d.down(Gh.data(), G, Gh.size() * sizeof(double)));
  CM M(nc, r);
  for (int a = 0; a < r; ++a) {
    M(2 * m->unit_of[a], a) = m->cre[a];
    M(2 * m->unit_of[a] + 1, a) = m->cim[a];
  }
  CM Gc(nc, nc);
  for (size_t i = 0; i < Gh.size(); ++i) Gc.a[i] = Gh[i];
  CM H = cmulH(M, cmul(Gc, M));
  for (int i = 0; i < r; ++i)
    for (int j = i; j < r; ++j) {
      const cd v = 0.5 * (H(i, j) + std::conj(H(j, i)));
      H(i, j) = v;
      H(j, i) = std::conj(v);
    }
  // H is Hermitian PSD: its SVD is its eigendecomposition
  CM Uh, Vh;
  std::vector<double> mu;
  csvd(H, Uh, mu, Vh);
  const double mu_max = mu.empty() ? 0.0 : mu[0];
  const double mu_min = mu.empty() ? 0.0 : mu.back();
  if (!(mu_min > 0) || mu_max / mu_min > 1e12) {
    // The Gram cannot resolve the reference's cut (sigma > 1e-12 sigma_max) for
    // cond(phi) > 1e6: QR of the table instead (modes.DeviceModes.pinv_rows'
    // ill-conditioned branch). phi = D M = D' M' over the nonzero raw columns
    // D' (a real mode's exactly-zero imaginary column carries nothing), D' = Q R
    // by Householder on the device and pinv(phi) = pinv(R M') Q^T: the model keeps
    // Q, and encode projects u onto it directly (Q^T u on the device) — going
    // through R^-T D'^T u instead would square cond(D').
    std::vector<int> keep;
    for (int k = 0; k < nc; ++k)
      if (Gh[(size_t)k * nc + k] > 0.0) keep.push_back(k);
    const int kc = (int)keep.size();
    if (kc == 0) return fail(FDMD_ERR_SOLVER, "pinv: empty mode table");
    const int64_t ldy = round_up(kc, 2);
    std::vector<double> Isel((size_t)nc * kc, 0.0);
    for (int j = 0; j < kc; ++j) Isel[(size_t)keep[j] * kc + j] = 1.0;
    double* Id = d.alloc<double>(Isel.size());
    double* Y = nullptr;
    if (!Id || cudaMalloc(&Y, (size_t)m->n * ldy * sizeof(double)) != cudaSuccess)
      return fail(FDMD_ERR_CUDA, "pinv: device allocation failed (QR route)");
    auto drop = [&](int rc) { cudaFree(Y); return rc; };
    if (int rc = d.up(Isel.data(), Id, Isel.size() * sizeof(double))) return drop(rc);
    if (int rc = fdmd_tall_gemm(m->raw, m->dt, FDMD_COL, m->ldr, Id, kc, Y, FDMD_F64, FDMD_ROW, ldy, m->n, nc, kc, 0,
                                nullptr, 0, nullptr, 0, d.s))
      return drop(rc);
    std::vector<double> fix, R;
    if (int rc = householder(d, Y, ldy, m->n, kc, fix, &R)) return drop(rc);
    if (cudaStreamSynchronize(d.s) != cudaSuccess) return drop(fail(FDMD_ERR_CUDA, "pinv: QR route"));
    auto pinv_small = [](const CM& A) {   // SVD pseudo-inverse, cut 1e-12 sigma_max (linalg.py:93-104)
      CM U, V;
      std::vector<double> sv;
      const bool tall = A.m >= A.n;
      CM B = A;
      if (!tall) {
        B = CM(A.n, A.m);
        for (int i = 0; i < A.m; ++i)
          for (int j = 0; j < A.n; ++j) B(j, i) = std::conj(A(i, j));
      }
      csvd(B, U, sv, V);               // B = U s V^H
      CM P(B.n, B.m);                  // pinv(B) = V s^-1 U^H
      for (int i = 0; i < B.n; ++i)
        for (int j = 0; j < B.m; ++j) {
          cd acc = 0.0;
          for (int k = 0; k < (int)sv.size(); ++k)
            if (sv[0] > 0 && sv[k] > 1e-12 * sv[0]) acc += V(i, k) * std::conj(U(j, k)) / sv[k];
          P(i, j) = acc;
        }
      if (tall) return P;
      CM Pt(P.n, P.m);                 // pinv(A) = pinv(A^H)^H
      for (int i = 0; i < P.m; ++i)
        for (int j = 0; j < P.n; ++j) Pt(j, i) = std::conj(P(i, j));
      return Pt;
    };
    CM RM(kc, r);
    for (int i = 0; i < kc; ++i)
      for (int a = 0; a < r; ++a) {
        cd acc = 0.0;
        for (int k = i; k < kc; ++k) acc += R[(size_t)i * kc + k] * M(keep[k], a);
        RM(i, a) = acc;
      }
    const CM P1 = pinv_small(RM);      // r x kc: pinv(phi) u = P1 (Q^T u)
    m->pinv = P1.a;
    m->qbuf = Y;
    m->ldq = ldy;
    m->qcols = kc;
    m->have_pinv = true;
    return FDMD_OK;
  }
  CM P(r, r);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) {
      cd acc = 0.0;
      for (int k = 0; k < r; ++k)
        if (mu[k] > 1e-14 * mu_max) acc += Uh(i, k) * std::conj(Uh(j, k)) / mu[k];
      P(i, j) = acc;
    }
  // pinv(phi) u = P phi^H u = P M^H (D^T u)
  CM Mh(r, nc);
  for (int i = 0; i < nc; ++i)
    for (int a = 0; a < r; ++a) Mh(a, i) = std::conj(M(i, a));
  CM PM = cmul(P, Mh);
  m->pinv = PM.a;
  m->have_pinv = true;
  return FDMD_OK;
}

int set_device(int dev) {
  CUDA_TRY(cudaSetDevice(dev));
  return FDMD_OK;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- fdmd_rsvd
int fdmd_rsvd(const void* X, int x_dtype, int64_t ldx, int64_t n, int T, int r, int l, int q, const double* omega_host,
              double* sigma_host, double* V_host, double* U, int64_t ldu, void* stream) {
  if (n < 1 || T < 1 || r < 1 || r > std::min<int64_t>(n, T))
    return fail(FDMD_ERR_INVALID, "rank r=%d must satisfy 1 <= r <= min(n, T) = %lld", r,
                (long long)std::min<int64_t>(n, T));
  if (!X || !omega_host || !sigma_host || !V_host || !U) return fail(FDMD_ERR_INVALID, "rsvd: null argument");
  if (x_dtype != FDMD_F32 && x_dtype != FDMD_F64) return fail(FDMD_ERR_INVALID, "rsvd: bad x_dtype");
  if (l < r || l > T || l > 256 || ldx < T || ldu < n || q < 0)
    return fail(FDMD_ERR_INVALID, "rsvd: need r <= l <= min(T, 256), ldx >= T, ldu >= n, q >= 0");
  Dev d((cudaStream_t)stream);
  d.trim = true;
  Sketch f;
  TRY(sketch(d, Tall{X, x_dtype, ldx}, n, T, T, l, q, omega_host, f));
  std::vector<double> M = lift_map(f, r);  // l x r
  std::vector<double> Vr((size_t)T * r);
  for (int j = 0; j < T; ++j)
    for (int k = 0; k < r; ++k) Vr[(size_t)j * r + k] = f.V[(size_t)j * l + k];
  // canonical signs (linalg.py:29-44): the first largest-|U| entry of each column positive
  std::vector<double> Mp((size_t)l * 2 * r, 0.0);
  for (int i = 0; i < l; ++i)
    for (int k = 0; k < r; ++k) Mp[(size_t)i * 2 * r + 2 * k] = M[(size_t)i * r + k];
  double* Bd = d.alloc<double>(Mp.size());
  double* st = d.alloc<double>((size_t)3 * r);
  const size_t sws_b = fdmd_tall_gemm_workspace(n, 2 * r);
  void* sws = d.alloc<unsigned char>(sws_b);
  if (!Bd || !st || !sws) return fail(FDMD_ERR_CUDA, "rsvd: device allocation failed");
  TRY(d.up(Mp.data(), Bd, Mp.size() * sizeof(double)));
  TRY(fdmd_tall_gemm(f.Q, FDMD_F64, FDMD_ROW, f.ldq, Bd, 2 * r, nullptr, FDMD_F64, FDMD_COL, n, n, l, 2 * r, 0, st, 0, sws,
                     sws_b, d.s));
  std::vector<double> sth((size_t)3 * r);
  TRY(d.down(sth.data(), st, sth.size() * sizeof(double)));
  std::vector<double> rows((size_t)r * l);
  for (int k = 0; k < r; ++k) {
    const double a = sth[(size_t)3 * k + 2];
    if (!std::isfinite(sth[(size_t)3 * k]) || !std::isfinite(sth[(size_t)3 * k + 1]) || !std::isfinite(a) || a < 0.0 ||
        a >= (double)n)
      return fail(FDMD_ERR_SOLVER, "randomized SVD: non-finite basis (degenerate sketch)");
    const int64_t piv = (int64_t)llround(a);
    CUDA_TRY(cudaMemcpyAsync(rows.data() + (size_t)k * l, f.Q + piv * f.ldq, sizeof(double) * l, cudaMemcpyDeviceToHost,
                             d.s));
  }
  CUDA_TRY(cudaStreamSynchronize(d.s));
  for (int k = 0; k < r; ++k) {
    const double* row = rows.data() + (size_t)k * l;
    double v = 0.0;
    for (int i = 0; i < l; ++i) v += row[i] * M[(size_t)i * r + k];
    if (v < 0) {
      for (int i = 0; i < l; ++i) M[(size_t)i * r + k] = -M[(size_t)i * r + k];
      for (int j = 0; j < T; ++j) Vr[(size_t)j * r + k] = -Vr[(size_t)j * r + k];
    }
  }
  TRY(d.up(M.data(), Bd, M.size() * sizeof(double)));
  TRY(fdmd_tall_gemm(f.Q, FDMD_F64, FDMD_ROW, f.ldq, Bd, r, U, FDMD_F64, FDMD_COL, ldu, n, l, r, 0, nullptr, 0, nullptr, 0,
                     d.s));  // lift (linalg.py:88)
  std::copy(f.s.begin(), f.s.begin() + r, sigma_host);
  std::copy(Vr.begin(), Vr.end(), V_host);
  CUDA_TRY(cudaStreamSynchronize(d.s));
  return FDMD_OK;
}

// ---------------------------------------------------------------- handles
int fdmd_ctx_create(int device, int n_streams, fdmd_ctx** out) {
  if (!out || n_streams < 1 || n_streams > 64) return fail(FDMD_ERR_INVALID, "ctx_create: 1 <= n_streams <= 64");
  *out = nullptr;
  int count = 0;
  CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(FDMD_ERR_INVALID, "ctx_create: no CUDA device %d", device);
  TRY(set_device(device));
  fdmd_ctx* c = new fdmd_ctx();
  c->device = device;
  for (int i = 0; i < n_streams; ++i) {
    cudaStream_t s;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      for (cudaStream_t t : c->streams) cudaStreamDestroy(t);
      delete c;
      return fail(FDMD_ERR_CUDA, "ctx_create: cudaStreamCreate failed");
    }
    c->streams.push_back(s);
  }
  c->busy.assign(n_streams, 0);
  *out = c;
  return FDMD_OK;
}

int fdmd_ctx_destroy(fdmd_ctx* ctx) {
  if (!ctx) return FDMD_OK;
  cudaSetDevice(ctx->device);
  for (cudaStream_t s : ctx->streams) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  delete ctx;
  return FDMD_OK;
}

int fdmd_mat_upload(fdmd_ctx* ctx, const void* host, int dtype, int64_t n, int64_t m, int64_t ld_host,
                    fdmd_mat** out) {
  if (!ctx || !host || !out) return fail(FDMD_ERR_INVALID, "mat_upload: null argument");
  *out = nullptr;
  if (dtype != FDMD_F32 && dtype != FDMD_F64) return fail(FDMD_ERR_INVALID, "mat_upload: bad dtype");
  // SnapshotMatrix validation (dmd.py:26-50)
  if (n < 1 || m < 2) return fail(FDMD_ERR_INVALID, "states must be a 2-D array with at least 2 columns");
  if (ld_host < m) return fail(FDMD_ERR_INVALID, "mat_upload: ld_host < m");
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m; ++j) {
      const double v = dtype == FDMD_F32 ? (double)((const float*)host)[i * ld_host + j]
                                         : ((const double*)host)[i * ld_host + j];
      if (!std::isfinite(v)) return fail(FDMD_ERR_INVALID, "states contain non-finite values");
    }
  TRY(set_device(ctx->device));
  StreamLease lease(ctx);
  fdmd_mat* M = new fdmd_mat();
  M->device = ctx->device;
  M->dt = dtype;
  M->n = n;
  M->m = m;
  M->ld = round_up(m, (int64_t)(16 / esize(dtype)));
  const size_t es = esize(dtype);
  if (cudaMalloc(&M->p, (size_t)n * M->ld * es) != cudaSuccess) {
    const long long ld = (long long)M->ld;
    delete M;
    return fail(FDMD_ERR_CUDA, "mat_upload: cudaMalloc of %lld x %lld failed", (long long)n, ld);
  }
  cudaError_t e = cudaMemsetAsync(M->p, 0, (size_t)n * M->ld * es, lease.s());
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(M->p, M->ld * es, host, ld_host * es, m * es, n, cudaMemcpyHostToDevice, lease.s());
  if (e == cudaSuccess) e = cudaStreamSynchronize(lease.s());
  if (e != cudaSuccess) {
    cudaFree(M->p);
    delete M;
    return fail(FDMD_ERR_CUDA, "mat_upload: %s", cudaGetErrorString(e));
  }
  *out = M;
  return FDMD_OK;
}

int fdmd_mat_free(fdmd_mat* mat) {
  if (!mat) return FDMD_OK;
  cudaSetDevice(mat->device);
  cudaFree(mat->p);
  delete mat;
  return FDMD_OK;
}

// ---------------------------------------------------------------- fits
int fdmd_dmd_fit(fdmd_ctx* ctx, const fdmd_mat* states, double dt, int r, int l, int q, const double* omega_host,
                 int method, int lm_max_iters, const double* init_lam_host, const double* jitter_host,
                 double* sigma_host, double* lam_host, fdmd_model** out) {
  if (!ctx || !states || !omega_host || !out) return fail(FDMD_ERR_INVALID, "dmd_fit: null argument");
  *out = nullptr;
  if (!(dt > 0) || !std::isfinite(dt)) return fail(FDMD_ERR_INVALID, "dt must be positive");
  if (method != FDMD_METHOD_EXACT && method != FDMD_METHOD_OPT) return fail(FDMD_ERR_INVALID, "dmd_fit: bad method");
  const int64_t n = states->n;
  const int m = (int)states->m, T = m - 1;
  if (r < 1 || r > std::min<int64_t>(n, T))
    return fail(FDMD_ERR_INVALID, "rank %d out of range [1, %lld]", r, (long long)std::min<int64_t>(n, T));
  if (l < r || l > T || l > 256 || q < 0)
    return fail(FDMD_ERR_INVALID, "dmd_fit: need r <= l <= min(T, 256) and q >= 0");
  if (method == FDMD_METHOD_OPT && lm_max_iters < 0) return fail(FDMD_ERR_INVALID, "dmd_fit: lm_max_iters < 0");
  TRY(set_device(ctx->device));
  StreamLease lease(ctx);
  Dev d(lease.s());
  d.trim = true;
  const Tall S{states->p, states->dt, states->ld};
  Sketch f;
  TRY(sketch(d, S, n, T, m, l, q, omega_host, f));
  // _check_sigma (dmd.py:225-230)
  if (f.s[r - 1] <= 1e-14 * f.s[0])
    return fail(FDMD_ERR_INVALID,
                "requested rank hits numerically zero singular value (sigma_r / sigma_1 = %.3e); lower the rank",
                f.s[r - 1] / f.s[0]);
  // U^T S = Ub_r^T (Q^T S); V S^-1; K = U^T X' V S^-1 (dmd.py:255-256)
  std::vector<double> UtS((size_t)r * m, 0.0);
  for (int k = 0; k < r; ++k)
    for (int i = 0; i < l; ++i) {
      const double u = f.Ub[(size_t)i * l + k];
      for (int j = 0; j < m; ++j) UtS[(size_t)k * m + j] += u * f.QtS[(size_t)i * m + j];
    }
  std::vector<double> VS((size_t)T * r);
  for (int j = 0; j < T; ++j)
    for (int k = 0; k < r; ++k) VS[(size_t)j * r + k] = f.V[(size_t)j * l + k] / f.s[k];
  std::vector<double> Kh((size_t)r * r, 0.0);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < T; ++j) {
      const double u = UtS[(size_t)i * m + 1 + j];
      for (int k = 0; k < r; ++k) Kh[(size_t)i * r + k] += u * VS[(size_t)j * r + k];
    }
  fdmd_model* model = new fdmd_model();
  model->device = ctx->device;
  model->n = n;
  model->r = r;
  model->step_dt = dt;
  model->sigma.assign(f.s.begin(), f.s.begin() + r);
  int rc = FDMD_OK;
  if (method == FDMD_METHOD_EXACT) {
    std::vector<cd> w;
    CM W;
    rc = eig_checked(d, Kh, r, true, w, W);
    if (rc == FDMD_OK) {
      PairPlan plan = pair_plan(w);
      // phi = X' (V/S) W = S [0; (V/S) W]  (dmd.py:255, 258)
      CM Cmap(T, r);
      for (int j = 0; j < T; ++j)
        for (int c = 0; c < r; ++c) {
          cd acc = 0.0;
          for (int k = 0; k < r; ++k) acc += VS[(size_t)j * r + k] * W(k, c);
          Cmap(j, c) = acc;
        }
      model->lam = plan.lam;
      rc = modes_pass(d, S, n, m, 1, Cmap, plan, states->dt, model);
    }
  } else {
    // D = conj(V) S (dmd.py:384); alpha0 = the exact-DMD eigenvalues (dmd.py:387)
    CM Dm(T, r);
    for (int j = 0; j < T; ++j)
      for (int k = 0; k < r; ++k) Dm(j, k) = f.V[(size_t)j * l + k] * f.s[k];
    std::vector<cd> alpha0(r);
    if (init_lam_host) {
      for (int k = 0; k < r; ++k) alpha0[k] = cd(init_lam_host[2 * k], init_lam_host[2 * k + 1]);
    } else {
      std::vector<cd> w;
      CM W;
      rc = eig_checked(d, Kh, r, false, w, W);
      if (rc == FDMD_OK) alpha0 = pair_plan(w).lam;
    }
    LMResult lm;
    if (rc == FDMD_OK && varpro_lm(Dm, alpha0, lm_max_iters, lm) == 1) {
      if (!jitter_host) {
        rc = fail(FDMD_ERR_SOLVER, "eigenvalue iterates collapsed below separation tolerance (no jitter given)");
      } else {
        // alpha0 + 1e-10 (1 + |alpha0|) exp(2 pi i u), u = default_rng(seed).random(r) (dmd.py:394-399)
        std::vector<cd> a1(r);
        for (int k = 0; k < r; ++k)
          a1[k] = alpha0[k] + 1e-10 * (1.0 + std::abs(alpha0[k])) * std::exp(cd(0.0, 2.0 * M_PI * jitter_host[k]));
        if (varpro_lm(Dm, a1, lm_max_iters, lm) == 1)
          rc = fail(FDMD_ERR_SOLVER, "eigenvalue iterates collapsed below separation tolerance twice");
      }
    }
    if (rc == FDMD_OK) {
      std::vector<cd> as = lm.alpha;
      CM Bs = lm.B;
      symmetrize(as, Bs);
      CM P = vander(as, T), PB = cmul(P, Bs), Rs(T, r);
      for (size_t i = 0; i < Rs.a.size(); ++i) Rs.a[i] = Dm.a[i] - PB.a[i];
      const double f_sym = cfro(Rs);
      std::vector<cd> alpha = lm.alpha;
      CM B = lm.B;
      if (f_sym <= lm.history.back() * (1 + 1e-9) && f_sym <= lm.history.front() * (1 + 1e-12)) {
        alpha = as;
        B = Bs;
      }
      PairPlan plan = pair_plan(alpha);
      // phi = U B^T (dmd.py:414) with U = Q_buffer (fix Ub_r): modes straight from Q
      std::vector<double> L = lift_map(f, r);  // l x r
      CM Cmap(l, r);
      for (int i = 0; i < l; ++i)
        for (int c = 0; c < r; ++c) {
          cd acc = 0.0;
          for (int k = 0; k < r; ++k) acc += L[(size_t)i * r + k] * B(c, k);
          Cmap(i, c) = acc;
        }
      model->lam = plan.lam;
      model->history = lm.history;
      model->converged = lm.converged ? 1 : 0;
      rc = modes_pass(d, Tall{f.Q, FDMD_F64, f.ldq}, n, l, 0, Cmap, plan, states->dt, model);
    }
  }
  if (rc != FDMD_OK) {
    free_model(model);
    return rc;
  }
  if (sigma_host) std::copy(model->sigma.begin(), model->sigma.end(), sigma_host);
  if (lam_host)
    for (int k = 0; k < r; ++k) lam_host[2 * k] = model->lam[k].real(), lam_host[2 * k + 1] = model->lam[k].imag();
  *out = model;
  return FDMD_OK;
}

// Augmented DMDc (Proctor et al. 2016; SURVEY §8(c) "C2 restatement"; the
// package's dmd.dmdc_fit): rank-r_aug sketch of [X; Upsilon], output basis
// U_hat = a rank-r sketch of X' (seed + 1), A~ = U_hat^T X' V S^-1 U1^T U_hat,
// B~ = U_hat^T X' V S^-1 U2^T, phi = X' V S^-1 U1^T U_hat W and the modal
// control matrix reduced_b = pinv(phi) U_hat B~ / dt (runtime.step_forced
// multiplies by dt, runtime.py:188).
int fdmd_dmdc_fit(fdmd_ctx* ctx, const fdmd_mat* states, const double* controls_host, int ell, double dt, int r_aug,
                  int l_aug, int r, int l, int q, const double* omega_aug_host, const double* omega_out_host,
                  double* sigma_aug_host, double* lam_host, double* reduced_b_host, fdmd_model** out) {
  if (!ctx || !states || !controls_host || !omega_aug_host || !omega_out_host || !out)
    return fail(FDMD_ERR_INVALID, "dmdc_fit: null argument");
  *out = nullptr;
  if (!(dt > 0) || !std::isfinite(dt)) return fail(FDMD_ERR_INVALID, "dt must be positive");
  const int64_t n = states->n;
  const int m = (int)states->m, T = m - 1;
  if (ell < 1) return fail(FDMD_ERR_INVALID, "controls must be ell x %d with ell >= 1", T);
  if (r_aug < 1 || r_aug > std::min<int64_t>(n + ell, T) || l_aug < r_aug || l_aug > T || l_aug > 256)
    return fail(FDMD_ERR_INVALID, "dmdc_fit: need 1 <= r_aug <= l_aug <= min(T, 256)");
  if (r < 1 || r > r_aug || r > std::min<int64_t>(n, T) || l < r || l > T || l > 256 || q < 0)
    return fail(FDMD_ERR_INVALID, "dmdc_fit: need 1 <= r <= min(r_aug, l), l <= min(T, 256), q >= 0");
  for (size_t i = 0; i < (size_t)ell * T; ++i)
    if (!std::isfinite(controls_host[i])) return fail(FDMD_ERR_INVALID, "controls contain non-finite values");
  TRY(set_device(ctx->device));
  StreamLease lease(ctx);
  Dev d(lease.s());
  d.trim = true;
  const size_t es = esize(states->dt);
  const int64_t ld = states->ld;
  // [S; Upsilon | 0]: the ell control rows below the n state rows
  void* aug = d.alloc<unsigned char>((size_t)(n + ell) * ld * es);
  if (!aug) return fail(FDMD_ERR_CUDA, "dmdc_fit: device allocation failed");
  CUDA_TRY(cudaMemcpyAsync(aug, states->p, (size_t)n * ld * es, cudaMemcpyDeviceToDevice, d.s));
  std::vector<unsigned char> tail((size_t)ell * ld * es, 0);
  for (int c = 0; c < ell; ++c)
    for (int j = 0; j < T; ++j) {
      const double v = controls_host[(size_t)c * T + j];
      if (states->dt == FDMD_F32)
        reinterpret_cast<float*>(tail.data())[(size_t)c * ld + j] = (float)v;
      else
        reinterpret_cast<double*>(tail.data())[(size_t)c * ld + j] = v;
    }
  TRY(d.up(tail.data(), (char*)aug + (size_t)n * ld * es, tail.size()));
  const Tall S{states->p, states->dt, ld};
  Sketch f1, f2;
  TRY(sketch(d, Tall{aug, states->dt, ld}, n + ell, T, m, l_aug, q, omega_aug_host, f1));
  TRY(sketch(d, S, n, T, m, l, q, omega_out_host, f2, 1));
  // U1^T U_hat = Ub1^T (Q1[:n]^T Q2) Ub2 with Q = buffer @ fix
  const size_t gws = std::max(fdmd_tall_gram_workspace(n, l_aug, l), fdmd_tall_gram_workspace(n, 2 * r + 2, l));
  double* Gd = d.alloc<double>((size_t)std::max(l_aug, 2 * r + 2) * l);
  void* ws = d.alloc<unsigned char>(gws);
  if (!Gd || !ws) return fail(FDMD_ERR_CUDA, "dmdc_fit: device allocation failed");
  TRY(fdmd_tall_gram(f1.Q, FDMD_F64, FDMD_ROW, f1.ldq, f2.Q, FDMD_F64, FDMD_ROW, f2.ldq, Gd, l, 0.0, n, l_aug, l, 0, ws, gws,
                     d.s));
  std::vector<double> M12((size_t)l_aug * l);
  TRY(d.down(M12.data(), Gd, M12.size() * sizeof(double)));
  if (!f1.fix.empty()) M12 = matmul(transpose(f1.fix, l_aug, l_aug), M12, l_aug, l_aug, l);
  if (!f2.fix.empty()) M12 = matmul(M12, f2.fix, l_aug, l, l);
  std::vector<double> Ub1((size_t)l_aug * r_aug), Ub2((size_t)l * r);
  for (int i = 0; i < l_aug; ++i)
    for (int k = 0; k < r_aug; ++k) Ub1[(size_t)i * r_aug + k] = f1.Ub[(size_t)i * l_aug + k];
  for (int i = 0; i < l; ++i)
    for (int k = 0; k < r; ++k) Ub2[(size_t)i * r + k] = f2.Ub[(size_t)i * l + k];
  std::vector<double> U1tUh = matmul(transpose(Ub1, l_aug, r_aug), matmul(M12, Ub2, l_aug, l, r), r_aug, l_aug, r);
  // control rows of U1: Q1[n:n+ell] (fix1 Ub1)
  std::vector<double> qrows((size_t)ell * l_aug);
  for (int c = 0; c < ell; ++c)
    CUDA_TRY(cudaMemcpyAsync(qrows.data() + (size_t)c * l_aug, f1.Q + (size_t)(n + c) * f1.ldq, l_aug * sizeof(double),
                             cudaMemcpyDeviceToHost, d.s));
  CUDA_TRY(cudaStreamSynchronize(d.s));
  const std::vector<double> R1 = lift_map(f1, r_aug);                       // l_aug x r_aug
  const std::vector<double> U2 = matmul(qrows, R1, ell, l_aug, r_aug);     // ell x r_aug
  // U_hat^T X' = Ub2^T (Q2^T S)[:, 1:]; core = U_hat^T X' V1 S1^-1
  std::vector<double> VS((size_t)T * r_aug);
  for (int j = 0; j < T; ++j)
    for (int k = 0; k < r_aug; ++k) VS[(size_t)j * r_aug + k] = f1.V[(size_t)j * l_aug + k] / f1.s[k];
  std::vector<double> UhtXp((size_t)r * T, 0.0);
  for (int k = 0; k < r; ++k)
    for (int i = 0; i < l; ++i) {
      const double u = f2.Ub[(size_t)i * l + k];
      for (int j = 0; j < T; ++j) UhtXp[(size_t)k * T + j] += u * f2.QtS[(size_t)i * m + 1 + j];
    }
  const std::vector<double> core = matmul(UhtXp, VS, r, T, r_aug);          // r x r_aug
  const std::vector<double> Atil = matmul(core, U1tUh, r, r_aug, r);        // r x r
  const std::vector<double> Btil = matmul(core, transpose(U2, ell, r_aug), r, r_aug, ell);   // r x ell
  fdmd_model* model = new fdmd_model();
  model->device = ctx->device;
  model->n = n;
  model->r = r;
  model->step_dt = dt;
  model->sigma.assign(f1.s.begin(), f1.s.begin() + r);
  std::vector<cd> w;
  CM W;
  int rc = eig_checked(d, Atil, r, true, w, W);
  PairPlan plan;
  if (rc == FDMD_OK) {
    plan = pair_plan(w);
    const std::vector<double> VU = matmul(VS, U1tUh, T, r_aug, r);          // T x r
    CM Cmap(T, r);
    for (int j = 0; j < T; ++j)
      for (int c = 0; c < r; ++c) {
        cd acc = 0.0;
        for (int k = 0; k < r; ++k) acc += VU[(size_t)j * r + k] * W(k, c);
        Cmap(j, c) = acc;
      }
    model->lam = plan.lam;
    rc = modes_pass(d, S, n, m, 1, Cmap, plan, states->dt, model);
  }
  std::vector<cd> red((size_t)r * ell, 0.0);
  if (rc == FDMD_OK) rc = ensure_pinv(d, model);
  if (rc == FDMD_OK) {
    // reduced_b = pinv(phi) U_hat B~ / dt with pinv(phi) = P D^T: y = (D^T Q2) (fix2 Ub2) B~
    // (ill-conditioned table: pinv(phi) = P Q^T with the table's Householder Q)
    const int nc = model->qbuf ? model->qcols : 2 * model->units;
    rc = model->qbuf ? fdmd_tall_gram(model->qbuf, FDMD_F64, FDMD_ROW, model->ldq, f2.Q, FDMD_F64, FDMD_ROW, f2.ldq, Gd,
                                      l, 0.0, n, nc, l, 0, ws, gws, d.s)
                     : fdmd_tall_gram(model->raw, model->dt, FDMD_COL, model->ldr, f2.Q, FDMD_F64, FDMD_ROW, f2.ldq, Gd,
                                      l, 0.0, n, nc, l, 0, ws, gws, d.s);
    std::vector<double> DtQ2((size_t)nc * l);
    if (rc == FDMD_OK) rc = d.down(DtQ2.data(), Gd, DtQ2.size() * sizeof(double));
    if (rc == FDMD_OK) {
      const std::vector<double> y = matmul(matmul(DtQ2, lift_map(f2, r), nc, l, r), Btil, nc, r, ell);   // nc x ell
      for (int a = 0; a < r; ++a)
        for (int c = 0; c < ell; ++c) {
          cd acc = 0.0;
          for (int k = 0; k < nc; ++k) acc += model->pinv[(size_t)a * nc + k] * y[(size_t)k * ell + c];
          red[(size_t)a * ell + c] = acc / dt;
        }
    }
  }
  if (rc != FDMD_OK) {
    free_model(model);
    return rc;
  }
  if (sigma_aug_host) std::copy(f1.s.begin(), f1.s.begin() + r_aug, sigma_aug_host);
  if (lam_host)
    for (int k = 0; k < r; ++k) lam_host[2 * k] = model->lam[k].real(), lam_host[2 * k + 1] = model->lam[k].imag();
  if (reduced_b_host)
    for (size_t i = 0; i < red.size(); ++i) reduced_b_host[2 * i] = red[i].real(), reduced_b_host[2 * i + 1] = red[i].imag();
  *out = model;
  return FDMD_OK;
}

int fdmd_model_info(const fdmd_model* model, int64_t* n, int* r, double* dt, int* converged) {
  if (!model) return fail(FDMD_ERR_INVALID, "model_info: null model");
  if (n) *n = model->n;
  if (r) *r = model->r;
  if (dt) *dt = model->step_dt;
  if (converged) *converged = model->converged;
  return FDMD_OK;
}

int fdmd_model_history(const fdmd_model* model, double* out, int cap) {
  if (!model) return fail(FDMD_ERR_INVALID, "model_history: null model");
  const int k = (int)model->history.size();
  if (out)
    for (int i = 0; i < std::min(k, cap); ++i) out[i] = model->history[i];
  return k;
}

int fdmd_model_phi_to_host(fdmd_ctx* ctx, const fdmd_model* model, int64_t row0, int64_t rows, double* out_c128) {
  if (!ctx || !model || !out_c128) return fail(FDMD_ERR_INVALID, "phi_to_host: null argument");
  if (row0 < 0 || rows < 0 || row0 + rows > model->n) return fail(FDMD_ERR_INVALID, "phi_to_host: rows out of range");
  if (rows == 0) return FDMD_OK;
  TRY(set_device(model->device));
  StreamLease lease(ctx);
  const int nc = 2 * model->units, r = model->r;
  const size_t es = esize(model->dt);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)(64 << 20) / (nc * es)));
  std::vector<unsigned char> buf((size_t)nc * chunk * es);
  for (int64_t c0 = 0; c0 < rows; c0 += chunk) {
    const int64_t cr = std::min(chunk, rows - c0);
    CUDA_TRY(cudaMemcpy2DAsync(buf.data(), cr * es, (const char*)model->raw + (size_t)(row0 + c0) * es,
                               model->ldr * es, cr * es, nc, cudaMemcpyDeviceToHost, lease.s()));
    CUDA_TRY(cudaStreamSynchronize(lease.s()));
    for (int64_t i = 0; i < cr; ++i) {
      double* o = out_c128 + (size_t)(c0 + i) * 2 * r;
      for (int a = 0; a < r; ++a) {
        const int u = model->unit_of[a];
        double re, im;
        if (model->dt == FDMD_F32) {
          re = ((const float*)buf.data())[(size_t)(2 * u) * cr + i];
          im = ((const float*)buf.data())[(size_t)(2 * u + 1) * cr + i];
        } else {
          re = ((const double*)buf.data())[(size_t)(2 * u) * cr + i];
          im = ((const double*)buf.data())[(size_t)(2 * u + 1) * cr + i];
        }
        const cd v = model->cre[a] * re + model->cim[a] * im;
        o[2 * a] = v.real();
        o[2 * a + 1] = v.imag();
      }
    }
  }
  return FDMD_OK;
}

int fdmd_encode(fdmd_ctx* ctx, const fdmd_model* cmodel, const double* u_host, double* z_host) {
  if (!ctx || !cmodel || !u_host || !z_host) return fail(FDMD_ERR_INVALID, "encode: null argument");
  fdmd_model* model = const_cast<fdmd_model*>(cmodel);  // the pseudo-inverse cache is internal state
  TRY(set_device(model->device));
  StreamLease lease(ctx);
  Dev d(lease.s());
  TRY(ensure_pinv(d, model));
  const int nc = 2 * model->units, r = model->r;
  const int64_t n = model->n;
  double* u = d.alloc<double>((size_t)n);
  double* y = d.alloc<double>((size_t)nc);
  const size_t wsb = fdmd_colmajor_dot_workspace(n, nc, 1);
  void* ws = d.alloc<unsigned char>(wsb);
  if (!u || !y || !ws) return fail(FDMD_ERR_CUDA, "encode: device allocation failed");
  TRY(d.up(u_host, u, (size_t)n * sizeof(double)));
  int ny = nc;
  if (model->qbuf) {   // ill-conditioned table: y = Q^T u (fdmd_tall_gram, K2 = 1)
    ny = model->qcols;
    const size_t gws = fdmd_tall_gram_workspace(n, ny, 1);
    void* gw = d.alloc<unsigned char>(gws);
    double* yq = d.alloc<double>((size_t)ny);
    if (!gw || !yq) return fail(FDMD_ERR_CUDA, "encode: device allocation failed");
    TRY(fdmd_tall_gram(model->qbuf, FDMD_F64, FDMD_ROW, model->ldq, u, FDMD_F64, FDMD_COL, n, yq, 1, 0.0, n, ny, 1,
                       0, gw, gws, d.s));
    y = yq;
  } else {
    TRY(fdmd_colmajor_dot(model->raw, model->dt, model->ldr, u, FDMD_F64, n, n, nc, 1, y, ws, wsb, d.s));
  }
  std::vector<double> yh(ny);
  TRY(d.down(yh.data(), y, ny * sizeof(double)));
  for (int a = 0; a < r; ++a) {
    cd acc = 0.0;
    for (int k = 0; k < ny; ++k) acc += model->pinv[(size_t)a * ny + k] * yh[k];
    z_host[2 * a] = acc.real();
    z_host[2 * a + 1] = acc.imag();
  }
  return FDMD_OK;
}

int fdmd_model_decode(fdmd_ctx* ctx, const fdmd_model* model, const double* z_host, int B, double* out_host) {
  if (!ctx || !model || !z_host || !out_host || B < 0) return fail(FDMD_ERR_INVALID, "model_decode: bad argument");
  if (B == 0) return FDMD_OK;
  TRY(set_device(model->device));
  StreamLease lease(ctx);
  Dev d(lease.s());
  const int nc = 2 * model->units, r = model->r;
  const int64_t n = model->n;
  const size_t es = esize(model->dt);
  // Re(phi z) = sum_k raw_k Re((M z)_k): coefficients in raw-table coordinates
  std::vector<double> coef((size_t)nc * B, 0.0);  // row-major nc x B (k*B + f)
  for (int f = 0; f < B; ++f)
    for (int a = 0; a < r; ++a) {
      const cd z(z_host[(size_t)f * 2 * r + 2 * a], z_host[(size_t)f * 2 * r + 2 * a + 1]);
      const int u = model->unit_of[a];
      coef[(size_t)(2 * u) * B + f] += (model->cre[a] * z).real();
      coef[(size_t)(2 * u + 1) * B + f] += (model->cim[a] * z).real();
    }
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(B, (int64_t)(256 << 20) / (n * (int64_t)es)));
  void* cd_ = d.alloc<unsigned char>((size_t)nc * B * es);
  void* fr = d.alloc<unsigned char>((size_t)chunk * n * es);
  if (!cd_ || !fr) return fail(FDMD_ERR_CUDA, "model_decode: device allocation failed");
  if (model->dt == FDMD_F32) {
    std::vector<float> c32(coef.begin(), coef.end());
    TRY(d.up(c32.data(), cd_, c32.size() * 4));
  } else {
    TRY(d.up(coef.data(), cd_, coef.size() * 8));
  }
  std::vector<float> tmp;
  for (int f0 = 0; f0 < B; f0 += (int)chunk) {
    const int fb = (int)std::min<int64_t>(chunk, B - f0);
    TRY(fdmd_decode(model->raw, model->dt, model->ldr, (const char*)cd_ + (size_t)f0 * es, B, fr, n, n, nc, fb, d.s));
    if (model->dt == FDMD_F64) {
      TRY(d.down(out_host + (size_t)f0 * n, fr, (size_t)fb * n * 8));
    } else {
      tmp.resize((size_t)fb * n);
      TRY(d.down(tmp.data(), fr, tmp.size() * 4));
      for (size_t i = 0; i < tmp.size(); ++i) out_host[(size_t)f0 * n + i] = tmp[i];
    }
  }
  return FDMD_OK;
}

int fdmd_model_free(fdmd_model* model) {
  free_model(model);
  return FDMD_OK;
}

}  // extern "C"
