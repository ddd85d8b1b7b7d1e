// Host driver: filtered subspace iteration with Rayleigh-Ritz on the GPU
// filter path -- the reference's subspace_iteration (eigensolver.hpp:154-217)
// and rayleigh_ritz (eigensolver.hpp:105-148), restated as a client of the
// C ABI exactly the way the reference's driver is a client of
// FilterOperator<S>. The N x n_v blocks never leave the device; only the
// n_v x n_v projections come to the host, where the small Hermitian
// eigenproblems are solved (north_star: "the n_v x n_v eig stays host-side").
//
// Reference correspondence:
//   start block        random_gaussian + mgs_orthonormalize (dense.hpp:193-229);
//                      here CholQR2 on the device, which yields the same unique
//                      QR factor (positive-diagonal R) up to rounding
//   filter             FilterOperator::apply_filter -> zolo_apply_filter_device
//   projections        adjoint_matmul(y, A y), (y, B y)  -> zolo_gram_device
//   small eigensolves  dense_hermitian_eig (dense_eig.hpp:194-202): a RESTATEMENT of
//                      the reference's routine (Householder tridiagonalisation,
//                      dense_eig.hpp:42-114, + implicit-shift QL, :118-172; see
//                      herm_eig below), kept so that the Ritz vectors -- whose
//                      phases / rotations within clusters are what iteration >= 2
//                      filters -- follow the reference's choice
//   refinement         residual correction of the shifted solves once the
//                      residual stalls (zolo_set_refinement; no reference
//                      equivalent, see run_solve)
//   Q = Y Q~           matmul (eigensolver.hpp:190)      -> zolo_block_gemm_device
//   residual           relative_residual (eigensolver.hpp:77-93)
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/zolo_b200.h"
#include "host.hpp"

namespace zolo {
cudaStream_t ctx_stream(const zolo_ctx* c);
void* device_alloc(size_t bytes, size_t* got, cudaStream_t st);
void device_free(void* p, size_t bytes, cudaStream_t st);
}

namespace {

using cplx = std::complex<double>;

inline double conj_s(double x) { return x; }
inline cplx conj_s(cplx x) { return std::conj(x); }
inline double abs2(double x) { return x * x; }
inline double abs2(cplx x) { return std::norm(x); }
inline double re(double x) { return x; }
inline double re(cplx x) { return x.real(); }

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// complex arithmetic by parts, the same operations as std::complex's operators (no fused
// multiply-adds in this translation unit), written out so the stride-1 loops below vectorise
inline double add(double a, double b) { return a + b; }
inline cplx add(cplx a, cplx b) { return cplx(a.real() + b.real(), a.imag() + b.imag()); }
inline double sub2(double a, double b) { return a - b; }
inline cplx sub2(cplx a, cplx b) { return cplx(a.real() - b.real(), a.imag() - b.imag()); }
inline double mul(double a, double b) { return a * b; }
inline cplx mul(cplx a, cplx b) {
  return cplx(a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real());
}
inline double mulc(double a, double b) { return a * b; }  // a conj(b)
inline cplx mulc(cplx a, cplx b) {
  return cplx(a.real() * b.real() + a.imag() * b.imag(), a.imag() * b.real() - a.real() * b.imag());
}

// Hermitian eigendecomposition of a dense n x n column-major matrix:
// A = Z diag(w) Z^H, w ascending. Restated from the reference's
// dense_hermitian_eig (dense_eig.hpp:42-172: Householder reduction with the
// reflectors accumulated into Z, unit-modulus rescaling to a real tridiagonal,
// implicit-shift QL) -- not a new algorithm: the n_v x n_v eigenproblem is
// host-side setup (north_star), and restating the reference's routine keeps the
// Ritz bases of iteration >= 2 on the reference's path. The changes: the extra absolute
// deflation test noted below, and loop nests running down the columns (stride-1, vectorised)
// with every sum in the reference's order -- the results are bit-identical to the row-wise form.
template <class S>
void herm_eig(int n, std::vector<S> a, std::vector<double>& w, std::vector<S>& z) {
  auto A = [&](int i, int j) -> S& { return a[static_cast<size_t>(j) * n + i]; };
  z.assign(static_cast<size_t>(n) * n, S(0));
  auto Z = [&](int i, int j) -> S& { return z[static_cast<size_t>(j) * n + i]; };
  for (int i = 0; i < n; ++i) Z(i, i) = S(1);
  std::vector<S> sub(std::max(n - 1, 0), S(0)), v(n), p(n), q(n), tvec(n);
  // Householder reduction to Hermitian tridiagonal form, Z accumulates the reflectors
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;
    double xn2 = 0.0;
    for (int i = 0; i < m; ++i) xn2 += abs2(A(k + 1 + i, k));
    const double xn = std::sqrt(xn2);
    if (xn == 0.0) continue;
    const S x0 = A(k + 1, k);
    const double ax0 = std::abs(x0);
    const S ph = ax0 == 0.0 ? S(1) : x0 / ax0;
    const S alpha = -ph * xn;
    double vn2 = 0.0;
    for (int i = 0; i < m; ++i) {
      v[i] = A(k + 1 + i, k) - (i == 0 ? alpha : S(0));
      vn2 += abs2(v[i]);
    }
    sub[k] = alpha;
    if (vn2 == 0.0) continue;
    const double tau = 2.0 / vn2;
    // p = tau A v, column by column (stride-1): every p[i] still sums over j in ascending order
    for (int i = 0; i < m; ++i) p[i] = S(0);
    for (int j = 0; j < m; ++j) {
      const S vj = v[j];
      const S* col = &A(k + 1, k + 1 + j);
      for (int i = 0; i < m; ++i) p[i] = add(p[i], mul(col[i], vj));
    }
    for (int i = 0; i < m; ++i) p[i] = tau * p[i];
    S vhp(0);
    for (int i = 0; i < m; ++i) vhp += conj_s(v[i]) * p[i];
    const S kc = 0.5 * tau * vhp;
    for (int i = 0; i < m; ++i) q[i] = p[i] - kc * v[i];
    for (int j = 0; j < m; ++j) {
      const S qj = q[j], vj = v[j];
      S* col = &A(k + 1, k + 1 + j);
      for (int i = 0; i < m; ++i) col[i] = sub2(col[i], add(mulc(v[i], qj), mulc(q[i], vj)));
    }
    for (int r = 0; r < n; ++r) tvec[r] = S(0);
    for (int j = 0; j < m; ++j) {
      const S vj = v[j];
      const S* col = &Z(0, k + 1 + j);
      for (int r = 0; r < n; ++r) tvec[r] = add(tvec[r], mul(col[r], vj));
    }
    for (int r = 0; r < n; ++r) tvec[r] = tau * tvec[r];
    for (int j = 0; j < m; ++j) {
      const S vj = v[j];
      S* col = &Z(0, k + 1 + j);
      for (int r = 0; r < n; ++r) col[r] = sub2(col[r], mulc(tvec[r], vj));
    }
  }
  if (n >= 2) sub[n - 2] = A(n - 1, n - 2);
  std::vector<double> d(n), e(std::max(n, 1), 0.0);
  for (int i = 0; i < n; ++i) d[i] = re(A(i, i));
  // unit-modulus diagonal scaling makes the subdiagonal real and nonnegative
  S phi(1);
  for (int i = 0; i + 1 < n; ++i) {
    const double mag = std::abs(sub[i]);
    e[i] = mag;
    if (mag > 0.0) phi = phi * (sub[i] / mag);
    for (int r = 0; r < n; ++r) Z(r, i + 1) *= phi;
  }
  // implicit-shift QL on (d, e), rotations applied to the columns of Z. Deflation:
  // relative to the neighbouring diagonal, or absolute at eps^2 ||T|| -- a filtered
  // block's projected B spans ~28 orders of magnitude and its bottom cluster would
  // otherwise iterate at the underflow level (those eigenvalues are dropped by the
  // 1e-13 mu_max cut of rayleigh_ritz anyway)
  const double eps = std::numeric_limits<double>::epsilon();
  double tnorm = 0.0;
  for (int i = 0; i < n; ++i) tnorm = std::max(tnorm, std::abs(d[i]) + std::abs(e[i]) + (i ? std::abs(e[i - 1]) : 0.0));
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    for (;;) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
        if (std::abs(e[m]) <= eps * dd || std::abs(e[m]) <= eps * eps * tnorm) break;
      }
      if (m == l) break;
      if (++iter > 100) throw Fail(ZOLO_ERR_NUMERICAL, "dense_hermitian_eig: QL did not converge");
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
      double s = 1.0, c = 1.0, pp = 0.0;
      int i = m - 1;
      for (; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= pp;
          e[m] = 0.0;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - pp;
        r = (d[i] - g) * s + 2.0 * c * b;
        pp = s * r;
        d[i + 1] = g + pp;
        g = c * r - b;
        {  // the rotation is real: it acts on the real and imaginary parts alike, as plain doubles
          double* __restrict__ za = reinterpret_cast<double*>(&Z(0, i));
          double* __restrict__ zb = reinterpret_cast<double*>(&Z(0, i + 1));
          const int len = n * static_cast<int>(sizeof(S) / sizeof(double));
          for (int k = 0; k < len; ++k) {
            const double zf = zb[k];
            zb[k] = s * za[k] + c * zf;
            za[k] = c * za[k] - s * zf;
          }
        }
      }
      if (r == 0.0 && i >= l) continue;
      d[l] -= pp;
      e[l] = g;
      e[m] = 0.0;
    }
  }
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return d[x] < d[y]; });
  w.resize(n);
  std::vector<S> zs(static_cast<size_t>(n) * n);
  for (int c = 0; c < n; ++c) {
    w[c] = d[idx[c]];
    for (int r = 0; r < n; ++r) zs[static_cast<size_t>(c) * n + r] = Z(r, idx[c]);
  }
  z.swap(zs);
}

template <class S>
void hermitianize(int n, std::vector<S>& m) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      const S v = 0.5 * (m[static_cast<size_t>(j) * n + i] + conj_s(m[static_cast<size_t>(i) * n + j]));
      m[static_cast<size_t>(j) * n + i] = v;
      m[static_cast<size_t>(i) * n + j] = conj_s(v);
    }
}

// Upper Cholesky G = R^H R and R^{-1} (upper), for the CholQR start block.
template <class S>
bool chol_inverse(int k, const std::vector<S>& g, std::vector<S>& rinv) {
  std::vector<S> r(static_cast<size_t>(k) * k, S(0));
  auto R = [&](int i, int j) -> S& { return r[static_cast<size_t>(j) * k + i]; };
  for (int j = 0; j < k; ++j) {
    for (int i = 0; i <= j; ++i) {
      S s = g[static_cast<size_t>(j) * k + i];
      for (int p = 0; p < i; ++p) s -= conj_s(R(p, i)) * R(p, j);
      if (i == j) {
        const double dv = re(s);
        if (!(dv > 0.0)) return false;
        R(j, j) = std::sqrt(dv);
      } else {
        R(i, j) = s / R(i, i);
      }
    }
  }
  rinv.assign(static_cast<size_t>(k) * k, S(0));
  for (int c = 0; c < k; ++c)
    for (int i = c; i >= 0; --i) {
      S s = (i == c) ? S(1) : S(0);
      for (int p = i + 1; p <= c; ++p) s -= R(i, p) * rinv[static_cast<size_t>(c) * k + p];
      rinv[static_cast<size_t>(c) * k + i] = s / R(i, i);
    }
  return true;
}

// fn(c) for c in [0, n) on the host cores (the n_v x n_v products of the Rayleigh-Ritz step);
// each c is computed by one thread in the serial order, so the result does not depend on threading
template <class F>
void par_for(int n, F&& fn) {
  const int nt = static_cast<int>(std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency())));
  if (n < 64 || nt < 2) {
    for (int c = 0; c < n; ++c) fn(c);
    return;
  }
  std::vector<std::thread> pool;
  for (int q = 0; q < nt; ++q)
    pool.emplace_back([&, q] {
      for (int c = q; c < n; c += nt) fn(c);
    });
  for (auto& t : pool) t.join();
}

void ck(zolo_ctx* ctx, int st) {
  if (st != ZOLO_OK) throw Fail(st, zolo_last_error(ctx));
}
void cuda_ck(cudaError_t e) {
  if (e != cudaSuccess) throw Fail(ZOLO_ERR_CUDA, cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  size_t got = 0;
  cudaStream_t st = nullptr;
  DevBuf(size_t bytes, cudaStream_t s) : st(s) {
    p = zolo::device_alloc(bytes ? bytes : 16, &got, st);  // capi.cu's caching allocator
    if (!p) throw Fail(ZOLO_ERR_CUDA, "cudaMalloc: out of device memory");
    if (std::getenv("ZOLO_ZERO_ALLOC")) {
      cuda_ck(cudaMemset(p, 0, bytes ? bytes : 16));
      cuda_ck(cudaDeviceSynchronize());
    }
  }
  ~DevBuf() {
    if (p) zolo::device_free(p, got, st);
  }
};

template <class S>
void run_solve(zolo_ctx* ctx, int64_t n, int scalar, const int64_t* a_rp, const int64_t* a_ci, const double* a_v,
               const int64_t* b_rp, const int64_t* b_ci, const double* b_v, const double* design, int r,
               int64_t n_lambda, int64_t oversample, double tol, int64_t max_iters, double gmres_tol,
               int64_t gmres_max, uint64_t seed, int refine, double* lambdas, int64_t* n_found, double* vectors,
               double* stats) {
  using clock = std::chrono::steady_clock;
  const auto secs = [](clock::time_point a, clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
  };
  if (n_lambda < 1) throw Fail(ZOLO_ERR_DOMAIN, "subspace_iteration: n_lambda must be >= 1");
  const int64_t n_ss = n_lambda + oversample;
  if (n_ss > n) throw Fail(ZOLO_ERR_DOMAIN, "subspace_iteration: subspace larger than the matrix");
  if (r < 1 || r > ZOLO_MAX_ORDER) throw Fail(ZOLO_ERR_DOMAIN, "subspace_iteration: order must be in [1,16]");

  const auto t0 = clock::now();
  // (development) ZOLO_SETUP_TIMES=1 prints the driver's phases
  const bool phases = std::getenv("ZOLO_SETUP_TIMES") != nullptr;
  auto tp = t0;
  const auto mark = [&](const char* what) {
    if (!phases) return;
    const auto now = clock::now();
    std::fprintf(stderr, "[solve] %-22s %8.2f ms\n", what, secs(tp, now) * 1e3);
    tp = now;
  };
  // the seeded start block (random_gaussian, dense.hpp:193-208) does not depend on the
  // factorization: a host thread generates it and uploads it on its own stream while the factors
  // are built
  const size_t es = sizeof(S);
  const cudaStream_t cst = zolo::ctx_stream(ctx);
  DevBuf q(es * n * n_ss, cst);
  cuda_ck(cudaStreamSynchronize(cst));  // the block's previous user (caching allocator) is done
  int dev = 0;
  cuda_ck(cudaGetDevice(&dev));
  cudaError_t up_err = cudaSuccess;
  std::thread rng([&] {
    // uninitialised host block: its pages are first touched by the generator's threads
    struct Free {
      void operator()(void* p) const { std::free(p); }
    };
    std::unique_ptr<void, Free> h0(std::malloc(es * n * n_ss));
    if (!h0) {
      up_err = cudaErrorMemoryAllocation;
      return;
    }
    zolo::random_block(scalar, n, n_ss, seed, false, static_cast<double*>(h0.get()));
    cudaStream_t us = nullptr;
    if ((up_err = cudaSetDevice(dev)) != cudaSuccess) return;
    if ((up_err = cudaStreamCreateWithFlags(&us, cudaStreamNonBlocking)) != cudaSuccess) return;
    up_err = cudaMemcpyAsync(q.p, h0.get(), es * n * n_ss, cudaMemcpyHostToDevice, us);
    if (up_err == cudaSuccess) up_err = cudaStreamSynchronize(us);
    cudaStreamDestroy(us);
  });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{rng};
  ck(ctx, zolo_set_refinement(ctx, refine == 1 ? 1 : 0));
  ck(ctx, zolo_filter_create(ctx, n, scalar, a_rp, a_ci, a_v, b_rp, b_ci, b_v, design, r, nullptr));
  const auto t1 = clock::now();
  mark("filter_create");
  const double wa = design[0], wb = design[1];
  const double scale = std::max(std::abs(wa), std::abs(wb));

  DevBuf y(es * n * n_ss, cst), t(es * n * n_ss, cst), u(es * n * n_ss, cst);
  {  // Q0: seeded Gaussian block, orthonormalised (CholQR2 == MGS's Q up to rounding)
    rng.join();
    cuda_ck(up_err);
    mark("start block upload");
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<S> g(static_cast<size_t>(n_ss) * n_ss), rinv;
      ck(ctx, zolo_gram_device(ctx, q.p, q.p, n_ss, n_ss, reinterpret_cast<double*>(g.data())));
      hermitianize(static_cast<int>(n_ss), g);
      if (!chol_inverse(static_cast<int>(n_ss), g, rinv))
        throw Fail(ZOLO_ERR_NUMERICAL, "subspace_iteration: random block failed to orthonormalize");
      ck(ctx, zolo_block_gemm_device(ctx, q.p, n_ss, reinterpret_cast<const double*>(rinv.data()), n_ss, t.p));
      std::swap(q.p, t.p);
      std::swap(q.got, t.got);  // block sizes travel with the blocks (caching allocator)
    }
  }

  mark("start block CholQR2");
  int64_t kq = n_ss;  // current subspace width
  int64_t n_iter = 0, n_gmres = 0, n_gmres_min = 0;
  double residual = std::numeric_limits<double>::infinity(), residual_lam = 0.0, filter_ms = 0.0;
  bool converged = false;
  std::vector<double> inside_vals;
  std::vector<int64_t> inside;
  std::vector<int64_t> cols(n_ss);
  int64_t refined_from = refine == 1 ? 1 : 0;
  double first_residual = 0.0;
  for (int64_t it = 1; it <= max_iters; ++it) {
    n_iter = it;
    zolo_report rep;
    rep.column_iterations = cols.data();
    const int st = zolo_apply_filter_device(ctx, q.p, y.p, kq, gmres_tol, gmres_max, &rep);
    if (st == ZOLO_ERR_GMRES) throw Fail(st, zolo_last_error(ctx));
    ck(ctx, st);
    double tm[8];
    zolo_last_timings(ctx, tm);
    filter_ms += tm[0];
    mark("apply_filter");
    n_gmres = std::max<int64_t>(n_gmres, rep.iterations);
    for (int64_t c = 0; c < kq; ++c) n_gmres_min = n_gmres_min == 0 ? cols[c] : std::min(n_gmres_min, cols[c]);

    // Rayleigh-Ritz (eigensolver.hpp:105-148)
    const int k = static_cast<int>(kq);
    std::vector<S> at(static_cast<size_t>(k) * k), bt(static_cast<size_t>(k) * k);
    ck(ctx, zolo_spmm_device(ctx, 0, y.p, t.p, kq));
    ck(ctx, zolo_gram_device(ctx, y.p, t.p, kq, kq, reinterpret_cast<double*>(at.data())));
    ck(ctx, zolo_spmm_device(ctx, 1, y.p, t.p, kq));
    ck(ctx, zolo_gram_device(ctx, y.p, t.p, kq, kq, reinterpret_cast<double*>(bt.data())));
    hermitianize(k, at);
    hermitianize(k, bt);
    mark("RR projections");
    std::vector<double> mu;
    std::vector<S> vb;
    herm_eig(k, bt, mu, vb);
    const double mu_max = mu.empty() ? 0.0 : mu.back();
    if (!(mu_max > 0.0))
      throw Fail(ZOLO_ERR_NUMERICAL, "rayleigh_ritz: projected B is numerically singular (rank-deficient subspace)");
    std::vector<int> kept;
    for (int i = 0; i < k; ++i)
      if (mu[i] > 1e-13 * mu_max) kept.push_back(i);
    const int kk = static_cast<int>(kept.size());
    std::vector<S> w(static_cast<size_t>(k) * kk);
    for (int c = 0; c < kk; ++c) {
      const double sc = 1.0 / std::sqrt(mu[kept[c]]);
      for (int i = 0; i < k; ++i) w[static_cast<size_t>(c) * k + i] = vb[static_cast<size_t>(kept[c]) * k + i] * sc;
    }
    std::vector<S> aw(static_cast<size_t>(k) * kk, S(0)), ar(static_cast<size_t>(kk) * kk, S(0));
    par_for(kk, [&](int c) {
      for (int p = 0; p < k; ++p) {
        const S wpc = w[static_cast<size_t>(c) * k + p];
        for (int i = 0; i < k; ++i) aw[static_cast<size_t>(c) * k + i] += at[static_cast<size_t>(p) * k + i] * wpc;
      }
    });
    par_for(kk, [&](int c) {
      for (int i = 0; i < kk; ++i) {
        S s(0);
        for (int p = 0; p < k; ++p) s += conj_s(w[static_cast<size_t>(i) * k + p]) * aw[static_cast<size_t>(c) * k + p];
        ar[static_cast<size_t>(c) * kk + i] = s;
      }
    });
    hermitianize(kk, ar);
    std::vector<double> ritz;
    std::vector<S> qa;
    herm_eig(kk, ar, ritz, qa);
    std::vector<S> small(static_cast<size_t>(k) * kk, S(0));
    par_for(kk, [&](int c) {
      for (int p = 0; p < kk; ++p) {
        const S v = qa[static_cast<size_t>(c) * kk + p];
        for (int i = 0; i < k; ++i) small[static_cast<size_t>(c) * k + i] += w[static_cast<size_t>(p) * k + i] * v;
      }
    });
    mark("RR host eigenproblems");
    ck(ctx, zolo_block_gemm_device(ctx, y.p, kq, reinterpret_cast<const double*>(small.data()), kk, q.p));
    kq = kk;
    mark("RR Q = Y Q~");

    // Ritz values inside (a,b) and their residual (eigensolver.hpp:193-207)
    inside.clear();
    inside_vals.clear();
    for (int i = 0; i < kk; ++i)
      if (wa < ritz[i] && ritz[i] < wb) {
        inside.push_back(i);
        inside_vals.push_back(ritz[i]);
      }
    if (inside.empty()) {
      residual = std::numeric_limits<double>::infinity();
      continue;
    }
    const int64_t ni = static_cast<int64_t>(inside.size());
    for (int64_t c = 0; c < ni; ++c)  // gather the inside columns (contiguous since ritz ascends)
      cuda_ck(cudaMemcpyAsync(static_cast<char*>(u.p) + es * n * c, static_cast<char*>(q.p) + es * n * inside[c],
                              es * n, cudaMemcpyDeviceToDevice, cst));
    cuda_ck(cudaStreamSynchronize(cst));
    ck(ctx, zolo_spmm_device(ctx, 0, u.p, t.p, ni));
    ck(ctx, zolo_spmm_device(ctx, 1, u.p, y.p, ni));
    std::vector<double> num(ni), den(ni);
    ck(ctx, zolo_residual_norms_device(ctx, t.p, y.p, ni, inside_vals.data(), num.data(), den.data()));
    residual = 0.0;
    residual_lam = 0.0;
    for (int64_t c = 0; c < ni; ++c) {
      residual = std::max(residual, std::sqrt(num[c]) / (scale * std::sqrt(den[c])));
      residual_lam = std::max(residual_lam, std::sqrt(num[c]) / (std::abs(inside_vals[c]) * std::sqrt(den[c])));
    }
    mark("residuals");
    if (it == 1) first_residual = residual;
    if (residual <= tol) {
      converged = true;
      break;
    }
    // Automatic refinement: once the subspace has converged to within a few orders of tol
    // (residual <= 1e-5) the remaining error is the shifted solves' rounding -- eps / min pivot
    // ratio of the unpivoted LU, injected afresh by every filter application (windows centred
    // near 0 sit far below ||A|| in the reference's residual scale max(|a|,|b|)). From then on
    // every solve gets one residual-correction step (zolo_set_refinement).
    if (refine < 0 && refined_from == 0 && residual <= 1e-5 && it < max_iters) {
      ck(ctx, zolo_set_refinement(ctx, 1));
      refined_from = it + 1;
    }
  }
  const auto t2 = clock::now();
  *n_found = static_cast<int64_t>(inside_vals.size());
  for (size_t i = 0; i < inside_vals.size(); ++i) lambdas[i] = inside_vals[i];
  if (vectors && !inside.empty())
    cuda_ck(cudaMemcpyAsync(vectors, u.p, es * n * inside.size(), cudaMemcpyDeviceToHost, cst));
  cuda_ck(cudaStreamSynchronize(cst));
  mark("vectors to host");
  int64_t inner = 0, gapps = 0;
  zolo_counters(ctx, &inner, &gapps);
  stats[0] = static_cast<double>(n_ss);
  stats[1] = static_cast<double>(n_iter);
  stats[2] = static_cast<double>(n_gmres);
  stats[3] = static_cast<double>(n_gmres_min);
  stats[4] = static_cast<double>(inner);
  stats[5] = secs(t0, t1);
  stats[6] = secs(t1, t2);
  stats[7] = residual;
  stats[8] = converged ? 1.0 : 0.0;
  stats[9] = r;
  stats[10] = residual_lam;
  stats[11] = filter_ms;
  stats[12] = static_cast<double>(refined_from);
  stats[13] = first_residual;
}

}  // namespace

extern "C" int zolo_subspace_iteration(zolo_ctx* ctx, int64_t n, int scalar, const int64_t* a_rp,
                                       const int64_t* a_ci, const double* a_v, const int64_t* b_rp,
                                       const int64_t* b_ci, const double* b_v, const double* design, int r,
                                       int64_t n_lambda, int64_t oversample, double tol, int64_t max_iters,
                                       double gmres_tol, int64_t gmres_max, uint64_t seed, int refine,
                                       double* lambdas, int64_t* n_found, double* vectors, double* stats) {
  try {
    if (scalar == ZOLO_C128)
      run_solve<cplx>(ctx, n, scalar, a_rp, a_ci, a_v, b_rp, b_ci, b_v, design, r, n_lambda, oversample, tol,
                      max_iters, gmres_tol, gmres_max, seed, refine, lambdas, n_found, vectors, stats);
    else
      run_solve<double>(ctx, n, scalar, a_rp, a_ci, a_v, b_rp, b_ci, b_v, design, r, n_lambda, oversample, tol,
                        max_iters, gmres_tol, gmres_max, seed, refine, lambdas, n_found, vectors, stats);
    return ZOLO_OK;
  } catch (const Fail& e) {
    zolo_set_error(ctx, e.what());
    return e.code;
  } catch (const std::exception& e) {
    zolo_set_error(ctx, e.what());
    return ZOLO_ERR_NUMERICAL;
  }
}
