// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A C-ABI harness over the *unmodified* reference library (header-only C++20,
// /root/reference/proj/include/zoloeig). It is compiled in place by
// oracle/Makefile into oracle/_ref/libzoloref.so; no reference source is
// copied into this repository. Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it.
//
// Every entry point calls the reference's own public API:
//   build_filter_design  filter_design.hpp:133-169
//   FilterOperator       filter_engine.hpp:37-165 (apply_g :56-82, apply_filter :86-155)
//   factorize / solve    band_factor.hpp:53-182, reorder_rcm rcm.hpp:69-115
//   rayleigh_ritz        eigensolver.hpp:105-148
//   subspace_iteration   eigensolver.hpp:154-217
//   random_gaussian/mgs  dense.hpp:193-229
// Status codes follow include/zolo_b200.h (0 ok, 1 domain, 2 numerical,
// 3 factorization, 4 gmres).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "zoloeig/zoloeig.hpp"
#include "zoloeig/serialize.hpp"  // needs <json.hpp> (nlohmann 3.11.3, see oracle/Makefile)

using namespace zoloeig;

namespace {

thread_local std::string g_err;

template <class S>
CsrMatrix<S> make_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
  CsrMatrix<S> m;
  m.n = static_cast<std::size_t>(n);
  const int64_t nnz = rp[n];
  m.row_offsets.assign(rp, rp + n + 1);
  m.col_indices.assign(ci, ci + nnz);
  m.values.resize(nnz);
  for (int64_t k = 0; k < nnz; ++k) {
    if constexpr (is_complex_v<S>)
      m.values[k] = Complex(v[2 * k], v[2 * k + 1]);
    else
      m.values[k] = v[k];
  }
  return m;
}

template <class S>
SparsePencil<S> make_pencil(int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
                            const int64_t* brp, const int64_t* bci, const double* bv) {
  SparsePencil<S> p;
  p.a_mat = make_csr<S>(n, arp, aci, av);
  if (brp) p.b_mat = make_csr<S>(n, brp, bci, bv);
  return p;
}

template <class S>
Matrix<S> load_block(int64_t n, int64_t k, const double* src) {
  Matrix<S> m(n, k);
  for (int64_t i = 0; i < n * k; ++i) {
    if constexpr (is_complex_v<S>)
      m.data()[i] = Complex(src[2 * i], src[2 * i + 1]);
    else
      m.data()[i] = src[i];
  }
  return m;
}

template <class S>
void store_block(const Matrix<S>& m, double* dst) {
  const std::size_t len = m.rows() * m.cols();
  for (std::size_t i = 0; i < len; ++i) {
    if constexpr (is_complex_v<S>) {
      dst[2 * i] = m.data()[i].real();
      dst[2 * i + 1] = m.data()[i].imag();
    } else {
      dst[i] = m.data()[i];
    }
  }
}

SpectralWindow window_of(const double* g) {
  return window_from_gaps(g[0], g[1], g[2], g[3]);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const FactorizationError& e) {
    g_err = e.what();
    return 3;
  } catch (const GmresError& e) {
    g_err = e.what();
    return 4;
  } catch (const DomainError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void fill_report(const ShiftedSolveReport& rep, int64_t* col_iters, double* residuals,
                 int32_t* converged, int64_t* iters, int64_t* op_apps) {
  if (col_iters)
    for (std::size_t c = 0; c < rep.column_iterations.size(); ++c)
      col_iters[c] = static_cast<int64_t>(rep.column_iterations[c]);
  for (std::size_t k = 0; k < rep.residuals.size(); ++k) {
    if (residuals) residuals[k] = rep.residuals[k];
    if (converged) converged[k] = rep.converged[k] ? 1 : 0;
  }
  if (iters) *iters = static_cast<int64_t>(rep.iterations);
  if (op_apps) *op_apps = static_cast<int64_t>(rep.operator_applications);
}

}  // namespace

extern "C" {

const char* zr_last_error() { return g_err.c_str(); }

/// Packed FilterDesign (layout shared with include/zolo_b200.h ZOLO_DESIGN_*):
/// [0..5] a b a- a+ b- b+, [6..9] gamma alpha beta ell1, [10..14] m_hat ell2
/// zmax constant_term delta0, [15..18] inner.M inner.delta outer.M
/// outer.delta, then inner_poles(2r) inner_weights(2r) inner_pf(r)
/// outer_pf(r) inner.c(2r-1) outer.c(2r-1). Length 17 + 10 r.
int zr_design(const double* gaps, int r, double* out) {
  return guarded([&] {
    const FilterDesign d = build_filter_design(window_of(gaps), r);
    double* o = out;
    const SpectralWindow& w = d.window;
    *o++ = w.a, *o++ = w.b, *o++ = w.a_minus, *o++ = w.a_plus, *o++ = w.b_minus, *o++ = w.b_plus;
    *o++ = d.mobius.gamma, *o++ = d.mobius.alpha, *o++ = d.mobius.beta, *o++ = d.mobius.ell1;
    *o++ = d.m_hat, *o++ = d.ell2, *o++ = d.zmax, *o++ = d.constant_term, *o++ = d.delta0;
    *o++ = d.inner.big_m, *o++ = d.inner.delta, *o++ = d.outer.big_m, *o++ = d.outer.delta;
    for (const Complex& p : d.inner_poles) *o++ = p.real(), *o++ = p.imag();
    for (const Complex& p : d.inner_weights) *o++ = p.real(), *o++ = p.imag();
    for (double a : d.inner_pf) *o++ = a;
    for (double a : d.outer_pf) *o++ = a;
    for (double c : d.inner.c) *o++ = c;
    for (double c : d.outer.c) *o++ = c;
  });
}

/// eval_g_scalar / eval_filter_scalar at npts points (filter_design.hpp:72-82).
int zr_eval_scalar(const double* gaps, int r, int64_t npts, const double* x, double* g_out,
                   double* filt_out) {
  return guarded([&] {
    const FilterDesign d = build_filter_design(window_of(gaps), r);
    for (int64_t i = 0; i < npts; ++i) {
      if (g_out) g_out[i] = eval_g_scalar(d, x[i]);
      if (filt_out) filt_out[i] = eval_filter_scalar(d, x[i]);
    }
  });
}

/// choose_order (filter_design.hpp:219-232): smallest r in [1,8] meeting eps (8 when capped).
int zr_choose_order(const double* gaps, double eps, int* r_out, double* bound) {
  return guarded([&] {
    const OrderChoice c = choose_order(window_of(gaps), eps);
    *r_out = c.r;
    if (bound) *bound = c.bound;
  });
}

/// n uniforms in [0,1) from raw mt19937_64 bits, (x >> 11) 2^-53 -- the reference's disorder
/// convention (hamiltonian.hpp:50-53): the seeded inputs of the BASELINE config generators, drawn
/// here so that a reference-side process needs no product library.
int zr_uniform_stream(uint64_t seed, int64_t n, double* out) {
  return guarded([&] {
    std::mt19937_64 gen(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
  });
}

/// read_matrix_market (matrix_market.hpp:106-159): pass 1 (rp == nullptr) returns n, nnz and
/// whether the file is complex; pass 2 fills the full-pattern CSR (values interleaved if complex).
int zr_read_mm(const char* path, int64_t* n, int64_t* nnz, int* cx, int64_t* rp, int64_t* ci, double* v) {
  return guarded([&] {
    const MatrixMarketInfo info = probe_matrix_market(path);
    *cx = info.complex_field ? 1 : 0;
    const auto fill = [&](auto tag) {
      using S = decltype(tag);
      const SparseHermitian<S> m = read_matrix_market<S>(path);
      *n = static_cast<int64_t>(m.n);
      *nnz = static_cast<int64_t>(m.values.size());
      if (!rp) return;
      for (std::size_t i = 0; i <= m.n; ++i) rp[i] = static_cast<int64_t>(m.row_offsets[i]);
      for (std::size_t k = 0; k < m.values.size(); ++k) {
        ci[k] = static_cast<int64_t>(m.col_indices[k]);
        if constexpr (is_complex_v<S>) {
          v[2 * k] = m.values[k].real();
          v[2 * k + 1] = m.values[k].imag();
        } else {
          v[k] = m.values[k];
        }
      }
    };
    if (*cx)
      fill(Complex{});
    else
      fill(double{});
  });
}

/// write_matrix_market (matrix_market.hpp:163-189) of a full-pattern CSR.
int zr_write_mm(const char* path, int cx, int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
  return guarded([&] {
    if (cx)
      write_matrix_market<Complex>(path, make_csr<Complex>(n, rp, ci, v));
    else
      write_matrix_market<double>(path, make_csr<double>(n, rp, ci, v));
  });
}

/// write_eigvec_binary / read_eigvec_binary (serialize.hpp:108-142), n x k column-major.
int zr_write_eigvec(const char* path, int cx, int64_t n, int64_t k, const double* x) {
  return guarded([&] {
    if (cx)
      write_eigvec_binary(path, load_block<Complex>(n, k, x));
    else
      write_eigvec_binary(path, load_block<double>(n, k, x));
  });
}

int zr_read_eigvec(const char* path, int cx, int64_t n, int64_t k, double* x) {
  return guarded([&] {
    const auto run = [&](auto tag) {
      using S = decltype(tag);
      const Matrix<S> m = read_eigvec_binary<S>(path);
      if (static_cast<int64_t>(m.rows()) != n || static_cast<int64_t>(m.cols()) != k)
        throw DomainError("eigenvector block shape mismatch");
      store_block(m, x);
    };
    if (cx)
      run(Complex{});
    else
      run(double{});
  });
}

/// random_gaussian (+ optional mgs_orthonormalize), dense.hpp:193-229.
int zr_random_block(int cx, int64_t n, int64_t k, uint64_t seed, int orthonormalize, double* out) {
  return guarded([&] {
    if (cx) {
      Matrix<Complex> q = random_gaussian<Complex>(n, k, seed);
      if (orthonormalize && !mgs_orthonormalize(q)) throw NumericalError("mgs failed");
      store_block(q, out);
    } else {
      Matrix<double> q = random_gaussian<double>(n, k, seed);
      if (orthonormalize && !mgs_orthonormalize(q)) throw NumericalError("mgs failed");
      store_block(q, out);
    }
  });
}

/// reorder_rcm + bandwidth_under + profile_under on a real pattern (rcm.hpp:69-147).
int zr_rcm(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* perm, int64_t* bw,
           int64_t* profile) {
  return guarded([&] {
    CsrMatrix<double> m;
    m.n = n;
    m.row_offsets.assign(rp, rp + n + 1);
    m.col_indices.assign(ci, ci + rp[n]);
    m.values.assign(rp[n], 1.0);
    const std::vector<std::size_t> p = reorder_rcm(m);
    for (int64_t i = 0; i < n; ++i) perm[i] = static_cast<int64_t>(p[i]);
    if (bw) *bw = static_cast<int64_t>(bandwidth_under(m, p));
    if (profile) *profile = static_cast<int64_t>(profile_under(m, p));
  });
}

/// Shifted factorization of the pencil at sigma with the ordering that
/// build_shifted_factors uses (band_factor.hpp:199-220), then solve and
/// adjoint_solve of an n x k complex rhs (band_factor.hpp:53-117).
int zr_shifted_solve(int cx, int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
                     const int64_t* brp, const int64_t* bci, const double* bv, double sig_re,
                     double sig_im, int64_t k, const double* rhs, double* x, double* xa,
                     int64_t* perm_out, int64_t* bw_out, double* min_ratio, int64_t* pivot_index) {
  if (pivot_index) *pivot_index = -1;
  return guarded([&] {
    const auto run = [&](auto tag) {
      using S = decltype(tag);
      const SparsePencil<S> p = make_pencil<S>(n, arp, aci, av, brp, bci, bv);
      const std::vector<Complex> shifts = {Complex(sig_re, sig_im)};
      try {
        const ShiftedFactorSet set = build_shifted_factors(p, shifts, 0);
        const ShiftedFactor& f = set.factors[0];
        if (perm_out)
          for (int64_t i = 0; i < n; ++i) perm_out[i] = static_cast<int64_t>(set.ordering[i]);
        if (bw_out) *bw_out = static_cast<int64_t>(f.profile.bandwidth);
        if (min_ratio) *min_ratio = f.profile.min_pivot_ratio;
        const Matrix<Complex> b = load_block<Complex>(n, k, rhs);
        if (x) store_block(f.solve(b), x);
        if (xa) store_block(f.adjoint_solve(b), xa);
      } catch (const FactorizationError& e) {
        if (pivot_index) *pivot_index = static_cast<int64_t>(e.pivot_index);
        throw;
      }
    };
    if (cx)
      run(Complex{});
    else
      run(double{});
  });
}

/// FilterOperator<S>::apply_g on an n x k block (filter_engine.hpp:56-82).
/// counters[0] = inner_solve_count, counters[1] = g_application_count.
int zr_apply_g(int cx, int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
               const int64_t* brp, const int64_t* bci, const double* bv, const double* gaps, int r,
               int64_t k, const double* v, double* out, int64_t* counters) {
  return guarded([&] {
    const auto run = [&](auto tag) {
      using S = decltype(tag);
      const FilterOperator<S> op(make_pencil<S>(n, arp, aci, av, brp, bci, bv),
                                 build_filter_design(window_of(gaps), r), 0);
      store_block(op.apply_g(load_block<S>(n, k, v)), out);
      counters[0] = op.inner_solve_count();
      counters[1] = op.g_application_count();
    };
    if (cx)
      run(Complex{});
    else
      run(double{});
  });
}

/// FilterOperator<S>::apply_filter (filter_engine.hpp:86-155). On GmresError
/// the report is still filled (status 4). counters: [inner_solves, g_apps].
/// seconds: [t_factor, t_filter] wall clock (steady_clock).
int zr_apply_filter(int cx, int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
                    const int64_t* brp, const int64_t* bci, const double* bv, const double* gaps,
                    int r, double gmres_tol, int64_t gmres_max, int threads, int64_t k,
                    const double* v, double* y, int64_t* col_iters, double* residuals,
                    int32_t* converged, int64_t* iters, int64_t* op_apps, int64_t* counters,
                    double* seconds) {
  return guarded([&] {
    const auto run = [&](auto tag) {
      using S = decltype(tag);
      using clock = std::chrono::steady_clock;
      const auto t0 = clock::now();
      const FilterOperator<S> op(make_pencil<S>(n, arp, aci, av, brp, bci, bv),
                                 build_filter_design(window_of(gaps), r), threads);
      const auto t1 = clock::now();
      try {
        auto [out, rep] = op.apply_filter(load_block<S>(n, k, v), gmres_tol,
                                          static_cast<std::size_t>(gmres_max));
        const auto t2 = clock::now();
        store_block(out, y);
        fill_report(rep, col_iters, residuals, converged, iters, op_apps);
        if (seconds) {
          seconds[0] = std::chrono::duration<double>(t1 - t0).count();
          seconds[1] = std::chrono::duration<double>(t2 - t1).count();
        }
      } catch (const GmresError& e) {
        // apply_filter rethrows the first worker's error; its report covers
        // that column only (filter_engine.hpp:134-137,153).
        fill_report(e.report, nullptr, residuals, converged, iters, op_apps);
        counters[0] = op.inner_solve_count();
        counters[1] = op.g_application_count();
        throw;
      }
      counters[0] = op.inner_solve_count();
      counters[1] = op.g_application_count();
    };
    if (cx)
      run(Complex{});
    else
      run(double{});
  });
}

/// Persistent reference operator (factorize once, apply many times) for the
/// timed CPU baseline: FilterOperator<S> built with `threads` workers.
struct ZrOp {
  int cx;
  void* op;
};

void* zr_op_create(int cx, int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
                   const int64_t* brp, const int64_t* bci, const double* bv, const double* gaps, int r,
                   int threads, double* t_factor) {
  ZrOp* h = nullptr;
  const int st = guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    h = new ZrOp{cx, nullptr};
    if (cx)
      h->op = new FilterOperator<Complex>(make_pencil<Complex>(n, arp, aci, av, brp, bci, bv),
                                          build_filter_design(window_of(gaps), r), threads);
    else
      h->op = new FilterOperator<double>(make_pencil<double>(n, arp, aci, av, brp, bci, bv),
                                         build_filter_design(window_of(gaps), r), threads);
    if (t_factor)
      *t_factor = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
  if (st != 0) {
    delete h;
    return nullptr;
  }
  return h;
}

void zr_op_free(void* p) {
  ZrOp* h = static_cast<ZrOp*>(p);
  if (!h) return;
  if (h->cx)
    delete static_cast<FilterOperator<Complex>*>(h->op);
  else
    delete static_cast<FilterOperator<double>*>(h->op);
  delete h;
}

/// apply_filter on a persistent operator; seconds = steady_clock wall time.
int zr_op_apply_filter(void* p, double gmres_tol, int64_t gmres_max, int64_t n, int64_t k, const double* v,
                       double* y, int64_t* iters, double* seconds) {
  ZrOp* h = static_cast<ZrOp*>(p);
  return guarded([&] {
    const auto run = [&](auto* op, auto tag) {
      using S = decltype(tag);
      const auto t0 = std::chrono::steady_clock::now();
      auto [out, rep] = op->apply_filter(load_block<S>(n, k, v), gmres_tol, static_cast<std::size_t>(gmres_max));
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (y) store_block(out, y);
      if (iters) *iters = static_cast<int64_t>(rep.iterations);
    };
    if (h->cx)
      run(static_cast<FilterOperator<Complex>*>(h->op), Complex{});
    else
      run(static_cast<FilterOperator<double>*>(h->op), double{});
  });
}

/// rayleigh_ritz (eigensolver.hpp:105-148). ritz has room for k values, q for
/// k*k entries; *kept receives the number of Ritz pairs returned.
int zr_rayleigh_ritz(int cx, int64_t n, const int64_t* arp, const int64_t* aci, const double* av,
                     const int64_t* brp, const int64_t* bci, const double* bv, int64_t k,
                     const double* y, double* ritz, double* q, int64_t* kept) {
  return guarded([&] {
    const auto run = [&](auto tag) {
      using S = decltype(tag);
      const SparsePencil<S> p = make_pencil<S>(n, arp, aci, av, brp, bci, bv);
      auto [vals, small_q] = rayleigh_ritz(load_block<S>(n, k, y), p);
      *kept = static_cast<int64_t>(vals.size());
      for (std::size_t i = 0; i < vals.size(); ++i) ritz[i] = vals[i];
      store_block(small_q, q);
    };
    if (cx)
      run(Complex{});
    else
      run(double{});
  });
}

/// subspace_iteration (eigensolver.hpp:154-217). lambdas has room for n_ss
/// values; vectors (optional) for n x n_ss entries. stats: [n_ss, n_iter,
/// n_gmres, n_gmres_min, n_solv, t_fact, t_iter, residual, converged, r].
int zr_subspace_iteration(int cx, int64_t n, const int64_t* arp, const int64_t* aci,
                          const double* av, const int64_t* brp, const int64_t* bci,
                          const double* bv, const double* gaps, int64_t n_lambda,
                          int64_t oversample, int r, double tol, int64_t max_iters,
                          double gmres_tol, int64_t gmres_max, uint64_t seed, int threads,
                          double* lambdas, int64_t* n_found, double* vectors, double* stats) {
  return guarded([&] {
    const auto run = [&](auto tag) {
      using S = decltype(tag);
      SolveConfig cfg;
      cfg.n_lambda = n_lambda;
      cfg.oversample_k = oversample;
      cfg.r = r;
      cfg.tol = tol;
      cfg.max_subspace_iters = max_iters;
      cfg.gmres_tol = gmres_tol;
      cfg.gmres_max = gmres_max;
      cfg.seed = seed;
      cfg.threads = threads;
      const EigResult<S> res = subspace_iteration(make_pencil<S>(n, arp, aci, av, brp, bci, bv),
                                                  window_of(gaps), cfg);
      *n_found = static_cast<int64_t>(res.lambdas.size());
      for (std::size_t i = 0; i < res.lambdas.size(); ++i) lambdas[i] = res.lambdas[i];
      if (vectors) store_block(res.vectors, vectors);
      stats[0] = res.stats.n_ss;
      stats[1] = res.stats.n_iter;
      stats[2] = res.stats.n_gmres;
      stats[3] = res.stats.n_gmres_min;
      stats[4] = static_cast<double>(res.stats.n_solv);
      stats[5] = res.stats.factorization_time;
      stats[6] = res.stats.iteration_time;
      stats[7] = res.residual;
      stats[8] = res.converged ? 1.0 : 0.0;
      stats[9] = res.r;
    };
    if (cx)
      run(Complex{});
    else
      run(double{});
  });
}

/// Dense generalized eigenvalues + filter_of_matrix_oracle (dense_eig.hpp:216-265),
/// for planted pencils given as dense column-major A, B (n <= 2048).
int zr_dense_filter_oracle(int cx, int64_t n, const double* a, const double* b, const double* gaps,
                           int r, int64_t k, const double* v, double* out, double* lambdas) {
  return guarded([&] {
    const auto run = [&](auto tag) {
      using S = decltype(tag);
      const DenseEig<S> eig =
          dense_generalized_eig(load_block<S>(n, n, a), load_block<S>(n, n, b));
      const FilterDesign d = build_filter_design(window_of(gaps), r);
      if (out) store_block(filter_of_matrix_oracle(d, eig, load_block<S>(n, k, v)), out);
      if (lambdas)
        for (int64_t i = 0; i < n; ++i) lambdas[i] = eig.lambdas[i];
    };
    if (cx)
      run(Complex{});
    else
      run(double{});
  });
}

}  // extern "C"
