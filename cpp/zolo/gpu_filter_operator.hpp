// GpuFilterOperator<S>: drop-in replacement for the reference's
// zoloeig::FilterOperator<S> (proj/include/zoloeig/filter_engine.hpp:37-165)
// on top of the C ABI in include/zolo_b200.h (libzolo_b200.so, sm_100a).
//
// Header-only; include it after the reference headers. Same public surface
// (ctor(pencil, design, threads), design(), pencil(), dim(),
// inner_solve_count(), g_application_count(), apply_g(), apply_filter()),
// same data types (Matrix<S>, SparsePencil<S>, FilterDesign,
// ShiftedSolveReport) and the same exceptions with the same fields
// (DomainError, NumericalError, FactorizationError{pivot_index},
// GmresError{report}). `threads` is accepted for signature compatibility:
// the GPU path parallelises over columns and poles itself.
#ifndef ZOLO_GPU_FILTER_OPERATOR_HPP
#define ZOLO_GPU_FILTER_OPERATOR_HPP

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "zoloeig/filter_engine.hpp"
#include "zolo_b200.h"

namespace zolo_b200 {

namespace detail {

// FilterDesign (filter_design.hpp:53-69) -> packed layout of zolo_b200.h.
inline std::vector<double> pack_design(const zoloeig::FilterDesign& d) {
  const int r = d.order();
  std::vector<double> o;
  o.reserve(ZOLO_DESIGN_LEN(r));
  const zoloeig::SpectralWindow& w = d.window;
  for (double v : {w.a, w.b, w.a_minus, w.a_plus, w.b_minus, w.b_plus}) o.push_back(v);
  for (double v : {d.mobius.gamma, d.mobius.alpha, d.mobius.beta, d.mobius.ell1}) o.push_back(v);
  for (double v : {d.m_hat, d.ell2, d.zmax, d.constant_term, d.delta0}) o.push_back(v);
  for (double v : {d.inner.big_m, d.inner.delta, d.outer.big_m, d.outer.delta}) o.push_back(v);
  for (const zoloeig::Complex& p : d.inner_poles) o.push_back(p.real()), o.push_back(p.imag());
  for (const zoloeig::Complex& p : d.inner_weights) o.push_back(p.real()), o.push_back(p.imag());
  for (double a : d.inner_pf) o.push_back(a);
  for (double a : d.outer_pf) o.push_back(a);
  for (double c : d.inner.c) o.push_back(c);
  for (double c : d.outer.c) o.push_back(c);
  return o;
}

template <class S>
struct Csr64 {
  std::vector<int64_t> rp, ci;
  const double* v = nullptr;
  explicit Csr64(const zoloeig::CsrMatrix<S>& m)
      : rp(m.row_offsets.begin(), m.row_offsets.end()),
        ci(m.col_indices.begin(), m.col_indices.end()),
        v(reinterpret_cast<const double*>(m.values.data())) {}
};

[[noreturn]] inline void raise(int st, const zolo_ctx* ctx, int64_t pivot = -1) {
  const std::string msg = zolo_last_error(ctx);
  switch (st) {
    case ZOLO_ERR_DOMAIN:
      throw zoloeig::DomainError(msg);
    case ZOLO_ERR_FACTORIZATION:
      throw zoloeig::FactorizationError(msg, static_cast<std::size_t>(pivot < 0 ? 0 : pivot));
    default:
      throw zoloeig::NumericalError(msg);
  }
}

}  // namespace detail

template <class S>
class GpuFilterOperator {
 public:
  GpuFilterOperator(zoloeig::SparsePencil<S> pencil, zoloeig::FilterDesign design, int threads = 0, int device = 0)
      : pencil_(std::move(pencil)), design_(std::move(design)), threads_(threads) {
    zolo_ctx* c = nullptr;
    const int st = zolo_ctx_create(device, &c);
    if (st != ZOLO_OK) detail::raise(st, nullptr);
    ctx_.reset(c);
    const int scalar = zoloeig::is_complex_v<S> ? ZOLO_C128 : ZOLO_F64;
    const detail::Csr64<S> a(pencil_.a_mat);
    std::unique_ptr<detail::Csr64<S>> b;
    if (!pencil_.b_is_identity()) b = std::make_unique<detail::Csr64<S>>(*pencil_.b_mat);
    const std::vector<double> packed = detail::pack_design(design_);
    const int r = design_.order();
    std::vector<zolo_factor_stats> stats(r);
    const int rc = zolo_filter_create(ctx_.get(), static_cast<int64_t>(pencil_.n()), scalar, a.rp.data(), a.ci.data(),
                                      a.v, b ? b->rp.data() : nullptr, b ? b->ci.data() : nullptr,
                                      b ? b->v : nullptr, packed.data(), r, stats.data());
    if (rc == ZOLO_ERR_FACTORIZATION) {
      int64_t piv = -1;
      for (const auto& s : stats)
        if (s.pivot_index >= 0 && (piv < 0 || s.pivot_index < piv)) piv = s.pivot_index;
      detail::raise(rc, ctx_.get(), piv);
    }
    if (rc != ZOLO_OK) detail::raise(rc, ctx_.get());
  }

  const zoloeig::FilterDesign& design() const { return design_; }
  const zoloeig::SparsePencil<S>& pencil() const { return pencil_; }
  std::size_t dim() const { return pencil_.n(); }
  std::int64_t inner_solve_count() const {
    int64_t a = 0, b = 0;
    zolo_counters(ctx_.get(), &a, &b);
    return a;
  }
  std::int64_t g_application_count() const {
    int64_t a = 0, b = 0;
    zolo_counters(ctx_.get(), &a, &b);
    return b;
  }

  /// filter_engine.hpp:56-82
  zoloeig::Matrix<S> apply_g(const zoloeig::Matrix<S>& v) const {
    if (v.rows() != dim()) throw zoloeig::DomainError("apply_g: dimension mismatch");
    zoloeig::Matrix<S> out(v.rows(), v.cols());
    const int st = zolo_apply_g(ctx_.get(), reinterpret_cast<const double*>(v.data()),
                                reinterpret_cast<double*>(out.data()), static_cast<int64_t>(v.cols()));
    if (st != ZOLO_OK) detail::raise(st, ctx_.get());
    return out;
  }

  /// filter_engine.hpp:86-155; throws GmresError carrying the merged report.
  std::pair<zoloeig::Matrix<S>, zoloeig::ShiftedSolveReport> apply_filter(const zoloeig::Matrix<S>& v,
                                                                          double gmres_tol = 1e-12,
                                                                          std::size_t gmres_max = 50) const {
    if (v.rows() != dim()) throw zoloeig::DomainError("apply_filter: dimension mismatch");
    zoloeig::Matrix<S> out(v.rows(), v.cols());
    std::vector<int64_t> cols(v.cols(), 0);
    zolo_report rep{};
    rep.column_iterations = cols.data();
    const int st = zolo_apply_filter(ctx_.get(), reinterpret_cast<const double*>(v.data()),
                                     reinterpret_cast<double*>(out.data()), static_cast<int64_t>(v.cols()), gmres_tol,
                                     static_cast<int64_t>(gmres_max), &rep);
    zoloeig::ShiftedSolveReport report;
    report.iterations = static_cast<std::size_t>(rep.iterations);
    report.operator_applications = static_cast<std::size_t>(rep.operator_applications);
    for (int k = 0; k < rep.n_shifts; ++k) {
      report.residuals.push_back(rep.residuals[k]);
      report.converged.push_back(rep.converged[k] != 0);
    }
    for (int64_t c : cols) report.column_iterations.push_back(static_cast<std::size_t>(c));
    if (st == ZOLO_ERR_GMRES) throw zoloeig::GmresError(zolo_last_error(ctx_.get()), report);
    if (st != ZOLO_OK) detail::raise(st, ctx_.get());
    return {std::move(out), std::move(report)};
  }

 private:
  struct CtxDel {
    void operator()(zolo_ctx* c) const { zolo_ctx_destroy(c); }
  };
  zoloeig::SparsePencil<S> pencil_;
  zoloeig::FilterDesign design_;
  int threads_ = 0;
  std::unique_ptr<zolo_ctx, CtxDel> ctx_;
};

}  // namespace zolo_b200

#endif  // ZOLO_GPU_FILTER_OPERATOR_HPP
