// TEST INFRASTRUCTURE ONLY: proves the drop-in boundary at the C++ level.
// Builds pencils with the reference's own types, then runs the reference's
// zoloeig::FilterOperator<S> and zolo_b200::GpuFilterOperator<S>
// (cpp/zolo/gpu_filter_operator.hpp over libzolo_b200.so) on the same block
// and prints one JSON line per case with the relative Frobenius difference,
// the counters of both, and the GPU-side exception behaviour.
// Compiled by oracle/Makefile (target dropin) into oracle/_ref/dropin_test.
#include <cmath>
#include <cstdio>
#include <random>
#include <tuple>
#include <vector>

#include "zolo/gpu_filter_operator.hpp"
#include "zoloeig/zoloeig.hpp"

using namespace zoloeig;

namespace {

// 7-point Laplacian + U[0,1] diagonal on k^3, B = mass matrix (config-2 shape)
SparsePencil<double> stencil3d(int k, std::uint64_t seed) {
  const int n = k * k * k;
  std::mt19937_64 rng(seed);
  std::vector<std::tuple<std::size_t, std::size_t, double>> ta, tb;
  auto id = [k](int x, int y, int z) { return static_cast<std::size_t>((x * k + y) * k + z); };
  for (int x = 0; x < k; ++x)
    for (int y = 0; y < k; ++y)
      for (int z = 0; z < k; ++z) {
        const std::size_t i = id(x, y, z);
        ta.emplace_back(i, i, 6.0 + static_cast<double>(rng() >> 11) * 0x1.0p-53);
        tb.emplace_back(i, i, 0.5);
        const int nb[6][3] = {{x - 1, y, z}, {x + 1, y, z}, {x, y - 1, z}, {x, y + 1, z}, {x, y, z - 1}, {x, y, z + 1}};
        for (const auto& q : nb)
          if (q[0] >= 0 && q[0] < k && q[1] >= 0 && q[1] < k && q[2] >= 0 && q[2] < k) {
            ta.emplace_back(i, id(q[0], q[1], q[2]), -1.0);
            tb.emplace_back(i, id(q[0], q[1], q[2]), 1.0 / 12.0);
          }
      }
  SparsePencil<double> p;
  p.a_mat = CsrMatrix<double>::from_triplets(n, ta);
  p.b_mat = CsrMatrix<double>::from_triplets(n, tb);
  return p;
}

// periodic tight binding with Peierls phases, B = I (config-5 shape)
SparsePencil<Complex> tight_binding(int k, std::uint64_t seed) {
  const int n = k * k * k;
  std::mt19937_64 rng(seed);
  auto u = [&rng] { return static_cast<double>(rng() >> 11) * 0x1.0p-53; };
  std::vector<std::tuple<std::size_t, std::size_t, Complex>> t;
  auto id = [k](int x, int y, int z) { return static_cast<std::size_t>((x * k + y) * k + z); };
  for (int x = 0; x < k; ++x)
    for (int y = 0; y < k; ++y)
      for (int z = 0; z < k; ++z) {
        const std::size_t i = id(x, y, z);
        t.emplace_back(i, i, Complex(4.0 * u() - 2.0, 0.0));
        const std::size_t js[3] = {id((x + 1) % k, y, z), id(x, (y + 1) % k, z), id(x, y, (z + 1) % k)};
        for (std::size_t j : js) {
          const Complex h = -std::polar(1.0, 2.0 * M_PI * u());
          t.emplace_back(i, j, h);
          t.emplace_back(j, i, std::conj(h));
        }
      }
  SparsePencil<Complex> p;
  p.a_mat = CsrMatrix<Complex>::from_triplets(n, t);
  return p;
}

template <class S>
SpectralWindow window_of(const SparsePencil<S>& p, int lo, int count) {
  const std::size_t n = p.n();
  Matrix<S> a(n, n), b = Matrix<S>::identity(n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t q = p.a_mat.row_offsets[i]; q < p.a_mat.row_offsets[i + 1]; ++q)
      a(i, p.a_mat.col_indices[q]) = p.a_mat.values[q];
  if (!p.b_is_identity()) {
    b = Matrix<S>(n, n);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t q = p.b_mat->row_offsets[i]; q < p.b_mat->row_offsets[i + 1]; ++q)
        b(i, p.b_mat->col_indices[q]) = p.b_mat->values[q];
  }
  const std::vector<double> ev = dense_generalized_eigenvalues(a, b);
  return window_from_gaps(ev[lo - 1], ev[lo], ev[lo + count - 1], ev[lo + count]);
}

template <class S>
void run_case(const char* name, const SparsePencil<S>& pencil, const SpectralWindow& w, int r, int ncols) {
  const FilterDesign design = build_filter_design(w, r);
  const FilterOperator<S> ref(pencil, design, 8);
  const zolo_b200::GpuFilterOperator<S> gpu(pencil, design);
  Matrix<S> v = random_gaussian<S>(pencil.n(), ncols, 1);
  mgs_orthonormalize(v);
  const auto [yr, rr] = ref.apply_filter(v);
  const auto [yg, rg] = gpu.apply_filter(v);
  const double diff = (yr - yg).norm_fro() / yr.norm_fro();
  const auto gr = ref.apply_g(v);
  const auto gg = gpu.apply_g(v);
  const double gdiff = (gr - gg).norm_fro() / gr.norm_fro();
  // exception behaviour: a dimension mismatch must surface as DomainError
  bool domain_ok = false;
  try {
    gpu.apply_filter(Matrix<S>(pencil.n() + 1, 1));
  } catch (const DomainError&) {
    domain_ok = true;
  }
  std::printf(
      "{\"case\": \"%s\", \"n\": %zu, \"r\": %d, \"cols\": %d, \"rel_fro_filter\": %.3e, \"rel_fro_apply_g\": %.3e, "
      "\"ref_iterations\": %zu, \"gpu_iterations\": %zu, \"ref_op_apps\": %zu, \"gpu_op_apps\": %zu, "
      "\"ref_inner_solves\": %lld, \"gpu_inner_solves\": %lld, \"ref_g_apps\": %lld, \"gpu_g_apps\": %lld, "
      "\"domain_error_ok\": %s}\n",
      name, pencil.n(), r, ncols, diff, gdiff, rr.iterations, rg.iterations, rr.operator_applications,
      rg.operator_applications, static_cast<long long>(ref.inner_solve_count()),
      static_cast<long long>(gpu.inner_solve_count()), static_cast<long long>(ref.g_application_count()),
      static_cast<long long>(gpu.g_application_count()), domain_ok ? "true" : "false");
}

}  // namespace

int main() {
  try {
    const SparsePencil<double> p = stencil3d(10, 2);
    run_case("stencil3d_k10_real", p, window_of(p, 500, 16), 4, 24);
    const SparsePencil<Complex> q = tight_binding(8, 3);
    run_case("tight_binding_k8_complex", q, window_of(q, 250, 12), 4, 18);
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
