// Host-side construction of the composed Zolotarev filter design -- the
// boundary input of the filter path (BASELINE.json north_star: "the
// Zolotarev pole/weight construction (elliptic functions) ... remain[s]
// host-side setup"). A restatement of the reference's published algorithm:
//
//   complete_elliptic_K_complement   specfun.hpp:53-63   (AGM)
//   jacobi_elliptic_complement       specfun.hpp:76-116  (Bulirsch descending Landen)
//   zolotarev_coeffs                 zolotarev.hpp:121-180 (c_j, 4096-point log scan +
//                                    golden section for M, delta, zmax)
//   partial_fraction_weights         zolotarev.hpp:192-220
//   fit_mobius                       mobius.hpp:50-147 (cross ratio, 3x3 LU, Newton polish)
//   build_filter_design              filter_design.hpp:133-169 (poles, weights, constant, delta0)
//   window_from_gaps / validate      window.hpp:28-68
//
// Output is the packed layout of include/zolo_b200.h (ZOLO_DESIGN_*).
#include <algorithm>
#include <cmath>
#include <complex>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "host.hpp"

namespace zolo {

namespace {

using cplx = std::complex<double>;

struct Window {
  double a, b, am, ap, bm, bp;
  bool left_open() const { return std::isinf(am); }
  bool right_open() const { return std::isinf(bp); }
};

void validate(const Window& w) {
  if (std::isnan(w.am) || std::isnan(w.ap) || std::isnan(w.bm) || std::isnan(w.bp) || std::isnan(w.a) ||
      std::isnan(w.b))
    throw DesignError(1, "SpectralWindow: NaN endpoint");
  if (std::isinf(w.ap) || std::isinf(w.bm)) throw DesignError(1, "SpectralWindow: interior gap endpoints must be finite");
  if (std::isinf(w.am) && w.am > 0) throw DesignError(1, "SpectralWindow: a_minus must be -inf");
  if (std::isinf(w.bp) && w.bp < 0) throw DesignError(1, "SpectralWindow: b_plus must be +inf");
  if (!(w.am < w.a && w.a < w.ap && w.ap <= w.bm && w.bm < w.b && w.b < w.bp))
    throw DesignError(1, "SpectralWindow: endpoints must satisfy a- < a < a+ <= b- < b < b+");
  if (std::isinf(w.am) && std::isinf(w.bp)) throw DesignError(1, "SpectralWindow: at most one endpoint may be infinite");
}

Window window_from_gaps(double am, double ap, double bm, double bp) {
  Window w;
  w.am = am;
  w.ap = ap;
  w.bm = bm;
  w.bp = bp;
  const double span = (bm > ap) ? (bm - ap) : 1.0;
  w.a = std::isinf(am) ? ap - span : 0.5 * (am + ap);
  w.b = std::isinf(bp) ? bm + span : 0.5 * (bm + bp);
  validate(w);
  return w;
}

double k_complement(double kc) {
  if (!(kc >= 0.0) || kc > 1.0) throw DesignError(1, "complete_elliptic_K_complement: kc outside [0,1]");
  if (kc == 0.0) return std::numeric_limits<double>::infinity();
  double a = 1.0, b = kc;
  for (int i = 0; i < 64 && std::abs(a - b) > 1e-17 * a; ++i) {
    const double am = 0.5 * (a + b);
    b = std::sqrt(a * b);
    a = am;
  }
  return M_PI / (2.0 * a);
}

struct Triple {
  double sn, cn, dn;
};

Triple jacobi_complement(double u, double kc) {
  if (kc == 0.0) {
    const double c = 1.0 / std::cosh(u);
    return {std::tanh(u), c, c};
  }
  constexpr int kMax = 32;
  double em[kMax], en[kMax];
  double a = 1.0, b = kc, dn = 1.0;
  int l = 0;
  for (int i = 0; i < kMax; ++i) {
    l = i;
    em[i] = a;
    en[i] = b;
    if (std::abs(a - b) <= 1e-15 * a) break;
    const double am = 0.5 * (a + b);
    b = std::sqrt(a * b);
    a = am;
  }
  const double c_final = 0.5 * (em[l] + en[l]);
  const double phi = c_final * u;
  double sn = std::sin(phi);
  double cn = std::cos(phi);
  if (sn != 0.0) {
    double aa = cn / sn;
    double c = c_final * aa;
    for (int i = l; i >= 0; --i) {
      const double bb = em[i];
      aa *= c;
      c *= dn;
      dn = (en[i] + aa) / (bb + aa);
      aa = c / bb;
    }
    const double inv = 1.0 / std::sqrt(c * c + 1.0);
    sn = (sn >= 0.0) ? inv : -inv;
    cn = c * sn;
  }
  return {sn, cn, dn};
}

struct Zolo {
  int r = 0;
  double ell = 0;
  std::vector<double> c;
  double big_m = 0, delta = 0, zmax = 0;
};

double product_raw(const std::vector<double>& c, double x) {
  const int r = static_cast<int>((c.size() + 1) / 2);
  if (std::abs(x) > 1e100) return 1.0 / x;
  const double x2 = x * x;
  double v = x / (x2 + c[2 * (r - 1)]);
  for (int j = 0; j + 1 < r; ++j) v *= (x2 + c[2 * j + 1]) / (x2 + c[2 * j]);
  return v;
}

double golden_max(const std::function<double(double)>& g, double a, double b) {
  constexpr double kInvPhi = 0.6180339887498949;
  double x1 = b - kInvPhi * (b - a);
  double x2 = a + kInvPhi * (b - a);
  double g1 = g(x1), g2 = g(x2);
  const double tol = 1e-15 * std::max({1.0, std::abs(a), std::abs(b)});
  for (int it = 0; it < 200 && (b - a) > tol; ++it) {
    if (g1 < g2) {
      a = x1;
      x1 = x2;
      g1 = g2;
      x2 = a + kInvPhi * (b - a);
      g2 = g(x2);
    } else {
      b = x2;
      x2 = x1;
      g2 = g1;
      x1 = b - kInvPhi * (b - a);
      g1 = g(x1);
    }
  }
  return 0.5 * (a + b);
}

std::vector<double> scan_extrema(const std::function<double(double)>& f, double lo, double hi, int samples) {
  std::vector<double> xs(samples), fs(samples);
  const double lr = std::log(hi / lo);
  for (int i = 0; i < samples; ++i) {
    xs[i] = lo * std::exp(lr * static_cast<double>(i) / (samples - 1));
    fs[i] = f(xs[i]);
  }
  xs.front() = lo;
  xs.back() = hi;
  std::vector<double> out;
  int prev_sign = 0, prev_at = 0;
  for (int i = 0; i + 1 < samples; ++i) {
    const double d = fs[i + 1] - fs[i];
    const int s = (d > 0) - (d < 0);
    if (s == 0) continue;
    if (prev_sign != 0 && s != prev_sign) {
      const double a = xs[prev_at], b = xs[i + 1];
      const double x = prev_sign > 0 ? golden_max(f, a, b) : golden_max([&](double t) { return -f(t); }, a, b);
      out.push_back(x);
    }
    prev_sign = s;
    prev_at = i;
  }
  return out;
}

Zolo zolotarev(int r, double ell) {
  if (r < 1 || r > 24) throw DesignError(1, "zolotarev_coeffs: order must be in [1,24]");
  if (!(ell > 1e-12) || !(ell < 1.0)) throw DesignError(1, "zolotarev_coeffs: ell outside (1e-12, 1)");
  Zolo z;
  z.r = r;
  z.ell = ell;
  const double kp = k_complement(ell);
  z.c.resize(2 * r - 1);
  for (int j = 1; j <= 2 * r - 1; ++j) {
    const Triple t = jacobi_complement(j * kp / (2 * r), ell);
    z.c[j - 1] = ell * ell * (t.sn * t.sn) / (t.cn * t.cn);
  }
  for (size_t j = 0; j + 1 < z.c.size(); ++j)
    if (!(z.c[j] < z.c[j + 1])) throw DesignError(2, "zolotarev_coeffs: coefficients not strictly increasing");
  const auto f = [&z](double x) { return product_raw(z.c, x); };
  std::vector<double> interior = scan_extrema(f, ell, 1.0, 4096);
  if (static_cast<int>(interior.size()) != 2 * r - 1) {
    const double f_lo = f(ell), f_hi = f(1.0);
    double fmin = std::min(f_lo, f_hi), fmax = std::max(f_lo, f_hi);
    for (double x : interior) {
      fmin = std::min(fmin, f(x));
      fmax = std::max(fmax, f(x));
    }
    if ((fmax - fmin) / fmax < 1e-10) {
      interior.resize(2 * r - 1);
      for (int i = 0; i < 2 * r - 1; ++i) interior[i] = ell * std::pow(1.0 / ell, (i + 1.0) / (2 * r));
    } else {
      throw DesignError(2, "zolotarev_coeffs: extremum scan found " + std::to_string(interior.size()) +
                               " interior extrema, expected " + std::to_string(2 * r - 1));
    }
  }
  std::vector<double> ext;
  ext.push_back(ell);
  ext.insert(ext.end(), interior.begin(), interior.end());
  ext.push_back(1.0);
  double fmin = f(ell), fmax = f(ell);
  for (double x : ext) {
    const double v = f(x);
    fmin = std::min(fmin, v);
    fmax = std::max(fmax, v);
  }
  z.big_m = 2.0 / (fmin + fmax);
  z.delta = (fmax - fmin) / (fmax + fmin);
  z.zmax = z.big_m * fmax;
  return z;
}

double zolo_eval(const Zolo& z, double x) {
  if (!std::isfinite(x)) throw DesignError(1, "zolotarev_eval: non-finite argument");
  return z.big_m * product_raw(z.c, x);
}

std::vector<double> pf_weights(const Zolo& z) {
  const int r = z.r;
  std::vector<double> d(r), e(r - 1);
  for (int j = 0; j < r; ++j) d[j] = z.c[2 * j];
  for (int j = 0; j + 1 < r; ++j) e[j] = z.c[2 * j + 1];
  std::vector<double> a(r, 0.0);
  if (r == 1) {
    a[0] = 1.0;
    return a;
  }
  double tail = 1.0;
  for (int j = 0; j + 1 < r; ++j) {
    double bj = e[j] - d[j];
    for (int k = 0; k + 1 < r; ++k) {
      if (k == j) continue;
      const double den = d[k] - d[j];
      if (std::abs(den) < 1e-300) throw DesignError(2, "partial_fraction_weights: coincident poles");
      bj *= (e[k] - d[j]) / den;
    }
    const double den = d[r - 1] - d[j];
    if (std::abs(den) < 1e-300) throw DesignError(2, "partial_fraction_weights: coincident poles");
    a[j] = bj / den;
    tail -= a[j];
  }
  a[r - 1] = tail;
  return a;
}

// Dense 3x3 LU with partial pivoting (dense.hpp:233-269), single rhs.
bool lu_solve3(double m[3][3], double rhs[3], double out[3]) {
  double a[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = m[i][j];
  int piv[3];
  for (int k = 0; k < 3; ++k) {
    int p = k;
    double best = std::abs(a[k][k]);
    for (int i = k + 1; i < 3; ++i)
      if (std::abs(a[i][k]) > best) {
        best = std::abs(a[i][k]);
        p = i;
      }
    if (best == 0.0) return false;
    piv[k] = p;
    if (p != k)
      for (int j = 0; j < 3; ++j) std::swap(a[k][j], a[p][j]);
    const double inv = 1.0 / a[k][k];
    for (int i = k + 1; i < 3; ++i) {
      a[i][k] *= inv;
      const double mm = a[i][k];
      for (int j = k + 1; j < 3; ++j) a[i][j] -= mm * a[k][j];
    }
  }
  double x[3] = {rhs[0], rhs[1], rhs[2]};
  for (int k = 0; k < 3; ++k)
    if (piv[k] != k) std::swap(x[k], x[piv[k]]);
  for (int k = 0; k < 3; ++k)
    for (int i = k + 1; i < 3; ++i) x[i] -= a[i][k] * x[k];
  for (int k = 3; k-- > 0;) {
    for (int j = k + 1; j < 3; ++j) x[k] -= a[k][j] * x[j];
    x[k] /= a[k][k];
  }
  for (int i = 0; i < 3; ++i) out[i] = x[i];
  return true;
}

struct Mobius {
  double gamma, alpha, beta, ell1;
  double apply(double x) const { return gamma * (x - alpha) / (x - beta); }
  double apply_ext(double x) const { return std::isinf(x) ? gamma : apply(x); }
};

Mobius fit_mobius(const Window& w) {
  validate(w);
  const double am = w.am, ap = w.ap, bm = w.bm, bp = w.bp;
  double excess;
  if (std::isinf(am))
    excess = (bp - bm) / (bm - ap);
  else if (std::isinf(bp))
    excess = (ap - am) / (bm - ap);
  else
    excess = ((ap - am) * (bp - bm)) / ((bp - am) * (bm - ap));
  if (!(excess > 0.0) || !std::isfinite(excess)) throw DesignError(1, "fit_mobius: window yields an infeasible cross ratio");
  const double root = std::sqrt(1.0 + excess);
  const double ell1 = excess / ((root + 1.0) * (root + 1.0));
  if (!(ell1 > 0.0 && ell1 < 1.0)) throw DesignError(2, "fit_mobius: ell1 outside (0,1)");
  const double targets[4] = {-1.0, 1.0, ell1, -ell1};
  const double points[4] = {am, ap, bm, bp};
  double m[3][3], rhs[3], sol[3];
  for (int i = 0; i < 3; ++i) {
    const double x = points[i], t = targets[i];
    if (std::isinf(x)) {
      m[i][0] = 1.0;
      m[i][1] = 0.0;
      m[i][2] = 0.0;
      rhs[i] = t;
    } else {
      m[i][0] = x;
      m[i][1] = -1.0;
      m[i][2] = t;
      rhs[i] = t * x;
    }
  }
  if (!lu_solve3(m, rhs, sol)) throw DesignError(2, "lu_solve: singular matrix");
  Mobius fit;
  fit.gamma = sol[0];
  fit.beta = sol[2];
  fit.ell1 = ell1;
  if (fit.gamma == 0.0) throw DesignError(2, "fit_mobius: degenerate transform (gamma = 0)");
  fit.alpha = sol[1] / fit.gamma;
  {
    double px[3], pt[3];
    int nf = 0;
    for (int i = 0; i < 4 && nf < 3; ++i) {
      if (std::isinf(points[i])) continue;
      px[nf] = points[i];
      pt[nf] = targets[i];
      ++nf;
    }
    for (int it = 0; it < 8 && nf == 3; ++it) {
      double jac[3][3], f[3], step[3];
      double worst = 0.0;
      for (int i = 0; i < 3; ++i) {
        const double dxa = px[i] - fit.alpha, dxb = px[i] - fit.beta;
        f[i] = fit.gamma * dxa / dxb - pt[i];
        worst = std::max(worst, std::abs(f[i]));
        jac[i][0] = dxa / dxb;
        jac[i][1] = -fit.gamma / dxb;
        jac[i][2] = fit.gamma * dxa / (dxb * dxb);
      }
      if (worst < 1e-15) break;
      if (!lu_solve3(jac, f, step)) break;
      fit.gamma -= step[0];
      fit.alpha -= step[1];
      fit.beta -= step[2];
    }
  }
  const double scale = std::max({1.0, std::abs(ap), std::abs(bm)});
  for (int i = 0; i < 4; ++i) {
    const double res = std::abs(fit.apply_ext(points[i]) - targets[i]);
    if (!(res <= 1e-10 * scale)) throw DesignError(2, "fit_mobius: residual of mapping condition exceeds tolerance");
  }
  const bool ai_a = fit.alpha > am && fit.alpha < ap, ai_b = fit.alpha > bm && fit.alpha < bp;
  const bool be_a = fit.beta > am && fit.beta < ap, be_b = fit.beta > bm && fit.beta < bp;
  if (!((ai_a && be_b) || (ai_b && be_a)))
    throw DesignError(2, "fit_mobius: alpha and beta do not occupy distinct eigengaps");
  return fit;
}

struct Design {
  Window w;
  Mobius mob;
  Zolo inner, outer;
  double zmax, m_hat, ell2, constant_term, delta0;
  std::vector<double> inner_pf, outer_pf;
  std::vector<cplx> poles, weights;
};

double eval_g(const Design& d, double x) {
  if (x == d.mob.beta) throw DesignError(1, "eval_g_scalar: x is the pole of T");
  const double t = d.mob.apply(x);
  if (!std::isfinite(t)) return 0.0;
  return zolo_eval(d.inner, t) / d.inner.zmax;
}

double eval_filter(const Design& d, double x) { return 0.5 * (zolo_eval(d.outer, eval_g(d, x)) + 1.0); }

double eval_filter_inf(const Design& d) {
  return 0.5 * (zolo_eval(d.outer, zolo_eval(d.inner, d.mob.gamma) / d.inner.zmax) + 1.0);
}

double measure_error(const Window& w, const Design& d, int per_branch = 2000) {
  double worst = std::abs(eval_filter_inf(d));
  const auto visit = [&](double x, double target) {
    const double v = std::abs(eval_filter(d, x) - target);
    if (v > worst) worst = v;
  };
  const double span = std::max(w.b - w.a, 1e-30);
  for (int i = 0; i <= per_branch; ++i) visit(w.ap + (w.bm - w.ap) * i / per_branch, 1.0);
  const int half = per_branch / 2, tail = std::max(per_branch / 8, 4);
  if (!w.left_open()) {
    const double lo = w.am - span;
    for (int i = 0; i <= half; ++i) visit(lo + (w.am - lo) * i / half, 0.0);
    for (int i = 0; i < tail; ++i) visit(w.am - span / ((i + 0.5) / tail), 0.0);
  }
  if (!w.right_open()) {
    const double hi = w.bp + span;
    for (int i = 0; i <= half; ++i) visit(w.bp + (hi - w.bp) * i / half, 0.0);
    for (int i = 0; i < tail; ++i) visit(w.bp + span / ((i + 0.5) / tail), 0.0);
  }
  return worst;
}

Design build(const double* gaps, int r) {
  if (r < 1 || r > 16) throw DesignError(1, "build_filter_design: order must be in [1,16]");
  Design d;
  d.w = window_from_gaps(gaps[0], gaps[1], gaps[2], gaps[3]);
  d.mob = fit_mobius(d.w);
  d.inner = zolotarev(r, d.mob.ell1);
  d.zmax = d.inner.zmax;
  d.m_hat = d.inner.big_m / d.zmax;
  d.ell2 = (1.0 - d.inner.delta) / (1.0 + d.inner.delta);
  d.outer = zolotarev(r, d.ell2);
  d.inner_pf = pf_weights(d.inner);
  d.outer_pf = pf_weights(d.outer);
  const double ga = d.mob.gamma, al = d.mob.alpha, be = d.mob.beta;
  double ct = 0.0;
  for (int j = 0; j < r; ++j) {
    const double c_odd = d.inner.c[2 * j];
    const double rt = std::sqrt(c_odd);
    const cplx den(ga, rt);
    cplx sigma = (ga * al + cplx(0.0, rt) * be) / den;
    cplx wj = d.inner_pf[j] * (sigma - be) / (2.0 * den);
    if (sigma.imag() < 0.0) {
      sigma = std::conj(sigma);
      wj = std::conj(wj);
    }
    d.poles.push_back(sigma);
    d.weights.push_back(wj);
    ct += d.inner_pf[j] * ga / (ga * ga + c_odd);
  }
  d.constant_term = d.m_hat * ct;
  d.delta0 = measure_error(d.w, d);
  return d;
}

}  // namespace

void build_filter_design(const double* gaps, int r, double* o) {
  const Design d = build(gaps, r);
  *o++ = d.w.a, *o++ = d.w.b, *o++ = d.w.am, *o++ = d.w.ap, *o++ = d.w.bm, *o++ = d.w.bp;
  *o++ = d.mob.gamma, *o++ = d.mob.alpha, *o++ = d.mob.beta, *o++ = d.mob.ell1;
  *o++ = d.m_hat, *o++ = d.ell2, *o++ = d.zmax, *o++ = d.constant_term, *o++ = d.delta0;
  *o++ = d.inner.big_m, *o++ = d.inner.delta, *o++ = d.outer.big_m, *o++ = d.outer.delta;
  for (const cplx& p : d.poles) *o++ = p.real(), *o++ = p.imag();
  for (const cplx& p : d.weights) *o++ = p.real(), *o++ = p.imag();
  for (double a : d.inner_pf) *o++ = a;
  for (double a : d.outer_pf) *o++ = a;
  for (double c : d.inner.c) *o++ = c;
  for (double c : d.outer.c) *o++ = c;
}

// choose_order (filter_design.hpp:219-232): smallest r in [1,8] whose Gonchar
// upper bound (goncar_rho / goncar_bracket, filter_design.hpp:180-196) meets eps.
int choose_order(const double* gaps, double eps) {
  if (!(eps >= 1e-16) || !(eps < 1.0)) throw DesignError(1, "choose_order: eps outside [1e-16, 1)");
  const Mobius fit = fit_mobius(window_from_gaps(gaps[0], gaps[1], gaps[2], gaps[3]));
  const double mu = (1.0 - std::sqrt(fit.ell1)) / (1.0 + std::sqrt(fit.ell1));
  const double mu_c = std::sqrt((1.0 - mu) * (1.0 + mu));
  const double rho = std::exp(M_PI * k_complement(mu) / (4.0 * k_complement(mu_c)));
  for (int r = 1; r <= 8; ++r) {
    const int deg = 2 * r;
    const double pw = std::exp(deg * deg * std::log(rho));
    const double upper = (pw > 1.0) ? 2.0 / (pw - 1.0) : std::numeric_limits<double>::infinity();
    if (upper <= eps) return r;
  }
  return 8;
}

void eval_filter_scalar(const double* gaps, int r, int64_t npts, const double* x, double* g_out, double* f_out) {
  const Design d = build(gaps, r);
  for (int64_t i = 0; i < npts; ++i) {
    if (g_out) g_out[i] = eval_g(d, x[i]);
    if (f_out) f_out[i] = eval_filter(d, x[i]);
  }
}

}  // namespace zolo
