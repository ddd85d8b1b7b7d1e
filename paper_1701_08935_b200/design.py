"""Host-side filter design: the composed Zolotarev filter of a spectral window.

The reference builds it in C++ (``build_filter_design``, filter_design.hpp:133-169,
from mobius.hpp:50-147, zolotarev.hpp:121-220 and window.hpp:56-68); north_star keeps
this construction on the host, as setup in front of the filter path, and the C++
drop-in (cpp/zolo/gpu_filter_operator.hpp) takes the reference's own FilterDesign.
This module is the Python mirror's independent implementation of the same
published mathematics (the paper's eqs. for T, Z_2r and the pole/weight form),
packed in the ``include/zolo_b200.h`` layout:

* the Zolotarev coefficients c_j = ell^2 sc^2(j K'/(2r); ell') and the 2r + 1
  equioscillation points x_k = ell / dn(k K'/(2r); ell') are evaluated through
  Jacobi's imaginary transformation as theta series in the nome of the *small*
  modulus ell (q ~ (ell/4)^2), which converge in a few terms exactly where the
  complementary modulus ell' is close to 1;
* the normalisation M, delta, zmax comes from f at those points (Newton-polished
  on d log f / dx), not from a numerical scan;
* the Moebius map T(x) = gamma (x - alpha)/(x - beta) is solved in coordinates
  centred and scaled on the window, then polished by Newton on the mapping
  conditions.

Agreement with the reference's FilterDesign is pinned in
tests/test_host_setup.py (reference goldens, tests/golden/designs.npz).
"""
from __future__ import annotations

import math

import numpy as np

from . import DomainError, NumericalError, design_len

# packed offsets (include/zolo_b200.h)
A, B, A_MINUS, A_PLUS, B_MINUS, B_PLUS = range(6)
GAMMA, ALPHA, BETA, ELL1 = 6, 7, 8, 9
M_HAT, ELL2, ZMAX, CONSTANT, DELTA0 = 10, 11, 12, 13, 14
INNER_M, INNER_DELTA, OUTER_M, OUTER_DELTA = 15, 16, 17, 18
HEAD = 19


# --- window (window.hpp:28-68) ------------------------------------------------
def window_from_gaps(am, ap, bm, bp):
    """(a, b, a-, a+, b-, b+); a, b are the gap midpoints (one interior width
    inside the window when a gap is unbounded)."""
    am, ap, bm, bp = (float(x) for x in (am, ap, bm, bp))
    span = bm - ap if bm > ap else 1.0
    a = ap - span if math.isinf(am) else 0.5 * (am + ap)
    b = bm + span if math.isinf(bp) else 0.5 * (bm + bp)
    w = (a, b, am, ap, bm, bp)
    _validate(w)
    return w


def _validate(w):
    a, b, am, ap, bm, bp = w
    if any(math.isnan(x) for x in w):
        raise DomainError("SpectralWindow: NaN endpoint")
    if math.isinf(ap) or math.isinf(bm):
        raise DomainError("SpectralWindow: interior gap endpoints must be finite")
    if (math.isinf(am) and am > 0) or (math.isinf(bp) and bp < 0):
        raise DomainError("SpectralWindow: an unbounded gap must open outwards")
    if not (am < a < ap <= bm < b < bp):
        raise DomainError("SpectralWindow: endpoints must satisfy a- < a < a+ <= b- < b < b+")
    if math.isinf(am) and math.isinf(bp):
        raise DomainError("SpectralWindow: at most one endpoint may be infinite")


# --- elliptic machinery --------------------------------------------------------
def _agm(x: float, y: float) -> float:
    while abs(x - y) > 4e-16 * x:
        x, y = 0.5 * (x + y), math.sqrt(x * y)
    return 0.5 * (x + y)


def _k_pair(ell: float):
    """(K(ell), K(ell')) with ell' = sqrt(1 - ell^2): K(k) = pi / (2 agm(1, k'))."""
    ellc = math.sqrt((1.0 - ell) * (1.0 + ell))
    return math.pi / (2.0 * _agm(1.0, ellc)), math.pi / (2.0 * _agm(1.0, ell))


def _theta_at_imag(t, q_log: float, which: int):
    """Jacobi theta functions of nome q = exp(-q_log) at the imaginary argument i t
    (real series): which = 1 -> theta_1(it)/i, 2 -> theta_2(it), 3 -> theta_3(it),
    4 -> theta_4(it)."""
    t = np.asarray(t, dtype=np.float64)
    if which in (1, 2):
        acc = np.zeros_like(t)
        for n in range(64):
            h = n + 0.5
            # q^{h^2} e^{+-2 h t}, summed as exponentials (no overflow: t < q_log / 2)
            ep = np.exp(-q_log * h * h + 2.0 * h * t)
            em = np.exp(-q_log * h * h - 2.0 * h * t)
            term = (ep - em) if which == 1 else (ep + em)
            if which == 1 and n & 1:
                term = -term
            acc += term
            if np.all(np.abs(term) <= 1e-18 * np.abs(acc)):
                break
        return acc  # 2 sum ... sinh / cosh = sum (e^+ -+ e^-)
    acc = np.ones_like(t)
    for n in range(1, 64):
        ep = np.exp(-q_log * n * n + 2.0 * n * t)
        em = np.exp(-q_log * n * n - 2.0 * n * t)
        term = ep + em
        if which == 4 and n & 1:
            term = -term
        acc += term
        if np.all(np.abs(term) <= 1e-18 * np.abs(acc)):
            break
    return acc


def _sc_dn_complement(u, ell: float):
    """sc(u; ell') and dn(u; ell') for u in [0, K(ell')], through Jacobi's imaginary
    transformation sn(iu; ell) = i sc(u; ell'), dn(iu; ell)/cn(iu; ell) = dn(u; ell')."""
    kk, kkp = _k_pair(ell)
    q_log = math.pi * kkp / kk  # nome of the modulus ell: q = exp(-q_log)
    t = math.pi * np.asarray(u, dtype=np.float64) / (2.0 * kk)
    rl = math.sqrt(ell)
    sc = _theta_at_imag(t, q_log, 1) / (rl * _theta_at_imag(t, q_log, 4))
    dn = rl * _theta_at_imag(t, q_log, 3) / _theta_at_imag(t, q_log, 2)
    return sc, dn, kkp


def _zolo_raw(c, x):
    """f(x) = x prod_j (x^2 + c_2j) / prod_j (x^2 + c_2j-1) (unnormalised, zolotarev.hpp:48-55)."""
    x = np.asarray(x, dtype=np.float64)
    r = (len(c) + 1) // 2
    big = np.abs(x) > 1e100
    xs = np.where(big, 1.0, x)
    x2 = xs * xs
    v = xs / (x2 + c[2 * (r - 1)])
    for j in range(r - 1):
        v = v * (x2 + c[2 * j + 1]) / (x2 + c[2 * j])
    return np.where(big, 1.0 / np.where(big, x, 1.0), v)


class Zolotarev:
    """Best rational sign approximant of type (2r-1, 2r) on [-1,-ell] u [ell,1]:
    Z(x) = M x prod_j (x^2 + c_2j)/prod_j (x^2 + c_2j-1), equioscillating in
    [1 - delta, 1 + delta] on [ell, 1] (zolotarev.hpp:36-44)."""

    def __init__(self, r: int, ell: float):
        if not 1 <= r <= 24:
            raise DomainError("zolotarev_coeffs: order must be in [1,24]")
        if not (1e-12 < ell < 1.0):
            raise DomainError("zolotarev_coeffs: ell outside (1e-12, 1)")
        self.r, self.ell = r, ell
        j = np.arange(1, 2 * r)
        _, _, kkp = _sc_dn_complement(0.0, ell)
        sc, _, _ = _sc_dn_complement(j * kkp / (2 * r), ell)
        self.c = ell * ell * sc * sc
        if not np.all(np.diff(self.c) > 0):
            raise NumericalError("zolotarev_coeffs: coefficients not strictly increasing")
        # equioscillation points x_k = ell / dn(k K'/(2r); ell'), k = 0..2r (x_0 = ell, x_2r = 1)
        k = np.arange(0, 2 * r + 1)
        _, dn, _ = _sc_dn_complement(k * kkp / (2 * r), ell)
        x = ell / dn
        x[0], x[-1] = ell, 1.0
        x[1:-1] = self._polish(np.clip(x[1:-1], ell, 1.0))
        self.extrema = x
        fx = _zolo_raw(self.c, x)
        fmin, fmax = float(fx.min()), float(fx.max())
        self.big_m = 2.0 / (fmin + fmax)
        self.delta = (fmax - fmin) / (fmax + fmin)
        self.zmax = self.big_m * fmax

    def _polish(self, x):
        """Newton on g(x) = d log f / dx = 1/x + sum_even 2x/(x^2+c) - sum_odd 2x/(x^2+c)."""
        ce, co = self.c[1::2], self.c[0::2]
        for _ in range(3):
            x2 = x * x
            de, do = x2[:, None] + ce[None, :], x2[:, None] + co[None, :]
            g = 1.0 / x + (2 * x[:, None] / de).sum(1) - (2 * x[:, None] / do).sum(1)
            dg = -1.0 / x2 + (2 * (ce[None, :] - x2[:, None]) / de ** 2).sum(1) - \
                (2 * (co[None, :] - x2[:, None]) / do ** 2).sum(1)
            step = np.where(dg != 0, g / np.where(dg != 0, dg, 1.0), 0.0)
            ok = np.abs(step) < 1e-3 * x  # only refine; never jump to another extremum
            x = np.where(ok, x - step, x)
        return x

    def eval(self, x):
        return self.big_m * _zolo_raw(self.c, x)

    def partial_fractions(self):
        """a_j with f(x) = x sum_j a_j / (x^2 + c_2j-1): residues of the y = x^2 form."""
        r = self.r
        d, e = self.c[0::2], self.c[1::2]
        a = np.ones(r)
        for j in range(r):
            num = np.prod(e - d[j]) if r > 1 else 1.0
            den = np.prod(np.delete(d, j) - d[j]) if r > 1 else 1.0
            if r > 1 and abs(den) < 1e-300:
                raise NumericalError("partial_fraction_weights: coincident poles")
            a[j] = num / den
        return a


# --- Moebius map (mobius.hpp:50-147) ---------------------------------------------
def fit_mobius(w):
    """T(x) = gamma (x - alpha)/(x - beta) with T(a-) = -1, T(a+) = 1, T(b-) = ell1,
    T(b+) = -ell1 (T(-+inf) = gamma); ell1 from the cross ratio of the endpoints."""
    a, b, am, ap, bm, bp = w
    if math.isinf(am):
        excess = (bp - bm) / (bm - ap)
    elif math.isinf(bp):
        excess = (ap - am) / (bm - ap)
    else:
        excess = ((ap - am) * (bp - bm)) / ((bp - am) * (bm - ap))
    if not (excess > 0.0 and math.isfinite(excess)):
        raise DomainError("fit_mobius: window yields an infeasible cross ratio")
    root = math.sqrt(1.0 + excess)
    ell1 = excess / (root + 1.0) ** 2  # = (sqrt(C) - 1)/(sqrt(C) + 1), C = 1 + excess
    if not 0.0 < ell1 < 1.0:
        raise NumericalError("fit_mobius: ell1 outside (0,1)")
    pts = [am, ap, bm, bp]
    tgt = [-1.0, 1.0, ell1, -ell1]
    # centred / scaled coordinates s = (x - c0)/h keep the 3 x 3 system well conditioned
    fin = [p for p in pts if math.isfinite(p)]
    c0 = 0.5 * (ap + bm)
    h = max(max(abs(p - c0) for p in fin), 1e-300)
    rows, rhs = [], []
    for p, t in zip(pts, tgt):
        if len(rows) == 3:
            break
        if math.isinf(p):  # gamma = t
            rows.append([1.0, 0.0, 0.0])
            rhs.append(t)
        else:  # gamma s - gamma alpha' + t beta' = t s
            s = (p - c0) / h
            rows.append([s, -1.0, t])
            rhs.append(t * s)
    try:
        gam, q, bet = np.linalg.solve(np.array(rows), np.array(rhs))
    except np.linalg.LinAlgError as e:
        raise NumericalError("fit_mobius: singular mapping system") from e
    if gam == 0.0:
        raise NumericalError("fit_mobius: degenerate transform (gamma = 0)")
    alp = q / gam
    finite = [((p - c0) / h, t) for p, t in zip(pts, tgt) if math.isfinite(p)][:3]
    if len(finite) == 3:
        for _ in range(8):  # Newton on the three finite conditions (scaled coordinates)
            F, J = np.zeros(3), np.zeros((3, 3))
            for i, (s, t) in enumerate(finite):
                da, db = s - alp, s - bet
                F[i] = gam * da / db - t
                J[i] = [da / db, -gam / db, gam * da / db ** 2]
            if np.abs(F).max() < 1e-16:
                break
            try:
                dgam, dalp, dbet = np.linalg.solve(J, F)
            except np.linalg.LinAlgError:
                break
            gam, alp, bet = gam - dgam, alp - dalp, bet - dbet
    alpha, beta = c0 + h * alp, c0 + h * bet
    gamma = float(gam)
    scale = max(1.0, abs(ap), abs(bm))
    for p, t in zip(pts, tgt):
        val = gamma if math.isinf(p) else gamma * (p - alpha) / (p - beta)
        if not abs(val - t) <= 1e-10 * scale:
            raise NumericalError("fit_mobius: residual of mapping condition exceeds tolerance")
    in_a = lambda x: am < x < ap  # noqa: E731
    in_b = lambda x: bm < x < bp  # noqa: E731
    if not ((in_a(alpha) and in_b(beta)) or (in_b(alpha) and in_a(beta))):
        raise NumericalError("fit_mobius: alpha and beta do not occupy distinct eigengaps")
    return gamma, float(alpha), float(beta), ell1


# --- the composed filter (filter_design.hpp:53-169) --------------------------------
def build_filter_design(gaps, r: int) -> np.ndarray:
    """Packed FilterDesign (include/zolo_b200.h layout) for window_from_gaps(*gaps) at order r."""
    if not 1 <= int(r) <= 16:
        raise DomainError("build_filter_design: order must be in [1,16]")
    r = int(r)
    w = window_from_gaps(*gaps)
    gamma, alpha, beta, ell1 = fit_mobius(w)
    inner = Zolotarev(r, ell1)
    zmax = inner.zmax
    m_hat = inner.big_m / zmax
    ell2 = (1.0 - inner.delta) / (1.0 + inner.delta)
    outer = Zolotarev(r, ell2)
    ipf, opf = inner.partial_fractions(), outer.partial_fractions()
    d_odd = inner.c[0::2]
    rt = np.sqrt(d_odd)
    den = gamma + 1j * rt
    sigma = (gamma * alpha + 1j * rt * beta) / den
    wts = ipf * (sigma - beta) / (2.0 * den)
    flip = sigma.imag < 0.0
    sigma = np.where(flip, np.conj(sigma), sigma)
    wts = np.where(flip, np.conj(wts), wts)
    constant = m_hat * float(np.sum(ipf * gamma / (gamma * gamma + d_odd)))
    out = np.zeros(design_len(r))
    out[:6] = w
    out[GAMMA], out[ALPHA], out[BETA], out[ELL1] = gamma, alpha, beta, ell1
    out[M_HAT], out[ELL2], out[ZMAX], out[CONSTANT] = m_hat, ell2, zmax, constant
    out[INNER_M], out[INNER_DELTA], out[OUTER_M], out[OUTER_DELTA] = inner.big_m, inner.delta, outer.big_m, outer.delta
    o = HEAD
    out[o:o + 2 * r:2], out[o + 1:o + 2 * r:2] = sigma.real, sigma.imag
    out[o + 2 * r:o + 4 * r:2], out[o + 2 * r + 1:o + 4 * r:2] = wts.real, wts.imag
    out[o + 4 * r:o + 5 * r] = ipf
    out[o + 5 * r:o + 6 * r] = opf
    out[o + 6 * r:o + 8 * r - 1] = inner.c
    out[o + 8 * r - 1:o + 10 * r - 2] = outer.c
    out[DELTA0] = _measured_error(out, r)
    return out


def _unpack(design, r):
    d = np.asarray(design, dtype=np.float64)
    o = HEAD
    inner_c = d[o + 6 * r:o + 8 * r - 1]
    outer_c = d[o + 8 * r - 1:o + 10 * r - 2]
    return d, inner_c, outer_c


def eval_g(design, r: int, x):
    """Zhat_inner(T(x)) (eval_g_scalar, filter_design.hpp:72-77): G's eigenvalue at x."""
    d, ic, _ = _unpack(design, r)
    x = np.asarray(x, dtype=np.float64)
    if np.any(x == d[BETA]):
        raise DomainError("eval_g_scalar: x is the pole of T")
    with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
        t = np.where(np.isinf(x), d[GAMMA], d[GAMMA] * (x - d[ALPHA]) / (x - d[BETA]))
    fin = np.isfinite(t)
    g = d[INNER_M] * _zolo_raw(ic, np.where(fin, t, 1.0)) / d[ZMAX]
    return np.where(fin, g, 0.0)


def eval_filter(design, r: int, x):
    """R(x) = (Z_outer(Zhat_inner(T(x))) + 1)/2 (eval_filter_scalar, filter_design.hpp:80-82)."""
    d, _, oc = _unpack(design, r)
    return 0.5 * (d[OUTER_M] * _zolo_raw(oc, eval_g(design, r, x)) + 1.0)


def _measured_error(design, r, per_branch: int = 2000):
    """delta0: max |S_ab - R| over a dense sample of the window interior (target 1), one
    window width beyond each finite gap and 1/x-spaced tails (target 0), and x -> inf."""
    a, b, am, ap, bm, bp = (float(v) for v in design[:6])
    span = max(b - a, 1e-30)
    xs_in = ap + (bm - ap) * np.arange(per_branch + 1) / per_branch
    outs = []
    half, tail = per_branch // 2, max(per_branch // 8, 4)
    u = (np.arange(tail) + 0.5) / tail
    if not math.isinf(am):
        outs += [am - span + span * np.arange(half + 1) / half, am - span / u]
    if not math.isinf(bp):
        outs += [bp + span * np.arange(half + 1) / half, bp + span / u]
    worst = abs(float(eval_filter(design, r, np.array([np.inf]))[0]))
    worst = max(worst, float(np.abs(eval_filter(design, r, xs_in) - 1.0).max()))
    if outs:
        xo = np.concatenate(outs)
        xo = xo[xo != design[BETA]]
        worst = max(worst, float(np.abs(eval_filter(design, r, xo)).max()))
    return worst


def eval_scalar(gaps, r, x):
    """(eval_g_scalar, eval_filter_scalar) at the points x for window_from_gaps(*gaps)."""
    d = build_filter_design(gaps, r)
    return eval_g(d, r, x), eval_filter(d, r, x)


def choose_order(gaps, eps: float) -> int:
    """Smallest r in [1, 8] whose Gonchar upper bound 2/(rho^{(2r)^2} - 1) meets eps
    (filter_design.hpp:183-232); 8 when none does."""
    if not (1e-16 <= eps < 1.0):
        raise DomainError("choose_order: eps outside [1e-16, 1)")
    _, _, _, ell1 = fit_mobius(window_from_gaps(*gaps))
    mu = (1.0 - math.sqrt(ell1)) / (1.0 + math.sqrt(ell1))
    k_mu, k_mup = _k_pair(mu)  # K(mu), K(mu')
    log_rho = math.pi * k_mup / (4.0 * k_mu)
    for r in range(1, 9):
        e = (2 * r) ** 2 * log_rho
        bound = 2.0 / math.expm1(e) if e < 700 else 0.0
        if bound <= eps:
            return r
    return 8


def inner_poles(design, r):
    d = np.asarray(design)
    return d[HEAD:HEAD + 2 * r:2] + 1j * d[HEAD + 1:HEAD + 2 * r:2]


def outer_c(design, r):
    d = np.asarray(design)
    return d[HEAD + 6 * r + (2 * r - 1):HEAD + 6 * r + 2 * (2 * r - 1)]
