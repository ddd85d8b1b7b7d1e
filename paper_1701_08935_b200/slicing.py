"""Spectrum slicing by Sylvester inertia.

The reference takes the window (a, b), its gap endpoints and the eigenvalue
count as inputs (the paper protocol needs the exact lambda_1,
lambda_88, lambda_89; the CLI screens gaps with a dense
eig, zoloeig.cpp:214-253). Here they come from eigenvalue counts on the GPU:
count_below(sigma) = number of negative pivots of the unpivoted LDL^H of
A - sigma B (InertiaCounter), and bisection on counts locates individual
eigenvalues to any tolerance.
"""
from __future__ import annotations

import math


def bracket(counter, k: int, center: float, width: float):
    """(lo, hi) with count_below(lo) <= k < count_below(hi), grown from center."""
    lo, hi = center - width, center + width
    while counter.count_below(lo) > k:
        lo = center - 2.0 * (center - lo)
    while counter.count_below(hi) <= k:
        hi = center + 2.0 * (hi - center)
    return lo, hi


def eigenvalue(counter, k: int, lo: float, hi: float, rtol: float = 1e-10) -> float:
    """The k-th smallest eigenvalue (0-based) inside the bracket (lo, hi) by
    bisection on counts: the smallest sigma with count_below(sigma) > k."""
    tol = rtol * max(1.0, abs(lo), abs(hi))
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if counter.count_below(mid) > k:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def window_at(counter, k0: int, count: int, center: float, width: float = 1e-2, rtol: float = 1e-10):
    """Gap endpoints [a_minus, a_plus, b_minus, b_plus] of the window holding the
    eigenvalues k0 .. k0 + count - 1 (0-based, ascending): a_minus / b_plus are
    the nearest eigenvalues outside, a_plus / b_minus the first and last inside --
    the `gaps` argument of build_filter_design (-inf when k0 = 0)."""
    out = []
    for k in (k0 - 1, k0, k0 + count - 1, k0 + count):
        if k < 0:
            out.append(-math.inf)
            continue
        lo, hi = bracket(counter, k, center, width)
        out.append(eigenvalue(counter, k, lo, hi, rtol))
    return out


def window_around(counter, center: float, count: int, width: float = 1e-2, rtol: float = 1e-10):
    """window_at for the `count` eigenvalues around `center` (count // 2 of them below it)."""
    k0 = max(counter.count_below(center) - count // 2, 0)
    return window_at(counter, k0, count, center, width, rtol)
