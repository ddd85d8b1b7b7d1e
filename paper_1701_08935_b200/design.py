"""Host-side filter design (filter_design.hpp:133-169) through the C ABI.

The design is the boundary input of the filter path; it is built on the CPU
(csrc/design.cpp restates the reference's elliptic-function construction)
and packed as include/zolo_b200.h describes.
"""
from __future__ import annotations

import numpy as np

from . import _check_host, _ptr, design_len, lib

# packed offsets (include/zolo_b200.h)
A, B, A_MINUS, A_PLUS, B_MINUS, B_PLUS = range(6)
GAMMA, ALPHA, BETA, ELL1 = 6, 7, 8, 9
M_HAT, ELL2, ZMAX, CONSTANT, DELTA0 = 10, 11, 12, 13, 14
INNER_M, INNER_DELTA, OUTER_M, OUTER_DELTA = 15, 16, 17, 18
HEAD = 19


def build_filter_design(gaps, r: int) -> np.ndarray:
    """Packed FilterDesign for window_from_gaps(*gaps) at order r."""
    g = np.asarray(gaps, dtype=np.float64)
    out = np.zeros(design_len(r))
    _check_host(lib().zolo_build_design(_ptr(g), int(r), _ptr(out)))
    return out


def inner_poles(design, r):
    d = np.asarray(design)
    return d[HEAD:HEAD + 2 * r:2] + 1j * d[HEAD + 1:HEAD + 2 * r:2]


def outer_c(design, r):
    d = np.asarray(design)
    return d[HEAD + 6 * r + (2 * r - 1):HEAD + 6 * r + 2 * (2 * r - 1)]


def eval_scalar(gaps, r, x):
    """(eval_g_scalar, eval_filter_scalar) at the points x."""
    g = np.asarray(gaps, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    gv = np.zeros_like(x)
    fv = np.zeros_like(x)
    _check_host(lib().zolo_eval_filter(_ptr(g), int(r), x.size, _ptr(x), _ptr(gv), _ptr(fv)))
    return gv, fv
