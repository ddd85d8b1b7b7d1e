"""Locate the spectral windows (gap endpoints) of BASELINE configs 2-5 once,
offline, by shift-invert Lanczos (scipy eigsh), and print the WINDOWS entries
recorded in paper_1701_08935_b200/configs.py.

The window is the run of `count` consecutive eigenvalues around `target`
whose smaller end gap relative to the interior width (relative_eigengap,
eigensolver.hpp:66-74) is largest -- the GMRES budget (gmres_max = 50, no
restart) needs delta_lambda >~ 3e-3 at r = 4.
"""
import sys
import time

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import eigsh

sys.path.insert(0, ".")
from paper_1701_08935_b200 import configs  # noqa: E402


def best_window(ev, count):
    ev = np.sort(ev)
    best = None
    for lo in range(1, len(ev) - count):
        inner = ev[lo + count - 1] - ev[lo]
        ga = ev[lo] - ev[lo - 1]
        gb = ev[lo + count] - ev[lo + count - 1]
        score = min(ga, gb) / inner
        if best is None or score > best[0]:
            best = (score, lo)
    score, lo = best
    return [ev[lo - 1], ev[lo], ev[lo + count - 1], ev[lo + count]], score


def run(name, pencil, cx, target, count, k):
    n, a, b = pencil
    am = sp.csr_matrix((a[2], a[1], a[0]), shape=(n, n))
    bm = sp.identity(n) if b is None else sp.csr_matrix((b[2], b[1], b[0]), shape=(n, n))
    t0 = time.time()
    ev = eigsh(am, k=k, M=bm, sigma=target, which="LM", return_eigenvectors=False)
    gaps, score = best_window(ev.real, count)
    print(f'    "{name}": {{"gaps": {[float(x) for x in gaps]}, "count": {count}, '
          f'"rel_gap": {score:.3e}}},  # eigsh k={k} sigma={target}, {time.time() - t0:.0f} s')


if __name__ == "__main__":
    which = sys.argv[1:] or ["cfg2"]
    if "cfg2" in which:
        run("cfg2", configs.stencil3d_pencil(32, seed=2), False, 6.0, 64, 140)
    if "cfg3" in which:
        run("cfg3", configs.tight_binding_pencil(48, seed=3, disorder=1.5), True, 0.0, 128, 260)
