"""subspace_iteration (eigensolver.hpp:154-217) on the GPU filter path.

Thin Python mirror of the C-ABI driver ``zolo_subspace_iteration``
(csrc/driver.cu), with the reference's SolveConfig defaults
(eigensolver.hpp:30-42) and EigResult / SolveStats fields
(eigensolver.hpp:44-62).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import CudaError, _check, _csr, _ptr, lib


@dataclass
class SolveConfig:
    n_lambda: int = 1
    oversample_k: int = 1
    r: int = 0
    tol: float = 1e-10
    max_subspace_iters: int = 5
    gmres_tol: float = 1e-12
    gmres_max: int = 50
    seed: int = 0
    refine: object = "auto"  # residual-correction refinement of the solves: "auto", True, False

    def subspace_size(self) -> int:
        return self.n_lambda + self.oversample_k


@dataclass
class SolveStats:
    n_ss: int = 0
    n_iter: int = 0
    n_gmres: int = 0
    n_gmres_min: int = 0
    n_solv: int = 0
    factorization_time: float = 0.0
    iteration_time: float = 0.0
    filter_device_ms: float = 0.0
    refined_from: int = 0  # first subspace iteration with refined solves (0: none)
    first_residual: float = 0.0  # residual after the first iteration


@dataclass
class EigResult:
    lambdas: np.ndarray
    vectors: Optional[np.ndarray]
    residual: float
    residual_rel_lambda: float
    stats: SolveStats = field(default_factory=SolveStats)
    converged: bool = False
    r: int = 0

    @property
    def time_to_all_eigenpairs(self) -> float:
        return self.stats.factorization_time + self.stats.iteration_time


def subspace_iteration(pencil, gaps, config: SolveConfig, is_complex: Optional[bool] = None, device: int = 0,
                       want_vectors: bool = False) -> EigResult:
    """subspace_iteration (eigensolver.hpp:154-217) through zolo_subspace_iteration. The filter
    design is built on the host (design.py, as the reference builds it inside its driver,
    eigensolver.hpp:168-172) and its time counts into t_fact like the reference's.
    config.refine: residual-correction refinement of the shifted solves -- "auto" (once the
    residual stalls below 1e-5 without meeting tol), True / False."""
    import time

    from .design import build_filter_design, choose_order

    L = lib()
    L.zolo_subspace_iteration.argtypes = [C.c_void_p, C.c_int64, C.c_int] + [C.c_void_p] * 7 + [
        C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_int64, C.c_double, C.c_int64, C.c_uint64, C.c_int,
        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    n, a, b = pencil
    cx = bool(is_complex) if is_complex is not None else np.iscomplexobj(a[2])
    ac = _csr(a, cx)
    bc = _csr(b, cx) if b is not None else (None, None, None)
    t0 = time.perf_counter()
    r = config.r if config.r > 0 else choose_order(gaps, max(config.tol * 1e-2, 1e-16))
    design = np.ascontiguousarray(build_filter_design(gaps, r))
    t_design = time.perf_counter() - t0
    refine = {"auto": -1, True: 1, False: 0}[config.refine]
    h = C.c_void_p()
    st = L.zolo_ctx_create(device, C.byref(h))
    if st != 0:
        raise CudaError(L.zolo_last_error(None).decode())
    try:
        n_ss = config.subspace_size()
        lam = np.zeros(n_ss)
        nf = np.zeros(1, dtype=np.int64)
        vec = np.zeros((n, n_ss), dtype=np.complex128 if cx else np.float64, order="F") if want_vectors else None
        stats = np.zeros(14)
        st = L.zolo_subspace_iteration(h, int(n), int(cx), *map(_ptr, ac), *map(_ptr, bc), _ptr(design), r,
                                       config.n_lambda, config.oversample_k, config.tol, config.max_subspace_iters,
                                       config.gmres_tol, config.gmres_max, config.seed, refine, _ptr(lam), _ptr(nf),
                                       _ptr(vec), _ptr(stats))
        _check(h, st)
        k = int(nf[0])
        vectors = None
        if want_vectors:
            vectors = np.asfortranarray(vec.reshape(-1, order="F")[: n * k].reshape(n, k, order="F"))
        s = SolveStats(n_ss=int(stats[0]), n_iter=int(stats[1]), n_gmres=int(stats[2]), n_gmres_min=int(stats[3]),
                       n_solv=int(stats[4]), factorization_time=float(stats[5]) + t_design,
                       iteration_time=float(stats[6]), filter_device_ms=float(stats[11]),
                       refined_from=int(stats[12]), first_residual=float(stats[13]))
        return EigResult(lambdas=lam[:k].copy(), vectors=vectors, residual=float(stats[7]),
                         residual_rel_lambda=float(stats[10]), stats=s, converged=bool(stats[8]), r=int(stats[9]))
    finally:
        L.zolo_ctx_destroy(h)
