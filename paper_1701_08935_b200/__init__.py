"""B200-native Zolotarev filter path (ZoloEig, arXiv 1701.08935).

Python mirror of the reference's hot-path API over the C ABI in
``include/zolo_b200.h`` (``libzolo_b200.so``, sm_100a):

* :class:`FilterOperator` -- ``FilterOperator<S>`` (filter_engine.hpp:37-165):
  ``apply_g``, ``apply_filter``, ``inner_solve_count``, ``g_application_count``.
* exceptions with the reference's names and fields (error.hpp:25-43,
  gmres.hpp:45-52): :class:`DomainError`, :class:`NumericalError`,
  :class:`FactorizationError` (``pivot_index``), :class:`GmresError` (``report``).
* :class:`ShiftedSolveReport` (gmres.hpp:31-43).
* :func:`subspace_iteration` (eigensolver.hpp:154-217) in ``driver.py``.

There is no CPU fallback: constructing an operator without a CUDA device or
without the built extension raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZOLO_LIB_PATH") or os.path.join(HERE, "libzolo_b200.so")  # (override: development builds)

ZOLO_OK, ZOLO_ERR_DOMAIN, ZOLO_ERR_NUMERICAL, ZOLO_ERR_FACTORIZATION, ZOLO_ERR_GMRES, ZOLO_ERR_CUDA = range(6)
MAX_ORDER = 16
# factor layouts (include/zolo_b200.h ZOLO_ORDER_*): nested-dissection block-sparse
# factors with DAG-scheduled sweeps, or the reference's RCM band.
ORDERINGS = {"nd": 0, "rcm": 1}


class DomainError(ValueError):
    """Invalid argument or out-of-domain input (error.hpp:25-29)."""


class NumericalError(RuntimeError):
    """Numerical breakdown inside an algorithm (error.hpp:32-35)."""


class FactorizationError(NumericalError):
    """Unpivoted elimination met a pivot below threshold (error.hpp:37-43)."""

    def __init__(self, what: str, pivot_index: int):
        super().__init__(what)
        self.pivot_index = pivot_index


class GmresError(NumericalError):
    """Multi-shift GMRES missed the tolerance (gmres.hpp:45-52)."""

    def __init__(self, what: str, report: "ShiftedSolveReport", y=None):
        super().__init__(what)
        self.report = report
        self.y = y


class CudaError(RuntimeError):
    """Device / driver failure (no silent CPU fallback exists)."""


@dataclass
class ShiftedSolveReport:
    """gmres.hpp:31-43, merged over columns as filter_engine.hpp:127-133."""

    iterations: int = 0
    residuals: List[float] = field(default_factory=list)
    converged: List[bool] = field(default_factory=list)
    column_iterations: List[int] = field(default_factory=list)
    operator_applications: int = 0

    def all_converged(self) -> bool:
        return all(self.converged)


class _Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64),
        ("operator_applications", C.c_int64),
        ("n_shifts", C.c_int32),
        ("all_converged", C.c_int32),
        ("residuals", C.c_double * (2 * MAX_ORDER)),
        ("converged", C.c_int32 * (2 * MAX_ORDER)),
        ("column_iterations", C.POINTER(C.c_int64)),
    ]


class FactorStats(C.Structure):
    """FactorProfile (band_factor.hpp:31-35) + the rejected pivot index."""

    _fields_ = [
        ("bandwidth", C.c_int64),
        ("stored_entries", C.c_int64),
        ("min_pivot_ratio", C.c_double),
        ("pivot_index", C.c_int64),
    ]


_lib = None
# zolo_collective_fn (include/zolo_b200.h): op, buffer of doubles, count, user
COLLECTIVE_FN = C.CFUNCTYPE(C.c_int, C.c_int, C.POINTER(C.c_double), C.c_int64, C.c_void_p)


def build() -> None:
    """Compile libzolo_b200.so for sm_100a (nvcc cross-compiles without a GPU)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(f"native extension missing: {LIB_PATH} (run paper_1701_08935_b200.build())")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        I64 = C.c_int64
        D = C.c_double
        L.zolo_last_error.restype = C.c_char_p
        L.zolo_last_error.argtypes = [P]
        L.zolo_version.restype = C.c_char_p
        L.zolo_ctx_create.argtypes = [C.c_int, C.POINTER(P)]
        L.zolo_ctx_destroy.argtypes = [P]
        L.zolo_pencil_upload.argtypes = [P, I64, C.c_int, P, P, P, P, P, P]
        L.zolo_set_design.argtypes = [P, P, C.c_int]
        L.zolo_set_ordering.argtypes = [P, C.c_int, I64]
        L.zolo_set_pole_shard.argtypes = [P, C.c_int, C.c_int, C.c_char_p]
        L.zolo_set_pole_shard_host.argtypes = [P, C.c_int, C.c_int, COLLECTIVE_FN, P]
        L.zolo_set_block_size.argtypes = [P, I64]
        L.zolo_nccl_unique_id.argtypes = [C.c_char_p]
        L.zolo_count_below.argtypes = [P, D, P, P]
        L.zolo_set_solve_mode.argtypes = [P, C.c_int, C.c_int, D, C.c_int]
        L.zolo_factorize.argtypes = [P, P, P]
        L.zolo_apply_g.argtypes = [P, P, P, I64]
        L.zolo_shifted_solve.argtypes = [P, C.c_int, C.c_int, P, P, I64]
        L.zolo_apply_filter.argtypes = [P, P, P, I64, D, I64, C.POINTER(_Report)]
        L.zolo_apply_filter_device.argtypes = [P, P, P, I64, D, I64, C.POINTER(_Report)]
        L.zolo_counters.argtypes = [P, P, P]
        L.zolo_rr_project.argtypes = [P, P, I64, P, P]
        L.zolo_block_update.argtypes = [P, P, I64, P, I64, P]
        L.zolo_last_timings.argtypes = [P, P]
        L.zolo_sweep_profile.argtypes = [P, P]
        L.zolo_timer.argtypes = [P, C.c_int, P]
        L.zolo_rcm.argtypes = [I64, P, P, P, P, P]
        L.zolo_random_block.argtypes = [C.c_int, I64, I64, C.c_uint64, C.c_int, P]
        L.zolo_uniform_stream.argtypes = [C.c_uint64, I64, P]
        L.zolo_set_refinement.argtypes = [P, C.c_int]
        L.zolo_pool_trim.argtypes = [C.c_int]
        _lib = L
    return _lib


NCCL_ID_BYTES = 128


def pool_trim(device: int = 0) -> None:
    """Return the device memory the library's allocator keeps cached to the driver."""
    lib().zolo_pool_trim(int(device))


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0), to broadcast to the pole-shard ranks."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    if lib().zolo_nccl_unique_id(buf) != ZOLO_OK:
        raise CudaError(lib().zolo_last_error(None).decode())
    return buf.raw


def shard_poles(r: int, rank: int, nranks: int):
    """Poles a pole-shard rank factors (zolo_set_pole_shard): j = rank, rank + nranks, ..."""
    return list(range(rank, r, nranks))


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def design_len(r: int) -> int:
    return 17 + 10 * r


def _check(ctx, st, pivot_index=-1):
    if st == ZOLO_OK:
        return
    msg = lib().zolo_last_error(ctx).decode()
    if st == ZOLO_ERR_DOMAIN:
        raise DomainError(msg)
    if st == ZOLO_ERR_FACTORIZATION:
        raise FactorizationError(msg, pivot_index)
    if st == ZOLO_ERR_NUMERICAL:
        raise NumericalError(msg)
    if st == ZOLO_ERR_CUDA:
        raise CudaError(msg)
    raise NumericalError(msg)


def _check_host(st):
    if st == ZOLO_OK:
        return
    msg = lib().zolo_last_error(None).decode()
    if st == ZOLO_ERR_DOMAIN:
        raise DomainError(msg)
    raise NumericalError(msg)


def rcm(n, rp, ci):
    """reorder_rcm (rcm.hpp:69-115): perm[new] = old, plus bandwidth/profile."""
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    perm = np.zeros(n, dtype=np.int64)
    bw = np.zeros(1, dtype=np.int64)
    prof = np.zeros(1, dtype=np.int64)
    lib().zolo_rcm(n, _ptr(rp), _ptr(ci), _ptr(perm), _ptr(bw), _ptr(prof))
    return perm, int(bw[0]), int(prof[0])


def random_block(n, k, seed, cx=False, orthonormalize=False):
    """random_gaussian<S> (+ mgs_orthonormalize), dense.hpp:181-229, bit-reproducible."""
    out = np.zeros((n, k), dtype=np.complex128 if cx else np.float64, order="F")
    st = lib().zolo_random_block(int(cx), n, k, seed, int(orthonormalize), _ptr(out))
    if st != ZOLO_OK:
        raise NumericalError("random block failed to orthonormalize")
    return out


def _csr(m, cx):
    rp = np.ascontiguousarray(m[0], dtype=np.int64)
    ci = np.ascontiguousarray(m[1], dtype=np.int64)
    v = np.ascontiguousarray(m[2], dtype=np.complex128 if cx else np.float64)
    return rp, ci, v


class InertiaCounter:
    """Eigenvalue counts of the pencil (A, B) by Sylvester inertia on the GPU
    (zolo_count_below): the unpivoted block LU of
    A - sigma B under the ND ordering has as many negative pivots as the pencil
    has eigenvalues below sigma (B positive definite)."""

    def __init__(self, pencil, is_complex: Optional[bool] = None, device: int = 0, nd_leaf: int = 192):
        L = lib()
        n, a, b = pencil
        cx = bool(is_complex) if is_complex is not None else np.iscomplexobj(a[2])
        self.n, self.cx = int(n), cx
        h = C.c_void_p()
        if L.zolo_ctx_create(device, C.byref(h)) != ZOLO_OK:
            raise CudaError(L.zolo_last_error(None).decode())
        self._h = h
        self._a = _csr(a, cx)
        self._b = _csr(b, cx) if b is not None else None
        bp = self._b if self._b is not None else (None, None, None)
        _check(h, L.zolo_pencil_upload(h, self.n, int(cx), *map(_ptr, self._a), *map(_ptr, bp)))
        _check(h, L.zolo_set_ordering(h, ORDERINGS["nd"], int(nd_leaf)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:
            lib().zolo_ctx_destroy(h)
            self._h = None

    def _count_once(self, s: float):
        out = np.zeros(1, dtype=np.int64)
        ratio = np.zeros(1)
        st = lib().zolo_count_below(self._h, C.c_double(s), _ptr(out), _ptr(ratio))
        return st, int(out[0]), float(ratio[0])

    def count_below(self, sigma: float, nudges: int = 3, growth_ratio: float = 1e-8) -> int:
        """Eigenvalues < sigma. A shift within rounding of an eigenvalue (rejected pivot) is
        nudged by 1e-12 relative, up to `nudges` times. The real-shift LU is unpivoted (the
        pencil A - sigma B is Hermitian indefinite): when its smallest pivot ratio is below
        `growth_ratio` -- where element growth could flip a pivot's sign -- the count is
        confirmed at two shifts 1e-10 (relative) to either side, which must agree (no eigenvalue
        lies that close); otherwise NumericalError."""
        s = float(sigma)
        for k in range(nudges + 1):
            st, cnt, ratio = self._count_once(s)
            if st != ZOLO_ERR_FACTORIZATION:
                _check(self._h, st)
                self.last_min_pivot_ratio = ratio
                if ratio < growth_ratio:
                    h = 1e-10 * max(1.0, abs(s))
                    lo, hi = self._count_once(s - h), self._count_once(s + h)
                    if lo[0] != ZOLO_OK or hi[0] != ZOLO_OK or not (lo[1] == cnt == hi[1]):
                        raise NumericalError(f"inertia count at {s!r} unstable (min pivot ratio {ratio:.2e}; "
                                             f"neighbouring counts {lo[1]}, {cnt}, {hi[1]})")
                return cnt
            s = float(sigma) + (k + 1) * 1e-12 * max(1.0, abs(float(sigma)))
        _check(self._h, st)

    def structure(self):
        """Block structure of the ND factors (zolo_sweep_profile; after a count)."""
        out = np.zeros(8, dtype=np.int64)
        _check(self._h, lib().zolo_sweep_profile(self._h, _ptr(out)))
        return dict(block_rows=int(out[0]), offdiag_tiles=int(out[1]), critical_path=int(out[5]))

    def count_in(self, a: float, b: float) -> int:
        """Eigenvalues in (a, b) = count_below(b) - count_below(a); an infinite end (the
        reference's SpectralWindow allows one, window.hpp:28-52) counts all or none."""
        n = self.n
        below_b = n if b == np.inf else self.count_below(b)
        below_a = 0 if a == -np.inf else self.count_below(a)
        return below_b - below_a


class FilterOperator:
    """GPU FilterOperator<S> (filter_engine.hpp:37-165).

    ``pencil`` = ``(n, A, B)`` with ``A``/``B`` = ``(rp, ci, vals)`` CSR (full
    pattern, sorted columns; B ``None`` = identity). ``design`` is the packed
    FilterDesign of ``include/zolo_b200.h`` (e.g. from
    :func:`paper_1701_08935_b200.design.build_filter_design`); ``r`` its order.
    ``is_complex`` selects S = complex128 (Hermitian pencil) vs float64.
    ``shard=(rank, nranks, unique_id)`` makes this operator one pole shard of a
    multi-GPU operator (zolo_set_pole_shard): it factors the poles
    :func:`shard_poles` gives and reduces every G application over NCCL (row-sharded
    Arnoldi by default); ``unique_id=None`` leaves G unreduced (``apply_g`` returns the
    partial sum). ``shard=(rank, nranks, fn)`` with a :data:`COLLECTIVE_FN` callback
    stages the group's collectives through the host instead (zolo_set_pole_shard_host;
    sharding.py builds them over torch.distributed or over threads of one process).
    ``block_size=b`` declares a BSR pencil (atoms of b rows, BASELINE config 4;
    zolo_set_block_size): the ordering keeps atoms whole and the SpMMs use BSR.
    ``solve="hybrid"`` factors only pole ``hybrid_pole`` and solves the other
    shifted systems by shift-invariant GMRES on K_p^{-1} B (zolo_set_solve_mode;
    BASELINE config 2) to ``inner_tol`` within ``inner_max`` iterations.
    ``refine=k`` adds k residual-correction steps to every shifted solve
    (zolo_set_refinement; 0 = the reference's plain solve).
    """

    def __init__(self, pencil, design, r: int, is_complex: Optional[bool] = None, device: int = 0, perm=None,
                 ordering: str = "nd", nd_leaf: int = 192, shard=None, solve: str = "direct", hybrid_pole: int = 0,
                 inner_tol: float = 1e-14, inner_max: int = 256, block_size: int = 1, refine: int = 0):
        L = lib()
        n, a, b = pencil
        cx = bool(is_complex) if is_complex is not None else np.iscomplexobj(a[2])
        self.n = int(n)
        self.cx = cx
        self.r = int(r)
        self.design = np.ascontiguousarray(design, dtype=np.float64)
        if self.design.size != design_len(self.r):
            raise DomainError("design length does not match order r")
        h = C.c_void_p()
        st = L.zolo_ctx_create(device, C.byref(h))
        if st != ZOLO_OK:
            raise CudaError(L.zolo_last_error(None).decode())
        self._h = h
        self._a = _csr(a, cx)
        self._b = _csr(b, cx) if b is not None else None
        bp = self._b if self._b is not None else (None, None, None)
        _check(h, L.zolo_pencil_upload(h, self.n, int(cx), *map(_ptr, self._a), *map(_ptr, bp)))
        _check(h, L.zolo_set_design(h, _ptr(self.design), self.r))
        if ordering not in ORDERINGS:
            raise DomainError(f"ordering must be one of {sorted(ORDERINGS)}")
        _check(h, L.zolo_set_ordering(h, ORDERINGS[ordering], int(nd_leaf)))
        if block_size != 1:  # BSR pencil: atoms of block_size rows (zolo_set_block_size)
            _check(h, L.zolo_set_block_size(h, int(block_size)))
        self.shard = (0, 1) if shard is None else (int(shard[0]), int(shard[1]))
        if shard is not None:
            uid = shard[2] if len(shard) > 2 else None
            if isinstance(uid, COLLECTIVE_FN):
                self._collective = uid  # keep the callback alive
                _check(h, L.zolo_set_pole_shard_host(h, self.shard[0], self.shard[1], uid, None))
            else:
                _check(h, L.zolo_set_pole_shard(h, self.shard[0], self.shard[1], uid))
        self.poles = shard_poles(self.r, *self.shard)
        if solve not in ("direct", "hybrid"):
            raise DomainError("solve must be 'direct' or 'hybrid'")
        self.solve = solve
        if solve == "hybrid":
            _check(h, L.zolo_set_solve_mode(h, 1, int(hybrid_pole), float(inner_tol), int(inner_max)))
            self.poles = [int(hybrid_pole)]
        if refine:
            _check(h, L.zolo_set_refinement(h, int(refine)))
        self.stats = (FactorStats * self.r)()
        perm_arr = None if perm is None else np.ascontiguousarray(perm, dtype=np.int64)
        st = L.zolo_factorize(h, _ptr(perm_arr), self.stats)
        if st == ZOLO_ERR_FACTORIZATION:
            piv = min((s.pivot_index for s in self.stats if s.pivot_index >= 0), default=-1)
            _check(h, st, piv)
        _check(h, st)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and lib is not None:  # (module globals may be gone at exit)
            lib().zolo_ctx_destroy(h)
            self._h = None

    # --- reference surface -------------------------------------------------
    def dim(self) -> int:
        return self.n

    def inner_solve_count(self) -> int:
        a = np.zeros(1, dtype=np.int64)
        b = np.zeros(1, dtype=np.int64)
        lib().zolo_counters(self._h, _ptr(a), _ptr(b))
        return int(a[0])

    def g_application_count(self) -> int:
        a = np.zeros(1, dtype=np.int64)
        b = np.zeros(1, dtype=np.int64)
        lib().zolo_counters(self._h, _ptr(a), _ptr(b))
        return int(b[0])

    def _block(self, v):
        v = np.asarray(v)
        if v.ndim == 1:
            v = v[:, None]
        if v.shape[0] != self.n:
            raise DomainError("dimension mismatch")
        return np.asfortranarray(v, dtype=np.complex128 if self.cx else np.float64)

    def apply_g(self, v):
        """G v (filter_engine.hpp:56-82)."""
        v = self._block(v)
        out = np.zeros_like(v)
        _check(self._h, lib().zolo_apply_g(self._h, _ptr(v), _ptr(out), v.shape[1]))
        return out

    def shifted_solve(self, b, pole: int = 0, adjoint: bool = False):
        """ShiftedFactor::solve / adjoint_solve (band_factor.hpp:53-117) of the factored pole
        `pole`: (A - sigma_pole B)^-1 b or its adjoint, b an n x k (complex) block."""
        b = np.asarray(b)
        if b.ndim == 1:
            b = b[:, None]
        if b.shape[0] != self.n:
            raise DomainError("dimension mismatch")
        b = np.asfortranarray(b, dtype=np.complex128)
        x = np.zeros_like(b)
        _check(self._h, lib().zolo_shifted_solve(self._h, int(pole), int(bool(adjoint)), _ptr(b), _ptr(x), b.shape[1]))
        return x

    def apply_filter(self, v, gmres_tol: float = 1e-12, gmres_max: int = 50):
        """(R_ab(B^-1 A) V, report) (filter_engine.hpp:86-155). Raises GmresError."""
        v = self._block(v)
        k = v.shape[1]
        y = np.zeros_like(v)
        cols = np.zeros(k, dtype=np.int64)
        rep = _Report()
        rep.column_iterations = cols.ctypes.data_as(C.POINTER(C.c_int64))
        st = lib().zolo_apply_filter(self._h, _ptr(v), _ptr(y), k, float(gmres_tol), int(gmres_max), C.byref(rep))
        report = self._report(rep, cols)
        if st == ZOLO_ERR_GMRES:
            raise GmresError(lib().zolo_last_error(self._h).decode(), report, y)
        _check(self._h, st)
        return y, report

    def apply_filter_device(self, d_v: int, d_y: int, ncols: int, gmres_tol=1e-12, gmres_max=50):
        """Device-resident variant: raw device pointers (original ordering, ld = n)."""
        cols = np.zeros(ncols, dtype=np.int64)
        rep = _Report()
        rep.column_iterations = cols.ctypes.data_as(C.POINTER(C.c_int64))
        st = lib().zolo_apply_filter_device(self._h, C.c_void_p(d_v), C.c_void_p(d_y), ncols, float(gmres_tol),
                                            int(gmres_max), C.byref(rep))
        report = self._report(rep, cols)
        if st == ZOLO_ERR_GMRES:
            raise GmresError(lib().zolo_last_error(self._h).decode(), report)
        _check(self._h, st)
        return report

    @staticmethod
    def _report(rep, cols):
        q = rep.n_shifts
        return ShiftedSolveReport(
            iterations=int(rep.iterations),
            residuals=[float(rep.residuals[k]) for k in range(q)],
            converged=[bool(rep.converged[k]) for k in range(q)],
            column_iterations=[int(c) for c in cols],
            operator_applications=int(rep.operator_applications),
        )

    # --- Rayleigh-Ritz helpers (eigensolver.hpp:105-148,190) ---------------
    def rr_project(self, y):
        y = self._block(y)
        k = y.shape[1]
        at = np.zeros((k, k), dtype=y.dtype, order="F")
        bt = np.zeros((k, k), dtype=y.dtype, order="F")
        _check(self._h, lib().zolo_rr_project(self._h, _ptr(y), k, _ptr(at), _ptr(bt)))
        return at, bt

    def block_update(self, y, q):
        y = self._block(y)
        q = np.asfortranarray(q, dtype=y.dtype)
        out = np.zeros((self.n, q.shape[1]), dtype=y.dtype, order="F")
        _check(self._h, lib().zolo_block_update(self._h, _ptr(y), y.shape[1], _ptr(q), q.shape[1], _ptr(out)))
        return out

    def set_refinement(self, steps: int):
        """Residual-correction steps per shifted solve from the next application on."""
        _check(self._h, lib().zolo_set_refinement(self._h, int(steps)))

    def set_refinement_relaxation(self, on: bool):
        """Relaxed refinement (the default): a refined apply_filter skips the correction of the G
        applications whose GMRES residuals are already small -- zolo_set_refinement_relaxation."""
        _check(self._h, lib().zolo_set_refinement_relaxation(self._h, int(bool(on))))

    def refinement_stats(self):
        """(relative residual of the unrefined solves measured at the first refined application or
        -1, G applications of the last apply_filter that skipped the correction) --
        zolo_refinement_stats."""
        out = np.zeros(2)
        lib().zolo_refinement_stats(self._h, _ptr(out))
        return float(out[0]), int(out[1])

    def last_timings(self):
        ms = np.zeros(8)
        lib().zolo_last_timings(self._h, _ptr(ms))
        return dict(filter_ms=ms[0], factor_ms=ms[1], trsm_ms=ms[2], trsm_launches=int(ms[3]),
                    kernel_launches=int(ms[4]), operator_applications=int(ms[5]), inner_steps=int(ms[6]),
                    iterations_ms=ms[7])

    def bsr_info(self):
        """(block size, atoms of the device BSR copies or 0) -- zolo_bsr_info."""
        out = np.zeros(2, dtype=np.int64)
        lib().zolo_bsr_info(self._h, _ptr(out))
        return int(out[0]), int(out[1])

    def sweep_profile(self):
        """Structure the triangular sweeps run over (zolo_sweep_profile)."""
        out = np.zeros(8, dtype=np.int64)
        _check(self._h, lib().zolo_sweep_profile(self._h, _ptr(out)))
        return dict(block_rows=int(out[0]), offdiag_tiles=int(out[1]), fwd_tasks=int(out[2]),
                    bwd_tasks=int(out[3]), chunk_slots=int(out[4]), critical_path=int(out[5]),
                    nonzero_entries=int(out[6]), executed_entries=int(out[7]))

    def timer_start(self):
        _check(self._h, lib().zolo_timer(self._h, 0, None))

    def timer_stop(self) -> float:
        ms = np.zeros(1)
        _check(self._h, lib().zolo_timer(self._h, 1, _ptr(ms)))
        return float(ms[0])

    def factor_profile(self):
        return [dict(bandwidth=s.bandwidth, stored_entries=s.stored_entries, min_pivot_ratio=s.min_pivot_ratio)
                for s in list(self.stats)[:len(self.poles)]]
