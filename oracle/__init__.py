"""TEST INFRASTRUCTURE ONLY: ctypes access to the two CPU checkers.

* ``Oracle``    -- our C restatement of the reference hot path (oracle/zolo_oracle.c
                   -> oracle/liboracle.so).
* ``Reference`` -- the unmodified reference library compiled in place
                   (oracle/ref_harness.cpp -> oracle/_ref/libzoloref.so, see
                   oracle/Makefile). Absent on machines without /root/reference
                   unless a prebuilt copy travelled with the repo.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package; the product never does.

Pencils are passed as ``(n, (rp, ci, vals), (rp, ci, vals) | None)`` with int64
CSR arrays (full pattern, sorted columns: sparse.hpp:31-91) and float64 or
complex128 values. Dense blocks are column-major (Fortran-ordered) numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libzoloref.so")

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double

STATUS = {0: "ok", 1: "domain", 2: "numerical", 3: "factorization", 4: "gmres"}


def design_len(r: int) -> int:
    return 17 + 10 * r


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _as_f(a, cx):
    """Column-major float64/complex128 copy, viewed as interleaved doubles."""
    dt = np.complex128 if cx else np.float64
    return np.asfortranarray(np.asarray(a, dtype=dt))


def _csr_args(pencil, cx):
    n, a, b = pencil
    keep = []

    def one(m):
        if m is None:
            return (None, None, None)
        rp = np.ascontiguousarray(m[0], dtype=np.int64)
        ci = np.ascontiguousarray(m[1], dtype=np.int64)
        v = np.ascontiguousarray(m[2], dtype=np.complex128 if cx else np.float64)
        keep.extend([rp, ci, v])
        return (_ptr(rp), _ptr(ci), _ptr(v))

    return (int(n),) + one(a) + one(b), keep


def build(ref: bool = True) -> None:
    """Compile the checkers (oracle/Makefile). Reference only if its headers exist."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class _Lib:
    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)


class Reference(_Lib):
    """The reference library itself (oracle/_ref/libzoloref.so)."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        self.lib.zr_last_error.restype = C.c_char_p

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def _check(self, st):
        if st != 0:
            raise RuntimeError(f"reference: {STATUS.get(st, st)}: {self.lib.zr_last_error().decode()}")

    def design(self, gaps, r):
        out = np.zeros(design_len(r))
        g = np.asarray(gaps, dtype=np.float64)
        self._check(self.lib.zr_design(_ptr(g), C.c_int(r), _ptr(out)))
        return out

    def eval_scalar(self, gaps, r, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.asarray(gaps, dtype=np.float64)
        gv = np.zeros_like(x)
        fv = np.zeros_like(x)
        self._check(self.lib.zr_eval_scalar(_ptr(g), C.c_int(r), _I64(x.size), _ptr(x), _ptr(gv), _ptr(fv)))
        return gv, fv

    def read_mm(self, path):
        """read_matrix_market through the reference: (n, (rp, ci, vals), is_complex)."""
        n, nnz = _I64(0), _I64(0)
        cx = C.c_int(0)
        p = str(path).encode()
        self._check(self.lib.zr_read_mm(p, C.byref(n), C.byref(nnz), C.byref(cx), None, None, None))
        rp = np.zeros(n.value + 1, dtype=np.int64)
        ci = np.zeros(nnz.value, dtype=np.int64)
        v = np.zeros(nnz.value, dtype=np.complex128 if cx.value else np.float64)
        self._check(self.lib.zr_read_mm(p, C.byref(n), C.byref(nnz), C.byref(cx), _ptr(rp), _ptr(ci), _ptr(v)))
        return int(n.value), (rp, ci, v), bool(cx.value)

    def write_mm(self, path, n, csr, cx):
        rp = np.ascontiguousarray(csr[0], dtype=np.int64)
        ci = np.ascontiguousarray(csr[1], dtype=np.int64)
        v = np.ascontiguousarray(csr[2], dtype=np.complex128 if cx else np.float64)
        self._check(self.lib.zr_write_mm(str(path).encode(), C.c_int(int(cx)), _I64(n), _ptr(rp), _ptr(ci), _ptr(v)))

    def write_eigvec(self, path, x):
        cx = np.iscomplexobj(x)
        x = _as_f(x, cx)
        self._check(self.lib.zr_write_eigvec(str(path).encode(), C.c_int(int(cx)), _I64(x.shape[0]), _I64(x.shape[1]),
                                             _ptr(x)))

    def read_eigvec(self, path, n, k, cx):
        x = np.zeros((n, k), dtype=np.complex128 if cx else np.float64, order="F")
        self._check(self.lib.zr_read_eigvec(str(path).encode(), C.c_int(int(cx)), _I64(n), _I64(k), _ptr(x)))
        return x

    def uniform_stream(self, seed, n):
        out = np.zeros(int(n))
        self._check(self.lib.zr_uniform_stream(C.c_uint64(seed), _I64(n), _ptr(out)))
        return out

    def choose_order(self, gaps, eps):
        g = np.asarray(gaps, dtype=np.float64)
        r = C.c_int(0)
        b = np.zeros(1)
        self._check(self.lib.zr_choose_order(_ptr(g), _D(eps), C.byref(r), _ptr(b)))
        return int(r.value), float(b[0])

    def random_block(self, n, k, seed, cx=False, orthonormalize=False):
        out = np.zeros((n, k), dtype=np.complex128 if cx else np.float64, order="F")
        self._check(self.lib.zr_random_block(C.c_int(int(cx)), _I64(n), _I64(k), C.c_uint64(seed),
                                             C.c_int(int(orthonormalize)), _ptr(out)))
        return out

    def rcm(self, n, rp, ci):
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.int64)
        perm = np.zeros(n, dtype=np.int64)
        bw = np.zeros(1, dtype=np.int64)
        prof = np.zeros(1, dtype=np.int64)
        self._check(self.lib.zr_rcm(_I64(n), _ptr(rp), _ptr(ci), _ptr(perm), _ptr(bw), _ptr(prof)))
        return perm, int(bw[0]), int(prof[0])

    def shifted_solve(self, pencil, cx, sigma, rhs):
        args, keep = _csr_args(pencil, cx)
        n = args[0]
        rhs = _as_f(rhs, True)
        k = rhs.shape[1]
        x = np.zeros((n, k), dtype=np.complex128, order="F")
        xa = np.zeros_like(x)
        perm = np.zeros(n, dtype=np.int64)
        bw = np.zeros(1, dtype=np.int64)
        mr = np.zeros(1)
        piv = np.zeros(1, dtype=np.int64)
        st = self.lib.zr_shifted_solve(C.c_int(int(cx)), _I64(args[0]), *args[1:], _D(sigma.real), _D(sigma.imag),
                                       _I64(k), _ptr(rhs), _ptr(x), _ptr(xa), _ptr(perm), _ptr(bw), _ptr(mr), _ptr(piv))
        return dict(status=st, x=x, xa=xa, perm=perm, bw=int(bw[0]), min_ratio=float(mr[0]), pivot_index=int(piv[0]))

    def apply_g(self, pencil, cx, gaps, r, v):
        args, keep = _csr_args(pencil, cx)
        v = _as_f(v, cx)
        out = np.zeros_like(v)
        cnt = np.zeros(2, dtype=np.int64)
        g = np.asarray(gaps, dtype=np.float64)
        self._check(self.lib.zr_apply_g(C.c_int(int(cx)), _I64(args[0]), *args[1:], _ptr(g), C.c_int(r),
                                        _I64(v.shape[1]), _ptr(v), _ptr(out), _ptr(cnt)))
        return out, cnt

    def apply_filter(self, pencil, cx, gaps, r, v, gmres_tol=1e-12, gmres_max=50, threads=0):
        args, keep = _csr_args(pencil, cx)
        v = _as_f(v, cx)
        k = v.shape[1]
        y = np.zeros_like(v)
        col = np.zeros(k, dtype=np.int64)
        res = np.zeros(2 * r)
        conv = np.zeros(2 * r, dtype=np.int32)
        it = np.zeros(1, dtype=np.int64)
        ops = np.zeros(1, dtype=np.int64)
        cnt = np.zeros(2, dtype=np.int64)
        sec = np.zeros(2)
        g = np.asarray(gaps, dtype=np.float64)
        st = self.lib.zr_apply_filter(C.c_int(int(cx)), _I64(args[0]), *args[1:], _ptr(g), C.c_int(r),
                                      _D(gmres_tol), _I64(gmres_max), C.c_int(threads), _I64(k), _ptr(v), _ptr(y),
                                      _ptr(col), _ptr(res), _ptr(conv), _ptr(it), _ptr(ops), _ptr(cnt), _ptr(sec))
        if st not in (0, 4):
            self._check(st)
        return dict(status=st, y=y, column_iterations=col, residuals=res, converged=conv.astype(bool),
                    iterations=int(it[0]), operator_applications=int(ops[0]), inner_solves=int(cnt[0]),
                    g_applications=int(cnt[1]), t_factor=float(sec[0]), t_filter=float(sec[1]))

    def operator(self, pencil, cx, gaps, r, threads=0):
        """Persistent reference FilterOperator<S> (factorized once)."""
        return RefOperator(self, pencil, cx, gaps, r, threads)

    def rayleigh_ritz(self, pencil, cx, y):
        args, keep = _csr_args(pencil, cx)
        y = _as_f(y, cx)
        k = y.shape[1]
        ritz = np.zeros(k)
        q = np.zeros((k, k), dtype=y.dtype, order="F")
        kept = np.zeros(1, dtype=np.int64)
        self._check(self.lib.zr_rayleigh_ritz(C.c_int(int(cx)), _I64(args[0]), *args[1:], _I64(k), _ptr(y),
                                              _ptr(ritz), _ptr(q), _ptr(kept)))
        kk = int(kept[0])
        return ritz[:kk], np.asfortranarray(q.reshape(-1, order="F")[: k * kk].reshape(k, kk, order="F"))

    def subspace_iteration(self, pencil, cx, gaps, n_lambda, oversample, r, tol=1e-10, max_iters=5,
                           gmres_tol=1e-12, gmres_max=50, seed=0, threads=0, want_vectors=False):
        args, keep = _csr_args(pencil, cx)
        n = args[0]
        n_ss = n_lambda + oversample
        lam = np.zeros(n_ss)
        nf = np.zeros(1, dtype=np.int64)
        vec = np.zeros((n, n_ss), dtype=np.complex128 if cx else np.float64, order="F") if want_vectors else None
        stats = np.zeros(10)
        g = np.asarray(gaps, dtype=np.float64)
        self._check(self.lib.zr_subspace_iteration(
            C.c_int(int(cx)), _I64(n), *args[1:], _ptr(g), _I64(n_lambda), _I64(oversample), C.c_int(r), _D(tol),
            _I64(max_iters), _D(gmres_tol), _I64(gmres_max), C.c_uint64(seed), C.c_int(threads), _ptr(lam),
            _ptr(nf), _ptr(vec), _ptr(stats)))
        k = int(nf[0])
        out = dict(lambdas=lam[:k], n_ss=int(stats[0]), n_iter=int(stats[1]), n_gmres=int(stats[2]),
                   n_gmres_min=int(stats[3]), n_solv=int(stats[4]), t_fact=float(stats[5]),
                   t_iter=float(stats[6]), residual=float(stats[7]), converged=bool(stats[8]), r=int(stats[9]))
        if want_vectors:
            out["vectors"] = np.asfortranarray(vec.reshape(-1, order="F")[: n * k].reshape(n, k, order="F"))
        return out

    def dense_filter_oracle(self, a, b, cx, gaps, r, v):
        a = _as_f(a, cx)
        b = _as_f(b, cx)
        v = _as_f(v, cx)
        n = a.shape[0]
        out = np.zeros_like(v)
        lam = np.zeros(n)
        g = np.asarray(gaps, dtype=np.float64)
        self._check(self.lib.zr_dense_filter_oracle(C.c_int(int(cx)), _I64(n), _ptr(a), _ptr(b), _ptr(g),
                                                    C.c_int(r), _I64(v.shape[1]), _ptr(v), _ptr(out), _ptr(lam)))
        return out, lam


class RefOperator:
    """The reference's own FilterOperator<S> (oracle/_ref), for timing."""

    def __init__(self, ref, pencil, cx, gaps, r, threads):
        self.ref = ref
        self.cx = bool(cx)
        self.n = int(pencil[0])
        args, self._keep = _csr_args(pencil, cx)
        g = np.asarray(gaps, dtype=np.float64)
        tf = np.zeros(1)
        ref.lib.zr_op_create.restype = _P
        self.h = ref.lib.zr_op_create(C.c_int(int(cx)), _I64(args[0]), *args[1:], _ptr(g), C.c_int(r),
                                      C.c_int(threads), _ptr(tf))
        if not self.h:
            raise RuntimeError("reference: " + ref.lib.zr_last_error().decode())
        self.t_factor = float(tf[0])

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.zr_op_free(_P(self.h))
            self.h = None

    def apply_filter(self, v, gmres_tol=1e-12, gmres_max=50):
        v = _as_f(v, self.cx)
        y = np.zeros_like(v)
        it = np.zeros(1, dtype=np.int64)
        sec = np.zeros(1)
        st = self.ref.lib.zr_op_apply_filter(_P(self.h), _D(gmres_tol), _I64(gmres_max), _I64(self.n),
                                             _I64(v.shape[1]), _ptr(v), _ptr(y), _ptr(it), _ptr(sec))
        if st != 0:
            raise RuntimeError("reference: " + self.ref.lib.zr_last_error().decode())
        return y, int(it[0]), float(sec[0])


class Oracle(_Lib):
    """Our C restatement (oracle/liboracle.so); designs are passed packed."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        super().__init__(path)
        self.lib.or_op_create.restype = _P

    def rcm(self, n, rp, ci):
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.int64)
        perm = np.zeros(n, dtype=np.int64)
        self.lib.or_rcm(_I64(n), _ptr(rp), _ptr(ci), _ptr(perm))
        return perm

    def spmv(self, csr, cx_mat, n, x):
        rp, ci, vals = csr
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        ci = np.ascontiguousarray(ci, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.complex128 if cx_mat else np.float64)
        cx_x = np.iscomplexobj(x)
        x = _as_f(x, cx_x)
        y = np.zeros(x.shape, dtype=np.complex128 if (cx_x or cx_mat) else np.float64, order="F")
        self.lib.or_spmv(C.c_int(int(cx_mat)), _I64(n), _ptr(rp), _ptr(ci), _ptr(vals), C.c_int(int(cx_x)),
                         _I64(x.shape[1]), _ptr(x), _ptr(y))
        return y

    def shifted_solve(self, pencil, cx, sigma, rhs):
        args, keep = _csr_args(pencil, cx)
        n = args[0]
        rhs = _as_f(rhs, True)
        k = rhs.shape[1]
        x = np.zeros((n, k), dtype=np.complex128, order="F")
        xa = np.zeros_like(x)
        perm = np.zeros(n, dtype=np.int64)
        bw = np.zeros(1, dtype=np.int64)
        mr = np.zeros(1)
        piv = np.zeros(1, dtype=np.int64)
        st = self.lib.or_shifted_solve(C.c_int(int(cx)), _I64(n), *args[1:], _D(sigma.real), _D(sigma.imag),
                                       _I64(k), _ptr(rhs), _ptr(x), _ptr(xa), _ptr(perm), _ptr(bw), _ptr(mr), _ptr(piv))
        return dict(status=st, x=x, xa=xa, perm=perm, bw=int(bw[0]), min_ratio=float(mr[0]), pivot_index=int(piv[0]))

    def operator(self, pencil, cx, design, r):
        return OracleOperator(self, pencil, cx, design, r)


class OracleOperator:
    """Mirror of FilterOperator<S> (filter_engine.hpp:37-165) over liboracle."""

    def __init__(self, oracle, pencil, cx, design, r):
        self.o = oracle
        self.cx = bool(cx)
        self.r = r
        self.n = int(pencil[0])
        args, self._keep = _csr_args(pencil, cx)
        self._design = np.ascontiguousarray(design, dtype=np.float64)
        st = C.c_int(0)
        piv = np.full(1, -1, dtype=np.int64)
        self.h = oracle.lib.or_op_create(C.c_int(int(cx)), _I64(args[0]), *args[1:], _ptr(self._design), C.c_int(r),
                                         C.byref(st), _ptr(piv))
        if not self.h:
            raise RuntimeError(f"oracle factorization failed at pivot {int(piv[0])}")

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.or_op_free(_P(self.h))
            self.h = None

    def counters(self):
        out = np.zeros(2, dtype=np.int64)
        self.o.lib.or_counters(_P(self.h), _ptr(out))
        return int(out[0]), int(out[1])

    def apply_g(self, v):
        v = _as_f(v, self.cx)
        out = np.zeros_like(v)
        self.o.lib.or_apply_g(_P(self.h), _I64(v.shape[1]), _ptr(v), _ptr(out))
        return out

    def apply_filter(self, v, gmres_tol=1e-12, gmres_max=50):
        v = _as_f(v, self.cx)
        k = v.shape[1]
        y = np.zeros_like(v)
        col = np.zeros(k, dtype=np.int64)
        res = np.zeros(2 * self.r)
        conv = np.zeros(2 * self.r, dtype=np.int32)
        it = np.zeros(1, dtype=np.int64)
        ops = np.zeros(1, dtype=np.int64)
        st = self.o.lib.or_apply_filter(_P(self.h), _D(gmres_tol), _I64(gmres_max), _I64(k), _ptr(v), _ptr(y),
                                        _ptr(col), _ptr(res), _ptr(conv), _ptr(it), _ptr(ops))
        return dict(status=st, y=y, column_iterations=col, residuals=res, converged=conv.astype(bool),
                    iterations=int(it[0]), operator_applications=int(ops[0]))
