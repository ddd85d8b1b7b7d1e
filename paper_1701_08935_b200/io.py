"""Host-side ingestion and result files.

Mirrors the reference's file formats so pencils and eigenvectors move between
the two implementations unchanged:

* Matrix Market coordinate files (matrix_market.hpp:48-190): real/complex
  field, symmetric/hermitian/general qualifier; symmetric files store the lower
  triangle and are expanded to the full pattern; duplicates are summed and exact
  zeros dropped (CsrMatrix::from_triplets, sparse.hpp:56-90); the result must be
  numerically Hermitian. Written back as the lower triangle with 17 significant
  digits (bit-exact round trip).
* BSR (block-sparse rows, the chemistry-shaped BASELINE config 4) expanded to
  the full-pattern CSR the filter path consumes.
* Eigenvector blocks: the "ZEIGVEC1" binary (serialize.hpp:108-140): magic,
  u64 n, u64 k, u32 scalar tag (0 real64, 1 complex128), column-major payload.
* Results: result_to_json / window_to_json of serialize.hpp:33-86.
"""
from __future__ import annotations

import json
import struct
from typing import List, Optional, Tuple

import numpy as np

from . import DomainError


class ParseError(DomainError):
    """Malformed Matrix Market input; the message names the line."""

    def __init__(self, what: str, line: int):
        super().__init__(f"{what} (line {line})")
        self.line = line


def _header(lines, path):
    if not lines:
        raise ParseError("matrix market: empty file", 1)
    tok = lines[0].split()
    if len(tok) < 5 or tok[0] != "%%MatrixMarket":
        raise ParseError("matrix market: missing banner", 1)
    obj, fmt, field, sym = (t.lower() for t in tok[1:5])
    if obj != "matrix" or fmt != "coordinate":
        raise ParseError("matrix market: only coordinate matrices are supported", 1)
    if field not in ("real", "complex"):
        raise ParseError(f"matrix market: unsupported field '{field}'", 1)
    if sym not in ("symmetric", "hermitian", "general"):
        raise ParseError(f"matrix market: unsupported symmetry '{sym}'", 1)
    comments, k = [], 1
    while k < len(lines):
        ln = lines[k]
        k += 1
        if ln.startswith("%"):
            comments.append(ln[1:])
            continue
        if not ln.strip():
            continue
        parts = ln.split()
        try:
            rows, cols, entries = int(parts[0]), int(parts[1]), int(parts[2])
        except (ValueError, IndexError):
            raise ParseError("matrix market: malformed size line", k) from None
        if rows == 0 or rows != cols:
            raise ParseError("matrix market: matrix must be square and nonempty", k)
        return dict(complex_field=field == "complex", symmetry=sym, n=rows, entries=entries, comments=comments), k
    raise ParseError("matrix market: missing size line", len(lines))


def probe_matrix_market(path: str) -> dict:
    """Header-only peek: field, symmetry, size, stored entry count, comments."""
    with open(path) as f:
        head = []
        for ln in f:
            head.append(ln.rstrip("\n"))
            if not ln.startswith("%") and ln.strip() and len(head) > 1:
                break
    return _header(head, path)[0]


def triplets_to_csr(n: int, i, j, v, cx: bool):
    """CsrMatrix::from_triplets: sort by (row, col), sum duplicates, drop exact zeros."""
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    v = np.asarray(v, dtype=np.complex128 if cx else np.float64)
    if i.size and (i.min() < 0 or j.min() < 0 or i.max() >= n or j.max() >= n):
        raise DomainError("CsrMatrix: triplet index out of range")
    order = np.lexsort((j, i))
    i, j, v = i[order], j[order], v[order]
    key = i * n + j
    if key.size:
        first = np.ones(key.size, dtype=bool)
        first[1:] = key[1:] != key[:-1]
        idx = np.flatnonzero(first)
        vs = np.add.reduceat(v, idx)
        i, j, v = i[idx], j[idx], vs
    keep = v != 0
    i, j, v = i[keep], j[keep], v[keep]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, i + 1, 1)
    return np.cumsum(rp), j, v


def is_hermitian(csr, n: int, tol: float = 1e-14) -> bool:
    import scipy.sparse as sp

    rp, ci, v = csr
    m = sp.csr_matrix((v, ci, rp), shape=(n, n))
    d = m - m.conj().T
    scale = max(1.0, float(np.abs(v).max()) if len(v) else 1.0)
    return (abs(d).max() if d.nnz else 0.0) <= tol * scale


def read_matrix_market(path: str, cx: Optional[bool] = None, comments: Optional[List[str]] = None):
    """Coordinate Matrix Market -> full-pattern CSR (rp, ci, vals) and n.
    cx=False on a complex file raises DomainError (as the reference)."""
    with open(path) as f:
        lines = [ln.rstrip("\n") for ln in f]
    info, k = _header(lines, path)
    n = info["n"]
    if info["complex_field"] and cx is False:
        raise DomainError("matrix market: complex file read into a real matrix")
    cxm = info["complex_field"] if cx is None else cx
    if comments is not None:
        comments[:] = info["comments"]
    ii, jj, vv = [], [], []
    seen = 0
    for ln_no in range(k + 1, len(lines) + 1):
        ln = lines[ln_no - 1]
        if not ln.strip() or ln.startswith("%"):
            continue
        p = ln.split()
        try:
            a, b = int(p[0]), int(p[1])
            re = float(p[2])
            im = float(p[3]) if info["complex_field"] else 0.0
        except (ValueError, IndexError):
            raise ParseError("matrix market: malformed entry", ln_no) from None
        if a < 1 or b < 1 or a > n or b > n:
            raise ParseError("matrix market: index out of range", ln_no)
        a, b = a - 1, b - 1
        val = complex(re, im) if cxm else re
        if info["symmetry"] != "general":
            if a < b:
                raise ParseError(f"matrix market: upper-triangle entry in a {info['symmetry']} file", ln_no)
            ii.append(a)
            jj.append(b)
            vv.append(val)
            if a != b:
                ii.append(b)
                jj.append(a)
                vv.append(val.conjugate() if cxm else val)
        else:
            ii.append(a)
            jj.append(b)
            vv.append(val)
        seen += 1
    if seen != info["entries"]:
        raise ParseError("matrix market: entry count does not match the size line", len(lines))
    csr = triplets_to_csr(n, ii, jj, vv, cxm)
    if not is_hermitian(csr, n):
        raise DomainError(f"matrix market: '{path}' is not numerically Hermitian")
    return n, csr


def write_matrix_market(path: str, n: int, csr, cx: bool, comments: Tuple[str, ...] = ()) -> None:
    """Lower triangle, symmetric (real) / hermitian (complex), 17 significant digits."""
    rp, ci, v = (np.asarray(x) for x in csr)
    rows = np.repeat(np.arange(n), np.diff(rp))
    low = ci <= rows
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate {'complex hermitian' if cx else 'real symmetric'}\n")
        for c in comments:
            f.write(f"%{c}\n")
        f.write(f"{n} {n} {int(low.sum())}\n")
        for r, c, x in zip(rows[low], ci[low], v[low]):
            if cx:
                f.write(f"{r + 1} {c + 1} {x.real:.17g} {x.imag:.17g}\n")
            else:
                f.write(f"{r + 1} {c + 1} {float(x):.17g}\n")


def bsr_to_csr(nb: int, bs: int, indptr, indices, blocks, cx: bool):
    """Block-sparse rows (nb block rows of bs x bs dense blocks, blocks[k] row-major)
    -> full-pattern CSR of order nb * bs (exact zeros inside blocks dropped)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    blocks = np.asarray(blocks, dtype=np.complex128 if cx else np.float64).reshape(-1, bs, bs)
    brow = np.repeat(np.arange(nb), np.diff(indptr))
    r = (brow[:, None, None] * bs + np.arange(bs)[None, :, None]) + 0 * np.arange(bs)[None, None, :]
    c = (indices[:, None, None] * bs + np.arange(bs)[None, None, :]) + 0 * np.arange(bs)[None, :, None]
    return triplets_to_csr(nb * bs, r.ravel(), c.ravel(), blocks.ravel(), cx)


def write_eigvec_binary(path: str, x: np.ndarray) -> None:
    """"ZEIGVEC1" file: u64 n, u64 k, u32 tag, column-major little-endian payload."""
    x = np.asarray(x)
    cx = np.iscomplexobj(x)
    n, k = x.shape
    with open(path, "wb") as f:
        f.write(b"ZEIGVEC1")
        f.write(struct.pack("<QQI", n, k, 1 if cx else 0))
        f.write(np.asfortranarray(x, dtype="<c16" if cx else "<f8").tobytes(order="F"))


def read_eigvec_binary(path: str, cx: Optional[bool] = None) -> np.ndarray:
    with open(path, "rb") as f:
        if f.read(8) != b"ZEIGVEC1":
            raise DomainError("bad eigenvector file magic")
        n, k, tag = struct.unpack("<QQI", f.read(20))
        if cx is not None and tag != (1 if cx else 0):
            raise DomainError("eigenvector scalar tag mismatch")
        dt = np.dtype("<c16" if tag == 1 else "<f8")
        buf = f.read(dt.itemsize * n * k)
        if len(buf) != dt.itemsize * n * k:
            raise DomainError("truncated eigenvector file")
    return np.frombuffer(buf, dtype=dt).reshape((n, k), order="F").copy()


def window_to_json(gaps) -> dict:
    """window_to_json (serialize.hpp:33-36) of window_from_gaps (window.hpp:56-68):
    a, b are the gap midpoints (an open end sits one interior width out);
    infinite endpoints serialize as null."""
    am, ap, bm, bp = (float(x) for x in gaps)
    span = bm - ap if bm > ap else 1.0
    a = ap - span if np.isinf(am) else 0.5 * (am + ap)
    b = bm + span if np.isinf(bp) else 0.5 * (bm + bp)
    fin = lambda x: None if np.isinf(x) else x  # noqa: E731
    return {"a": a, "b": b, "a_minus": fin(am), "a_plus": ap, "b_minus": bm, "b_plus": fin(bp)}


def result_to_json(res, gaps) -> str:
    """result_to_json (serialize.hpp:67-86) of an EigResult."""
    s = res.stats
    return json.dumps({
        "lambdas": [float(x) for x in res.lambdas],
        "residual": float(res.residual),
        "converged": bool(res.converged),
        "stats": {"n_ss": s.n_ss, "n_iter": s.n_iter, "n_gmres": s.n_gmres, "n_solv": s.n_solv,
                  "t_fact_s": s.factorization_time, "t_iter_s": s.iteration_time,
                  "t_total_s": s.factorization_time + s.iteration_time},
        "window": window_to_json(gaps),
        "r": int(res.r),
    }, indent=1)
