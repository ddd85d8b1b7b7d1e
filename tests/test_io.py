"""Host-side file formats (paper_1701_08935_b200/io.py):
Matrix Market semantics of matrix_market.hpp:48-190 (symmetric expansion,
duplicate summation, zero dropping, Hermitian check, line-numbered parse
errors, bit-exact round trip), BSR expansion, the ZEIGVEC1 eigenvector file and
the result JSON of serialize.hpp."""
import json

import numpy as np
import pytest

from conftest import golden_pencil, load_golden


@pytest.fixture(scope="module")
def io():
    from paper_1701_08935_b200 import io

    return io


def dense(n, csr):
    import scipy.sparse as sp

    return sp.csr_matrix((csr[2], csr[1], csr[0]), shape=(n, n)).toarray()


@pytest.mark.parametrize("case", ["filter_cfg2_k6", "filter_planted30_cx", "filter_cfg3_k5"])
def test_round_trip_bit_exact(io, tmp_path, case):
    g = load_golden(case)
    n, a, b = golden_pencil(g)
    cx = np.iscomplexobj(a[2])
    p = tmp_path / "a.mtx"
    io.write_matrix_market(str(p), n, a, cx, comments=(" pencil A of " + case,))
    com = []
    n2, a2 = io.read_matrix_market(str(p), comments=com)
    assert n2 == n and com == [" pencil A of " + case]
    assert (a2[0] == a[0]).all() and (a2[1] == a[1]).all() and (a2[2] == a[2]).all()
    info = io.probe_matrix_market(str(p))
    assert info["n"] == n and info["complex_field"] == cx and info["symmetry"] == ("hermitian" if cx else "symmetric")


def test_symmetric_expansion_duplicates_and_zeros(io, tmp_path):
    p = tmp_path / "d.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 5\n1 1 2\n2 1 -1\n2 1 -0.5\n"
                 "3 3 1\n3 2 0\n")
    n, csr = io.read_matrix_market(str(p))
    want = np.array([[2, -1.5, 0], [-1.5, 0, 0], [0, 0, 1]])
    assert n == 3 and np.array_equal(dense(n, csr), want)
    assert len(csr[2]) == 4  # the summed duplicates and the explicit zero are not stored


def test_general_hermitian_check_and_complex_into_real(io, tmp_path):
    p = tmp_path / "g.mtx"
    p.write_text("%%MatrixMarket matrix coordinate complex general\n2 2 3\n1 1 1 0\n1 2 0 1\n2 1 0 -1\n")
    n, csr = io.read_matrix_market(str(p))
    assert np.allclose(dense(n, csr), [[1, 1j], [-1j, 0]])
    with pytest.raises(io.DomainError):
        io.read_matrix_market(str(p), cx=False)
    q = tmp_path / "ng.mtx"
    q.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n2 1 2\n")
    with pytest.raises(io.DomainError, match="not numerically Hermitian"):
        io.read_matrix_market(str(q))


@pytest.mark.parametrize("text,line", [
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", 1),
    ("%MatrixMarket matrix coordinate real general\n2 2 0\n", 1),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 5\n", 3),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n3 1 5\n", 3),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 5\n", 2),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 5\n", 3),
])
def test_parse_errors_name_the_line(io, tmp_path, text, line):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(io.ParseError) as ei:
        io.read_matrix_market(str(p))
    assert ei.value.line == line


def test_bsr_expansion(io):
    rng = np.random.default_rng(3)
    bs, nb = 3, 4
    indptr = [0, 2, 3, 5, 6]
    indices = [0, 2, 1, 0, 2, 3]
    blocks = rng.standard_normal((6, bs, bs)) + 1j * rng.standard_normal((6, bs, bs))
    csr = io.bsr_to_csr(nb, bs, indptr, indices, blocks, True)
    import scipy.sparse as sp

    ref = sp.bsr_matrix((blocks, indices, indptr), shape=(nb * bs, nb * bs)).toarray()
    assert np.array_equal(dense(nb * bs, csr), ref)


def test_eigvec_binary_round_trip(io, tmp_path):
    x = np.asfortranarray(np.arange(12.0).reshape(4, 3) + 1j * np.ones((4, 3)))
    p = tmp_path / "v.bin"
    io.write_eigvec_binary(str(p), x)
    raw = p.read_bytes()
    assert raw[:8] == b"ZEIGVEC1" and len(raw) == 8 + 20 + 16 * 12
    assert np.array_equal(io.read_eigvec_binary(str(p), cx=True), x)
    with pytest.raises(io.DomainError):
        io.read_eigvec_binary(str(p), cx=False)


def test_window_json_matches_window_from_gaps(io):
    w = io.window_to_json([-np.inf, 1.0, 2.0, 3.0])
    assert w == {"a": 0.0, "b": 2.5, "a_minus": None, "a_plus": 1.0, "b_minus": 2.0, "b_plus": 3.0}
    json.dumps(w)


# ---- interoperability with the reference's own readers / writers (oracle/_ref) ----
REF_DIAG10 = "/root/reference/proj/data/diag10.mtx"


def _ref():
    import oracle

    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built")
    return oracle.Reference()


def test_reads_the_reference_fixture_diag10(io):
    """proj/data/diag10.mtx, the reference CLI's own fixture: our reader and the reference's
    (matrix_market.hpp:106-159) return the same CSR."""
    import os

    if not os.path.exists(REF_DIAG10):
        pytest.skip("reference tree absent")
    ref = _ref()
    n, csr, cx = ref.read_mm(REF_DIAG10)
    ours = io.read_matrix_market(REF_DIAG10)
    assert ours[0] == n == 10 and not cx
    for x, y in zip(ours[1], csr):
        assert (np.asarray(x) == np.asarray(y)).all()
    assert (np.asarray(ours[1][2]) == np.arange(1.0, 11.0)).all()


@pytest.mark.parametrize("case", ["filter_cfg2_k6", "filter_planted30_cx", "filter_cfg3_k5"])
def test_matrix_market_files_cross_read(io, tmp_path, case):
    """A file the reference wrote (write_matrix_market) read by us, and one we wrote read by the
    reference: identical CSR arrays, bit for bit."""
    ref = _ref()
    g = load_golden(case)
    n, a, b = golden_pencil(g)
    cx = bool(g["cx"])
    ref.write_mm(tmp_path / "ref.mtx", n, a, cx)
    ours = io.read_matrix_market(str(tmp_path / "ref.mtx"))
    for x, y in zip(ours[1], a):
        assert (np.asarray(x) == np.asarray(y)).all()
    io.write_matrix_market(str(tmp_path / "ours.mtx"), n, a, cx)
    n2, back, cx2 = ref.read_mm(tmp_path / "ours.mtx")
    assert n2 == n and cx2 == cx
    for x, y in zip(back, a):
        assert (np.asarray(x) == np.asarray(y)).all()


@pytest.mark.parametrize("cx", [False, True])
def test_eigvec_files_cross_read(io, tmp_path, cx):
    """ZEIGVEC1 eigenvector blocks (serialize.hpp:108-142) written by either side and read by the
    other, bit for bit."""
    ref = _ref()
    rng = np.random.default_rng(7)
    x = rng.standard_normal((37, 5)) + (1j * rng.standard_normal((37, 5)) if cx else 0)
    io.write_eigvec_binary(str(tmp_path / "ours.bin"), x)
    assert (ref.read_eigvec(tmp_path / "ours.bin", 37, 5, cx) == x).all()
    ref.write_eigvec(tmp_path / "ref.bin", x)
    assert (io.read_eigvec_binary(str(tmp_path / "ref.bin")) == x).all()
