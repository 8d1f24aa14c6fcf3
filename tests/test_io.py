"""File IO of the path, CPU: Matrix Market coordinate files and
permutation files against the reference's own readers/writers (matrix_market.hpp,
compiled unmodified in oracle/_ref), including the reference's error cases, and the
external-permutation reorder (ReorderSpec::file, reorder.hpp:183-192)."""
import numpy as np
import pytest

import oracle as O
import paper_2507_21253_b200 as B
from helpers import assert_csr_identical

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


MM_CASES = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% comment\n\n3 4 4\n"
                    "1 1 1.5\n3 4 -2e-3\n2 2 7\n1 3 0.25\n",
    "symmetric_pattern": "%%MatrixMarket matrix coordinate pattern symmetric\n4 4 4\n"
                         "1 1\n2 1\n4 2\n3 3\n",
    "integer_dups_crlf": "\ufeff%%MatrixMarket matrix coordinate integer general\r\n"
                         "2 2 4\r\n1 2 3\r\n1 2 4\r\n2 1 -1\r\n\r\n2 2 5\r\n",
    "upper_case_banner": "%%MatrixMarket MATRIX Coordinate REAL Symmetric\n3 3 3\n"
                         "2 1 0.5\n3 3 1.25\n3 1 -4\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n5 3 0\n",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(MM_CASES))
def test_load_matrix_market_matches_reference(tmp_path, case):
    path = _write(tmp_path, case + ".mtx", MM_CASES[case])
    assert_csr_identical(B.load_matrix_market(path), O.ref_load_matrix_market(path), case)


BAD_MM = {
    "no_banner": "MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n",
    "array_format": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
    "row_oob": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "truncated": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n",
    "missing_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(BAD_MM))
def test_load_matrix_market_errors_like_reference(tmp_path, case):
    path = _write(tmp_path, case + ".mtx", BAD_MM[case])
    with pytest.raises(RuntimeError):  # reference io_error
        O.ref_load_matrix_market(path)
    with pytest.raises(B.BspIOError):
        B.load_matrix_market(path)
    with pytest.raises(B.BspIOError):
        B.load_matrix_market(str(tmp_path / "does_not_exist.mtx"))


@needs_ref
def test_write_matrix_market_byte_identical_and_round_trips(tmp_path):
    a = B.make_config(2, 64)
    ours, ref = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    B.write_matrix_market(a, str(ours))
    O.ref_write_matrix_market(O.Csr(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values), ref)
    assert ours.read_bytes() == ref.read_bytes()
    assert_csr_identical(B.load_matrix_market(str(ours)), a, "round trip")


@needs_ref
def test_permutation_files(tmp_path):
    perm = B.reorder_random(1000, 7)
    path = tmp_path / "p.txt"
    B.write_permutation(perm, str(path))
    assert np.array_equal(B.load_permutation(str(path), 1000).perm, perm.perm)
    assert np.array_equal(O.ref_load_permutation(path, 1000), perm.perm)
    # blank lines and CRLF tolerated, as the reference
    p2 = _write(tmp_path, "p2.txt", "2\r\n\r\n0\n1\n")
    assert np.array_equal(B.load_permutation(p2, 3).perm, O.ref_load_permutation(p2, 3))
    for bad, n in (("0\n1\n", 3), ("0\n0\n1\n", 3), ("0\nx\n1\n", 3), ("0\n1\n3\n", 3)):
        pb = _write(tmp_path, "bad.txt", bad)
        with pytest.raises(RuntimeError):
            O.ref_load_permutation(pb, n)
        with pytest.raises(B.BspIOError):
            B.load_permutation(pb, n)


def test_reorder_spec_file_equals_in_process_orders(tmp_path):
    """An external permutation file (e.g. a GP/HP ordering computed elsewhere) drives
    the same reorder as the in-process methods (bench.hpp:119-127)."""
    a = B.make_config(4, 12)
    for spec in (B.ReorderSpec("rcm"), B.ReorderSpec("random", seed=3), B.ReorderSpec("degree")):
        p = B.make_permutation(spec, a)
        path = tmp_path / f"{spec.method}.perm"
        B.write_permutation(p, str(path))
        q = B.make_permutation(B.ReorderSpec("file", path=str(path)), a)
        assert np.array_equal(p.perm, q.perm)
        assert B.ReorderSpec("file", path=str(path)).name() == f"file:{path}"
    assert np.array_equal(B.make_permutation(B.ReorderSpec(), a).perm, np.arange(a.nrows))
