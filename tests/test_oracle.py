"""CPU: pin the oracle restatement (oracle/oracle.c) to the reference.

1. Against the committed golden vectors (generated from the UNMODIFIED
   reference by tests/golden/make_golden.py) — always runs.
2. Against oracle/_ref (the reference headers compiled here) on seeded
   random inputs — runs wherever oracle/_ref was built.
3. The reference's own known-answer tests, evaluated on the oracle.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import paper_2507_21253_b200 as B
from helpers import csr_from_rows, grouped_identical_rows, identity_csr, random_assignment, random_csr

G = np.load(Path(__file__).with_name("golden") / "golden.npz")
CFGS = [1, 2, 3, 4, 5]


def golden_A(cfg):
    p = f"cfg{cfg}_"
    rp = G[p + "A_rp"]
    return O.Csr(rp.size - 1, int(rp.size - 1), rp, G[p + "A_ci"], G[p + "A_v"])


def bits(x):
    return np.ascontiguousarray(x, np.float64).view(np.uint64)


@pytest.mark.parametrize("cfg", CFGS)
def test_rowwise_matches_golden(cfg):
    a = golden_A(cfg)
    c = O.spgemm_rowwise(a, a)
    p = f"cfg{cfg}_"
    assert np.array_equal(c.row_ptr, G[p + "C_rp"])
    assert np.array_equal(c.col_idx, G[p + "C_ci"])
    assert np.array_equal(bits(c.values), bits(G[p + "C_v"]))
    assert np.array_equal(O.spgemm_symbolic(a, a), G[p + "sym"])


@pytest.mark.parametrize("cfg", CFGS)
def test_topk_and_hierarchical_match_golden(cfg):
    a = golden_A(cfg)
    p = f"cfg{cfg}_"
    tk = O.spgemm_topk(a, 7, 0.3)
    assert np.array_equal(tk["i"], G[p + "topk_i"]) and np.array_equal(tk["j"], G[p + "topk_j"])
    assert np.array_equal(bits(tk["score"]), bits(G[p + "topk_s"]))
    ptr, rows = O.merge_candidates(a, tk, 0.3, 8)
    assert np.array_equal(ptr, G[p + "hier_ptr"]) and np.array_equal(rows, G[p + "hier_rows"])


@pytest.mark.parametrize("cfg", CFGS)
def test_clusterwise_matches_golden(cfg):
    a = golden_A(cfg)
    p = f"cfg{cfg}_"
    csr, d, st = O.spgemm_clusterwise(a, G[p + "hier_ptr"], G[p + "hier_rows"], a)
    assert np.array_equal(np.array(st, np.uint64), G[p + "cw_stats"])
    assert d["values"].size == G[p + "cw_slots"][0] and d["col_idx"].size == G[p + "cw_slots"][1]
    assert np.array_equal(csr.col_idx, G[p + "C_ci"])
    assert np.array_equal(bits(csr.values), bits(G[p + "C_v"]))  # cluster-wise == row-wise bitwise


def test_dense_oracle_corpus():
    """reference spgemm_rowwise_test.cpp:53-75 / acceptance 2 on the oracle."""
    rng = np.random.default_rng(5)
    for seed in range(30):
        n, m, k = (int(x) for x in rng.integers(1, 60, size=3))
        a = random_csr(n, k, 0.01 + 0.2 * rng.random(), 2 * seed + 1, nonnegative=False)
        b = random_csr(k, m, 0.01 + 0.2 * rng.random(), 2 * seed + 2, nonnegative=False)
        c = O.spgemm_rowwise(a, b)
        cc = B.CsrMatrix(c.nrows, c.ncols, c.row_ptr, c.col_idx, c.values)
        assert np.allclose(cc.to_dense(), a.to_dense() @ b.to_dense(), atol=1e-9, rtol=0)


def test_reference_kats_on_oracle():
    """spgemm_rowwise_test.cpp:85-97,148-169; clustering_test.cpp:109-127."""
    a = B.coo_to_csr(1, 2, [0, 0], [0, 1], [1.0, 1.0])
    b = B.coo_to_csr(2, 1, [0, 1], [0, 0], [1.0, -1.0])
    c = O.spgemm_rowwise(a, b)
    assert c.col_idx.size == 1 and c.values[0] == 0.0  # structural zero kept
    assert O.spgemm_topk(identity_csr(9), 7, 0.3).size == 0
    t = O.spgemm_topk(csr_from_rows(6, [[0, 1, 2], [0, 1, 2], [5]]), 7, 0.3)
    assert t.size == 1 and (t[0]["i"], t[0]["j"], t[0]["score"]) == (0, 1, 1.0)
    two = csr_from_rows(3, [[0, 1], [1, 2]])
    assert O.spgemm_topk(two, 7, 0.3).size == 1 and O.spgemm_topk(two, 7, 0.4).size == 0
    m = csr_from_rows(6, [[0, 1, 2], [5], [0, 1, 2]])
    ptr, rows = O.merge_candidates(m, O.spgemm_topk(m, 7, 0.3), 0.3, 8)
    assert ptr.tolist() == [0, 2, 3] and rows.tolist() == [0, 2, 1]
    ten = grouped_identical_rows(1, 10, 4)
    ptr, rows = O.merge_candidates(ten, O.spgemm_topk(ten, 7, 0.3), 0.3, 8)
    assert sorted(np.diff(ptr).tolist(), reverse=True)[:3] == [8, 1, 1]


def test_format_roundtrip_oracle():
    """acceptance 6: cluster_to_csr(build_csr_cluster(a, asg)) == a, exactly."""
    for seed in range(20):
        a = random_csr(40, 30, 0.15, seed)
        asg = random_assignment(40, 8, seed)
        d = O.build_csr_cluster(a, asg.cluster_ptr, asg.rows)
        csr, _, _ = O.spgemm_clusterwise(a, asg.cluster_ptr, asg.rows, identity_csr(30))
        assert np.array_equal(csr.row_ptr, a.row_ptr) and np.array_equal(csr.col_idx, a.col_idx)
        assert np.array_equal(bits(csr.values), bits(a.values))
        assert d["values"].size == int(np.sum(np.diff(d["cluster_col_ptr"]) * d["cluster_sizes"]))


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_matches_reference_build_random():
    rng = np.random.default_rng(9)
    for seed in range(12):
        n = int(rng.integers(20, 120))
        a = random_csr(n, n, 0.02 + 0.1 * rng.random(), 100 + seed)
        r = O.ref_spgemm_rowwise(a, a)
        o = O.spgemm_rowwise(a, a)
        assert np.array_equal(r.row_ptr, o.row_ptr) and np.array_equal(r.col_idx, o.col_idx)
        assert np.array_equal(bits(r.values), bits(o.values))
        rt, ot = O.ref_spgemm_topk(a, 7, 0.3), O.spgemm_topk(a, 7, 0.3)
        assert np.array_equal(rt, ot)
        asg = random_assignment(n, 8, seed)
        rc, rst, _, _ = O.ref_spgemm_clusterwise(a, asg.cluster_ptr, asg.rows, a)
        oc, _, ost = O.spgemm_clusterwise(a, asg.cluster_ptr, asg.rows, a)
        assert tuple(rst) == tuple(ost)
        assert np.array_equal(bits(rc.values), bits(oc.values))


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (needs /root/reference)")
def test_row_block_oracle_equals_full():
    """The row-block decomposition used for cfg3/cfg5 (int32 C offsets) gives
    the same rows as one call."""
    a = B.make_config(5, 10)
    full = O.ref_spgemm_rowwise(a, a)
    r0, r1 = 100, 700
    blk = O.ref_spgemm_rowwise(a, a, r0, r1)
    s, e = full.row_ptr[r0], full.row_ptr[r1]
    assert np.array_equal(blk.row_ptr, full.row_ptr[r0:r1 + 1] - s)
    assert np.array_equal(blk.col_idx, full.col_idx[s:e])
    assert np.array_equal(bits(blk.values), bits(full.values[s:e]))
