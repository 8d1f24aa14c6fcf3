"""GPU parity of the cluster-wise path, CSR_Cluster format and candidate
generation against the oracle / reference (cluster_spgemm_test.cpp,
cluster_format_test.cpp, clustering_test.cpp, spgemm_rowwise_test.cpp:148-207).
"""
import numpy as np
import pytest

import oracle as O
import paper_2507_21253_b200 as B
from helpers import (assert_csr_identical, csr_from_rows, grouped_identical_rows, identity_csr,
                     random_assignment, random_csr)

pytestmark = pytest.mark.gpu


def clusterwise(engine, a, asg, b=None):
    A = engine.upload(a)
    Bd = A if b is None else engine.upload(b)
    Ac = engine.build_csr_cluster(A, asg)
    return engine.spgemm_clusterwise(Ac, Bd).download()


@pytest.mark.parametrize("cfg,scale", [(2, 512), (2, 2048), (4, 16), (5, 13), (3, 12)])
def test_hierarchical_clusterwise_equals_rowwise(engine, cfg, scale):
    a = B.make_config(cfg, scale)
    asg = engine.hierarchical_clusters(a)
    c = clusterwise(engine, a, asg)
    assert_csr_identical(c, O.spgemm_rowwise(a, a), f"cfg{cfg} cluster-wise")


def test_strategies_corpus(engine):
    """acceptance_main.cpp:53-77 style: random matrices x 4 strategies."""
    rng = np.random.default_rng(11)
    for seed in range(24):
        n = int(rng.integers(1, 101))
        a = random_csr(n, n, 0.01 + 0.29 * rng.random(), seed)
        for asg in (B.fixed_length_clusters(n, 1), B.fixed_length_clusters(n, 4),
                    B.variable_length_clusters(a), engine.hierarchical_clusters(a),
                    random_assignment(n, 8, seed)):
            assert_csr_identical(clusterwise(engine, a, asg), O.spgemm_rowwise(a, a), f"seed {seed}")


def test_singletons_equal_rowwise_exactly(engine):
    """cluster_spgemm_test.cpp:20-26."""
    a = random_csr(40, 40, 0.15, 5)
    assert_csr_identical(clusterwise(engine, a, B.ClusterAssignment.singletons(40)),
                         O.spgemm_rowwise(a, a))


def test_identity_times_b(engine):
    """cluster_spgemm_test.cpp:28-36."""
    b = random_csr(12, 9, 0.3, 8)
    c = clusterwise(engine, identity_csr(12), B.fixed_length_clusters(12, 4), b)
    assert B.csr_equal_canonical(c, b, 0.0)


def test_format_matches_oracle(engine):
    """CSR_Cluster layout: merged columns, values, valid bits, slots
    (cluster_format_test.cpp:44-101)."""
    for seed in range(6):
        a = random_csr(50, 45, 0.12, 100 + seed)
        asg = random_assignment(50, 8, seed)
        Ac = engine.build_csr_cluster(engine.upload(a), asg)
        got = Ac.download()
        ref = O.build_csr_cluster(a, asg.cluster_ptr, asg.rows)
        for k in ("cluster_sizes", "cluster_col_ptr", "col_idx", "value_ptr", "row_map"):
            assert np.array_equal(got[k], ref[k]), k
        assert np.array_equal(got["values"].view(np.uint64), ref["values"].view(np.uint64))
        assert np.array_equal(got["valid"], ref["valid"])
        back = engine.cluster_to_csr(Ac).download()
        assert B.csr_equal_canonical(back, a, 0.0)  # round trip (acceptance 6)


def test_fig5_padding_kat(engine):
    """cluster_format_test.cpp: cluster {0,5},{0},{0,5} -> 2 cols x 3 members, 1 placeholder."""
    a = csr_from_rows(6, [[0, 5], [0], [0, 5]])
    Ac = engine.build_csr_cluster(engine.upload(a), B.ClusterAssignment.from_lists([[0, 1, 2]]))
    d = Ac.download()
    assert list(d["col_idx"]) == [0, 5] and Ac.value_slots() == 6 and d["placeholders"] == 1


def test_cluster_output_format(engine):
    """Optional CSR_Cluster C equals the reference's C format."""
    a = B.make_config(2, 256)
    asg = engine.hierarchical_clusters(a)
    A = engine.upload(a)
    Ac = engine.build_csr_cluster(A, asg)
    c, cc = engine.spgemm_clusterwise(Ac, A, want_cluster=True)
    csr, d, _ = O.spgemm_clusterwise(a, asg.cluster_ptr, asg.rows, a)
    got = cc.download()
    for k in ("cluster_sizes", "cluster_col_ptr", "col_idx", "value_ptr", "row_map", "valid"):
        assert np.array_equal(got[k], d[k]), k
    assert np.array_equal(got["values"].view(np.uint64), d["values"].view(np.uint64))


def test_access_stats_match_oracle(engine):
    """cluster_spgemm_test.cpp:86-130 / acceptance 5: exact counters."""
    a = grouped_identical_rows(6, 8, 5)
    asg = engine.hierarchical_clusters(a)
    A = engine.upload(a)
    st = engine.cluster_access_stats(engine.build_csr_cluster(A, asg), A)
    rw = engine.rowwise_access_stats(A, A)
    assert st.b_row_loads * 8 == rw.b_row_loads == a.nnz()
    b = B.make_config(2, 512)
    asg = engine.hierarchical_clusters(b)
    Bd = engine.upload(b)
    st = engine.cluster_access_stats(engine.build_csr_cluster(Bd, asg), Bd)
    _, _, ost = O.spgemm_clusterwise(b, asg.cluster_ptr, asg.rows, b)
    assert (st.b_row_loads, st.a_inner_iters, st.placeholder_skips) == ost


# ----------------------------------------------------------------- candidates
@pytest.mark.parametrize("cfg,scale", [(2, 512), (2, 4096), (4, 16), (5, 13), (3, 12), (3, 14)])
def test_topk_identical_to_reference(engine, cfg, scale):
    a = B.make_config(cfg, scale)
    A = engine.upload(B.binarize(a))
    got = engine.spgemm_topk(A, engine.transpose(A), 7, 0.3)
    ref = O.spgemm_topk(a, 7, 0.3)
    assert got.size == ref.size
    assert np.array_equal(got["i"], ref["i"]) and np.array_equal(got["j"], ref["j"])
    assert np.array_equal(got["score"].view(np.uint64), ref["score"].view(np.uint64))


def test_topk_kats(engine):
    """spgemm_rowwise_test.cpp:148-169."""
    e = engine
    i9 = identity_csr(9)
    I = e.upload(i9)
    assert e.spgemm_topk(I, e.transpose(I), 7, 0.3).size == 0
    a = csr_from_rows(6, [[0, 1, 2], [0, 1, 2], [5]])
    A = e.upload(a)
    p = e.spgemm_topk(A, e.transpose(A), 7, 0.3)
    assert p.size == 1 and (p[0]["i"], p[0]["j"], p[0]["score"]) == (0, 1, 1.0)
    a = csr_from_rows(3, [[0, 1], [1, 2]])
    A = e.upload(a)
    assert e.spgemm_topk(A, e.transpose(A), 7, 0.3).size == 1
    assert e.spgemm_topk(A, e.transpose(A), 7, 0.4).size == 0


def test_hierarchical_identical_to_reference(engine):
    """clustering_test.cpp:109-137 KATs + seeded recipes vs the reference merge."""
    a = csr_from_rows(6, [[0, 1, 2], [5], [0, 1, 2]])
    assert engine.hierarchical_clusters(a).clusters == [[0, 2], [1]]
    ten = grouped_identical_rows(1, 10, 4)
    sizes = sorted(engine.hierarchical_clusters(ten).sizes().tolist(), reverse=True)[:3]
    assert sizes == [8, 1, 1]
    for cfg, sc in [(2, 1024), (4, 16), (5, 13)]:
        m = B.make_config(cfg, sc)
        ptr, rows = O.merge_candidates(m, O.spgemm_topk(m, 7, 0.3), 0.3, 8)
        got = engine.hierarchical_clusters(m)
        assert np.array_equal(got.cluster_ptr, ptr) and np.array_equal(got.rows, rows)


def test_minhash_invariants(engine):
    """Minhash/LSH (north-star item 4; unpinned): partition, size cap, every
    candidate's score is the exact Jaccard >= threshold, planted clusters found."""
    a = B.make_config(2, 1024)
    A = engine.upload(a)
    pairs = engine.minhash_candidates(A, 64, 32, 1, 7, 0.3)
    assert pairs.size > 0
    for p in pairs[:: max(1, pairs.size // 200)]:
        assert p["score"] >= 0.3
        assert p["score"] == O.jaccard(a, int(p["i"]), int(p["j"]))
    asg = engine.hierarchical_clusters(a, method="minhash")
    asg.validate(a.nrows)
    assert asg.sizes().max() <= 8
    c = clusterwise(engine, a, asg)
    assert_csr_identical(c, O.spgemm_rowwise(a, a), "minhash cluster-wise")


@pytest.mark.parametrize("k,ncols", [(2, 64), (8, 33), (20, 64), (32, 7)])
def test_clusterwise_narrow_b_large_clusters(engine, k, ncols):
    """B with <= 64 columns: tiled clusters on the warp-per-cluster mask
    kernel (members taken 8 at a time, so K = 20 / 32 take several passes),
    the remaining rows on the row-wise mask kernel; identical to the oracle."""
    rng = np.random.default_rng(k * 100 + ncols)
    a = B.make_config(5, 12)
    r, c = [], []
    for i in range(a.nrows):
        if i % 5 == 0:
            continue  # empty B rows
        d = 1 + int(rng.integers(0, ncols))
        cs = np.sort(rng.choice(ncols, size=d, replace=False))
        r += [i] * cs.size
        c += cs.tolist()
    b = B.coo_to_csr(a.nrows, ncols, np.array(r), np.array(c), rng.uniform(-2, 2, size=len(r)))
    asg = B.fixed_length_clusters(a.nrows, k)
    got = clusterwise(engine, a, asg, b)
    assert_csr_identical(got, O.spgemm_rowwise(a, b), f"narrow cluster-wise K={k}")
    # CSR_Cluster output requested: the general path, same C
    A, Bd = engine.upload(a), engine.upload(b)
    Ac = engine.build_csr_cluster(A, asg)
    res = engine.spgemm_clusterwise(Ac, Bd, want_cluster=True)
    cc = res[0] if isinstance(res, tuple) else res
    assert_csr_identical(cc.download(), O.spgemm_rowwise(a, b), "narrow, CSR_Cluster requested")


@pytest.mark.parametrize("k", [33, 64, 200])
def test_clusters_beyond_32_members(engine, k):
    """fixed_length_clusters(n, k) with k > 32 (the reference accepts any k,
    clustering.hpp:59-69): the device CSR_Cluster holds them (valid bits; the
    32-bit member masks only serve the cluster kernels), the format equals the
    oracle's, cluster-wise C equals row-wise bit for bit (those clusters run
    through the row view), cluster_to_csr round-trips, access stats are exact,
    and the cluster split covers them."""
    a = random_csr(420, 420, 0.03, 900 + k)
    asg = B.fixed_length_clusters(a.nrows, k)
    A = engine.upload(a)
    Ac = engine.build_csr_cluster(A, asg)
    got = Ac.download()
    ref = O.build_csr_cluster(a, asg.cluster_ptr, asg.rows)
    for key in ("cluster_sizes", "cluster_col_ptr", "col_idx", "value_ptr", "row_map", "valid"):
        assert np.array_equal(got[key], ref[key]), key
    assert np.array_equal(got["values"].view(np.uint64), ref["values"].view(np.uint64))
    assert B.csr_equal_canonical(engine.cluster_to_csr(Ac).download(), a, 0.0)
    want, _, st = O.spgemm_clusterwise(a, asg.cluster_ptr, asg.rows, a)
    assert_csr_identical(engine.spgemm_clusterwise(Ac, A).download(), O.spgemm_rowwise(a, a),
                         f"k={k}")
    s = engine.cluster_access_stats(Ac, A)
    assert (s.b_row_loads, s.a_inner_iters, s.placeholder_skips) == tuple(st)
    b = engine.partition_clusters(Ac, A, 3)
    assert b[0] == 0 and b[-1] == asg.nclusters
    big = random_csr(1100, 50, 0.05, 7)
    with pytest.raises(B.ContractError):  # the format's limit: 1024 rows per cluster
        engine.build_csr_cluster(engine.upload(big), B.fixed_length_clusters(big.nrows, 1025))


_KNOB_SCRIPT = r"""
import sys, numpy as np
import oracle as O
import paper_2507_21253_b200 as B
e = B.default_engine()
for cfg, scale in ((2, 512), (2, 2048), (4, 16), (5, 13)):
    a = B.make_config(cfg, scale)
    asg = e.hierarchical_clusters(a)
    A = e.upload(a)
    c = e.spgemm_clusterwise(e.build_csr_cluster(A, asg), A).download()
    o = O.spgemm_rowwise(a, a)
    assert np.array_equal(c.row_ptr, o.row_ptr) and np.array_equal(c.col_idx, o.col_idx), cfg
    assert np.array_equal(c.values.view(np.uint64), o.values.view(np.uint64)), cfg
names = set(e.profile_names()) if hasattr(e, "profile_names") else set()
print("ok")
"""


@pytest.mark.parametrize("env", [{"BSP_CLUSTER_TMA": "1"},
                                 {"BSP_CLUSTER_TMA": "1", "BSP_CLUSTER_MIN_REUSE": "0"},
                                 {"BSP_CLUSTER_MIN_REUSE": "0"},
                                 {"BSP_CLUSTER_MIN_REUSE": "40"}])
def test_cluster_knobs_bit_identical(env):
    """The bulk-copy (TMA) staged union tile and the reuse routing threshold are read once
    per process: each setting runs in its own process and must reproduce the oracle's C."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **env)
    e["PYTHONPATH"] = root + os.pathsep + os.path.join(root, "tests") + os.pathsep + e.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", _KNOB_SCRIPT], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
