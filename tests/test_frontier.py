"""Square x tall-skinny workload: frontier operands (reference frontier.hpp:20-77)
and the multiply over them (bench.hpp:129-193).

CPU: the oracle restatement (oracle.generate_frontiers, with its own
std::mt19937_64) against golden vectors made from the UNMODIFIED reference.
GPU: bsp_generate_frontiers (batched device BFS) against the golden vectors
and the oracle, its edge cases, and A_variant x permute_rows(F_t, perm)
row-wise and cluster-wise against the oracle, as prepare_bench builds it.
"""
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import paper_2507_21253_b200 as B
from helpers import assert_csr_identical

G = np.load(Path(__file__).with_name("golden") / "golden.npz")
# (cfg, num_frontiers, batch, seed) — tests/golden/make_golden.py FRONTIER_CASES
CASES = [(5, 10, 16, 0), (2, 10, 64, 3), (1, 4, 100, 1), (4, 1, 8, 5)]


def golden_A(cfg):
    p = f"cfg{cfg}_"
    rp = G[p + "A_rp"]
    return O.Csr(rp.size - 1, rp.size - 1, rp, G[p + "A_ci"], G[p + "A_v"])


def golden_frontiers(case):
    q = "fr_{}_{}_{}_{}_".format(*case)
    return [(G[q + f"{t}_rp"], G[q + f"{t}_ci"]) for t in range(int(G[q + "count"][0]))]


def as_matrix(o):
    return B.CsrMatrix(o.nrows, o.ncols, np.asarray(o.row_ptr, np.int64),
                       np.asarray(o.col_idx, np.int32), np.asarray(o.values, np.float64))


def test_mt19937_64_known_answer():
    """[rand.predef]: the 10000th output of a default-constructed mt19937_64."""
    r = O._MT19937_64(5489)
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042


def test_oracle_shuffle_matches_golden():
    for k in G.files:
        if k.startswith("perm_"):
            _, n, seed = k.split("_")
            assert np.array_equal(O.random_permutation(int(n), int(seed)), G[k]), k


@pytest.mark.parametrize("case", CASES)
def test_oracle_frontiers_match_golden(case):
    cfg, nf, bt, sd = case
    got = O.generate_frontiers(golden_A(cfg), nf, bt, sd)
    ref = golden_frontiers(case)
    assert len(got) == len(ref)
    for f, (rp, ci) in zip(got, ref):
        assert f.ncols == min(bt, f.nrows)
        assert np.array_equal(f.row_ptr, rp) and np.array_equal(f.col_idx, ci)


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
def gpu_frontiers(engine, a, nf, bt, sd):
    A = engine.upload(as_matrix(a) if isinstance(a, O.Csr) else a)
    fs = engine.generate_frontiers(A, nf, bt, sd)
    out = []
    for f in fs:
        out.append(f.download())
        f.free()
    A.free()
    return out


def assert_frontiers_equal(got, ref, width):
    assert len(got) == len(ref)
    for t, (f, r) in enumerate(zip(got, ref)):
        rp, ci = (r.row_ptr, r.col_idx) if hasattr(r, "row_ptr") else r
        assert f.ncols == width, t
        assert np.array_equal(f.row_ptr, rp), f"frontier {t} row_ptr"
        assert np.array_equal(f.col_idx, ci), f"frontier {t} col_idx"
        assert np.all(f.values == 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_frontiers_match_golden(engine, case):
    cfg, nf, bt, sd = case
    a = golden_A(cfg)
    assert_frontiers_equal(gpu_frontiers(engine, a, nf, bt, sd), golden_frontiers(case),
                           min(bt, a.nrows))


@pytest.mark.gpu
def test_gpu_frontier_edge_cases(engine):
    # two components + isolated vertices: searches end early (shorter list)
    n = 300
    r = np.concatenate([np.arange(0, 99), np.arange(1, 100), np.arange(150, 249),
                        np.arange(151, 250)])
    c = np.concatenate([np.arange(1, 100), np.arange(0, 99), np.arange(151, 250),
                        np.arange(150, 249)])
    a = B.coo_to_csr(n, n, r, c, np.ones(r.size))
    o = O.Csr(n, n, a.row_ptr, a.col_idx, a.values)
    for nf, bt, sd in [(500, 32, 9), (3, 300, 1), (1, 1, 0), (200, 5, 77)]:
        assert_frontiers_equal(gpu_frontiers(engine, a, nf, bt, sd),
                               O.generate_frontiers(o, nf, bt, sd), min(bt, n))
    # directed path 0 -> 1 -> ... -> n-1 from every vertex: n frontiers
    n = 64
    p = B.coo_to_csr(n, n, np.arange(n - 1), np.arange(1, n), np.ones(n - 1))
    got = gpu_frontiers(engine, p, n + 5, n, 3)
    assert len(got) == n
    assert_frontiers_equal(got, O.generate_frontiers(O.Csr(n, n, p.row_ptr, p.col_idx, p.values),
                                                     n + 5, n, 3), n)
    # a larger R-MAT with hub rows
    a = B.make_config(5, 11)
    assert_frontiers_equal(gpu_frontiers(engine, a, 10, 64, 0),
                           O.generate_frontiers(O.Csr(a.nrows, a.ncols, a.row_ptr, a.col_idx,
                                                      a.values), 10, 64, 0), 64)


@pytest.mark.gpu
def test_gpu_frontier_contract(engine):
    rect = engine.upload(B.coo_to_csr(3, 4, [0], [1], [1.0]))
    with pytest.raises(B.ContractError):
        engine.generate_frontiers(rect, 2, 2, 0)
    sq = engine.upload(B.coo_to_csr(3, 3, [0], [1], [1.0]))
    with pytest.raises(B.ContractError):
        engine.generate_frontiers(sq, 0, 2, 0)
    with pytest.raises(B.ContractError):
        engine.generate_frontiers(sq, 2, 0, 0)
    empty = engine.upload(B.coo_to_csr(0, 0, [], [], []))
    assert engine.generate_frontiers(empty, 3, 4, 0) == []


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,scale,reorder", [(4, 12, "rcm"), (5, 12, "random"), (2, 256, None)])
def test_tall_skinny_multiply(engine, cfg, scale, reorder):
    """prepare_bench (bench.hpp:129-169): frontiers of the ORIGINAL A, rows
    co-permuted with A; C_t = A_variant * B_t row-wise and cluster-wise
    (hierarchical clusters of A_variant), bit-identical to the oracle."""
    a = B.make_config(cfg, scale)
    if reorder == "rcm":
        perm = B.reorder_rcm(a)
    elif reorder == "random":
        perm = B.reorder_random(a.nrows, 11)
    else:
        perm = B.Permutation(np.arange(a.nrows, dtype=np.int32))
    av = B.permute_symmetric(a, perm)
    fs = B.generate_frontiers(a, 10, 64, 0)
    assert len(fs) >= 2
    asg = engine.hierarchical_clusters(av)
    Av = engine.upload(av)
    Ac = engine.build_csr_cluster(Av, asg)
    for f in fs:
        bv = B.permute_rows(f, perm)
        Bv = engine.upload(bv)
        ref = O.spgemm_rowwise(av, bv)
        assert_csr_identical(engine.spgemm_rowwise(Av, Bv).download(), ref, "tall-skinny row-wise")
        assert_csr_identical(engine.spgemm_clusterwise(Ac, Bv).download(), ref,
                             "tall-skinny cluster-wise")
        Bv.free()
