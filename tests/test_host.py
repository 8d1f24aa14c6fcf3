"""CPU: the C-ABI library and the host side of the product.

- libbsp.so loads and exports every symbol include/bsp.h declares;
- host preprocessing (reorder_random / reorder_rcm / reorder_degree,
  permutations, transpose, clustering scans, the heap/union-find merge,
  Jaccard) is identical to the reference (golden vectors + KATs from
  reorder_test.cpp, clustering_test.cpp, sparse_core_test.cpp);
- contract errors surface as ContractError.
No GPU compute is called here.
"""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2507_21253_b200 as B
from paper_2507_21253_b200 import _lib
from helpers import csr_from_rows, grouped_identical_rows, identity_csr, random_csr

ROOT = Path(__file__).resolve().parents[1]
G = np.load(Path(__file__).with_name("golden") / "golden.npz")


def golden_A(cfg):
    p = f"cfg{cfg}_"
    rp = G[p + "A_rp"]
    return B.CsrMatrix(rp.size - 1, rp.size - 1, rp, G[p + "A_ci"], G[p + "A_v"])


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    hdr = (ROOT / "include" / "bsp.h").read_text()
    names = set(re.findall(r"^\s*(?:const char\*|void\*|int64_t|int|void)\s+(bsp_\w+)\(", hdr, re.M))
    assert len(names) > 50
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} missing from the ctypes binding"
    assert lib.bsp_version().startswith(b"bsp")


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


@pytest.mark.parametrize("n,seed", [(1, 7), (5, 3), (100, 42), (4096, 4)])
def test_reorder_random_identical(n, seed):
    """reorder.hpp:20-30 (reorder_test.cpp:9-15 determinism)."""
    assert np.array_equal(B.reorder_random(n, seed).perm, G[f"perm_{n}_{seed}"])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_rcm_and_degree_identical(cfg):
    a = golden_A(cfg)
    assert np.array_equal(B.reorder_rcm(a).perm, G[f"cfg{cfg}_rcm"])
    assert np.array_equal(B.reorder_degree(a).perm, G[f"cfg{cfg}_degree"])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_merge_and_scans_identical(cfg):
    a = golden_A(cfg)
    p = f"cfg{cfg}_"
    pairs = np.zeros(G[p + "topk_i"].size, dtype=B.CandidatePair)
    pairs["i"], pairs["j"], pairs["score"] = G[p + "topk_i"], G[p + "topk_j"], G[p + "topk_s"]
    asg, trace = B.merge_candidates(a, pairs)
    assert np.array_equal(asg.cluster_ptr, G[p + "hier_ptr"])
    assert np.array_equal(asg.rows, G[p + "hier_rows"])
    for t in trace:  # every union joined rows whose Jaccard was >= 0.3
        assert t["score"] >= 0.3
    var = B.variable_length_clusters(a)
    assert np.array_equal(var.cluster_ptr, G[p + "var_ptr"])
    assert np.array_equal(var.rows, G[p + "var_rows"])


def test_rcm_kats():
    """reorder_test.cpp:60-142: path, star, banded-shuffled bandwidth <= 2b."""
    path = B.coo_to_csr(4, 4, [2, 0, 0, 3, 3, 1], [0, 2, 3, 0, 1, 3], np.ones(6))
    assert B.bandwidth(B.permute_symmetric(path, B.reorder_rcm(path))) == 1
    star = B.coo_to_csr(6, 6, [0] * 5 + list(range(1, 6)), list(range(1, 6)) + [0] * 5, np.ones(10))
    sp = B.reorder_rcm(star)  # reorder_test.cpp:84-98
    assert sp.perm[-1] == 1 and sp.perm[4] == 0 and sp.inv[0] >= 4
    for seed in range(10):
        n, b = 20 + 15 * seed, 1 + seed % 5
        r, c = zip(*[(i, j) for i in range(n) for j in range(max(0, i - b), min(n, i + b + 1))])
        band = B.coo_to_csr(n, n, r, c, np.ones(len(r)))
        shuf = B.permute_symmetric(band, B.reorder_random(n, seed))
        assert B.bandwidth(B.permute_symmetric(shuf, B.reorder_rcm(shuf))) <= 2 * b


def test_clustering_kats():
    """clustering_test.cpp:28-80 and acceptance 3/4."""
    assert B.ClusterParams().jacc_th == 0.3 and B.ClusterParams().max_cluster_th == 8
    assert B.fixed_length_clusters(7, 3).clusters == [[0, 1, 2], [3, 4, 5], [6]]
    with pytest.raises(B.ContractError):
        B.fixed_length_clusters(5, 0)
    # walkthrough: similarities vs representative 0.5, 0.5, 0.0, 0.5, 0.25
    rows = [[0, 1], [0, 2], [0, 1, 2, 3], [4, 5], [4, 6], [7, 8, 9, 4]]
    a = csr_from_rows(10, rows)
    assert B.variable_length_clusters(a).clusters == [[0, 1, 2], [3, 4], [5]]
    twenty = grouped_identical_rows(1, 20, 3)
    assert B.variable_length_clusters(twenty).sizes().tolist()[:3] == [8, 8, 4]


def test_jaccard_and_errors():
    a = csr_from_rows(8, [[0, 2, 5], [0, 3, 5], [0, 2, 5], [1, 4], []])
    assert B.jaccard_similarity(a, 0, 2) == 1.0
    assert B.jaccard_similarity(a, 0, 1) == 0.5
    assert B.jaccard_similarity(a, 4, 4) == 0.0
    with pytest.raises(B.ContractError):
        B.jaccard_similarity(a, 0, 7)
    with pytest.raises(B.ContractError):
        B.Permutation.from_perm([2, 2, 0])
    with pytest.raises(B.ContractError):
        B.permute_symmetric(random_csr(3, 4, 0.5, 1), B.Permutation.identity(3))


def test_transpose_permute_roundtrips():
    a = random_csr(30, 30, 0.2, 3, nonnegative=False)
    assert B.csr_equal_canonical(B.transpose(B.transpose(a)), a, 0.0)
    p = B.reorder_random(30, 11)
    assert B.csr_equal_canonical(B.permute_symmetric(B.permute_symmetric(a, p), p.inverse()), a, 0.0)
    r = B.permute_rows(a, p)
    assert np.allclose(r.to_dense()[p.inv], a.to_dense())
    d = B.permute_symmetric(a, p).to_dense()
    assert np.allclose(d[np.ix_(p.inv, p.inv)], a.to_dense())


def test_generators_pinned():
    """Seeded generators are deterministic and valid CSR."""
    for cfg, sc in [(1, 512), (2, 64), (3, 9), (4, 8), (5, 10)]:
        x, y = B.make_config(cfg, sc), B.make_config(cfg, sc)
        x.check_invariants()
        assert np.array_equal(x.col_idx, y.col_idx) and np.array_equal(x.values, y.values)
    s = B.make_config(4, 8)
    assert s.nnz() == (3 * 8 - 2) ** 3  # 27-point stencil, boundary truncated
    rm = B.make_config(5, 10)
    assert B.csr_equal_canonical(B.transpose(B.binarize(rm)), B.binarize(rm), 0.0)  # symmetric
