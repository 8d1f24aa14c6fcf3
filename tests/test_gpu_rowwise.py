"""GPU parity of the row-wise hot path (bsp_spgemm_rowwise) against the oracle.

Mirrors the reference's spgemm_rowwise_test.cpp checks (file:line cited per
test) and adds per-config parity on seeded inputs of every BASELINE recipe.
The bar is bit-exact row_ptr / col_idx and bit-identical values.
"""
import numpy as np
import pytest

import oracle as O
import paper_2507_21253_b200 as B
from helpers import (assert_csr_identical, csr_from_rows, identity_csr, random_csr,
                     same_bits)

pytestmark = pytest.mark.gpu


def gpu_mul(engine, a, b):
    A = engine.upload(a)
    Bd = A if b is a else engine.upload(b)
    return engine.spgemm_rowwise(A, Bd).download()


@pytest.mark.parametrize("cfg,scale", [(1, None), (1, 4096), (2, 512), (2, 4096), (3, 12),
                                       (3, 14), (4, 16), (4, 24), (5, 13), (5, 15)])
def test_config_recipes_match_oracle(engine, cfg, scale):
    a = B.make_config(cfg, scale)
    c = gpu_mul(engine, a, a)
    o = O.spgemm_rowwise(a, a)
    assert_csr_identical(c, o, f"cfg{cfg} scale {scale}")


def test_heavy_rows_exercise_windows(engine):
    """R-MAT 16 (ef 16, a=.57) has rows far above the on-chip tile capacity:
    both sparse and dense column windows must run and stay bit-exact."""
    a = B.make_config(3, 15)
    A = engine.upload(a)
    c = engine.spgemm_rowwise(A, A).download()
    st = engine.exec_stats()
    assert st["units"][7] > 0, "no heavy rows"
    assert st["units"][8] > 0 and st["units"][9] > 0, st
    assert_csr_identical(c, O.spgemm_rowwise(a, a), "rmat15 heavy")


def test_identity_is_unit(engine):
    """reference spgemm_rowwise_test.cpp:45-51 (tolerance 0.0)."""
    b = random_csr(20, 14, 0.2, 3, nonnegative=False)
    assert B.csr_equal_canonical(gpu_mul(engine, identity_csr(20), b), b, 0.0)
    assert B.csr_equal_canonical(gpu_mul(engine, b, identity_csr(14)), b, 0.0)


def test_structural_zero_kept(engine):
    """reference spgemm_rowwise_test.cpp:85-97."""
    a = B.coo_to_csr(1, 2, [0, 0], [0, 1], [1.0, 1.0])
    b = B.coo_to_csr(2, 1, [0, 1], [0, 0], [1.0, -1.0])
    c = gpu_mul(engine, a, b)
    assert c.nnz() == 1 and c.values[0] == 0.0


@pytest.mark.parametrize("narrow", ["1", "0"])
def test_dense_oracle_corpus(engine, monkeypatch, narrow):
    """reference spgemm_rowwise_test.cpp:53-75 / acceptance_main.cpp:80-97; B of
    <= 100 columns runs the narrow-B kernel, BSP_NARROW=0 forces the tiles."""
    monkeypatch.setenv("BSP_NARROW", narrow)
    rng = np.random.default_rng(7)
    for seed in range(40):
        n, m, k = (int(x) for x in rng.integers(1, 101, size=3))
        dens = 0.01 + 0.19 * rng.random()
        a = random_csr(n, k, dens, 2 * seed + 1, nonnegative=False)
        b = random_csr(k, m, dens, 2 * seed + 2, nonnegative=False)
        c = gpu_mul(engine, a, b)
        c.check_invariants()
        assert np.allclose(c.to_dense(), a.to_dense() @ b.to_dense(), atol=1e-9, rtol=0)
        assert_csr_identical(c, O.spgemm_rowwise(a, b), f"corpus seed {seed}")


def test_symbolic_matches_oracle(engine):
    """reference spgemm_rowwise_test.cpp:25-43,77-83."""
    for seed in range(5):
        a = random_csr(60, 50, 0.12, seed)
        b = random_csr(50, 70, 0.12, seed + 50)
        A, Bd = engine.upload(a), engine.upload(b)
        assert np.array_equal(engine.spgemm_symbolic(A, Bd), O.spgemm_symbolic(a, b))
    a = B.make_config(5, 14)
    A = engine.upload(a)
    assert np.array_equal(engine.spgemm_symbolic(A, A), O.spgemm_symbolic(a, a))


def test_empty_and_ragged(engine):
    """Empty rows, empty matrix, all-empty B rows."""
    a = csr_from_rows(5, [[], [0, 4], [], [1], []])
    b = csr_from_rows(3, [[0, 2], [], [], [], [1]])
    assert_csr_identical(gpu_mul(engine, a, b), O.spgemm_rowwise(a, b), "ragged")
    z = B.coo_to_csr(4, 4, [], [], [])
    c = gpu_mul(engine, z, z)
    assert c.nnz() == 0 and np.all(c.row_ptr == 0)


def test_dimension_mismatch_rejected(engine):
    """reference spgemm_rowwise_test.cpp:99-104."""
    a = random_csr(4, 5, 0.5, 1)
    b = random_csr(4, 4, 0.5, 2)
    with pytest.raises(B.ContractError):
        engine.spgemm_rowwise(engine.upload(a), engine.upload(b))


def test_aat_symmetric_with_nnz_diagonal(engine):
    """reference spgemm_rowwise_test.cpp:106-121."""
    a = B.binarize(random_csr(26, 19, 0.25, 31))
    at = B.transpose(a)
    c = gpu_mul(engine, a, at)
    ct = B.transpose(c)
    assert B.csr_equal_canonical(c, ct, 1e-12)
    d = c.to_dense()
    for i in range(a.nrows):
        if a.row_nnz(i):
            assert d[i, i] == a.row_nnz(i)


def test_row_range_shards_concatenate(engine):
    """Row shards (multi-GPU split) concatenate to the full product, bitwise."""
    a = B.make_config(5, 14)
    A = engine.upload(a)
    full = engine.spgemm_rowwise(A, A).download()
    bounds = engine.partition_rows(A, A, 4)
    assert bounds[0] == 0 and bounds[-1] == a.nrows and np.all(np.diff(bounds) >= 0)
    # the device split follows the documented cost rule (distributed.product_split)
    deg = np.diff(a.row_ptr)
    prods = np.add.reduceat(deg[a.col_idx], a.row_ptr[:-1].clip(max=a.nnz() - 1))
    prods[np.diff(a.row_ptr) == 0] = 0
    from paper_2507_21253_b200 import distributed as D
    assert np.array_equal(bounds, D.product_split(prods, 4))
    parts = [engine.spgemm_rowwise_range(A, A, int(bounds[g]), int(bounds[g + 1])).download()
             for g in range(4)]
    assert np.array_equal(np.concatenate([p.col_idx for p in parts]), full.col_idx)
    assert same_bits(np.concatenate([p.values for p in parts]), full.values)
    off = 0
    for p, g in zip(parts, range(4)):
        assert np.array_equal(p.row_ptr + off, full.row_ptr[bounds[g]:bounds[g + 1] + 1])
        off += p.nnz()


def test_host_buffer_entry_point(engine):
    """bsp_spgemm_rowwise_host: host in, host out (the reference-shaped call)."""
    a = B.make_config(2, 1024)
    c = B.spgemm_rowwise(a, a)
    assert_csr_identical(c, O.spgemm_rowwise(a, a), "host entry")


def test_host_entry_point_chunks_rows_when_c_exceeds_budget(engine, monkeypatch):
    """When C's bound exceeds the device budget (cfg3: ~285 GB), the reference-shaped
    host call splits A's rows into chunks itself (exact counts first, each chunk's C
    downloaded into place).  A small forced budget exercises that path: same bits as
    the oracle, several chunks reported, heavy (windowed) rows included."""
    a = B.make_config(5, 14)
    want = O.spgemm_rowwise(a, a)
    monkeypatch.setenv("BSP_CHUNK_BYTES", str(4 << 20))
    c = engine.spgemm_rowwise_host(a, a)
    st = engine.exec_stats()
    assert st["chunks"] > 4, st
    assert st["nnz_out"] == want.col_idx.size
    assert_csr_identical(c, want, "chunked host entry")
    monkeypatch.delenv("BSP_CHUNK_BYTES")
    c1 = engine.spgemm_rowwise_host(a, a)
    assert engine.exec_stats()["chunks"] == 1
    assert_csr_identical(c1, want, "unchunked host entry")


def test_heavy_rows_over_empty_b_rows(engine):
    """Heavy rows (windowed) whose segments include empty B rows — the shape
    of A x frontier operands: every start-table entry must still be filled."""
    rng = np.random.default_rng(5)
    n, m = 600, 3000
    r, c = [], []
    for i in range(n):
        d = 1500 if i % 50 == 0 else int(rng.integers(1, 12))
        cols = np.sort(rng.choice(n, size=min(d, n), replace=False))
        r += [i] * cols.size
        c += cols.tolist()
    a = B.coo_to_csr(n, n, np.array(r), np.array(c), rng.random(len(r)))
    br, bc = [], []
    for k in range(n):
        if k % 3 == 0:
            continue  # empty B row
        cols = np.sort(rng.choice(m, size=int(rng.integers(5, 40)), replace=False))
        br += [k] * cols.size
        bc += cols.tolist()
    b = B.coo_to_csr(n, m, np.array(br), np.array(bc), rng.random(len(br)))
    A, Bd = engine.upload(a), engine.upload(b)
    c = engine.spgemm_rowwise(A, Bd).download()
    assert engine.exec_stats()["units"][7] > 0, "no heavy rows"
    assert_csr_identical(c, O.spgemm_rowwise(a, b), "heavy rows over empty B rows")
    # tall-skinny: every heavy row's window is one dense 64-column window
    r64, c64 = [], []
    for k in range(n):
        if k % 3:
            cols = np.sort(rng.choice(64, size=int(rng.integers(1, 20)), replace=False))
            r64 += [k] * cols.size
            c64 += cols.tolist()
    b64 = B.coo_to_csr(n, 64, np.array(r64), np.array(c64), np.ones(len(r64)))
    B64 = engine.upload(b64)
    assert_csr_identical(engine.spgemm_rowwise(A, B64).download(), O.spgemm_rowwise(a, b64),
                         "dense windows over empty B rows")


@pytest.mark.parametrize("ncols", [1, 31, 33, 63, 64, 65, 200, 256, 257])
def test_narrow_b_matches_oracle(engine, ncols):
    """Narrow B (<= 64 columns: 64-bit row masks, sums in registers; <= 256:
    one warp per row, dense accumulator) against
    the oracle, with heavy rows, hub B rows, empty rows and empty B rows;
    257 columns takes the tile path."""
    rng = np.random.default_rng(ncols)
    n = 3000
    a = B.make_config(5, 12)
    r, c = [], []
    for k in range(a.nrows):
        if k % 4 == 0:
            continue
        d = 1 + int(rng.integers(0, min(ncols, 40)))
        cols = np.sort(rng.choice(ncols, size=min(d, ncols), replace=False))
        r += [k] * cols.size
        c += cols.tolist()
    b = B.coo_to_csr(a.nrows, ncols, np.array(r), np.array(c), rng.random(len(r)) - 0.5)
    A, Bd = engine.upload(a), engine.upload(b)
    got = engine.spgemm_rowwise(A, Bd).download()
    assert_csr_identical(got, O.spgemm_rowwise(a, b), f"narrow {ncols}")
    assert engine.exec_stats()["products"] == int(np.diff(b.row_ptr)[a.col_idx].sum())


def test_counting_sort_wide_and_duplicate_tiles(engine):
    """The tile sort's paths at a 2^22 + 123-column B (cfg5's width): light
    rows whose columns span all 22 bits (counting sort with a bucket array),
    windows of heavy rows (packed-word counting sort), and rows whose products
    pile >128 copies of a few columns into one bucket (fallback to the merge /
    radix sorts after the deferred fix-up).  Ties must still sum in k order."""
    rng = np.random.default_rng(2025)
    ncols = (1 << 22) + 123
    nb = 700
    rows_b = []
    for k in range(nb):
        if k < 64:  # duplicate group: every row shares columns 100..110
            cols = np.arange(100, 111)
        else:
            cols = rng.choice(ncols, size=int(rng.integers(4, 48)), replace=False)
        rows_b.append(np.unique(cols))
    rb = np.concatenate([[k] * len(c) for k, c in enumerate(rows_b)])
    cb = np.concatenate(rows_b)
    b = B.coo_to_csr(nb, ncols, rb, cb, rng.uniform(-4.0, 4.0, size=cb.size))
    ra, ca = [], []
    for i, d in enumerate([3, 20, 40, 70, 110, 150, 400, 690]):  # light .. heavy rows
        ks = rng.choice(np.arange(64, nb), size=min(d, nb - 64), replace=False)
        ra += [i] * len(ks)
        ca += list(ks)
    for i in range(8, 12):  # duplicate-heavy rows: 64 x 11 products on 11 columns
        ks = np.concatenate([np.arange(64), rng.choice(np.arange(64, nb), 30, replace=False)])
        ra += [i] * len(ks)
        ca += list(ks)
    a = B.coo_to_csr(12, nb, np.array(ra), np.array(ca), rng.uniform(-4.0, 4.0, size=len(ra)))
    c = gpu_mul(engine, a, b)
    o = O.spgemm_rowwise(a, b)
    assert_csr_identical(c, o, "wide / duplicate tiles")
    assert engine.exec_stats()["units"][7] > 0, "no heavy rows"


def test_duplicate_heavy_rows_hash_accumulator(engine):
    """Rows whose products repeat columns (compression factor >= 2, <= 256
    outputs) run on the warp hash accumulator, summed in k order; rows with
    more outputs stay on the sort tiles.  Mixed signs make any reordering of a
    sum visible in the bits."""
    rng = np.random.default_rng(77)
    n = 4000
    rows, cols = [], []
    for i in range(n):
        if i % 7 == 0:  # wide rows: > 256 distinct outputs through the tiles
            cs = rng.choice(n, size=40, replace=False)
        else:  # stencil-like: neighbours in a small window
            cs = np.unique(np.clip(i + rng.integers(-12, 13, size=20), 0, n - 1))
        rows += [i] * len(cs)
        cols += list(cs)
    a = B.coo_to_csr(n, n, np.array(rows), np.array(cols), rng.uniform(-4, 4, size=len(rows)))
    A = engine.upload(a)
    engine.profile(True)
    c = engine.spgemm_rowwise(A, A).download()
    prof = engine.profile_report()
    engine.profile(False)
    assert_csr_identical(c, O.spgemm_rowwise(a, a), "duplicate-heavy rows")
    assert "hashacc_kernel" in prof, sorted(prof)


@pytest.mark.parametrize("nout", [255, 256, 257])
def test_hash_accumulator_output_bound(engine, nout):
    """Rows right at the hash accumulator's 256-output bound (routed when
    <= 256, tiles above), each column hit by 4 segments in k order."""
    rng = np.random.default_rng(nout)
    kseg = 4
    rows_b = [np.sort(rng.choice(nout, size=nout // 2, replace=False)) for _ in range(kseg * 8)]
    for r in range(kseg):  # make sure all nout columns occur
        rows_b[r] = np.arange(nout)
    rb_ = np.concatenate([[k] * len(cs) for k, cs in enumerate(rows_b)])
    # the nout columns spread over 5000 (B wider than the narrow kernels' 256)
    colmap = np.sort(rng.choice(5000, size=nout, replace=False))
    b = B.coo_to_csr(len(rows_b), 5000, rb_, colmap[np.concatenate(rows_b)],
                     rng.uniform(-3, 3, size=rb_.size))
    ra = np.repeat(np.arange(40), 12)
    ca = np.concatenate([np.sort(rng.choice(len(rows_b), 12, replace=False)) for _ in range(40)])
    ca[:12] = np.arange(12)  # row 0 covers the full columns (4 full B rows)
    a = B.coo_to_csr(40, len(rows_b), ra, ca, rng.uniform(-3, 3, size=ra.size))
    A, Bd = engine.upload(a), engine.upload(b)
    engine.profile(True)
    c = engine.spgemm_rowwise(A, Bd).download()
    prof = engine.profile_report()
    engine.profile(False)
    assert_csr_identical(c, O.spgemm_rowwise(a, b), f"{nout} outputs")
    assert "hashacc_kernel" in prof  # rows with fewer outputs are routed in every case


@pytest.mark.parametrize("cfg,scale", [(5, 14), (2, 512), (4, 16)])
def test_device_transpose_matches_host(engine, cfg, scale):
    """bsp_transpose (csr.hpp:115-135): a stable radix sort of the entries by column,
    so rows of A^T come out sorted and identical to the host counting-sort transpose,
    hub columns (R-MAT) and unsymmetric patterns (cfg2) included."""
    a = B.make_config(cfg, scale)
    want = B.transpose(a)
    got = engine.transpose(engine.upload(a)).download()
    assert_csr_identical(got, want, f"transpose cfg{cfg}")


_LB_KNOB_SCRIPT = r"""
import numpy as np
import oracle as O
import paper_2507_21253_b200 as B
e = B.default_engine()
for cfg, scale in ((5, 15), (3, 15), (5, 16)):
    a = B.make_config(cfg, scale)
    A = e.upload(a)
    c = e.spgemm_rowwise(A, A).download()
    assert e.exec_stats()["units"][8] > 0, "no sparse windows"
    o = O.spgemm_rowwise(a, a)
    assert np.array_equal(c.row_ptr, o.row_ptr) and np.array_equal(c.col_idx, o.col_idx), cfg
    assert np.array_equal(c.values.view(np.uint64), o.values.view(np.uint64)), cfg
print("ok")
"""


@pytest.mark.parametrize("env", [{"BSP_LB_V2": "1"}, {"BSP_LB_DMAX": "64"},
                                 {"BSP_LB_V2": "1", "BSP_LB_DMAX": "128"},
                                 {"BSP_LOOKBACK": "0"}, {"BSP_BLOCK_CACHE": "0"}, {"BSP_LB_V2": "0"}])
def test_lookback_knobs_bit_identical(env):
    """The look-back tile's second form (values gathered after the count is published), the
    split of long-row windows onto the two-pass path, the two-pass path alone and the block
    cache switch are read once per process: each runs in its own process against the oracle."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **env)
    e["PYTHONPATH"] = root + os.pathsep + os.path.join(root, "tests") + os.pathsep + e.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", _LB_KNOB_SCRIPT], env=e, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_repeated_multiply_makes_no_driver_allocation(engine):
    """A repeated multiply is served from the handle's block cache: after the first calls no
    allocation reaches the driver (exec_stats units[14]); such calls wait on the driver's
    locks whenever a GPU monitor polls, which showed as 5-300 % long steps in the bench."""
    a = B.make_config(5, 15)
    engine = B.Engine(0)  # a fresh handle: its first multiply has to allocate
    A = engine.upload(a)
    misses = []
    for _ in range(4):
        c = engine.spgemm_rowwise(A, A)
        misses.append(engine.exec_stats()["units"][14])
        c.free()
    assert misses[0] > 0 and misses[2] == 0 and misses[3] == 0, misses
    asg = engine.hierarchical_clusters(a)
    Ac = engine.build_csr_cluster(A, asg)
    misses = []
    for _ in range(4):
        c = engine.spgemm_clusterwise(Ac, A)
        misses.append(engine.exec_stats()["units"][14])
        c.free()
    assert misses[2] == 0 and misses[3] == 0, misses
