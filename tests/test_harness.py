"""The report harness (reference bench.hpp): CSV schema 1 byte for byte
against the reference's own writer (bench_csv_row / bench_csv_header, std::to_chars
doubles), parse round trip, csr_first_mismatch; and on the GPU run_bench / verify_mode
on a Matrix Market file (row-wise and cluster-wise variants, a file-driven reorder)."""
import math
import random

import numpy as np
import pytest

import oracle as O
import paper_2507_21253_b200 as B
from paper_2507_21253_b200 import harness as H

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")


@needs_ref
def test_fmt_double_is_to_chars():
    rng = random.Random(5)
    vals = [0.0, -0.0, 1.0, 100.0, 1e16, 1e15, 123456.0, 0.5, 1e-4, 1e-5, 0.0001234, 1.5e-7,
            3.14159, 2.0 ** 60, 1e21, 1e22, 5e-324, 1.7976931348623157e308, math.inf, -math.inf,
            0.1 + 0.2, 1e300, 12345678901234567.0, 0.001, 1234.5]
    vals += [rng.uniform(-1e6, 1e6) for _ in range(300)]
    vals += [10.0 ** rng.uniform(-30, 30) for _ in range(300)]
    vals += [float(rng.randint(0, 10 ** 18)) for _ in range(100)]
    for v in vals:
        assert H.fmt_double(v) == O.ref_fmt_double(v), v


def _report():
    cfg = H.BenchConfig(matrix_path="/data/m.mtx", workload="tallskinny", num_frontiers=7,
                        frontier_batch=32, frontier_seed=9,
                        reorder=B.ReorderSpec("file", 0, "/tmp/gp.perm"),
                        clustering=H.ClusteringSpec("hierarchical",
                                                    B.ClusterParams(0.35, 6, 4)),
                        repetitions=10, threads=16, warmup=True)
    return H.BenchReport(cfg, 0.25, 1.5e-3, 0.01, 0.009, 0.0125, 0.007, 0.0065, 0.0081,
                         0.01 / 0.007, 123456, 234567, 234567 / 123456, 1000, 600, 4000, 17,
                         1.75e-1 / 3e-3)


@needs_ref
def test_csv_row_and_header_identical_to_reference(tmp_path):
    r = _report()
    c = r.config
    row, header = O.ref_bench_csv_row(
        c.matrix_path, 1, 4, c.reorder.seed, c.reorder.path, 3, c.clustering.params.jacc_th,
        c.clustering.params.max_cluster_th, c.clustering.params.fixed_len, c.num_frontiers,
        c.frontier_batch, c.frontier_seed, c.repetitions, c.threads, 1,
        [r.reorder_seconds, r.cluster_build_seconds, r.baseline_mean_s, r.baseline_min_s,
         r.baseline_max_s, r.variant_mean_s, r.variant_min_s, r.variant_max_s,
         r.speedup_vs_baseline],
        [r.csr_bytes, r.cluster_bytes, r.baseline_b_row_loads, r.b_row_loads, r.a_inner_iters,
         r.placeholder_skips], r.footprint_ratio, r.amortization_iters)
    assert H.CSV_HEADER == header
    assert H.csv_row(r) == row
    # append (header once) and parse back to the identical report
    path = str(tmp_path / "r.csv")
    H.append_csv(r, path)
    r2 = _report()
    r2.config.reorder = B.ReorderSpec("rcm", 3)
    r2.amortization_iters = math.inf
    H.append_csv(r2, path)
    back = H.parse_csv(path)
    assert [H.csv_row(x) for x in back] == [H.csv_row(r), H.csv_row(r2)]
    lines = open(path).read().splitlines()
    assert lines[0] == header and len(lines) == 3


def test_parse_csv_rejects_bad_files(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("schema,oops\n")
    with pytest.raises(B.BspIOError):
        H.parse_csv(str(p))
    p.write_text(H.CSV_HEADER + "\n1,a,b\n")
    with pytest.raises(B.BspIOError):
        H.parse_csv(str(p))


def test_csr_first_mismatch():
    a = B.coo_to_csr(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 2.0, 3.0])
    assert H.csr_first_mismatch(a, a, 1e-9) is None
    b = B.coo_to_csr(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 2.0 + 1e-6, 3.0])
    assert H.csr_first_mismatch(b, a, 1e-9)[:2] == (1, 1)
    assert H.csr_first_mismatch(b, a, 1e-9)[4] == "value mismatch"
    c = B.coo_to_csr(3, 3, [0, 1, 2], [0, 2, 2], [1.0, 2.0, 3.0])
    assert H.csr_first_mismatch(c, a, 1e-9)[4] == "structure mismatch"
    d = B.coo_to_csr(3, 3, [0, 1, 1, 2], [0, 1, 2, 2], [1.0, 2.0, 5.0, 3.0])
    assert H.csr_first_mismatch(d, a, 1e-9)[4] == "row nnz mismatch"


@pytest.mark.gpu
def test_run_bench_and_verify_on_matrix_market_file(engine, tmp_path):
    a = B.make_config(2, 256)
    path = str(tmp_path / "hidden.mtx")
    B.write_matrix_market(a, path)
    perm_path = str(tmp_path / "rcm.perm")
    B.write_permutation(B.reorder_rcm(a), perm_path)
    csv = str(tmp_path / "report.csv")
    specs = [
        H.BenchConfig(matrix_path=path, repetitions=3, output_path=csv),
        H.BenchConfig(matrix_path=path, reorder=B.ReorderSpec("file", path=perm_path),
                      repetitions=3, output_path=csv),
        H.BenchConfig(matrix_path=path, clustering=H.ClusteringSpec("hierarchical"),
                      repetitions=3, warmup=True, output_path=csv),
        H.BenchConfig(matrix_path=path, workload="tallskinny", num_frontiers=3,
                      reorder=B.ReorderSpec("random", 1),
                      clustering=H.ClusteringSpec("fixed"), repetitions=2, output_path=csv),
    ]
    for cfg in specs:
        ok, msg = H.verify_mode(cfg, engine)
        assert ok, msg
        r = H.run_bench(cfg, engine)
        assert r.baseline_mean_s > 0 and r.variant_mean_s > 0 and r.speedup_vs_baseline > 0
        assert r.baseline_b_row_loads > 0 and r.b_row_loads > 0
    clustered = H.parse_csv(csv)[2]
    assert clustered.b_row_loads < clustered.baseline_b_row_loads  # B rows shared in clusters
    assert clustered.footprint_ratio > 1.0  # padded CSR_Cluster slots
    assert len(H.parse_csv(csv)) == len(specs)
