"""Benchmark / verify harness with the reference's report format.

Mirrors reference bench.hpp: an experiment (BenchConfig: matrix file, workload a2 or
tall-skinny, reorder, clustering, repetitions) is prepared (prepare_bench,
bench.hpp:128-171), timed as baseline = row-wise on the original order vs variant =
row-wise on the reordered A or cluster-wise on its CSR_Cluster (run_bench,
bench.hpp:390-460; the GPU times each execution with CUDA events on the engine's
stream), and reported as a BenchReport / CSV schema-1 row (bench.hpp:260-387, same
header, same field order, doubles in the shortest round-trip form of std::to_chars).
verify_mode (bench.hpp:227-252) checks the variant against the row-wise result on the
original order transported through the permutation (csr_first_mismatch, tol 1e-9).
"""
from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import (AccessStats, ClusterAssignment, ClusterParams, CsrMatrix, Engine, ReorderSpec,
               default_engine, fixed_length_clusters, load_matrix_market, make_permutation,
               permute_rows, permute_symmetric, variable_length_clusters)

CSV_SCHEMA = 1
CSV_HEADER = ("schema,matrix,workload,reorder,reorder_seed,cluster,jacc_th,max_cluster,fixed_len,"
              "num_frontiers,frontier_batch,frontier_seed,reps,threads,warmup,"
              "reorder_seconds,cluster_build_seconds,"
              "baseline_mean_s,baseline_min_s,baseline_max_s,"
              "variant_mean_s,variant_min_s,variant_max_s,speedup_vs_baseline,"
              "csr_bytes,cluster_bytes,footprint_ratio,"
              "baseline_b_row_loads,b_row_loads,a_inner_iters,placeholder_skips,"
              "amortization_iters")


@dataclass
class ClusteringSpec:
    """reference ClusteringSpec (bench.hpp:33-49): none / fixed / variable /
    hierarchical (+ candidates: "topk" as the reference, or "minhash")."""
    method: str = "none"
    params: ClusterParams = field(default_factory=ClusterParams)
    candidates: str = "topk"

    def name(self) -> str:
        return self.method if self.method in ("none", "fixed", "variable") else "hierarchical"


@dataclass
class BenchConfig:
    """reference BenchConfig (bench.hpp:62-75)."""
    matrix_path: str = ""
    workload: str = "a2"  # "a2" | "tallskinny"
    num_frontiers: int = 10
    frontier_batch: int = 64
    frontier_seed: int = 0
    reorder: ReorderSpec = field(default_factory=ReorderSpec)
    clustering: ClusteringSpec = field(default_factory=ClusteringSpec)
    repetitions: int = 10
    threads: int = 0
    warmup: bool = False
    output_path: str = ""


@dataclass
class BenchReport:
    """reference BenchReport (bench.hpp:80-97)."""
    config: BenchConfig
    reorder_seconds: float = 0.0
    cluster_build_seconds: float = 0.0
    baseline_mean_s: float = 0.0
    baseline_min_s: float = 0.0
    baseline_max_s: float = 0.0
    variant_mean_s: float = 0.0
    variant_min_s: float = 0.0
    variant_max_s: float = 0.0
    speedup_vs_baseline: float = 0.0
    csr_bytes: int = 0
    cluster_bytes: int = 0
    footprint_ratio: float = 0.0
    baseline_b_row_loads: int = 0
    b_row_loads: int = 0
    a_inner_iters: int = 0
    placeholder_skips: int = 0
    amortization_iters: float = 0.0


@dataclass
class Prepared:
    a_original: CsrMatrix
    a_variant: CsrMatrix
    perm: object
    b_original: List[CsrMatrix]
    b_variant: List[CsrMatrix]
    assignment: Optional[ClusterAssignment]
    reorder_seconds: float
    cluster_build_seconds: float


# ------------------------------------------------------------------ doubles
def fmt_double(v: float) -> str:
    """std::to_chars(double) with no format: the shortest round-trip digits, in
    fixed or scientific notation, whichever is shorter (fixed on a tie)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    a = abs(v)
    if a == 0.0:
        return sign + "0"
    r = repr(a)  # shortest round-trip digits
    mant, _, ex = r.partition("e")
    exp = int(ex) if ex else 0
    ip, _, fp = mant.partition(".")
    fp = "" if fp == "0" and not ex else fp
    digits = (ip + fp).lstrip("0")
    # value = 0.<digits> x 10^point, point = position of the decimal point
    point = len(ip.lstrip("0")) + exp if ip.strip("0") else exp - (len(fp) - len(fp.lstrip("0")))
    digits = digits.rstrip("0") or "0"
    # scientific: d[.ddd]e±XX
    e10 = point - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + \
        ("e-" if e10 < 0 else "e+") + f"{abs(e10):02d}"
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= len(digits):
        # an integer: %f prints its exact decimal expansion (same length)
        fixed = str(int(a))
    else:
        fixed = digits[:point] + "." + digits[point:]
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def csv_row(r: BenchReport) -> str:
    c = r.config
    f = fmt_double
    return ",".join(str(x) for x in (
        CSV_SCHEMA, c.matrix_path, c.workload, c.reorder.name(), c.reorder.seed,
        c.clustering.name(), f(c.clustering.params.jacc_th), c.clustering.params.max_cluster_th,
        c.clustering.params.fixed_len, c.num_frontiers, c.frontier_batch, c.frontier_seed,
        c.repetitions, c.threads, 1 if c.warmup else 0, f(r.reorder_seconds),
        f(r.cluster_build_seconds), f(r.baseline_mean_s), f(r.baseline_min_s),
        f(r.baseline_max_s), f(r.variant_mean_s), f(r.variant_min_s), f(r.variant_max_s),
        f(r.speedup_vs_baseline), r.csr_bytes, r.cluster_bytes, f(r.footprint_ratio),
        r.baseline_b_row_loads, r.b_row_loads, r.a_inner_iters, r.placeholder_skips,
        f(r.amortization_iters)))


def append_csv(r: BenchReport, path: str) -> None:
    """reference append_bench_csv (bench.hpp:293-302)."""
    need_header = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a") as out:
        if need_header:
            out.write(CSV_HEADER + "\n")
        out.write(csv_row(r) + "\n")


def parse_csv(path: str) -> List[BenchReport]:
    """reference parse_bench_csv (bench.hpp:305-387)."""
    from . import BspIOError

    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise BspIOError(f"{path}: empty report file")
    if lines[0] != CSV_HEADER:
        raise BspIOError(f"{path}: unrecognized report header (schema mismatch)")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 32:
            raise BspIOError(f"{path}: malformed row (expected 32 fields, got {len(f)})")
        if int(f[0]) != CSV_SCHEMA:
            raise BspIOError(f"{path}: unsupported schema version {f[0]}")
        rn = f[3]
        if rn in ("original", "random", "degree", "rcm"):
            ro = ReorderSpec(rn, int(f[4]))
        else:
            ro = ReorderSpec("file", int(f[4]), rn[rn.find(":") + 1:])
        cn = f[5] if f[5] in ("none", "fixed", "variable") else "hierarchical"
        cs = ClusteringSpec(cn, ClusterParams(jacc_th=float(f[6]), max_cluster_th=int(f[7]),
                                              fixed_len=int(f[8])))
        cfg = BenchConfig(matrix_path=f[1], workload="a2" if f[2] == "a2" else "tallskinny",
                          num_frontiers=int(f[9]), frontier_batch=int(f[10]),
                          frontier_seed=int(f[11]), reorder=ro, clustering=cs,
                          repetitions=int(f[12]), threads=int(f[13]), warmup=f[14] == "1")
        d = [float(x) for x in f[15:24]]
        out.append(BenchReport(cfg, *d, int(f[24]), int(f[25]), float(f[26]), int(f[27]),
                               int(f[28]), int(f[29]), int(f[30]), float(f[31])))
    return out


# ------------------------------------------------------------------ harness
def prepare_bench(cfg: BenchConfig, engine: Optional[Engine] = None,
                  a: Optional[CsrMatrix] = None) -> Prepared:
    """reference detail::prepare_bench (bench.hpp:128-171).  `a` (optional) skips
    loading cfg.matrix_path."""
    from . import ContractError

    e = engine or default_engine()
    a0 = a if a is not None else load_matrix_market(cfg.matrix_path)
    if a0.nrows != a0.ncols:
        raise ContractError("bench: both workloads require a square A matrix")
    t0 = time.perf_counter()
    perm = make_permutation(cfg.reorder, a0)
    t_re = time.perf_counter() - t0
    av = permute_symmetric(a0, perm)
    if cfg.workload == "a2":
        b0, bv = [a0], [av]
    else:
        A0 = e.upload(a0)
        fs = e.generate_frontiers(A0, cfg.num_frontiers, cfg.frontier_batch, cfg.frontier_seed)
        b0 = [f.download() for f in fs]
        bv = [permute_rows(f, perm) for f in b0]
    asg, t_cl = None, 0.0
    if cfg.clustering.method != "none":
        t0 = time.perf_counter()
        prm = cfg.clustering.params
        if cfg.clustering.method == "fixed":
            asg = fixed_length_clusters(av.nrows, prm.fixed_len)
        elif cfg.clustering.method == "variable":
            asg = variable_length_clusters(av, prm)
        else:
            asg = e.hierarchical_clusters(av, prm, method=cfg.clustering.candidates)
        t_cl = time.perf_counter() - t0
    return Prepared(a0, av, perm, b0, bv, asg, t_re, t_cl)


def _timer(e: Engine):
    import torch

    s = torch.cuda.ExternalStream(e.stream_ptr()) if e.stream_ptr() else None

    def run(fn) -> float:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if s is not None:
            ev0.record(s)
        else:
            ev0.record()
        fn()
        if s is not None:
            ev1.record(s)
        else:
            ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) * 1e-3

    return run


def run_bench(cfg: BenchConfig, engine: Optional[Engine] = None,
              a: Optional[CsrMatrix] = None) -> BenchReport:
    """reference run_bench (bench.hpp:390-460), timed on the GPU."""
    from . import ContractError

    if cfg.repetitions < 1:
        raise ContractError("bench: repetitions must be >= 1")
    e = engine or default_engine()
    p = prepare_bench(cfg, e, a)
    r = BenchReport(cfg, p.reorder_seconds, p.cluster_build_seconds)
    A0, AV = e.upload(p.a_original), e.upload(p.a_variant)
    B0 = [e.upload(b) for b in p.b_original]
    BV = [e.upload(b) for b in p.b_variant]
    t_build = time.perf_counter()
    Ac = e.build_csr_cluster(AV, p.assignment) if p.assignment is not None else None
    if Ac is not None:
        e.synchronize()
        r.cluster_build_seconds += time.perf_counter() - t_build
    timed = _timer(e)

    def rowwise(A, Bs):
        for b in Bs:
            e.spgemm_rowwise(A, b).free()

    def clusterwise(Bs):
        for b in Bs:
            e.spgemm_clusterwise(Ac, b).free()

    tb, tv = [], []
    for rep in range(cfg.repetitions + (1 if cfg.warmup else 0)):
        x = timed(lambda: rowwise(A0, B0))
        y = timed(lambda: clusterwise(BV)) if Ac is not None else timed(lambda: rowwise(AV, BV))
        if cfg.warmup and rep == 0:
            continue
        tb.append(x)
        tv.append(y)
    r.baseline_mean_s, r.baseline_min_s, r.baseline_max_s = \
        float(np.mean(tb)), float(min(tb)), float(max(tb))
    r.variant_mean_s, r.variant_min_s, r.variant_max_s = \
        float(np.mean(tv)), float(min(tv)), float(max(tv))
    r.speedup_vs_baseline = r.baseline_mean_s / r.variant_mean_s
    for b in B0:
        s = e.rowwise_access_stats(A0, b)
        r.baseline_b_row_loads += s.b_row_loads
    for b in BV:
        s = e.cluster_access_stats(Ac, b) if Ac is not None else e.rowwise_access_stats(AV, b)
        r.b_row_loads += s.b_row_loads
        r.a_inner_iters += s.a_inner_iters
        r.placeholder_skips += s.placeholder_skips
    # footprint (cluster_format.hpp:247-267), 4-byte indices
    w = 4
    r.csr_bytes = (p.a_variant.nrows + 1) * w + p.a_variant.nnz() * (w + 8)
    if Ac is not None:
        s = Ac.s
        r.cluster_bytes = (s.nclusters * w + (s.nclusters + 1) * w + s.ncolslots * w +
                           (s.nclusters + 1) * w + s.nslots * 8 + ((s.nslots + 63) // 64) * 8 +
                           s.nrows * w)
    else:
        r.cluster_bytes = r.csr_bytes
    r.footprint_ratio = r.cluster_bytes / r.csr_bytes
    gain = r.baseline_mean_s - r.variant_mean_s
    pre = r.reorder_seconds + r.cluster_build_seconds
    r.amortization_iters = pre / gain if gain > 0 else math.inf
    if cfg.output_path:
        append_csv(r, cfg.output_path)
    return r


def csr_first_mismatch(a: CsrMatrix, b: CsrMatrix, tol: float) -> Optional[Tuple]:
    """reference csr_first_mismatch (csr.hpp:215-241): (row, col, lhs, rhs, what) or None."""
    if a.nrows != b.nrows or a.ncols != b.ncols:
        return (-1, -1, 0.0, 0.0, "shape mismatch")
    la, lb = np.diff(a.row_ptr), np.diff(b.row_ptr)
    for i in range(a.nrows):
        ca, cb = a.row_cols(i), b.row_cols(i)
        n = min(ca.size, cb.size)
        bad = np.flatnonzero(ca[:n] != cb[:n])
        vbad = np.flatnonzero(np.abs(a.row_vals(i)[:n] - b.row_vals(i)[:n]) > tol)
        k = min(bad[0] if bad.size else n, vbad[0] if vbad.size else n)
        if k < n:
            if bad.size and bad[0] == k:
                return (i, int(ca[k]), 0.0, 0.0, "structure mismatch")
            return (i, int(ca[k]), float(a.row_vals(i)[k]), float(b.row_vals(i)[k]),
                    "value mismatch")
        if la[i] != lb[i]:
            return (i, -1, 0.0, 0.0, "row nnz mismatch")
    return None


def verify_mode(cfg: BenchConfig, engine: Optional[Engine] = None,
                a: Optional[CsrMatrix] = None) -> Tuple[bool, str]:
    """reference verify_mode (bench.hpp:227-252): (pass, message)."""
    try:
        e = engine or default_engine()
        p = prepare_bench(cfg, e, a)
        Ac = e.build_csr_cluster(e.upload(p.a_variant), p.assignment) \
            if p.assignment is not None else None
        AV = e.upload(p.a_variant)
        A0 = e.upload(p.a_original)
        for t, (b0, bv) in enumerate(zip(p.b_original, p.b_variant)):
            ref = e.spgemm_rowwise(A0, e.upload(b0)).download()
            tr = permute_symmetric(ref, p.perm) if cfg.workload == "a2" else permute_rows(ref, p.perm)
            Bv = e.upload(bv)
            act = (e.spgemm_clusterwise(Ac, Bv) if Ac is not None
                   else e.spgemm_rowwise(AV, Bv)).download()
            mm = csr_first_mismatch(act, tr, 1e-9)
            if mm is not None:
                msg = "mismatch"
                if len(p.b_original) > 1:
                    msg += f" at frontier {t}"
                msg += f": {mm[4]} at ({mm[0]}, {mm[1]})"
                if mm[4] == "value mismatch":
                    msg += f" got {mm[2]!r} want {mm[3]!r}"
                return False, msg
        return True, "ok"
    except Exception as ex:  # the reference returns the exception text
        return False, str(ex)
