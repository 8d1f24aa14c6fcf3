#!/usr/bin/env python
"""bench.py — A·B SpGEMM GFLOP/s (2 x intermediate products / s) and % of the
HBM roofline on B200 (BASELINE.json metric).

Workload (N=1): BASELINE cfg5, R-MAT scale 22 / edge factor 8 /
(0.45, 0.22, 0.22, 0.11), symmetrised, C = A·A row-wise (the largest
single-GPU configuration).  N>1 (torchrun): the same matrix,
A rows sharded by cumulative products, B replicated with an NCCL broadcast
(outside the timed region), no collective during the multiply.

One step = one complete multiply (products/binning, symbolic, int64 scan,
C allocation from the stream-ordered pool, numeric) on inputs already
resident in HBM.  Inputs (A = B, 0.81 GB) exceed the 126 MB L2, so no L2
flush is needed between steps.

Keys beyond the driver contract:
  e2e          the same metric through the reference-shaped host-buffer
               pipeline (pinned host A -> H2D -> multiply in row chunks ->
               D2H of every chunk of C into pinned host buffers), timed per
               step on the wall clock with the copies inside.
  roofline     bytes_alg = 12(nnzA+nnzB+nnzC) + 8(rowsA+rowsB+rowsC+3)
                / measured step time vs MEASURED_PEAKS hbm_gbs.
  cpu_baseline the UNMODIFIED reference (oracle/_ref, OpenMP, all host cores)
               on a bounded strided row sample of the same matrix.

--impl reference: times the reference's CPU row-wise SpGEMM (oracle/_ref)
on bounded row samples of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CFG = 5
PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        d = json.loads(PEAKS.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def bytes_alg(nnz_a, nnz_b, nnz_c, rows_a, rows_b, rows_c):
    return 12 * (nnz_a + nnz_b + nnz_c) + 8 * (rows_a + rows_b + rows_c + 3)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    The sampler is started BEFORE the warm-up steps: nvidia-smi's start-up holds
    driver locks for tens of ms, and a multiply whose allocation or launch waits
    on them ran 40-90 ms long when the sampler started with the first timed step.
    `mark()` is called at the start of the timed region; only the samples taken
    after it (nvidia-smi's own timestamps) are summarised."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.t_mark = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "250"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def mark(self):
        import datetime
        self.t_mark = datetime.datetime.now()

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.proc.kill()

    def summary(self):
        import datetime
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if self.t_mark is not None:
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f")
                    if ts < self.t_mark:
                        continue
                except ValueError:
                    pass
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# The workload (BASELINE cfg5), shared by both arms.  The reference arm builds
# its input with the oracle's C restatement of the generator (oracle/gen.c,
# pinned bit-for-bit to the product's in tests/test_oracle.py), so that
# process never loads the product library.
CFG5 = dict(scale=22, ef=8, a=0.45, b=0.22, c=0.22, seed=5)
PINNED_NNZ_C = {22: 11522129996}  # nnz(C) of cfg5, pinned by tests/test_gpu_fullsize.py


def workload_config(n, nnz_a, products, nnz_c, world, scale):
    """The `config` object of both arms' JSON lines (identical by construction)."""
    return {"workload": "cfg5_rmat22_ef8_AxA_rowwise" if scale is None
            else f"rmat{scale}_ef8_AxA_rowwise",
            "n": n, "nnz_a": nnz_a, "products": products, "nnz_c": nnz_c,
            "parallelism": f"row-shard x{world}", "l2": "inputs larger than L2"}


def row_products(a):
    """Intermediate products per row of A·A (row_upper_bound, spgemm.hpp:31-36)."""
    cs = np.concatenate([[0], np.cumsum(np.diff(a.row_ptr)[a.col_idx], dtype=np.int64)])
    return cs[a.row_ptr[1:]] - cs[a.row_ptr[:-1]]


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sub_rows(a, rows):
    """The rows `rows` of A as a CSR (the reference-side sample operand)."""
    import oracle as O

    rows = np.asarray(rows, np.int64)
    lens = np.diff(a.row_ptr)[rows]
    rp = np.zeros(rows.size + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    idx = (np.concatenate([np.arange(a.row_ptr[r], a.row_ptr[r + 1]) for r in rows])
           if rows.size else np.zeros(0, np.int64))
    return O.Csr(rows.size, a.ncols, rp, a.col_idx[idx], a.values[idx])


def ref_rowwise_samples(a, stride, offsets, threads):
    """The unmodified reference's spgemm_rowwise (oracle/_ref, OpenMP on `threads`
    cores) on strided row samples {o, o+stride, ...} of A against the full B = A.
    Operands are converted to the reference's own types outside the timed call;
    only spgemm_rowwise is timed.  Returns [(seconds, products)] per offset."""
    import oracle as O

    bref = O.RefCsr(a)
    blen = np.diff(a.row_ptr)
    out = []
    for off in offsets:
        sub = sub_rows(a, np.arange(off, a.nrows, stride, dtype=np.int64))
        aref = O.RefCsr(sub)
        secs, _ = O.ref_time_rowwise(aref, bref, threads)
        out.append((secs, int(blen[sub.col_idx].sum())))
        del aref
    return out


def ref_clusterwise_sample(a, cluster_ptr, rows, stride, threads):
    """The reference's row-wise and cluster-wise paths (bench.hpp:176-193) on the
    same rows: every `stride`-th cluster of the assignment (its rows, in cluster
    order), B = full A; build_csr_cluster outside the timing.  Returns (row-wise s,
    cluster-wise s, products, clusters, rows)."""
    import oracle as O

    cp = np.asarray(cluster_ptr, np.int64)
    sel = np.arange(0, cp.size - 1, stride)
    lens = cp[sel + 1] - cp[sel]
    sptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    srows = np.concatenate([rows[cp[c]:cp[c + 1]] for c in sel]).astype(np.int64)
    sub = sub_rows(a, srows)  # sample rows, renumbered 0..R-1 in cluster order
    bref = O.RefCsr(a)
    aref = O.RefCsr(sub)
    acl = O.RefCluster(aref, sptr, np.arange(srows.size, dtype=np.int32))
    t_row, _ = O.ref_time_rowwise(aref, bref, threads)
    t_cl, _ = O.ref_time_clusterwise(acl, bref, threads)
    prods = int(np.diff(a.row_ptr)[sub.col_idx].sum())
    return t_row, t_cl, prods, int(sel.size), int(srows.size)


def run_reference(args, world: int):
    """--impl reference: the reference's own CPU row-wise SpGEMM (oracle/_ref, the
    unmodified headers) on the host cores, on this workload — each step a bounded
    sample (1/stride of A's rows against the full B = A, a different offset per
    step), the throughput being products / time over the timed steps."""
    import oracle as O

    if not O.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    scale = CFG5["scale"] if args.scale is None else args.scale
    a = O.gen_rmat(scale, CFG5["ef"], CFG5["a"], CFG5["b"], CFG5["c"], CFG5["seed"])
    products = int(row_products(a).sum())
    nnz_c = PINNED_NNZ_C.get(scale)
    if nnz_c is None:
        nnz_c = int(O.ref_spgemm_symbolic(a, a).sum())
    threads = os.cpu_count() or 1
    stride = args.ref_stride
    res = ref_rowwise_samples(a, stride, [s % stride for s in range(args.warmup + args.steps)],
                              threads)[args.warmup:]
    secs = sum(t for t, _ in res)
    prods = sum(p for _, p in res)
    value = 2.0 * prods / secs / 1e9
    sample = (f"per step 1/{stride} of A's rows (i = s mod {stride}, step s) x full B = A; "
              f"{prods} products in {secs:.2f} s over {args.steps} steps; only "
              f"spgemm_rowwise timed; {cpu_model()}, {threads} threads")
    line = {
        "impl": "reference", "metric": "A·B SpGEMM GFLOP/s (2×products/s)", "value": value,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded R-MAT, BASELINE cfg5; inputs 0.81 GB > L2, no flush)",
        "config": workload_config(a.nrows, int(a.row_ptr[-1]), products, nnz_c, world, args.scale),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "cpu": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=None, help="override R-MAT scale (debug)")
    ap.add_argument("--ref-stride", type=int, default=512)
    ap.add_argument("--cpu-stride", type=int, default=128)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--workload", default="a2", choices=["a2", "ts", "cfg2", "cfg4"],
                    help="a2: C = A*A (headline); ts: A x 10 BFS frontiers of 64 sources "
                         "(square x tall-skinny, SURVEY 8(f)-1); cfg2 / cfg4: row-wise vs "
                         "cluster-wise on the clustered configs (BASELINE targets)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # plumbing check only (not a measurement): BSP_BENCH_SHARED_GPU=1 puts every
    # rank on cuda:0 and talks gloo, so the N-rank code path runs on one GPU
    shared_gpu = os.environ.get("BSP_BENCH_SHARED_GPU") == "1"
    if shared_gpu:
        local = 0

    if args.impl == "reference":
        if rank != 0:
            return
        os.environ.setdefault("OMP_PROC_BIND", "spread")
        os.environ.setdefault("OMP_PLACES", "cores")
        run_reference(args, world)
        return

    import paper_2507_21253_b200 as B

    import torch

    torch.cuda.set_device(local)
    if args.workload == "ts":
        if rank == 0:
            run_tall_skinny(B, args)
        return
    if args.workload in ("cfg2", "cfg4"):
        if rank == 0:
            run_clustered(B, args)
        return
    dist = None
    if world > 1:
        import torch.distributed as dist

        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    # ---- input: generated on rank 0, replicated by the engine's own NCCL ----
    # communicator (bsp_comm_init + bsp_csr_broadcast, NVLink); the broadcast is
    # timed on the device and reported, outside the multiply's timed region.
    engine_comm = world > 1 and not shared_gpu
    a = B.make_config(CFG, args.scale) if rank == 0 else None
    eng = B.Engine(local)
    stream = torch.cuda.Stream()
    eng.set_stream(stream.cuda_stream)
    bcast_ms = 0.0
    if engine_comm:
        # the engine's own NCCL communicator; if it cannot be set up on every rank
        # (checked with an all-reduce), fall back to torch.distributed + row ranges
        ok = torch.ones(1, device="cuda")
        try:
            uid = torch.zeros(B.L.BSP_NCCL_ID_BYTES, dtype=torch.uint8, device="cuda")
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(B.Engine.nccl_unique_id()),
                                           dtype=torch.uint8))
            dist.broadcast(uid, 0)
            eng.comm_init(world, rank, bytes(uid.cpu().numpy().tobytes()))
        except Exception as ex:  # reported; the torch path below still measures
            print(f"[bench] engine NCCL communicator unavailable ({ex}); "
                  "falling back to torch.distributed", file=sys.stderr)
            ok.zero_()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        engine_comm = bool(ok.item() > 0)
    if engine_comm:
        A_root = eng.upload(a) if rank == 0 else None
        eng.synchronize()
        A, bcast_ms = eng.broadcast(A_root, 0)
        rp_t, ci_t, v_t = A.torch_views()
        n, ncols, nnz = A.nrows, A.ncols, A.nnz()
    else:
        if rank == 0:
            meta = torch.tensor([a.nrows, a.ncols, a.nnz()], dtype=torch.int64, device="cuda")
        else:
            meta = torch.zeros(3, dtype=torch.int64, device="cuda")
        if dist:
            dist.broadcast(meta, 0)
        n, ncols, nnz = (int(x) for x in meta.tolist())
        if rank == 0:
            rp_t = torch.from_numpy(a.row_ptr).cuda()
            ci_t = torch.from_numpy(a.col_idx).cuda()
            v_t = torch.from_numpy(a.values).cuda()
        else:
            rp_t = torch.empty(n + 1, dtype=torch.int64, device="cuda")
            ci_t = torch.empty(nnz, dtype=torch.int32, device="cuda")
            v_t = torch.empty(nnz, dtype=torch.float64, device="cuda")
        if dist:
            for t in (rp_t, ci_t, v_t):
                dist.broadcast(t, 0)
        torch.cuda.synchronize()
        A = eng.view_torch(n, ncols, rp_t, ci_t, v_t)
    total_products = eng.spgemm_products(A, A)
    bounds = eng.partition_rows(A, A, world) if world > 1 else np.array([0, n])
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])

    def step():
        if world == 1:
            return eng.spgemm_rowwise(A, A)
        if engine_comm:  # bsp_spgemm_rowwise_sharded: this rank's row block, no gather
            return eng.spgemm_rowwise_sharded(A, A, gather=False)[0]
        return eng.spgemm_rowwise_range(A, A, r0, r1)

    with ClockSampler(local) as clk:  # started before the warm-up (see ClockSampler)
        for _ in range(args.warmup):
            C = step()
            C.free()
        torch.cuda.synchronize()

        # ---- timed region: exactly K steps, events on the engine's stream ----
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        nnz_c_local = 0
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = eng.kernel_launches()
        clk.mark()
        t_wall0 = time.perf_counter()
        for s in range(args.steps):
            evs[s][0].record(stream)
            C = step()
            evs[s][1].record(stream)
            nnz_c_local = C.nnz()
            C.free()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    launches = eng.kernel_launches() - l0
    step_ms = [s.elapsed_time(e) for s, e in evs]
    local_ms = float(sum(step_ms))
    # per-kernel breakdown of one extra (untimed) profiled step
    eng.profile(True)
    C = step()
    C.free()
    kprof = eng.profile_report()
    eng.profile(False)

    t = torch.tensor([local_ms, float(nnz_c_local)], dtype=torch.float64, device="cuda")
    if dist:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum[1:], op=dist.ReduceOp.SUM)
        total_ms, nnz_c = float(tmax[0]), int(tsum[1])
    else:
        total_ms, nnz_c = local_ms, nnz_c_local
    ms_per_step = total_ms / args.steps
    value = 2.0 * total_products / (ms_per_step * 1e-3) / 1e9

    # ---- e2e: host-buffer pipeline through the public API (all ranks) ----
    e2e = None
    if not args.no_e2e:
        host = [t_.cpu().numpy() for t_ in (rp_t, ci_t, v_t)]
        e2e = run_e2e(B, eng, host, n, ncols, args, total_products, rank, world, dist)

    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_kind = hbm_peak()
    bal = bytes_alg(nnz, nnz, nnz_c, n, n, n)
    achieved = bal / (ms_per_step * 1e-3) / 1e9
    ktot = sum(v[1] for v in kprof.values()) or 1.0
    top = max(kprof.items(), key=lambda kv: kv[1][1]) if kprof else ("none", (0, 0.0))
    kernels = {k: {"launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / ktot, 4)}
               for k, v in sorted(kprof.items(), key=lambda kv: -kv[1][1])}
    traffic = None
    tf = ROOT / "profiles" / "traffic_cfg5.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("dram_bytes_per_step")
        except Exception:
            traffic = None

    line = {
        "metric": "A·B SpGEMM GFLOP/s (2×products/s)",
        "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step,
        "step_ms": [round(x, 3) for x in step_ms], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded R-MAT, BASELINE cfg5; inputs 0.81 GB > L2, no flush)",
        "config": workload_config(n, nnz, total_products, nnz_c, world, args.scale),
        "gpu_launches": launches,
        "b_broadcast_ms": round(bcast_ms, 3) if engine_comm else None,
        "wall_ms_per_step": 1e3 * t_wall / args.steps,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                     "frac": achieved / (peak * world), "traffic": traffic,
                     "bytes_alg_per_step": bal, "peak_source": peak_kind,
                     "unit_of_work": "one full multiply (all kernels of the step)",
                     "dominant_kernel": top[0], "dominant_share": round(top[1][1] / ktot, 4)},
        "kernels": kernels,
        "clocks": clk.summary(),
    }

    if e2e is not None:
        line["e2e"] = e2e
    # ---- cpu baseline (rank 0, N=1) --------------------------------------
    if not args.no_cpu and world == 1:
        import oracle as O

        if O.have_ref():
            threads = os.cpu_count() or 1
            (secs, prods), = ref_rowwise_samples(a, args.cpu_stride, [0], threads)
            cb = {"value": 2.0 * prods / secs / 1e9, "unit": "GFLOP/s", "cores": threads,
                  "kind": "reference", "cpu": cpu_model(),
                  "sample": f"rows i = 0 mod {args.cpu_stride} (1/{args.cpu_stride} of rows) x "
                            f"full B = A, {prods} products, {secs:.2f} s; only the reference's "
                            f"spgemm_rowwise timed"}
            # the reference's cluster-wise path beside it (bench.hpp:185-193), on the
            # rows of every cpu_stride-th cluster of the hierarchical clustering
            # (clusters from the GPU top-k candidates + the reference's merge rule)
            try:
                t0 = time.perf_counter()
                asg = eng.hierarchical_clusters(a)
                t_clu = time.perf_counter() - t0
                t_row, t_cl, cp, ncl, nrw = ref_clusterwise_sample(
                    a, asg.cluster_ptr, asg.rows, args.cpu_stride, threads)
                cb["clusterwise"] = {
                    "rowwise_value": 2.0 * cp / t_row / 1e9,
                    "clusterwise_value": 2.0 * cp / t_cl / 1e9, "unit": "GFLOP/s",
                    "sample": f"every {args.cpu_stride}-th cluster of {asg.nclusters} "
                              f"(hierarchical, GPU clustering {t_clu:.1f} s): {ncl} clusters, "
                              f"{nrw} rows, {cp} products; row-wise {t_row:.2f} s, "
                              f"cluster-wise {t_cl:.2f} s on the same rows"}
            except Exception as ex:  # reported, never fatal for the bench line
                cb["clusterwise"] = {"error": str(ex)[:200]}
            line["cpu_baseline"] = cb
        else:
            line["cpu_baseline"] = None
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_tall_skinny(B, args, num_frontiers=10, batch=64, seed=0):
    """Square x tall-skinny (bench.hpp:129-193 with Workload::tall_skinny):
    B_t = the BFS frontiers of A (generate_frontiers, frontier.hpp:20-77; 10 x
    64 sources, seed 0, original order), one step = C_t = A * B_t for every
    t (time_rowwise / time_clusterwise, bench.hpp:172-193), A clustered once
    (hierarchical) and reused — the paper's amortisation scenario."""
    import torch

    a = B.make_config(CFG, args.scale)
    eng = B.Engine(0)
    stream = torch.cuda.Stream()
    eng.set_stream(stream.cuda_stream)
    A = eng.upload(a)
    fs = eng.generate_frontiers(A, num_frontiers, batch, seed)
    products = sum(eng.spgemm_products(A, f) for f in fs)
    asg = eng.hierarchical_clusters(a)
    Ac = eng.build_csr_cluster(A, asg)

    def timed(fn):
        for _ in range(args.warmup):
            for f in fs:
                fn(f).free()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = eng.kernel_launches()
        e0.record(stream)
        for _ in range(args.steps):
            for f in fs:
                fn(f).free()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps, eng.kernel_launches() - l0

    with ClockSampler(0) as clk:
        ms_row, launches = timed(lambda f: eng.spgemm_rowwise(A, f))
        ms_cl, _ = timed(lambda f: eng.spgemm_clusterwise(Ac, f))
    nnz_c = 0
    for f in fs:
        C = eng.spgemm_rowwise(A, f)
        nnz_c += C.nnz()
        C.free()
    peak, peak_kind = hbm_peak()
    bal = sum(bytes_alg(a.nnz(), f.nnz(), 0, a.nrows, f.nrows, a.nrows) for f in fs) + 12 * nnz_c
    line = {
        "metric": "A·B SpGEMM GFLOP/s (2×products/s)",
        "value": 2.0 * products / (ms_row * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_row,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded R-MAT, BASELINE cfg5; frontiers by device BFS)",
        "config": {"workload": f"cfg5_rmat22_x_{len(fs)}_frontiers_b{batch}_rowwise",
                   "n": a.nrows, "nnz_a": a.nnz(), "frontiers": len(fs), "batch": batch,
                   "nnz_b": [f.nnz() for f in fs], "products": products, "nnz_c": nnz_c,
                   "parallelism": "x1"},
        "clusterwise": {"value": 2.0 * products / (ms_cl * 1e-3) / 1e9, "ms_per_step": ms_cl,
                        "clusters": asg.nclusters},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": bal / (ms_row * 1e-3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": bal / (ms_row * 1e-3) / 1e9 / peak,
                     "traffic": None, "bytes_alg_per_step": bal, "peak_source": peak_kind,
                     "unit_of_work": "all frontier multiplies of one step"},
        "clocks": clk.summary(),
    }
    if not args.no_cpu:
        import oracle as O

        if O.have_ref():
            stride = args.cpu_stride
            sub = sub_rows(a, np.arange(0, a.nrows, stride, dtype=np.int64))
            aref = O.RefCsr(sub)
            secs, prods = 0.0, 0
            for f in fs:
                fh = f.download()
                prods += int(np.diff(fh.row_ptr)[sub.col_idx].sum())
                fref = O.RefCsr(O.Csr(fh.nrows, fh.ncols, fh.row_ptr, fh.col_idx, fh.values))
                t, _ = O.ref_time_rowwise(aref, fref, os.cpu_count() or 1)
                secs += t
            line["cpu_baseline"] = {"value": 2.0 * prods / secs / 1e9, "unit": "GFLOP/s",
                                    "cores": os.cpu_count(), "kind": "reference",
                                    "cpu": cpu_model(),
                                    "sample": f"rows i = 0 mod {stride} of A x every frontier; "
                                              f"only spgemm_rowwise timed"}
    for f in fs:
        f.free()
    print(json.dumps(line), flush=True)


def run_clustered(B, args):
    """BASELINE's cluster-wise comparisons: cfg2 = row-wise vs cluster-wise
    on the permuted hidden-cluster matrix (hierarchical clustering; the row-wise line is the
    value); cfg4 = row-wise unreordered, row-wise after RCM, cluster-wise after RCM +
    hierarchical.  All timed in the same run with CUDA events on the engine's stream;
    C checked identical across the variants (cluster-wise C == row-wise C bit for bit)."""
    import torch
    import numpy as np

    cfg = 2 if args.workload == "cfg2" else 4
    a0 = B.make_config(cfg, args.scale)
    eng = B.Engine(0)
    stream = torch.cuda.Stream()
    eng.set_stream(stream.cuda_stream)

    def timed(fn):
        for _ in range(args.warmup):
            fn().free()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            C = fn()
            e1.record(stream)
            C.free()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        # per-kernel times of one more multiply (CUDA events around every launch)
        eng.profile(True)
        fn().free()
        torch.cuda.synchronize()
        kern = {k: round(v[1], 4) for k, v in
                sorted(eng.profile_report().items(), key=lambda kv: -kv[1][1])[:12]}
        eng.profile(False)
        variant_kernels[len(variant_kernels)] = kern
        return float(np.mean(ts)), float(min(ts))

    variants = {}
    variant_kernels = {}
    t0 = time.perf_counter()
    a = a0
    if cfg == 4:
        A0 = eng.upload(a0)
        products = eng.spgemm_products(A0, A0)
        variants["rowwise_unreordered"] = timed(lambda: eng.spgemm_rowwise(A0, A0))
        ref_c = eng.spgemm_rowwise(A0, A0).download()
        A0.free()
        t0 = time.perf_counter()
        perm = B.reorder_rcm(a0)
        a = B.permute_symmetric(a0, perm)
    t_reorder = time.perf_counter() - t0 if cfg == 4 else 0.0
    A = eng.upload(a)
    products = eng.spgemm_products(A, A)
    name = "rowwise" if cfg == 2 else "rowwise_rcm"
    variants[name] = timed(lambda: eng.spgemm_rowwise(A, A))
    t0 = time.perf_counter()
    # cfg2: "hierarchical clustering (minhash, 64 hashes, max cluster size 8)" (BASELINE);
    # cfg4: the reference's hierarchical top-k
    asg = (eng.hierarchical_clusters(a, method="minhash", nhash=64) if cfg == 2
           else eng.hierarchical_clusters(a))
    Ac = eng.build_csr_cluster(A, asg)
    eng.synchronize()
    t_cluster = time.perf_counter() - t0
    cname = "clusterwise" if cfg == 2 else "clusterwise_rcm_hier"
    variants[cname] = timed(lambda: eng.spgemm_clusterwise(Ac, A))
    c_row = eng.spgemm_rowwise(A, A).download()
    c_cl = eng.spgemm_clusterwise(Ac, A).download()
    same = (np.array_equal(c_row.row_ptr, c_cl.row_ptr) and
            np.array_equal(c_row.col_idx, c_cl.col_idx) and
            np.array_equal(c_row.values.view(np.uint64), c_cl.values.view(np.uint64)))
    if cfg == 4:  # the reordered product is the original one, permuted
        same = same and B.csr_equal_canonical(B.permute_symmetric(ref_c, perm), c_row, 0.0)
    ms_row = variants[name][0]
    peak, peak_kind = hbm_peak()
    bal = bytes_alg(a.nnz(), a.nnz(), c_row.nnz(), a.nrows, a.nrows, a.nrows)
    line = {
        "metric": "A·B SpGEMM GFLOP/s (2×products/s)",
        "value": 2.0 * products / (ms_row * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_row,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (seeded BASELINE cfg{cfg})",
        "config": {"workload": f"cfg{cfg}_AxA_rowwise_vs_clusterwise", "n": a.nrows,
                   "nnz_a": a.nnz(), "products": products, "nnz_c": c_row.nnz(),
                   "clusters": asg.nclusters,
                   "clustering": "hierarchical, minhash-64 candidates" if cfg == 2
                   else "RCM + hierarchical (top-k candidates)", "parallelism": "x1"},
        "variants_ms": {k: {"mean": round(v[0], 4), "best": round(v[1], 4),
                            "gflops": round(2.0 * products / (v[0] * 1e-3) / 1e9, 2)}
                        for k, v in variants.items()},
        "variant_kernels_ms": {k: variant_kernels[i] for i, k in enumerate(variants)},
        "clusterwise_speedup_vs_" + name: round(ms_row / variants[cname][0], 3),
        "c_bit_identical_across_variants": bool(same),
        "preprocessing_s": {"reorder": round(t_reorder, 3), "cluster": round(t_cluster, 3)},
        "roofline": {"bound": "hbm", "achieved": bal / (ms_row * 1e-3) / 1e9, "peak": peak,
                     "unit": "GB/s", "frac": bal / (ms_row * 1e-3) / 1e9 / peak,
                     "traffic": None, "bytes_alg_per_step": bal, "peak_source": peak_kind,
                     "unit_of_work": "one full row-wise multiply"},
    }
    print(json.dumps(line), flush=True)


def run_e2e(B, eng, host, n, ncols, args, total_products, rank=0, world=1, dist=None):
    """Reference-shaped call with HOST buffers: pinned A -> device (H2D), the
    multiply in row chunks, each chunk of C copied back (D2H) into a pinned
    host ring by a second engine handle whose stream waits on the compute
    stream, so the copy engine overlaps the next chunk's kernels.  With N
    ranks each rank copies A in, multiplies its row shard (the chunks of the
    same cost split, so shard bounds coincide with bench's) and copies its
    shard of C out; the step time is the max over ranks."""
    import torch

    nchunks = args.e2e_chunks
    hp = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in host]
    h2d = sum(x.numel() * x.element_size() for x in hp)
    ce = B.Engine(eng.device)  # copy handle (own stream)
    cstream = torch.cuda.ExternalStream(ce.stream_ptr())
    # size the pinned ring from one untimed pass
    dev = [x.cuda() for x in hp]
    torch.cuda.synchronize()
    A = eng.view_torch(n, ncols, *dev)
    allb = eng.partition_rows(A, A, nchunks * world)
    bounds = allb[rank * nchunks:(rank + 1) * nchunks + 1]
    sizes = []
    for g in range(nchunks):
        C = eng.spgemm_rowwise_range(A, A, int(bounds[g]), int(bounds[g + 1]))
        sizes.append((C.nrows, C.nnz()))
        C.free()
    max_rows = max(r for r, _ in sizes)
    max_nnz = max(z for _, z in sizes)
    ring = [(torch.empty(max_rows + 1, dtype=torch.int64).pin_memory(),
             torch.empty(max(max_nnz, 1), dtype=torch.int32).pin_memory(),
             torch.empty(max(max_nnz, 1), dtype=torch.float64).pin_memory()) for _ in range(2)]
    del dev, A
    torch.cuda.synchronize()
    times, d2h = [], 0
    steps = max(1, min(args.steps, 3))
    mstream = torch.cuda.ExternalStream(eng.stream_ptr())
    for s in range(1 + steps):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(mstream):
            dev = [x.cuda(non_blocking=True) for x in hp]
        A = eng.view_torch(n, ncols, *dev)
        slot_ev = [None, None]
        d2h = 0
        for g in range(nchunks):
            C = eng.spgemm_rowwise_range(A, A, int(bounds[g]), int(bounds[g + 1]))
            slot = g % 2
            if slot_ev[slot] is not None:
                slot_ev[slot].synchronize()  # host ring slot free again
            ce.wait_for(eng)
            rp, ci, v = ring[slot]
            C.download_async(rp.data_ptr(), ci.data_ptr(), v.data_ptr(), engine=ce)
            d2h += (C.nrows + 1) * 8 + C.nnz() * 12
            ev = torch.cuda.Event()
            ev.record(cstream)
            slot_ev[slot] = ev
            C.free(engine=ce)  # stream-ordered after its copy
        ce.synchronize()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt, float(d2h)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
            dt, d2h = float(t[0]), int(t[1])
        if s > 0:
            times.append(dt)
        del dev, A
    # The copy floor of this box: the same bytes (every chunk's three arrays, same sizes)
    # device -> pinned host on the copy stream with nothing else running — what the PCIe
    # link allows for this step's output, measured beside the pipeline it bounds.
    floor_ms = None
    try:
        src_i = torch.empty(max(max_nnz, 1), dtype=torch.int32, device="cuda")
        src_v = torch.empty(max(max_nnz, 1), dtype=torch.float64, device="cuda")
        src_r = torch.empty(max_rows + 1, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fstream = torch.cuda.Stream()  # torch's own stream (it outlives the copy handle)
        with torch.cuda.stream(fstream):
            f0.record(fstream)
            for g, (r_, z_) in enumerate(sizes):
                rp, ci, v = ring[g % 2]
                rp[:r_ + 1].copy_(src_r[:r_ + 1], non_blocking=True)
                ci[:z_].copy_(src_i[:z_], non_blocking=True)
                v[:z_].copy_(src_v[:z_], non_blocking=True)
            f1.record(fstream)
        torch.cuda.synchronize()
        floor_ms = f0.elapsed_time(f1)
        del src_i, src_v, src_r
    except Exception:
        floor_ms = None
    ce.close()
    t = statistics.median(times)
    return {"value": 2.0 * total_products / t / 1e9, "unit": "GFLOP/s",
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * t,
            "chunks": nchunks * world, "d2h_copy_floor_ms": floor_ms,
            "path": "pinned H2D of A + bsp_spgemm_rowwise_range per row chunk + "
                    "bsp_csr_download_async of every chunk of C into a pinned host ring"
                    + (f" (per rank, {world} ranks, max over ranks)" if world > 1 else "")}


if __name__ == "__main__":
    main()
