#!/usr/bin/env python
"""Strong-scaling projection for the row-sharded multiply, measured on ONE GPU.

For N in (1, 2, 4, 8) the rows of A are split by cumulative products exactly as
bench.py's multi-rank path does (bsp_partition_rows), and every shard's
multiply (bsp_spgemm_rowwise_range, the call each rank makes) is timed alone on
the GPU with CUDA events.  The projected N-GPU step time is the slowest shard
(ranks do not communicate during the multiply; B is broadcast beforehand), so
projected efficiency = T1 / (N * max shard time).  This measures load balance
and per-shard fixed costs; it does not measure NVLink or NCCL.

usage: python tools/shard_projection.py [--cfg 5] [--reps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2507_21253_b200 as B

    a = B.make_config(args.cfg, args.scale)
    torch.cuda.set_device(0)
    eng = B.Engine(0)
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)
    rp = torch.from_numpy(a.row_ptr).cuda()
    ci = torch.from_numpy(a.col_idx).cuda()
    v = torch.from_numpy(a.values).cuda()
    A = eng.view_torch(a.nrows, a.ncols, rp, ci, v)
    P = eng.spgemm_products(A, A)

    def timed(r0, r1):
        C = eng.spgemm_rowwise_range(A, A, r0, r1)  # warm-up
        C.free()
        ts = []
        for _ in range(args.reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            C = eng.spgemm_rowwise_range(A, A, r0, r1)
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            C.free()
        return min(ts)

    out = {"cfg": args.cfg, "products": P, "runs": []}
    t1 = None
    for n in (1, 2, 4, 8):
        bounds = [int(x) for x in eng.partition_rows(A, A, n)]
        shard_ms = [timed(bounds[g], bounds[g + 1]) for g in range(n)]
        tmax = max(shard_ms)
        if n == 1:
            t1 = tmax
        out["runs"].append({"n": n, "bounds": bounds, "shard_ms": [round(x, 2) for x in shard_ms],
                            "projected_ms": round(tmax, 2),
                            "projected_gflops": 2 * P / tmax / 1e6,
                            "projected_efficiency": t1 / (n * tmax)})
        print(json.dumps(out["runs"][-1]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
