"""(Lives under tests/: --check uses the oracle as the checker.)
Time row-wise / cluster-wise / row-chunked multiplies of a BASELINE config on cuda:0
(CUDA events on the engine stream, per step), with an optional per-kernel event profile and
an oracle check.  Used for the A/B runs and ncu captures recorded in profiles/.

usage: python tests/tools/time_multiply.py [--cfg 5] [--scale S] [--steps K] [--warmup W] [--prof]
       [--cluster] [--rcm] [--chunks N] [--check] [--tag T]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2507_21253_b200 as B
ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5); ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--steps", type=int, default=3); ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--prof", action="store_true"); ap.add_argument("--tag", default="")
ap.add_argument("--check", action="store_true"); ap.add_argument("--cluster", action="store_true"); ap.add_argument("--rcm", action="store_true"); ap.add_argument("--chunks", type=int, default=0)
a_ = ap.parse_args()
a = B.make_config(a_.cfg, a_.scale)
if a_.rcm:
    a = B.permute_symmetric(a, B.reorder_rcm(a))
torch.cuda.set_device(0)
eng = B.Engine(0); st = torch.cuda.Stream(); eng.set_stream(st.cuda_stream)
rp = torch.from_numpy(a.row_ptr).cuda(); ci = torch.from_numpy(a.col_idx).cuda(); v = torch.from_numpy(a.values).cuda()
A = eng.view_torch(a.nrows, a.ncols, rp, ci, v)
P = eng.spgemm_products(A, A)
if a_.cluster:
    asg = eng.hierarchical_clusters(a)
    Ac = eng.build_csr_cluster(A, asg)
    mult = lambda: eng.spgemm_clusterwise(Ac, A)
elif a_.chunks:
    bnd = [int(x) for x in eng.partition_rows(A, A, a_.chunks)]
    class _Sum:
        def __init__(s, n): s.n = n
        def nnz(s): return s.n
        def free(s): pass
    def mult():
        tot = 0
        for g in range(a_.chunks):
            Cg = eng.spgemm_rowwise_range(A, A, bnd[g], bnd[g + 1]); tot += Cg.nnz(); Cg.free()
        return _Sum(tot)
else:
    mult = lambda: eng.spgemm_rowwise(A, A)
for _ in range(a_.warmup):
    C = mult(); C.free()
torch.cuda.synchronize()
ts = []
for _ in range(a_.steps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st); C = mult(); e1.record(st); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1)); nnzc = C.nnz()
    if a_.check and _ == a_.steps - 1:
        c = C.download()
    C.free()
out = {"tag": a_.tag, "cfg": a_.cfg, "ms": ts, "best": min(ts), "gflops": 2 * P / min(ts) / 1e6, "nnzc": nnzc}
if a_.prof:
    eng.profile(True); C = mult(); C.free()
    out["kernels"] = {k: round(v_[1], 2) for k, v_ in sorted(eng.profile_report().items(), key=lambda kv: -kv[1][1])}
    eng.profile(False)
if a_.check:
    import oracle as O
    o = O.spgemm_rowwise(a, a)
    out["exact"] = bool(np.array_equal(c.row_ptr, o.row_ptr) and np.array_equal(c.col_idx, o.col_idx)
                        and np.array_equal(c.values.view(np.uint64), o.values.view(np.uint64)))
print(json.dumps(out))
