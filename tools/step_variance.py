"""Per-step kernel-time profile of the cfg5 multiply (diagnoses step-to-step spread):
K steps with bsp_profile on, then per kernel the min / max / spread over steps and the
steps' host-visible gaps (step time minus the sum of its kernels).

usage: python tools/step_variance.py [--steps 12] [--scale S]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_21253_b200 as B

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=12)
ap.add_argument("--scale", type=int, default=None)
a_ = ap.parse_args()
a = B.make_config(5, a_.scale)
torch.cuda.set_device(0)
eng = B.Engine(0)
st = torch.cuda.Stream()
eng.set_stream(st.cuda_stream)
A = eng.view_torch(a.nrows, a.ncols, *(torch.from_numpy(x).cuda() for x in (a.row_ptr, a.col_idx, a.values)))
for _ in range(2):
    eng.spgemm_rowwise(A, A).free()
torch.cuda.synchronize()
rows, steps = [], []
eng.profile(True)
for s in range(a_.steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    C = eng.spgemm_rowwise(A, A)
    e1.record(st)
    C.free()
    torch.cuda.synchronize()
    rep = eng.profile_report()
    steps.append(e0.elapsed_time(e1))
    rows.append({k: v[1] for k, v in rep.items()})
eng.profile(False)
names = sorted(rows[0], key=lambda k: -rows[0][k])
out = {"step_ms": [round(x, 2) for x in steps],
       "gap_ms": [round(s - sum(r.values()), 2) for s, r in zip(steps, rows)],
       "kernels": {k: [round(r.get(k, 0.0), 2) for r in rows] for k in names[:14]}}
print(json.dumps(out))
