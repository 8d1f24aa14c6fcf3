"""Step-time spread of the cfg5 multiply with BSP_GAP_LOG=1 markers: prints a marker line per
step on stderr so [gap] / [slow] lines can be attributed to the step they fall in.

usage: BSP_GAP_LOG=1 python tools/step_gaps.py [--steps 16] [--smi]   (--smi: nvidia-smi -lms 250 beside)
"""
import argparse, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_21253_b200 as B
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=16); ap.add_argument("--smi", action="store_true")
ap.add_argument("--scale", type=int, default=None)
a_ = ap.parse_args()
a = B.make_config(5, a_.scale)
torch.cuda.set_device(0)
eng = B.Engine(0); st = torch.cuda.Stream(); eng.set_stream(st.cuda_stream)
A = eng.view_torch(a.nrows, a.ncols, *(torch.from_numpy(x).cuda() for x in (a.row_ptr, a.col_idx, a.values)))
proc = None
if a_.smi:
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "250"],
                            stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
for _ in range(3):
    eng.spgemm_rowwise(A, A).free()
torch.cuda.synchronize()
ts = []
for s in range(a_.steps):
    sys.stderr.write(f"--- step {s}\n"); sys.stderr.flush()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(st); C = eng.spgemm_rowwise(A, A); e1.record(st)
    C.nnz(); C.free()
    torch.cuda.synchronize()
    ts.append((round(e0.elapsed_time(e1), 1), round((time.perf_counter() - w0) * 1e3, 1)))
    sys.stderr.write(f"    step {s}: device {ts[-1][0]} ms wall {ts[-1][1]} ms\n")
if proc: proc.terminate()
print(ts)
