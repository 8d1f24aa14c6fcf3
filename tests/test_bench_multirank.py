"""The bench's N-rank path (row shards, B broadcast, max-over-ranks timing,
per-rank e2e) run end to end with two ranks.  Only one GPU exists here, so
BSP_BENCH_SHARED_GPU=1 puts both ranks on cuda:0 over gloo: this checks the
plumbing and the sharded result (total nnz(C) equals one rank's), not speed."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(nproc, port):
    env = dict(os.environ, BSP_BENCH_SHARED_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "bench.py"), "--gpus", str(nproc), "--steps", "1", "--warmup", "3",
           "--scale", "14", "--no-cpu", "--e2e-chunks", "2"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 prints one line
    return json.loads(lines[0])


def test_two_rank_bench_matches_one_rank():
    one = _run(1, 29541)
    two = _run(2, 29542)
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["config"]["nnz_c"] == one["config"]["nnz_c"]
    assert two["config"]["products"] == one["config"]["products"]
    assert two["e2e"]["d2h_bytes_per_step"] >= one["e2e"]["d2h_bytes_per_step"]
    assert two["e2e"]["chunks"] == 4


def test_tall_skinny_workload_runs():
    """bench.py --workload ts (A x BFS frontiers) at a small scale."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--workload", "ts", "--steps", "1",
           "--warmup", "3", "--scale", "12", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["value"] > 0 and line["clusterwise"]["value"] > 0
    assert line["config"]["frontiers"] >= 1


@pytest.mark.parametrize("wl,scale", [("cfg2", 512), ("cfg4", 16)])
def test_clustered_workloads_run(wl, scale):
    """bench.py --workload cfg2 / cfg4: row-wise and cluster-wise timed in one run, C identical."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--workload", wl, "--steps", "2",
           "--warmup", "3", "--scale", str(scale)]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["c_bit_identical_across_variants"] is True
    assert len(line["variants_ms"]) == (2 if wl == "cfg2" else 3)
