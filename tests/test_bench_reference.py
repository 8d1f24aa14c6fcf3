"""bench.py's reference arm (CPU, no GPU needed).

- The oracle's C restatement of the R-MAT recipe (oracle/gen.c) builds the same matrix,
  bit for bit, as the product's generator (host_gen.cpp gen_rmat), so the reference arm
  times the reference on exactly the bench workload without loading the product library.
- The reference arm's process never maps libbsp.so, and its `config` equals the GPU
  arm's (same workload keys and values), so the driver can compare the two lines.
"""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import paper_2507_21253_b200 as B

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


@pytest.mark.parametrize("scale,ef,abc,seed", [(10, 8, (0.45, 0.22, 0.22), 5),
                                               (12, 16, (0.57, 0.19, 0.19), 3),
                                               (15, 8, (0.45, 0.22, 0.22), 5)])
def test_oracle_rmat_generator_bit_identical(scale, ef, abc, seed):
    x = O.gen_rmat(scale, ef, *abc, seed)
    y = B.gen_rmat(scale, ef, *abc, seed)
    assert np.array_equal(x.row_ptr, y.row_ptr)
    assert np.array_equal(x.col_idx, y.col_idx)
    assert np.array_equal(x.values.view(np.uint64), y.values.view(np.uint64))


def test_bench_workload_is_cfg5():
    c = B.CONFIGS[5]
    assert bench.CFG5 == dict(scale=c["scale"], ef=c["ef"], a=c["a"], b=c["b"], c=c["c"],
                              seed=c["seed"])


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_reference_arm_never_loads_the_product_and_shares_the_config():
    code = (
        "import runpy, sys, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--scale', '12', '--steps', '2',"
        " '--warmup', '1']\n"
        "runpy.run_path('bench.py', run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'libbsp': 'libbsp.so' in maps, 'ref': 'libcspgemm_ref' in maps}))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, check=True).stdout.strip().splitlines()
    line = json.loads(out[-2])
    maps = json.loads(out[-1])
    assert maps == {"libbsp": False, "ref": True}
    assert line["impl"] == "reference" and line["value"] > 0
    a = B.gen_rmat(12, 8, 0.45, 0.22, 0.22, 5)
    products = int(bench.row_products(a).sum())
    nnz_c = int(O.spgemm_symbolic(a, a).sum())
    assert line["config"] == bench.workload_config(a.nrows, a.nnz(), products, nnz_c, 1, 12)
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
