"""A/B builds: python tools/build_variant.py NAME -DFLAG[=V] ... compiles csrc/ with the extra
defines into paper_2507_21253_b200/libbsp_NAME.so (loaded when BSP_LIB_VARIANT=NAME).  The
variant libraries are git-ignored experiments; the product is libbsp.so."""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_21253_b200 import build as b

name, defs = sys.argv[1], sys.argv[2:]
obj = b.ROOT / "build" / f"obj_{name}"
obj.mkdir(parents=True, exist_ok=True)
base = b.ROOT / "build" / "obj"

def comp(src):
    if src.suffix != ".cu" or src.name not in ("rowwise.cu", "cluster.cu"):
        return base / (src.name + ".o")  # untouched sources: the product's objects
    o = obj / (src.name + ".o")
    r = subprocess.run([b.NVCC, *b.CU_FLAGS, *defs, "-c", str(src), "-o", str(o)], capture_output=True, text=True)
    (obj / (src.name + ".log")).write_text(r.stdout + r.stderr)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr); raise SystemExit(1)
    return o

b.build(verbose=False)
srcs = sorted(b.CSRC.glob("*.cu")) + sorted(b.CSRC.glob("*.cpp"))
with ThreadPoolExecutor(4) as ex:
    objs = list(ex.map(comp, srcs))
lib = b.PKG / f"libbsp_{name}.so"
r = subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-Xcompiler", "-fopenmp", "-lgomp", "-cudart", "static"], capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr); raise SystemExit(1)
print(lib)
