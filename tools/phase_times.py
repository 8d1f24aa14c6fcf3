"""Phase shares of the look-back window tile (experiment build: python tools/build_variant.py
phase -DBSP_X_PHASE; run with BSP_LIB_VARIANT=phase).  Thread 0 of each tile accumulates the
cycles between phase marks; the table is the share of tile residency per phase on cfg5."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BSP_LIB_VARIANT", "phase")
import numpy as np, torch
import paper_2507_21253_b200 as B
from paper_2507_21253_b200 import _lib
lib = _lib.load()
lib.bsp_debug_phases.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
a = B.make_config(5, int(sys.argv[1]) if len(sys.argv) > 1 else None)
eng = B.Engine(0)
A = eng.upload(a)
eng.spgemm_rowwise(A, A).free()
buf = (C.c_ulonglong * 32)()
lib.bsp_debug_phases(buf, 1)
eng.spgemm_rowwise(A, A).free()
lib.bsp_debug_phases(buf, 0)
names = {1: "segment ranges + scan + compaction", 2: "gather (cp.async) + wait", 3: "fix-up a*b",
         4: "expansion end", 5: "csort: min/max", 6: "csort: bucket atomics + cost", 7: "csort: bucket scan",
         8: "csort: scatter packed", 9: "csort: rank + write (narrow)", 10: "csort: rank + write (wide)",
         11: "radix fallback", 12: "merge fallback", 13: "heads + scan + publish", 14: "run sums",
         15: "look-back (wait)", 16: "store C"}
tiles = buf[0]
tot = sum(buf[i] for i in range(1, 32))
print(f"tiles {tiles}  cycles/tile {tot / max(tiles, 1):.0f}")
for i in range(1, 17):
    print(f"  {names[i]:40s} {100 * buf[i] / max(tot, 1):6.2f}%  {buf[i] / max(tiles, 1):8.0f} cyc/tile")
print("time from tile start to its count being published, by A-row length d:")
for c, nm in enumerate(["<=256", "<=512", "<=1024", "<=2048", "<=4096", ">4096"]):
    if buf[26 + c]:
        print(f"  d {nm:7s}: {100 * buf[26 + c] / max(tiles, 1):5.1f}% of tiles, {buf[20 + c] / buf[26 + c]:9.0f} cycles to publish")
