"""Per-source-line summary of an `ncu --page source --csv --print-source cuda,sass` export:
thread instructions, warp instructions, stall samples and the top stall reasons per line.

usage: python tools/ncu_source_lines.py export.csv [top_n] [products]
"""
import csv, sys, collections
path = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
products = float(sys.argv[3]) if len(sys.argv) > 3 else None
rows = list(csv.reader(open(path)))
cur_file = None; hdr = None
agg = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] in ("Function Name", "File Name", "Kernel Name"): continue
    if hdr is None or len(r) != len(hdr) or not r[0]: continue   # SASS rows have an empty line number
    try: line = int(r[0])
    except ValueError: continue
    d = dict(zip(hdr[4:], r[4:]))
    def f(k):
        try: return float(d.get(k, 0) or 0)
        except ValueError: return 0.0
    stalls = {k[6:]: f(k) for k in d if k.startswith("stall_") and "Not Issued" not in k}
    agg[(cur_file, line)] = dict(src=r[1].strip()[:90], inst=f("Instructions Executed"),
                                 tinst=f("Thread Instructions Executed"), samples=f("# Samples"), stalls=stalls)
ti = sum(v["tinst"] for v in agg.values()); wi = sum(v["inst"] for v in agg.values()); sm = sum(v["samples"] for v in agg.values())
print(f"total thread inst {ti:.4g}  warp inst {wi:.4g}  samples {sm:.0f}" + (f"  thread inst/product {ti/products:.1f}  warp inst/product {wi/products:.2f}" if products else ""))
tot_st = collections.Counter()
for v in agg.values(): tot_st.update(v["stalls"])
print("stall mix:", ", ".join(f"{k} {100*x/sm:.1f}%" for k, x in tot_st.most_common(8)))
for (fn, ln), v in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:topn]:
    top = ", ".join(f"{k} {x:.0f}" for k, x in sorted(v["stalls"].items(), key=lambda kv: -kv[1])[:3] if x > 0)
    print(f"{fn}:{ln:<5d} smp {100*v['samples']/sm:5.2f}%  tinst {100*v['tinst']/ti:5.2f}%  thr/warp {v['tinst']/max(v['inst'],1):4.1f} | {top} | {v['src']}")
