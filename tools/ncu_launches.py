#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) of `bench.py --steps 1 --warmup 1 --no-e2e --no-cpu`:
per-kernel time / DRAM bytes of ONE multiply (the second; multiplies start at
products_kernel), as a markdown table, plus the traffic JSON bench.py reads.

usage: tools/ncu_launches.py launches.csv traffic.json [bytes_alg]
"""
import collections
import csv
import json
import re
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    balg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ii, kn, mn, mv, mu = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {"name": r[kn]})
        v = float(r[mv].replace(",", ""))
        unit = r[mu]
        if r[mn] == "gpu__time_duration.sum":
            v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
        elif unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        d[r[mn]] = v
    ids = list(launches)
    starts = [i for i in ids if "products_kernel" in launches[i]["name"]]
    lo = starts[1] if len(starts) > 1 else starts[0]
    hi = starts[2] if len(starts) > 2 else ids[-1] + 1
    agg = collections.OrderedDict()
    for i in ids:
        if lo <= i < hi:
            d = launches[i]
            name = re.sub(r"\(.*$", "", d["name"]).replace("bsp::<unnamed>::", "").replace("(int)", "")
            a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
            a[0] += 1
            a[1] += d.get("gpu__time_duration.sum", 0.0)
            a[2] += d.get("dram__bytes_read.sum", 0.0)
            a[3] += d.get("dram__bytes_write.sum", 0.0)
    tms = sum(a[1] for a in agg.values())
    rd = sum(a[2] for a in agg.values())
    wr = sum(a[3] for a in agg.values())
    print(f"one multiply: launches {hi - lo}  time {tms:.1f} ms  read {rd / 1e9:.1f} GB  write {wr / 1e9:.1f} GB"
          + (f" (bytes_alg = {balg / 1e9:.1f} GB => traffic = {(rd + wr) / balg:.2f} x bytes_alg)" if balg else ""))
    print()
    print("| kernel | launches | ms (ncu, serialized, cold) | share | DRAM read GB | DRAM write GB |")
    print("|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k[:70]}` | {a[0]} | {a[1]:.2f} | {100 * a[1] / tms:.1f}% | {a[2] / 1e9:.2f} | {a[3] / 1e9:.2f} |")
    json.dump({"dram_bytes_per_step": rd + wr, "dram_read_gb": rd / 1e9, "dram_write_gb": wr / 1e9,
               "ncu_serialized_ms": tms,
               "source": f"{src} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                         f"--clock-control none, bench.py --steps 1 --warmup 1 --no-e2e --no-cpu; the second of the "
                         f"multiplies, launches {lo}-{hi - 1})"},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
