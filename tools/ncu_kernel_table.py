#!/usr/bin/env python
"""Per-kernel ncu metric table for one multiply (the second products_kernel onwards, or the
first if only one): duration, DRAM GB/s, L2 hit rate, shared-memory bank conflicts (share of
wavefronts), issue-slot use, occupancy.  Input: `ncu --metrics <below> --csv --log-file`.

usage: tools/ncu_kernel_table.py metrics.csv
metrics: gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
  lts__t_sector_hit_rate.pct,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,
  l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,
  smsp__issue_active.avg.pct_of_peak_sustained_active,
  sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
"""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
        "s": 1.0, "second": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
    h = rows[0]
    ii, kn, mn, mu, mv = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                               "Metric Value"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {"name": r[kn]})
        v = float(r[mv].replace(",", "")) * UNIT.get(r[mu], 1.0)
        d[r[mn]] = v
    agg = collections.OrderedDict()
    for d in launches.values():
        name = re.sub(r"\(.*$", "", d["name"]).replace("bsp::<unnamed>::", "").replace("(int)", "")
        name = name.replace("void ", "")
        a = agg.setdefault(name, collections.defaultdict(float))
        t = d.get("gpu__time_duration.sum", 0.0)
        a["n"] += 1
        a["t"] += t
        a["rd"] += d.get("dram__bytes_read.sum", 0.0)
        a["wr"] += d.get("dram__bytes_write.sum", 0.0)
        a["bc"] += d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 0.0)
        a["wf"] += d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0.0)
        a["inst"] += d.get("smsp__inst_executed.sum", 0.0)
        for k in ("lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__warps_active.avg.pct_of_peak_sustained_active"):
            a[k] += d.get(k, 0.0) * t  # time-weighted
    tot = sum(a["t"] for a in agg.values()) or 1.0
    print("| kernel | launches | ms | share | DRAM GB/s | L2 hit | smem conflict wavefronts | issue busy | warps active | warp instr |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        if a["t"] / tot < 0.003:
            continue
        t = a["t"] or 1e-30
        print(f"| `{k[:48]}` | {int(a['n'])} | {1e3 * a['t']:.2f} | {100 * a['t'] / tot:.1f}% | "
              f"{(a['rd'] + a['wr']) / t / 1e9:.0f} | {a['lts__t_sector_hit_rate.pct'] / t:.0f}% | "
              f"{100 * a['bc'] / max(a['wf'], 1):.0f}% | "
              f"{a['smsp__issue_active.avg.pct_of_peak_sustained_active'] / t:.0f}% | "
              f"{a['sm__warps_active.avg.pct_of_peak_sustained_active'] / t:.0f}% | {a['inst']:.2e} |")


if __name__ == "__main__":
    main()
