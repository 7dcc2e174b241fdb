#!/usr/bin/env python3
"""Summarise an ncu launch list (CSV from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv --log-file X.csv python bench.py ...`) over the
last iteration (from the last control_advance_kernel launch on): per-kernel total time, share,
launch count, average time and DRAM bytes per launch. With --traffic, also writes
profiles/traffic.json (the bench's roofline.traffic: DRAM bytes per launch of each GEMM family).

    python tools/launch_summary.py profiles/r1/v19_launches.csv > profiles/r1/v19_launch_summary.txt
"""
import argparse
import collections
import csv
import json
import os


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic", help="write the GEMM DRAM bytes per launch to this JSON file")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    launches = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[0], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    seq = list(launches.values())
    # iterations start at control_advance_kernel; take the last complete one (a trailing
    # control_advance with almost nothing after it belongs to a call ncu cut short)
    marks = [i for i, d in enumerate(seq) if "control_advance_kernel" in d["name"]]
    if len(seq) - marks[-1] < 10 and len(marks) > 1:
        it = seq[marks[-2]:marks[-1]]
    else:
        it = seq[marks[-1]:]
    agg = collections.OrderedDict()
    for d in it:
        name = d["name"].split("(")[0].replace("void ", "").replace("ppo::<unnamed>::", "")
        g = agg.setdefault(name, {"ns": 0.0, "n": 0, "dram": 0.0})
        g["ns"] += d.get("gpu__time_duration.sum", 0.0)
        g["n"] += 1
        g["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(g["ns"] for g in agg.values())
    for name, g in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        print(f"{g['ns'] / 1e3:9.1f}us {100 * g['ns'] / total:5.1f}% n={g['n']:3d} avg={g['ns'] / g['n'] / 1e3:8.2f}us "
              f"dram={g['dram'] / g['n'] / 1e6:8.2f}MB {name}")
    print(f"total {total / 1e3:.1f} us {len(it)} launches (one iteration, ncu-serialised, cold caches between kernels)")
    if a.traffic:
        # per GEMM family (template = <BN, A_MN, B_MN, EPI, WS, CS>): forward = EPI 0 (bias + ELU),
        # input gradient = EPI 1 (elu' product), weight gradient = EPI 2 (split-K fp32 slabs)
        fam = {"fwd": ", 0>", "dx": "1, 1, 0>", "dw": "2, 0, 1>"}
        kernels = {}
        for key in fam:
            epi = {"fwd": 0, "dx": 1, "dw": 2}[key]
            sel = [d for d in it if d["name"].startswith("void gemm_tcgen05_kernel")
                   and d["name"].split("<")[1].split(",")[3].strip() == str(epi)]
            byt = sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in sel)
            kernels[key] = {"dram_bytes_per_launch": byt / max(1, len(sel)), "launches": len(sel),
                            "templates": sorted({d["name"].split("(")[0].replace("void ", "") for d in sel})}
        with open(a.traffic, "w") as f:
            json.dump({"source": f"{os.path.relpath(a.csv)} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                                 "dram__bytes_write.sum --clock-control none over `python bench.py --steps 2 --warmup 1`;"
                                 " the GEMM launches of the last iteration, caches flushed between kernels)",
                       "kernels": kernels}, f, indent=1)
            f.write("\n")

if __name__ == "__main__":
    main()
