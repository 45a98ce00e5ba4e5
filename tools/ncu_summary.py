"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv --log-file X.csv ...`) into per-kernel totals, and write the
GEMM DRAM traffic per launch that bench.py reports as roofline.traffic.

  python tools/ncu_summary.py gpurun_out/launches.csv --out profiles/round1_launches_summary.json \
      --gemm-traffic profiles/gemm_traffic.json
ncu times are cold-cache and serialised: use the SHARES, not the absolute numbers.
"""
import argparse
import collections
import csv
import json

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3, "ms": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", default=None)
    ap.add_argument("--gemm-traffic", default=None)
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = collections.OrderedDict()
    for r in rows[1:]:
        rec = launches.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "").replace("pds::", "")})
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        rec[r[mi]] = v
    agg = collections.OrderedDict()
    for rec in launches.values():
        if rec["name"].startswith("at::"):
            continue                       # torch plumbing (input generation, L2 flush)
        g = agg.setdefault(rec["name"], {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
        g["launches"] += 1
        g["us"] += rec.get("gpu__time_duration.sum", 0.0)
        g["dram_bytes"] += rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0)
    tot = sum(g["us"] for g in agg.values())
    for g in agg.values():
        g["share"] = g["us"] / tot if tot else 0.0
        g["dram_gbs"] = g["dram_bytes"] / (g["us"] * 1e-6) / 1e9 if g["us"] else 0.0
    agg = dict(sorted(agg.items(), key=lambda kv: -kv[1]["us"]))
    out = {"source": a.csv, "note": "ncu launch list, cold-cache serialised launches; compare shares",
           "total_us": tot, "kernels": agg}
    for k, g in list(agg.items())[:12]:
        print(f"{g['launches']:4d} {g['us']:10.1f} us {100 * g['share']:5.1f}% {g['dram_gbs']:7.0f} GB/s  {k[:70]}")
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)
    if a.gemm_traffic:
        gem = [g for k, g in agg.items() if k.startswith("gemm")]
        n = sum(g["launches"] for g in gem)
        byt = sum(g["dram_bytes"] for g in gem)
        json.dump({"source": a.csv, "kernels": [k for k in agg if k.startswith("gemm")], "launches": n,
                   "dram_bytes_per_launch": byt / n if n else None}, open(a.gemm_traffic, "w"), indent=1)
        print("gemm dram bytes / launch", byt / n if n else None)


if __name__ == "__main__":
    main()
