"""Key metrics of an `ncu --set full` report, one record per profiled launch.

  python tools/ncu_full_summary.py gpurun_out/x.ncu-rep --out profiles/round1_ncu_x.json
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("pds::", "")}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = r[i] + (" " + units[i] if units[i] else "")
        recs.append(rec)
        print(rec["kernel"][:40], {k.split(".")[0].split("__")[-1]: rec.get(k) for k in KEYS[:5]})
    if a.out:
        json.dump({"report": a.rep, "clock_control": "none", "launches": recs}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
