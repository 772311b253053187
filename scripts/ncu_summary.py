"""Summarise one kernel of an ncu --set full report into profiles/*.json.

    python scripts/ncu_summary.py REPORT.ncu-rep|REPORT_raw.csv OUT.json "<kernel title>" "<config>" "<capture cmd>"
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__registers_per_thread", "smsp__inst_executed.sum")


def main():
    rep, out, title, config, cmd = sys.argv[1:6]
    # REPORT may also be the csv already exported on the GPU box
    # (ncu -i X.ncu-rep --page raw --csv > X_raw.csv: reports exceed gpurun's copy-back cap)
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = [r[i], units[i]]
        d["kernel"] = r[hdr.index("Kernel Name")][:120] if "Kernel Name" in hdr else ""
        launches.append(d)
    mul = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    l0 = launches[0]
    dram = sum(float(l0[k][0].replace(",", "")) * mul.get(l0[k][1], 1.0)
               for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in l0)
    json.dump({"kernel": title, "config": config, "capture": cmd,
               "dram_bytes_per_launch": dram, "launches": launches},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
