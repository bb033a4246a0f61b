#!/bin/bash
# ncu --set full capture of one kernel launch and a grep of the metrics that
# explain a memory-bound kernel's time (throughputs, issue, stalls).
# usage: tools/ncu_metrics.sh <name> <ncu_target loop> <kernel regex> [env...]
name=$1; loop=$2; kre=$3; shift 3
env "$@" timeout 900 ncu --set full --clock-control none -k "regex:$kre" -s 2 -c 1 -o gpurun_out/m_$name -f python tools/ncu_target.py $loop 3 > gpurun_out/m_$name.log 2>&1
ncu -i gpurun_out/m_$name.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/m_$name.csv
python - "$name" <<'PY'
import csv, sys
name = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/m_{name}.csv")))
h, u, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in h:
        i = h.index(k); print(f"{name} {k} = {v[i]} {u[i]}")
stalls = [(float(v[i].replace(",", "")), h[i]) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled_") and h[i].endswith("_per_issue_active.ratio")
          and v[i].replace(",", "").replace(".", "").isdigit()]
for val, k in sorted(stalls, reverse=True)[:6]:
    print(f"{name} {k} = {val}")
PY
rm -f gpurun_out/m_$name.ncu-rep
