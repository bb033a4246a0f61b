"""Summarise ncu captures brought back in gpurun_out/ into profiles/.

    python tools/summarize_ncu.py r01

reads gpurun_out/prof_<kernel>.ncu-rep (ncu --set full) and
gpurun_out/launches.csv (gpu__time_duration.sum launch list), writes
profiles/ncu_summary_<tag>.json and profiles/launches_<tag>.md.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_theoretical",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "sm__maximum_warps_per_active_cycle_pct": "theoretical_occupancy_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "warp_instructions",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
         "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def _num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(unit, 1)


def read_rep(path):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = {"kernel": row[h.index("Kernel Name")].split("(")[0]}
        for m, key in METRICS.items():
            if m in h:
                i = h.index(m)
                d[key] = _num(row[i], units[i])
        out.append(d)
    return out


def launches(path):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rows[1:]:
        if r[ki] == "Kernel Name":
            continue
        name = r[ki].split("(")[0]
        tot[name] += _num(r[vi], r[ui])
        cnt[name] += 1
    return tot, cnt


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    summary = {"tag": tag, "how": "ncu --set full --clock-control none --import-source on, "
               "1 launch per kernel after 2 warm-up launches (tools/ncu_target.py); "
               "dram bytes are per launch", "kernels": {}}
    for name in sorted(os.listdir(OUT)):
        if name.startswith("prof_") and name.endswith(".ncu-rep"):
            key = name[5:-8]
            recs = read_rep(os.path.join(OUT, name))
            for rec in recs:
                kk = rec["kernel"].replace("void ", "").replace("unnamed>::", "")
                rec["dram_bytes_per_launch"] = rec.get("dram_read", 0) + rec.get("dram_write", 0)
                summary["kernels"][key if key != "jacobi" else "jacobi2d"] = dict(rec, kernel=kk)
    with open(os.path.join(PROF, f"ncu_summary_{tag}.json"), "w") as f:
        json.dump(summary, f, indent=1)
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        tot, cnt = launches(lp)
        T = sum(tot.values())
        with open(os.path.join(PROF, f"launches_{tag}.md"), "w") as f:
            f.write(f"# Launch list {tag}\n\n`ncu --metrics gpu__time_duration.sum --clock-control none` "
                    "over `python bench.py --steps 1 --warmup 1 --no-extra --no-cpu-baseline` "
                    "(cold-cache, serialised: compare shares, not absolutes)\n\n")
            f.write("| kernel | launches | avg us | share of kernel time |\n|---|---|---|---|\n")
            for k in sorted(tot, key=lambda k: -tot[k]):
                f.write(f"| `{k}` | {cnt[k]} | {tot[k] / cnt[k] * 1e6:.1f} | {tot[k] / T * 100:.1f} % |\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
