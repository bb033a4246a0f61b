#!/bin/bash
# round-2 call c: paged single-pass binned scatter -- parity, stress, timing, ncu
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 -k "scatter or graph" > gpurun_out/gpu_tests_c.log 2>&1
tail -5 gpurun_out/gpu_tests_c.log
for l in scat_f64 scat_i32; do timeout 300 python tools/time_loop.py $l 10 >> gpurun_out/time_c.jsonl 2>> gpurun_out/time_c.err; done
cat gpurun_out/time_c.jsonl; tail -3 gpurun_out/time_c.err
timeout 900 python tools/stress_scatter.py 50 i32_1 f64_1 i32_3 f64_2 > gpurun_out/stress_c.jsonl 2> gpurun_out/stress_c.err
timeout 600 python tools/stress_scatter.py 8 full_f64 full_i32 >> gpurun_out/stress_c.jsonl 2>> gpurun_out/stress_c.err
cat gpurun_out/stress_c.jsonl; tail -3 gpurun_out/stress_c.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_scat_c.csv python tools/ncu_target.py scatter 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_scat_i32_c.csv python tools/ncu_target.py scatter_i32 3 > /dev/null 2>&1
for k in scat_part scat_apply; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f -o gpurun_out/prof_c_$k python tools/ncu_target.py scatter 2 > gpurun_out/ncu_c_$k.log 2>&1
done
python - <<'PY'
import csv
for f in ("gpurun_out/launches_scat_c.csv", "gpurun_out/launches_scat_i32_c.csv"):
    rows = [r for r in csv.reader(l for l in open(f) if l.startswith('"'))]
    h = rows[0]; ki = h.index("Kernel Name"); mi = h.index("Metric Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
    for r in rows[1:]:
        print(f.split("/")[-1], r[ki].split("(")[0][-40:], r[mi], r[vi], r[ui])
PY
