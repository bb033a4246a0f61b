#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for l in scat_f64 scat_i32; do timeout 300 python tools/time_loop.py $l 5 >> gpurun_out/time_f.jsonl 2>> gpurun_out/time_f.err; done
cat gpurun_out/time_f.jsonl; tail -3 gpurun_out/time_f.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_scat_f.csv python tools/ncu_target.py scatter 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launches_scat_f.csv') if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
for r in rows[1:]: print(r[ki].split("(")[0][-32:], r[mi], r[vi])
PY
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/gpu_tests_f.log 2>&1
tail -5 gpurun_out/gpu_tests_f.log
timeout 900 python tools/stress_scatter.py 20 i32_1 i32_3 f64_2 > gpurun_out/stress_f.jsonl 2> gpurun_out/stress_f.err
timeout 600 python tools/stress_scatter.py 4 full_f64 full_i32 >> gpurun_out/stress_f.jsonl 2>> gpurun_out/stress_f.err
cat gpurun_out/stress_f.jsonl
timeout 1200 python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
tail -2 gpurun_out/bench_f.err
