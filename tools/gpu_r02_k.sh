#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for l in scat_f64 scat_i32 scat_f64 scat_i32; do timeout 300 python tools/time_loop.py $l 8; done
for m in scatter scatter_i32; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_k_$m.csv python tools/ncu_target.py $m 2 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launches_k_$m.csv') if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
for r in rows[-15:]: print(r[ki].split("(")[0][-30:], r[mi], r[vi])
PY
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 -k "scatter or graph" > gpurun_out/gpu_tests_k.log 2>&1; tail -2 gpurun_out/gpu_tests_k.log
timeout 600 python tools/stress_scatter.py 20 i32_1 i32_3 f64_2 > gpurun_out/stress_k.jsonl 2> gpurun_out/stress_k.err
timeout 600 python tools/stress_scatter.py 4 full_f64 full_i32 >> gpurun_out/stress_k.jsonl 2>> gpurun_out/stress_k.err; cat gpurun_out/stress_k.jsonl
