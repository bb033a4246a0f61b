#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 -k "scatter or graph or merge or gemm" > gpurun_out/gpu_tests_e.log 2>&1
tail -3 gpurun_out/gpu_tests_e.log
for l in scat_f64 scat_i32 gemm; do timeout 300 python tools/time_loop.py $l 5 >> gpurun_out/time_e.jsonl 2>> gpurun_out/time_e.err; done
JACC_GEMM_VARIANT=4 timeout 300 python tools/time_loop.py gemm 3 >> gpurun_out/time_e.jsonl 2>> gpurun_out/time_e.err
cat gpurun_out/time_e.jsonl; tail -3 gpurun_out/time_e.err
timeout 600 python tools/stress_scatter.py 20 i32_3 f64_2 > gpurun_out/stress_e.jsonl 2> gpurun_out/stress_e.err
timeout 600 python tools/stress_scatter.py 4 full_f64 full_i32 >> gpurun_out/stress_e.jsonl 2>> gpurun_out/stress_e.err
cat gpurun_out/stress_e.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_scat_e.csv python tools/ncu_target.py scatter 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launches_scat_e.csv') if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
for r in rows[1:]: print(r[ki].split("(")[0][-32:], r[mi], r[vi])
PY
bash tools/ncu_brief.sh e_part scat_part 1 python tools/ncu_target.py scatter 2
bash tools/ncu_brief.sh e_apply scat_apply 1 python tools/ncu_target.py scatter 2
bash tools/ncu_brief.sh e_gemm gemm_tma 1 python tools/ncu_target.py gemm 2
du -sh gpurun_out
