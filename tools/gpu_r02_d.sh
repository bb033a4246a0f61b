#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 -k "scatter or graph or merge" > gpurun_out/gpu_tests_d.log 2>&1
tail -3 gpurun_out/gpu_tests_d.log
for l in scat_f64 scat_i32; do timeout 300 python tools/time_loop.py $l 10 >> gpurun_out/time_d.jsonl 2>> gpurun_out/time_d.err; done
cat gpurun_out/time_d.jsonl; tail -3 gpurun_out/time_d.err
timeout 600 python tools/stress_scatter.py 30 i32_3 f64_2 > gpurun_out/stress_d.jsonl 2> gpurun_out/stress_d.err
timeout 600 python tools/stress_scatter.py 5 full_f64 >> gpurun_out/stress_d.jsonl 2>> gpurun_out/stress_d.err
cat gpurun_out/stress_d.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_scat_d.csv python tools/ncu_target.py scatter 2 > /dev/null 2>&1
grep -E "scat_" gpurun_out/launches_scat_d.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | cut -c1-160
bash tools/ncu_brief.sh d_part scat_part 1 python tools/ncu_target.py scatter 2
bash tools/ncu_brief.sh d_apply scat_apply 1 python tools/ncu_target.py scatter 2
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/merge_probe tools/merge_probe.cu && timeout 300 /tmp/merge_probe > gpurun_out/merge_probe.txt 2>&1
cat gpurun_out/merge_probe.txt
du -sh gpurun_out
