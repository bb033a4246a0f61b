#!/bin/bash
# multi-device readiness: virtual-device J16K runs (single process graph
# replay and one process per device) vs n=1 -- the per-launch cross-device
# sync overhead probe; isolated ncu of the BK5 merge kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for l in scat_f64 scat_i32; do timeout 300 python tools/time_loop.py $l 5 >> gpurun_out/time_g.jsonl 2>> gpurun_out/time_g.err; done
cat gpurun_out/time_g.jsonl; tail -2 gpurun_out/time_g.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_scat_g.csv python tools/ncu_target.py scatter 2 > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 -k "scatter or graph" > gpurun_out/gpu_tests_g.log 2>&1; tail -2 gpurun_out/gpu_tests_g.log
timeout 600 python tools/stress_scatter.py 20 i32_3 f64_2 > gpurun_out/stress_g.jsonl 2> gpurun_out/stress_g.err
timeout 600 python tools/stress_scatter.py 4 full_f64 full_i32 >> gpurun_out/stress_g.jsonl 2>> gpurun_out/stress_g.err; cat gpurun_out/stress_g.jsonl
for n in 1 2 4 8; do
  timeout 900 python bench.py --gpus $n --steps 3 --warmup 2 --no-extra --no-cpu-baseline > gpurun_out/bench_sp$n.json 2> gpurun_out/bench_sp$n.err
  tail -1 gpurun_out/bench_sp$n.err
done
for n in 2 8; do
  timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 3 --warmup 2 --no-extra --no-cpu-baseline > gpurun_out/bench_mp$n.json 2> gpurun_out/bench_mp$n.err
  tail -1 gpurun_out/bench_mp$n.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_[sm]p*.json")):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "no line", e); continue
    r = j["roofline"]; c = j["config"]
    print(f.split("/")[-1], j["n_gpus"], round(j["ms_per_step"], 2), "ms/step", round(j["value"]), "GB/s",
          c.get("issue"), "plain", round(c.get("ms_per_step_plain_launches", 0), 2),
          "host_us", round(c.get("host_us_per_launch", 0), 1), "kavg_us", round(r["kernel_avg_us"], 1))
PY
NCU_NDEV=2 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:merge --csv --log-file gpurun_out/launches_merge.csv python tools/ncu_target.py merge 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launches_merge.csv') if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
for r in rows[1:]: print(r[ki].split("(")[0][-30:], r[mi], r[vi])
PY
