#!/bin/bash
# one gpurun session: full-size parity, bench, launch list, ncu full captures
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -k "full_size" > gpurun_out/gpu_full.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
for k in jacobi dot gemm scatter; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'(jacobi2d|reduce|gemm|scatter)' -s 2 -c 1 -o gpurun_out/prof_$k -f python tools/ncu_target.py $k 3 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
