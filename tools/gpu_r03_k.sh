#!/bin/bash
# dense-word bitmap merge: EAGER parity, merge timings vs previous build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x -k "scatter or eager or random_programs or multiprocess" > gpurun_out/tests_k.log 2>&1; tail -2 gpurun_out/tests_k.log
LIB=paper_2110_14340_b200/libjacc.so
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_k_new.json 2> gpurun_out/bench_k_new.err
cp $LIB /tmp/new.so; cp variants/libjacc.prev.so $LIB
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_k_prev.json 2> gpurun_out/bench_k_prev.err
cp /tmp/new.so $LIB
for f in new prev; do python - $f <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/bench_k_{sys.argv[1]}.json').read().strip().splitlines()[-1])
m=d.get('merge',{})
print(sys.argv[1], {k:(round(v.get('us') or v.get('push_cost_us') or 0,1), v.get('bytes_pushed')) for k,v in m.items()})
PY
done
