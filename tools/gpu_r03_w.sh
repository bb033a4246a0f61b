#!/bin/bash
# repeat the one-process-per-device random programs (world 3) with full logs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for r in 1 2 3 4; do
  timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port $((29600 + r)) \
    tests/workers/mp_random.py --seeds 24 --first 5300 > gpurun_out/mpr_$r.out 2> gpurun_out/mpr_$r.err
  echo "run $r rc=$? $(grep -c 'ok 24' gpurun_out/mpr_$r.out)"
done
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -m gpu > gpurun_out/mp_tests_w.log 2>&1; tail -2 gpurun_out/mp_tests_w.log
