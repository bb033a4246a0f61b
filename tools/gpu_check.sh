#!/bin/bash
# parity + multi-process + bench smoke on one GPU
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1
tail -15 gpurun_out/gpu_tests.log
timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_mp2.json 2> gpurun_out/bench_mp2.err
tail -3 gpurun_out/bench_mp2.err
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/bench_sp2.json 2> gpurun_out/bench_sp2.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
