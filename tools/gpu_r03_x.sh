#!/bin/bash
# repeat the one-process-per-device random programs (world 3 and 2) with full logs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for r in 1 2 3 4 5 6 7 8; do
  w=$(( r % 2 == 0 ? 2 : 3 ))
  timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port $((29700 + r)) \
    tests/workers/mp_random.py --seeds 24 --first $((5000 + 100 * w)) > gpurun_out/mpx_$r.out 2> gpurun_out/mpx_$r.err
  echo "run $r world $w rc=$? ok=$(grep -c 'ok 24' gpurun_out/mpx_$r.out)"
done
