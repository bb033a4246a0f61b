#!/bin/bash
# repeat the one-process-per-GPU tests; keep the output of failing runs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
mkdir -p gpurun_out/stress
for i in $(seq 1 ${ITERS:-4}); do
  timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -x > gpurun_out/stress/pytest$i.txt 2>&1
  rc=$?
  echo "iter $i rc=$rc $(tail -1 gpurun_out/stress/pytest$i.txt)"
  if [ $rc = 0 ]; then rm gpurun_out/stress/pytest$i.txt; fi
done
