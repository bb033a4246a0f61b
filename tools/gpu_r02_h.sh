#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for r in 1 2; do
for l in scat_f64 scat_i32; do
  timeout 300 python tools/time_loop.py $l 8 | sed "s/^/concurrent /"
  JACC_SCATTER_BITS_SERIAL=1 timeout 300 python tools/time_loop.py $l 8 | sed "s/^/serial /"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_scat_h.csv python tools/ncu_target.py scatter 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open('gpurun_out/launches_scat_h.csv') if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); mi=h.index("Metric Name"); vi=h.index("Metric Value")
for r in rows[-15:]: print(r[ki].split("(")[0][-32:], r[mi], r[vi])
PY
