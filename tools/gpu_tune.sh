#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
true
cat gpurun_out/tune_jacobi.txt
JACC_SCATTER_BINNED=1 timeout 900 python -m pytest tests -q -m gpu -x -k "scatter and not full" > gpurun_out/scat_tests.log 2>&1; tail -3 gpurun_out/scat_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:scat --csv --log-file gpurun_out/scat_launches.csv python tools/ncu_target.py scatter 2 > gpurun_out/scat_ncu.log 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/scat_launches.csv')) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    print(r[h.index('Kernel Name')].split('(')[0][-40:], r[h.index('Metric Name')], r[h.index('Metric Unit')], r[h.index('Metric Value')])
P
