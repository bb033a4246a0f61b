#!/bin/bash
# bits-pass item size variants; Himeno stencil DRAM diagnosis (no-coefficient build)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
VARIANTS="b18:-DSBITS_LB=18,-DSBITS_T=512,-DSBITS_GRID=0 b18t1k:-DSBITS_LB=18,-DSBITS_T=1024,-DSBITS_GRID=0 b19:-DSBITS_LB=19,-DSBITS_T=1024,-DSBITS_GRID=0" LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh 2>&1 | tee gpurun_out/bits_ab_g.log
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum"
echo "== default"; timeout 600 ncu --metrics $M --clock-control none -k regex:himeno_stencil -c 2 --csv python tools/ncu_target.py himeno 2 2>/dev/null | grep himeno_stencil | awk -F'","' '{print $(NF-2), $NF}' | tail -7
python paper_2110_14340_b200/build.py --out /tmp/libjacc.nocoef.so -DHIMENO_DIAG_NOCOEF=1 > /dev/null; cp paper_2110_14340_b200/libjacc.so /tmp/libjacc.def.so; cp /tmp/libjacc.nocoef.so paper_2110_14340_b200/libjacc.so
echo "== nocoef"; timeout 600 ncu --metrics $M --clock-control none -k regex:himeno_stencil -c 2 --csv python tools/ncu_target.py himeno 2 2>/dev/null | grep himeno_stencil | awk -F'","' '{print $(NF-2), $NF}' | tail -7
cp /tmp/libjacc.def.so paper_2110_14340_b200/libjacc.so
for l in scat_f64 scat_i32; do python tools/time_loop.py $l 8; done 2>&1 | tail -2
