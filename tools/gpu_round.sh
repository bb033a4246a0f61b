#!/bin/bash
# one gpurun session of measurements of record: bench (both arms), the
# headline launch list, ncu --set full captures of every loop kernel
# (summarised on the box into profiles/ncu_summary_$TAG.json; reports
# deleted so gpurun_out stays small), a range-replay total of the binned
# scatter launch (kernels concurrent as in the product)
TAG=${ROUND_TAG:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-graph > gpurun_out/bench_ncu.log 2>&1
cap() {  # name loop regex [env]
  timeout 900 env $4 ncu --set full --clock-control none --import-source on -k regex:"$3" -s 2 -c 1 -o gpurun_out/prof_$1 -f python tools/ncu_target.py $2 3 > gpurun_out/ncu_$1.log 2>&1
}
cap jacobi jacobi jacobi2d
cap dot dot reduce_kernel
cap gemm gemm gemm_tma
# (the speculative partition is the first scat_part launch of each scatter
# launch; the histogram pass only runs after an overflow, never here)
for k in part apply bits; do cap scat_$k scatter scat_$k; cap scat_${k}_i32 scatter_i32 scat_$k; done
cap himeno_stencil himeno himeno_stencil
cap himeno_copy himeno himeno_copy
cap merge_range merge merge_range NCU_NDEV=2
cap merge_bitmap merge merge_bitmap NCU_NDEV=2
python tools/summarize_ncu.py $TAG > gpurun_out/summary_print.txt 2>&1
mkdir -p gpurun_out/profiles_new && cp profiles/ncu_summary_$TAG.json profiles/launches_$TAG.md gpurun_out/profiles_new/ 2>/dev/null
ncu -i gpurun_out/prof_gemm.ncu-rep --page source --csv > gpurun_out/ncu_gemm_source.csv 2>/dev/null
rm -f gpurun_out/prof_*.ncu-rep
# the binned scatter launch as one NVTX range: total DRAM bytes of the whole launch
timeout 600 ncu --replay-mode app-range --nvtx --nvtx-include "scatter_add_f64/" \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
    --log-file gpurun_out/range_scat.csv python tools/ncu_target.py scatter 3 > gpurun_out/range_scat.log 2>&1
du -sh gpurun_out
