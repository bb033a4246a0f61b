#!/bin/bash
# one gpurun session: bench, launch list, ncu --set full captures of every loop kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu-baseline --no-graph > gpurun_out/bench_ncu.log 2>&1
cap() {  # name loop regex
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$3" -s 2 -c 1 -o gpurun_out/prof_$1 -f python tools/ncu_target.py $2 3 > gpurun_out/ncu_$1.log 2>&1
}
cap jacobi jacobi jacobi2d
cap dot dot reduce_kernel
cap gemm gemm gemm_f64
cap scat_part scatter scat_part
cap scat_apply scatter scat_apply
cap scat_bits scatter scat_bits
cap himeno_stencil himeno himeno_stencil
cap himeno_copy himeno himeno_copy
ls gpurun_out/*.ncu-rep
# summarise on the box (ncu -i), keep the dominant kernel's report only
python tools/summarize_ncu.py ${ROUND_TAG:-r01} > gpurun_out/summary_print.txt 2>&1
mkdir -p gpurun_out/profiles_new && cp profiles/ncu_summary_${ROUND_TAG:-r01}.json profiles/launches_${ROUND_TAG:-r01}.md gpurun_out/profiles_new/ 2>/dev/null
for f in gpurun_out/prof_*.ncu-rep; do
  case "$f" in *prof_jacobi.ncu-rep) ;; *) rm -f "$f" ;; esac
done
du -sh gpurun_out
