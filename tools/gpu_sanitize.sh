#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small parity cases
# that reach every shared-memory kernel:
# Jacobi (BK1), reductions (BK2 + combine), GEMM (BK3), scatter direct /
# binned (hist/part/apply/bits, byte-map) / owner-slice (BK4, BK4b, BK4c),
# iteration-split scatter + combine, Himeno stencil/copy, Fig. 4, merges
# (range/box/bitmap under EAGER), graphs and async queues.
mkdir -p gpurun_out
TAG=${ROUND_TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
T=tests/test_gpu_parity.py
K='J256 or test_jacobi_multi_device and 17- or test_scatter_exact and 100- or test_square_multi and 1000- or test_dot_sum_dyadic_exact and 4096 or test_gemm_random_tolerance or himeno_multi_device and shape1 or test_fig4_chain and 257 or test_scatter_iteration_split and sizes0 or test_iteration_split_back_to_back_halo or test_graph_capture or async_queues or test_scatter_paths_and_misaligned_ranges or test_scatter_binned_extreme_skew or test_scatter_binned_overflow and late or test_jacobi_column_split'
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 2400 compute-sanitizer --tool $tool $extra --error-exitcode 9 python -m pytest $T -q -m gpu -k "$K" \
      > gpurun_out/san_${tool}_${TAG}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_${tool}_${TAG}.log
  tail -3 gpurun_out/san_${tool}_${TAG}.log
done
# kernels each test reached (names from the memcheck run's --print-level info would be verbose;
# the launch list of the same subset gives them)
timeout 900 ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/san_kernels_${TAG}.csv \
    python -m pytest $T -q -m gpu -k "$K" > /dev/null 2>&1
python - <<EOF
import csv, collections
c = collections.Counter()
for r in csv.DictReader(l for l in open("gpurun_out/san_kernels_${TAG}.csv") if l.startswith('"')):
    c[r["Kernel Name"].split("(")[0].split("<")[0]] += 1
open("gpurun_out/san_kernels_${TAG}.txt", "w").write("\n".join(f"{k} {v}" for k, v in sorted(c.items())) + "\n")
print(len(c), "distinct kernels under the sanitizer subset")
EOF
