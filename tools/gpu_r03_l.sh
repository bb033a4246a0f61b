#!/bin/bash
# EAGER push of the binned scatter: fused (words per round) vs separate merge_bitmap
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
LIB=paper_2110_14340_b200/libjacc.so; cp $LIB /tmp/def.so
for v in "pw8:-DSBITS_PW=8" "pw16:-DSBITS_PW=16" "unfused:-DSCAT_FUSED_PUSH=0"; do
  n=${v%%:*}; d=${v#*:}; python paper_2110_14340_b200/build.py --out /tmp/$n.so $d > /dev/null
done
for r in 1 2; do for n in def pw8 pw16 unfused; do
  cp /tmp/$n.so $LIB; echo -n "$n "; timeout 600 python tools/merge_time.py 2>/dev/null | tail -1
done; done | tee gpurun_out/push_ab_l.log
cp /tmp/def.so $LIB
