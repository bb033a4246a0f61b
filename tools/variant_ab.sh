#!/bin/bash
# A/B of compile-time kernel variants: build each into /tmp, swap it in as
# the package's libjacc.so, time the loops; the default build is restored.
#   VARIANTS="name:-DX=1,-DY=2 name2:@prebuilt.so ..." LOOPS="scat_f64 scat_i32" REPS=8 ROUNDS=2 bash tools/variant_ab.sh
set -u
LIB=paper_2110_14340_b200/libjacc.so
cp $LIB /tmp/libjacc.default.so
for v in $VARIANTS; do
  name=${v%%:*}; defs=${v#*:}
  if [ "${defs:0:1}" = "@" ]; then cp ${defs:1} /tmp/libjacc.$name.so; continue; fi  # prebuilt library
  python paper_2110_14340_b200/build.py --out /tmp/libjacc.$name.so $(echo $defs | tr ',' ' ') > /dev/null || echo "build $name failed"
done
for r in $(seq ${ROUNDS:-2}); do
  for v in default $VARIANTS; do
    name=${v%%:*}
    cp /tmp/libjacc.$name.so $LIB
    for l in $LOOPS; do
      echo -n "$name "; timeout 300 python tools/time_loop.py $l ${REPS:-8}
    done
  done
done
cp /tmp/libjacc.default.so $LIB
