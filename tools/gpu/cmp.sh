#!/bin/bash
# kprof workloads for the current library and variants: WL="chain naive" VARIANTS="r1" bash tools/gpu/cmp.sh
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for w in ${WL:-chain}; do
  for v in base ${VARIANTS}; do
    if [ "$v" = base ]; then unset DFAKIT_LIB_VARIANT; else export DFAKIT_LIB_VARIANT=$v; fi
    echo "== $w $v" >> gpurun_out/cmp.log
    timeout -s KILL 300 python tools/kprof.py $w --reps 3 >> gpurun_out/cmp.log 2>&1
  done
done
