#!/bin/bash
# per-kernel breakdown of the bench step for each library variant (make variant V=...)
#   VARIANTS="a b" KPROF_ARGS="synth" bash tools/gpu/variants.sh
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset DFAKIT_LIB_VARIANT; else export DFAKIT_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/variants.log
  timeout -s KILL 300 python tools/kprof.py ${KPROF_ARGS:-synth} --reps 5 >> gpurun_out/variants.log 2>&1
done
