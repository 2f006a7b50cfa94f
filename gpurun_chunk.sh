#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/chunk.log
for v in with without; do
  cp exp/$v.so paper_2508_20735_b200/lib/libdfakit_b200.so
  echo "$v" >> gpurun_out/chunk.log
  timeout -s KILL 120 python tools/kprof.py chain --reps 2 2>&1 | grep -E "wall" >> gpurun_out/chunk.log
  timeout -s KILL 120 python tools/kprof.py naive --reps 1 2>&1 | grep -E "wall" >> gpurun_out/chunk.log
  timeout -s KILL 120 python tools/kprof.py naive --algo naive_pr_fused --reps 1 2>&1 | grep -E "wall" >> gpurun_out/chunk.log
done
