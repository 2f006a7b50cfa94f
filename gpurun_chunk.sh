#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 120 python tools/kprof.py naive --algo naive_pr_fused --reps 1 2>&1 | grep -E "wall" > gpurun_out/chunk.log
