#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "regex:naive_persistent_kernel" -c 1 -o /tmp/chain_naive -f python tools/profile_step.py --workload chain --reps 1 > gpurun_out/prof_chain_naive.log 2>&1
cp /tmp/chain_naive.ncu-rep gpurun_out/
