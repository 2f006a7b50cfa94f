#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/prof_all.log
bash tools/gpu/prof_all.sh
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --reps 2 > gpurun_out/launches.log 2>&1
