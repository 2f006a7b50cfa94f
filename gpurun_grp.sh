#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 120 python tools/kprof.py synth --reps 5 > gpurun_out/grp8.log 2>&1
