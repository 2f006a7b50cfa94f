#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/qb$i.log 2>&1; done
