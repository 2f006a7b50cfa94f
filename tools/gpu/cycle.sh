#!/bin/bash
# GPU tests + quick bench + per-kernel breakdown of the bench step
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/qb.log 2>&1
timeout -s KILL 300 python tools/kprof.py synth --reps 5 > gpurun_out/kprof_synth.log 2>&1
