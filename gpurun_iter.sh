#!/bin/bash
# quick iteration: GPU tests (fail fast) + short bench without extras
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
