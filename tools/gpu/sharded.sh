#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_sharded.py -q -m gpu -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/pytest_sh.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sh.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --engine sharded --no-extras --no-cpu-baseline > gpurun_out/bench_sharded.log 2> gpurun_out/bench_sharded.err
