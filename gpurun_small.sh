#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_minimize.py tests/test_gpu_sharded.py -q -m gpu -p no:cacheprovider --timeout 800 -rf -x > gpurun_out/pytest_min.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_min.log
timeout -s KILL 600 python tools/family_timing.py > gpurun_out/family.log 2>&1
