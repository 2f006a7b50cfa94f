#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_sharded.py -q -m gpu -p no:cacheprovider --timeout 800 -rf -x > gpurun_out/pytest_sharded.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sharded.log
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 400 -rf -x --deselect tests/test_gpu_sharded.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
