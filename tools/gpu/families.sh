#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 600 python tools/family_timing.py > gpurun_out/families.jsonl 2> gpurun_out/families.err
