#!/bin/bash
# smoke + every -m gpu test (no -x: the whole failure list) + a quick bench line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout -s KILL 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 900 -rf ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/qb.log 2>&1; echo "bench rc=$?" >> gpurun_out/qb.log
