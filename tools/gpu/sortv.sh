#!/bin/bash
# radix sort primitive: parity vs numpy + per-digit timing for each library variant
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_prims.py -q -m gpu -p no:cacheprovider --timeout 500 -x > gpurun_out/sort_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sort_pytest.log
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset DFAKIT_LIB_VARIANT; else export DFAKIT_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/sortv.log
  timeout -s KILL 300 python tools/sort_bench.py >> gpurun_out/sortv.log 2>&1
done
