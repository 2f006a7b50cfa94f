#!/bin/bash
# product BFS: parity tests + per-kernel breakdown for each variant
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_product.py -q -m gpu -p no:cacheprovider --timeout 800 -x > gpurun_out/bfs_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bfs_pytest.log
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset DFAKIT_LIB_VARIANT; else export DFAKIT_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/bfs.log
  timeout -s KILL 300 python tools/kprof.py equiv --reps 5 >> gpurun_out/bfs.log 2>&1
done
