#!/bin/bash
# radix-sort grouping: parity tests + per-kernel breakdown (default lib and variants)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_minimize.py -q -m gpu -p no:cacheprovider --timeout 500 -x -k "exact_paths or grouping or config0" > gpurun_out/radix_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/radix_pytest.log
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset DFAKIT_LIB_VARIANT; else export DFAKIT_LIB_VARIANT=$v; fi
  echo "== $v" >> gpurun_out/radix.log
  timeout -s KILL 300 python tools/kprof.py synth --grouping 1 --reps 5 >> gpurun_out/radix.log 2>&1
done
