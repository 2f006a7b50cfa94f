#!/bin/bash
# quick perf loop: grouping parity tests, bench line (no extras), per-kernel breakdown
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_minimize.py -q -m gpu -p no:cacheprovider --timeout 500 -x -k "${PERF_TESTS:-grouping or exact_paths or sweep or config1}" > gpurun_out/perf_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/perf_pytest.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/perf_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/perf_bench.log
for w in ${KPROF:-synth}; do timeout -s KILL 300 python tools/kprof.py $w --reps 5 > gpurun_out/kprof_$w.log 2>&1; done
