#!/bin/bash
# one build->measure cycle: GPU tests, bench (no extras), launch list, ncu --set full of the sort_pr kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -p no:cacheprovider --timeout 400 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --reps 2 > gpurun_out/launches.log 2>&1
K=${PROF_KERNELS:-'regex:sig_table_kernel|sig_bucket_kernel|bucket_group_kernel|table_apply_kernel|compact_flags_kernel|slot_apply_kernel'}
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "$K" -c 12 \
  -o /tmp/prof_full -f python tools/profile_step.py --reps 2 > gpurun_out/prof_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/prof_full.log; cp /tmp/prof_full.ncu-rep gpurun_out/
