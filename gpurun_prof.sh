#!/bin/bash
# ncu --set full of the sort_pr kernels on the bench workload (1 GPU).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
K=${1:-'regex:signature_kernel|bucket_refine_kernel|sig_table_kernel|radix_scatter_kernel|radix_hist_kernel|table_apply_kernel|prefix_count_kernel'}
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "$K" -c 24 \
  -o gpurun_out/prof_full -f python tools/profile_step.py --reps 2 > gpurun_out/prof_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof_full.log
