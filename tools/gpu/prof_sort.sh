#!/bin/bash
# ncu --set full of the bench step's kernels only (the sort workload of prof_all.sh) + the launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/prof
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:sig_table_kernel|sig_bucket_kernel|bucket_group_kernel|table_apply_vec_kernel|table_counts_kernel|iota_kernel|leader_info_kernel|fill_regions_kernel" -c 12 \
  -o /tmp/prof/sort -f python tools/profile_step.py --workload synth --reps 1 > gpurun_out/prof_sort.log 2>&1
echo "sort rc=$?"
ncu -i /tmp/prof/sort.ncu-rep --page raw --csv > gpurun_out/prof_sort.csv 2>/dev/null
cp /tmp/prof/sort.ncu-rep gpurun_out/prof_sort.ncu-rep
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --reps 2 > gpurun_out/launches.log 2>&1
echo "launches rc=$?"
