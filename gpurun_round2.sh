#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash gpurun_round.sh
mkdir -p /tmp/prof
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k 'regex:sig_table_kernel|sig_bucket_kernel|bucket_group_kernel|table_apply_kernel|tile_apply_kernel|tile_count_kernel|dense2_kernel|relabel_kernel|leader_info_kernel|init_labels_kernel|gather_probe' -c 14 -o /tmp/prof/sort -f python tools/profile_step.py --workload synth --reps 1 > gpurun_out/prof_sort.log 2>&1
ncu -i /tmp/prof/sort.ncu-rep --page raw --csv > gpurun_out/prof_sort.csv 2>/dev/null
cp /tmp/prof/sort.ncu-rep gpurun_out/prof_sort.ncu-rep
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --reps 2 > gpurun_out/launches.log 2>&1
