cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/prof
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:sig_part_all_kernel|sig_part_vec_kernel|sig_bucket_kernel|bucket_group_kernel|sig_table_kernel|pack1" -c 7 -o /tmp/prof/sliced -f python tools/profile_step.py --workload synth --states 100000000 --reps 1 > gpurun_out/prof_sliced.log 2>&1
echo "sliced rc=$?"
ncu -i /tmp/prof/sliced.ncu-rep --page raw --csv > gpurun_out/prof_sliced.csv 2>/dev/null
