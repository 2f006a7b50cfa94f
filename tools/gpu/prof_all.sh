#!/bin/bash
# ncu --set full of every kernel family (1 GPU).  Reports stay in /tmp on the
# box; their raw pages come back as CSV (the merge limit is 64 MiB).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/prof
run() {  # name regex count skip workload-args...
  local name=$1 re=$2 cnt=$3 skip=$4; shift 4
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c $cnt \
    -o /tmp/prof/$name -f python tools/profile_step.py "$@" > gpurun_out/prof_$name.log 2>&1
  echo "$name rc=$?" >> gpurun_out/prof_all.log
  ncu -i /tmp/prof/$name.ncu-rep --page raw --csv > gpurun_out/prof_$name.csv 2>/dev/null
}
run sort 'sig_table_kernel|sig_bucket_kernel|bucket_group_kernel|table_apply_vec_kernel|tile_apply_kernel|tile_count_kernel|acc_dense2_kernel|iota_kernel|leader_info_kernel|table_occupied_kernel' 12 0 --workload synth --reps 1
cp /tmp/prof/sort.ncu-rep gpurun_out/prof_sort.ncu-rep
run radix 'signature_kernel|radix_hist_all_kernel|radix_onesweep_kernel|radix_bins_kernel|run_heads_kernel|run_apply_kernel|run_min_kernel|verify_runs_kernel' 14 0 --workload radix --reps 1
run naive 'naive_persistent_kernel|fused_persistent_kernel' 2 0 --workload naive
run chain 'double_kernel|naive_persistent_kernel' 6 0 --workload chain --reps 1
cp /tmp/prof/chain.ncu-rep gpurun_out/prof_chain.ncu-rep
run equiv 'bfs_persistent_kernel|uf_persistent_kernel|reinsert_kernel' 8 0 --workload equiv
run sharded 'sig_owner_kernel|owner_apply_kernel|bucket_group_kernel|owner_counts_kernel' 10 0 --workload sharded --reps 1
run sliced 'sig_part_all_kernel|sig_part_vec_kernel|sig_bucket_kernel|bucket_group_kernel|sig_table_kernel' 6 0 --workload synth --states 100000000 --reps 1
run trans 'trans_' 6 0 --workload trans --reps 1
run fib 'naive_one_kernel|fused_one_kernel|small_persistent_kernel' 3 0 --workload fib
run calib 'gather_probe_kernel' 2 0 --workload calib
du -sh gpurun_out >> gpurun_out/prof_all.log
