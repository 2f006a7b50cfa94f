cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/prof
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k "regex:bfs_persistent_kernel|uf_persistent_kernel|reinsert_kernel|bfs_init_kernel" -c 8 -o /tmp/prof/equiv -f python tools/profile_step.py --workload equiv > gpurun_out/prof_equiv.log 2>&1
echo "equiv rc=$?"
ncu -i /tmp/prof/equiv.ncu-rep --page raw --csv > gpurun_out/prof_equiv.csv 2>/dev/null
