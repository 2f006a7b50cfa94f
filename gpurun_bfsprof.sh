#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/prof
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent_kernel -s 0 -c 1 -o /tmp/prof/bfs -f python tools/profile_step.py --workload equiv > gpurun_out/prof_bfs.log 2>&1
ncu -i /tmp/prof/bfs.ncu-rep --page raw --csv > gpurun_out/prof_bfs.csv 2>/dev/null
ncu -i /tmp/prof/bfs.ncu-rep --page source --csv > gpurun_out/prof_bfs_source.csv 2>/dev/null
ncu -i /tmp/prof/bfs.ncu-rep --page details --csv > gpurun_out/prof_bfs_details.csv 2>/dev/null
