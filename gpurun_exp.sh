#!/bin/bash
# development experiments: DSMEM gather probe, per-kernel breakdowns of the secondary workloads
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 120 ./bin/dsmem_probe > gpurun_out/dsmem_probe.log 2>&1
for w in chain fib equiv; do timeout -s KILL 300 python tools/kprof.py $w > gpurun_out/kprof_$w.log 2>&1; done
timeout -s KILL 300 python tools/kprof.py fib --algo naive_pr > gpurun_out/kprof_fib_naive.log 2>&1
timeout -s KILL 300 python tools/kprof.py fib --param 15 --algo naive_pr > gpurun_out/kprof_fib15_naive.log 2>&1
timeout -s KILL 300 python tools/kprof.py fib --param 15 > gpurun_out/kprof_fib15.log 2>&1
