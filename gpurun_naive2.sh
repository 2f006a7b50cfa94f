#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_minimize.py -q -m gpu -p no:cacheprovider -x -k "sweep or golden or fibonacci or chain or transitive or edge" > gpurun_out/pytest_naive.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_naive.log
timeout -s KILL 300 python tools/kprof.py chain > gpurun_out/kprof_chain.log 2>&1
timeout -s KILL 300 python tools/kprof.py naive > gpurun_out/kprof_naive.log 2>&1
timeout -s KILL 300 python tools/kprof.py naive --algo naive_pr_fused > gpurun_out/kprof_naive_fused.log 2>&1
timeout -s KILL 300 python tools/kprof.py fib --algo naive_pr > gpurun_out/kprof_fib_naive.log 2>&1
