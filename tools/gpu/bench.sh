#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --engine sharded --no-extras --no-cpu-baseline > gpurun_out/bench_sharded.log 2> gpurun_out/bench_sharded.err; echo "rc=$?" >> gpurun_out/bench_sharded.err
timeout -s KILL 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
nproc > gpurun_out/nproc.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --engine sharded-py --no-extras --no-cpu-baseline > gpurun_out/bench_shardedpy.log 2> gpurun_out/bench_shardedpy.err; echo "rc=$?" >> gpurun_out/bench_shardedpy.err
