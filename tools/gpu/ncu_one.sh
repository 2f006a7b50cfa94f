#!/bin/bash
# ncu --set full of one kernel family with source correlation:
#   NCU_RE='regex' NCU_COUNT=3 NCU_ARGS='--workload synth --reps 1' NCU_TAG=x bash tools/gpu/ncu_one.sh
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/prof
tag=${NCU_TAG:-one}
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_RE}" -c ${NCU_COUNT:-3} \
  -o /tmp/prof/$tag -f python tools/profile_step.py ${NCU_ARGS:---workload synth --reps 1} > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$tag.log
ncu -i /tmp/prof/$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>/dev/null
ncu -i /tmp/prof/$tag.ncu-rep --page details --csv > gpurun_out/ncu_${tag}_details.csv 2>/dev/null
n=$(ncu -i /tmp/prof/$tag.ncu-rep --page raw --csv 2>/dev/null | tail -n +3 | wc -l)
for i in $(seq 0 $((n-1))); do
  ncu -i /tmp/prof/$tag.ncu-rep --page source --csv --print-source cuda,sass --launch-skip $i --launch-count 1 > gpurun_out/ncu_${tag}_src$i.csv 2>/dev/null
done
cp /tmp/prof/$tag.ncu-rep gpurun_out/
