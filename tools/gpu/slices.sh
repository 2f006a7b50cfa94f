#!/bin/bash
# sliced-pass geometry: label-array size x number of slices (no L2 pin)
cd "$GRAFT_REPO_ROOT"
for n in 50000000 70000000 100000000; do
  for sb in 1073741824 115343360 75497472 52428800; do
    echo "== n=$n slice_bytes=$sb"
    DFAKIT_TEST_SLICE_BYTES=$sb timeout 300 python tools/kprof.py synth --states $n --reps 3 2>&1 | grep -E "wall|sig_part|sig_bucket"
  done
done
