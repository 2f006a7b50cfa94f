cd "$GRAFT_REPO_ROOT"
python -m pytest tests/test_gpu_minimize.py tests/test_gpu_prims.py -m gpu -x -q 2>&1 | tail -2
python tools/kprof.py synth --reps 5 2>&1 | grep -E "wall|leader|#pass"
for v in base m4 i8m4 t512; do
  if [ "$v" = base ]; then unset DFAKIT_LIB_VARIANT; else export DFAKIT_LIB_VARIANT=$v; fi
  echo "== $v"; python tools/sort_bench.py 2>&1 | grep onesweep
done
unset DFAKIT_LIB_VARIANT
python tools/kprof.py synth --grouping 1 --reps 5 2>&1 | tail -17
