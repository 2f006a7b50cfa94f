#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_minimize.py -q -m gpu -p no:cacheprovider --timeout 500 -rf -x > gpurun_out/pytest_min.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_min.log
timeout -s KILL 300 python - > gpurun_out/naive_timing.log 2>&1 <<'PY'
import ctypes as C, time, torch, sys
sys.path.insert(0, '.')
import paper_2508_20735_b200 as dk
from paper_2508_20735_b200 import _native as nat
ctx = dk.Context(0)
for n in (20000, 100000, 1000000):
    k = 10
    d = torch.empty(k*n, dtype=torch.int32, device='cuda'); a = torch.empty(n, dtype=torch.uint8, device='cuda'); b = torch.empty(n, dtype=torch.int32, device='cuda')
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, 7, d.data_ptr(), a.data_ptr(), ctx.stream))
    view = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), -1)
    for algo in ('naive_pr', 'naive_pr_fused'):
        rep = nat.CReport(); opts = nat.COptions(0,0,0,0,0,64,0)
        f = lambda: nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm[algo]), C.byref(opts), b.data_ptr(), C.byref(rep), ctx.stream))
        f(); torch.cuda.synchronize(); t0=time.perf_counter(); f(); torch.cuda.synchronize(); dt=time.perf_counter()-t0
        print(n, algo, rep.passes, f"{dt*1e3:.1f} ms", f"{dt/rep.passes*1e6:.2f} us/pass")
PY
