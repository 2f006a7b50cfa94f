import torch, time
n=10_000_000; k=10
h=torch.empty(k*n,dtype=torch.int32,pin_memory=True); h.fill_(1)
d=torch.empty(k*n,dtype=torch.int32,device='cuda')
o=torch.empty(n,dtype=torch.int32,pin_memory=True); od=torch.empty(n,dtype=torch.int32,device='cuda')
def t(f,reps=10):
    f(); torch.cuda.synchronize()
    s=time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter()-s)/reps
x=t(lambda: d.copy_(h,non_blocking=True)); print(f"1D H2D 400MB: {x*1e3:.3f} ms {400e6/x/1e9:.1f} GB/s")
hv=h.view(k,n); dv=d.view(k,n)
def chunked(c):
    for i in range(c):
        q0=n*i//c; q1=n*(i+1)//c
        dv[:,q0:q1].copy_(hv[:,q0:q1],non_blocking=True)
for c in (1,8):
    x=t(lambda: chunked(c)); print(f"2D chunks={c}: {x*1e3:.3f} ms {400e6/x/1e9:.1f} GB/s")
x=t(lambda: o.copy_(od,non_blocking=True)); print(f"D2H 40MB: {x*1e3:.3f} ms {40e6/x/1e9:.1f} GB/s")
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
def dual():
    with torch.cuda.stream(s1): d[:k*n//2].copy_(h[:k*n//2],non_blocking=True)
    with torch.cuda.stream(s2): d[k*n//2:].copy_(h[k*n//2:],non_blocking=True)
x=t(dual); print(f"2 streams H2D 400MB: {x*1e3:.3f} ms {400e6/x/1e9:.1f} GB/s")
def both():
    with torch.cuda.stream(s1): d.copy_(h,non_blocking=True)
    with torch.cuda.stream(s2): o.copy_(od,non_blocking=True)
x=t(both); print(f"H2D 400 + D2H 40 concurrent: {x*1e3:.3f} ms")
