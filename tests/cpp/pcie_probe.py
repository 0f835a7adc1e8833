import torch, time
n = 8192*6144
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(3)]
d = [torch.empty(n, dtype=torch.float32, device='cuda') for _ in range(3)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    t0=time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter()-t0)/reps*1e3
def h2d():
    with torch.cuda.stream(s1): d[0].copy_(h[0], non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h[1].copy_(d[1], non_blocking=True)
def both():
    h2d(); d2h()
def h2d2():
    with torch.cuda.stream(s1): d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s2): d[2].copy_(h[2], non_blocking=True)
B=n*4/1e9
for name,fn,by in (("h2d",h2d,B),("d2h",d2h,B),("h2d+d2h",both,B),("2x h2d two streams",h2d2,2*B)):
    ms=t(fn); print(f"{name}: {ms:.2f} ms, {by/ms*1e3:.1f} GB/s")
