import torch, time
dev='cuda'
def t(fn, R=8, iters=50):
    s=torch.cuda.Stream()
    gs=[]
    for r in range(R):
        g=torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            fn(r); torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s): fn(r)
        gs.append(g)
    torch.cuda.synchronize()
    for i in range(10): gs[i%R].replay()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for i in range(iters): gs[i%R].replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b)/iters*1e3
for mb in [16, 33.6, 67, 101, 400]:
    n=int(mb*1e6/2)
    R=max(2, int(4*132e6/(mb*1e6))+1)
    xs=[torch.randn(n, device=dev, dtype=torch.bfloat16) for _ in range(R)]
    ys=[torch.empty(n//2, device=dev, dtype=torch.bfloat16) for _ in range(R)]
    out=torch.empty(1, device=dev)
    us=t(lambda r: torch.sum(xs[r].view(torch.float32), out=out), R)
    us2=t(lambda r: ys[r].copy_(xs[r][:n//2]), R)
    print(f"read {mb} MB: sum {us:.2f} us = {mb*1e6/us/1e3:.0f} GB/s | copy {mb/2}MB->{mb/2}MB {us2:.2f} us = {mb*1e6/us2/1e3:.0f} GB/s", flush=True)
