"""Graph-replay time vs kernel duration (development tool): is the per-replay time quantised?"""
import torch
dev = torch.device("cuda:0"); s = torch.cuda.Stream()
def timeit(fn, iters=300, per_graph=1):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(per_graph): fn()
    torch.cuda.synchronize()
    for _ in range(10): g.replay()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    n = iters // per_graph
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(n): g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (n * per_graph) * 1e3
for cyc in [0, 2000, 4000, 8000, 12000, 16000, 20000, 24000, 28000, 32000, 40000]:
    print(f"sleep {cyc:6d} cyc: 1/graph {timeit(lambda: torch.cuda._sleep(cyc)):7.2f} us; 10/graph {timeit(lambda: torch.cuda._sleep(cyc), per_graph=10):7.2f} us per kernel", flush=True)
