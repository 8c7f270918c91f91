"""Measurement tool (not part of the product): event-to-event time of a CUDA graph of 1-3 tiny
kernels (optionally PDL-free), with the same L2 flush between launches as bench.py, to bound the
fixed launch cost inside a bench step."""
import torch

torch.cuda.init()
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
x = torch.zeros(1024, device=dev)


def run(nk):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            for _ in range(nk):
                x.add_(1.0)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(nk):
                x.add_(1.0)
    ts = []
    for _ in range(50):
        flush.zero_()
        _ = flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort()
    print(f"graph of {nk} tiny kernels: min {ts[0]:.2f} us, median {ts[len(ts)//2]:.2f} us")


for nk in (1, 2, 3):
    run(nk)
