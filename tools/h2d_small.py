"""Latency of small pinned host->device copies (one TTI group ~570 KB), alone and
4 concurrent streams: what bounds the upload stage of the streaming run."""
import torch

n = 570_000 // 2
hs = [torch.zeros(n, dtype=torch.int16).pin_memory() for _ in range(4)]
ds = [torch.zeros(n, dtype=torch.int16, device="cuda") for _ in range(4)]
ss = [torch.cuda.Stream() for _ in range(4)]


def run(k):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
    e0.record()
    for i in range(k):
        ss[i].wait_event(e0)
        with torch.cuda.stream(ss[i]):
            ds[i].copy_(hs[i], non_blocking=True)
            ends[i].record(ss[i])
    torch.cuda.synchronize()
    return [round(e0.elapsed_time(e) * 1e3, 1) for e in ends]


for k in (1, 4):
    for _ in range(3):
        r = run(k)
    print(k, "copies of 570 KB: completion us", r)
