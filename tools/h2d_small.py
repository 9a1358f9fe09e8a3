"""Latency of pinned host->device copies of one TTI's inputs: the 4 cell groups'
~570 KB each (alone and on 4 concurrent streams) against one 2.27 MB copy --
what bounds the upload stage of the streaming run."""
import torch

n = 570_000 // 2
hs = [torch.zeros(n, dtype=torch.int16).pin_memory() for _ in range(4)]
ds = [torch.zeros(n, dtype=torch.int16, device="cuda") for _ in range(4)]
hb = torch.zeros(4 * n, dtype=torch.int16).pin_memory()
db = torch.zeros(4 * n, dtype=torch.int16, device="cuda")
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


def one():
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    db.copy_(hb, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3, 1)


for k in (1, 4):
    for _ in range(3):
        r = run(k)
    print(k, "copies of 570 KB: completion us", r)
for _ in range(3):
    r = one()
print("one 2.28 MB copy: us", r)
for sz in (64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20):
    h = torch.zeros(sz // 2, dtype=torch.int16).pin_memory()
    d = torch.zeros(sz // 2, dtype=torch.int16, device="cuda")
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
    print(sz >> 10, "KB:", round(e0.elapsed_time(e1) * 1e3, 1), "us", round(sz / e0.elapsed_time(e1) / 1e6, 1), "GB/s")
