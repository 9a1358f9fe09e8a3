import torch, time
n = 2_417_491_968 // 2
h = torch.empty(n, dtype=torch.int16).pin_memory()
d = torch.empty(n, dtype=torch.int16, device="cuda")
for ns in (1, 2, 3, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n + ns - 1) // ns
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(ss):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i*chunk:(i+1)*chunk].copy_(h[i*chunk:(i+1)*chunk], non_blocking=True)
        for s in ss:
            e1.wait_stream(s) if hasattr(e1,'wait_stream') else None
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(ns, "streams", round(n*2/ms/1e6, 1), "GB/s")
# D2H
h2 = torch.empty(n // 16, dtype=torch.int16).pin_memory()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); h2.copy_(d[:n//16], non_blocking=True); e1.record(); torch.cuda.synchronize()
print("d2h", round(n//16*2/e0.elapsed_time(e1)/1e6,1), "GB/s")
