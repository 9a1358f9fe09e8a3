"""Per-task timeline of one decode launch from a -DCRN_TASK_TRACE build
(CRN_LIB=.../libcrn_trace.so): for cfg5 TTIs (or cfg3 / cfg4 cells) the start / end
of every task relative to the first start, its SM, group (0 = whole CTA, 1-3 = a
group of four warps), K, pairs and its CBs' max iteration count.
usage: CRN_LIB=... python tools/task_trace.py [cfg] [n_ttis]"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import batch as bmod  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402
from paper_1905_01141_b200 import workload as wlmod  # noqa: E402


def one(cfg, cells):
    L = crn.lib()
    f = L.crn_trace_read
    f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int32]
    b = bmod.build(wlmod.make_workload(cfg, seed=0, cells=cells, device="cuda"))
    p = crn.Plan(b.desc)
    bits, ok, it, _ = bmod.outputs(b, want_ext=False)
    et = cfg != 4
    for _ in range(3):
        p.decode(*b.llr, 8, et, bits, ok, it)
    torch.cuda.synchronize()
    tof, info, _ = crn.task_layout(b.desc, spread_to=crn.device_info()["num_sms"])   # the plan's own spreading
    nt = info.shape[0]
    buf = (C.c_ulonglong * (4 * nt))()
    f(buf, nt)
    tr = np.array(list(buf), dtype=np.int64).reshape(nt, 4)
    its = it[:b.n_cb].cpu().numpy()
    t0 = tr[:, 0].min()
    rows = []
    for t in range(nt):
        cbs = np.flatnonzero(tof == t)
        rows.append({"task": t, "start_us": (tr[t, 0] - t0) / 1e3, "end_us": (tr[t, 1] - t0) / 1e3, "sm": int(tr[t, 2]),
                     "group": int(tr[t, 3]), "K": int(info[t, 0]), "pairs": int(info[t, 1]),
                     "max_iters": int(its[cbs].max()) if cbs.size else 0})
    span = max(r["end_us"] for r in rows)
    return {"cfg": cfg, "n_cb": b.n_cb, "n_tasks": nt, "span_us": span, "tasks": rows}


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    out = []
    for t in range(n):
        cells = range(20 * t, 20 * t + 20) if cfg == 5 else None
        out.append(one(cfg, cells))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
