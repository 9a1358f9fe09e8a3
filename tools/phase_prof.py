"""Phase breakdown of the decode kernel from a -DCRN_PHASE_PROF build
(CRN_LIB=.../libcrn_prof.so): clock64 cycles a head warp (warp 0) and a tail
warp (warp 6) spend per phase, summed over CTAs, on cfg4 (8 fixed iterations).
usage: CRN_LIB=... python tools/phase_prof.py [n_cells] [cfg]   (cfg 4: fixed 8 iterations; cfg 3 / 5:
the pooled TTI / a latency TTI with CRC early termination, all cells)"""
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

NAMES = ["fetch", "stage", "chunk", "phase1", "bar1", "phase2", "bar2", "hard_dec", "st_loads", "st_bar1", "st_gather",
         "hd_lapp", "hd_bar1", "hd_crc", "hd_bar2", "hd_decide", "fetch_bars", "st_mbar_wait"]


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    L = crn.lib()
    f = L.crn_prof_read
    f.argtypes = [C.POINTER(C.c_ulonglong)]
    wl = wlmod.make_workload(cfg, seed=0, cells=range(cells) if cfg == 4 else None, device="cuda")
    b = bmod.build(wl)
    p = crn.Plan(b.desc)
    bits, ok, it, _ = bmod.outputs(b, want_ext=False)
    buf = (C.c_ulonglong * (2 * len(NAMES)))()
    et = cfg != 4
    p.decode(*b.llr, 8, et, bits, ok, it)
    torch.cuda.synchronize()
    f(buf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p.decode(*b.llr, 8, et, bits, ok, it)
    e1.record()
    torch.cuda.synchronize()
    f(buf)
    v = np.array(list(buf), dtype=np.float64).reshape(2, len(NAMES))
    its = it[:b.n_cb].cpu().numpy()
    out = {"cfg": cfg, "n_cb": b.n_cb, "ms": e0.elapsed_time(e1), "mean_iters": float(its.mean()),
           "sum_K": int(b.K.sum()), "counted_ops": crn.counted_ops(b.K, 8, its)}
    for k, who in enumerate(("head_warp0", "tail_warp6")):
        tot = v[k].sum()
        out[who] = {n: round(100 * x / tot, 2) for n, x in zip(NAMES, v[k])}
        out[who + "_cycles_per_task"] = {n: round(x / (b.n_cb / 2), 1) for n, x in zip(NAMES, v[k])}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
