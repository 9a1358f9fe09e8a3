"""Latency probe: device time of one decode launch for single CBs of chosen K
(8 fixed iterations) and for cfg5-sized TTIs, to see what bounds the per-TTI
latency.  usage: python tools/lat_probe.py > out.json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import batch as bmod  # noqa: E402
from paper_1905_01141_b200 import build as crn_build  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402
from paper_1905_01141_b200 import workload as wlmod  # noqa: E402


def time_plan(b, iters, et, reps=20):
    p = crn.Plan(b.desc)
    bits, ok, it, _ = bmod.outputs(b, want_ext=False)
    for _ in range(3):
        p.decode(*b.llr, iters, et, bits, ok, it)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p.decode(*b.llr, iters, et, bits, ok, it)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts)), it[:b.n_cb].cpu().numpy()


def main():
    crn_build.build()
    out = {"single_cb_8it_us": {}, "pair_8it_us": {}}
    for K in (40, 56, 120, 504, 752, 1008, 1024, 1056, 2048, 4096, 6144):
        b = bmod.build(wlmod.make_cb_workload([K], device="cuda"))
        out["single_cb_8it_us"][K] = time_plan(b, 8, False)[0]
        b = bmod.build(wlmod.make_cb_workload([K, K], device="cuda"))
        out["pair_8it_us"][K] = time_plan(b, 8, False)[0]
    for I in (1, 2, 4, 8):
        b = bmod.build(wlmod.make_cb_workload([6144], device="cuda"))
        out[f"K6144_{I}it_us"] = time_plan(b, I, False)[0]
    tt = []
    for s in range(5):
        b = bmod.build(wlmod.make_workload(5, seed=s, device="cuda"))
        t_et, its = time_plan(b, 8, True)
        t_fx, _ = time_plan(b, 8, False)
        tt.append(dict(n_cb=b.n_cb, et_us=t_et, fixed8_us=t_fx, max_iters=int(its.max()),
                       mean_iters=float(its.mean()), n_generic=int((b.desc["K"] % 32 != 0).sum())))
    out["cfg5_tti_one_launch"] = tt
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
