"""Quick A/B timing of one libcrn build (CRN_LIB=...): device time of cfg4 (full,
8 fixed iterations), cfg3 (one pooled TTI, CRC ET), cfg5 (20 distinct latency TTIs,
one launch each, CRC ET) and cfg1; one JSON line.  Also checks that the outputs
equal the ones in --ref (a .pt written by a previous run) when given.
usage: CRN_LIB=... python tools/ab_quick.py [--save out.pt] [--ref ref.pt] [--cfg4-cells N]"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import batch as bmod  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402
from paper_1905_01141_b200 import workload as wlmod  # noqa: E402


def timed(plan, b, iters, et, reps, warm=2):
    bits, ok, it, _ = bmod.outputs(b, want_ext=False)
    st = torch.cuda.current_stream()
    for _ in range(warm):
        plan.decode(*b.llr, iters, et, bits, ok, it, stream=st)
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        plan.decode(*b.llr, iters, et, bits, ok, it, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return statistics.median(t), (bits.clone(), ok.clone(), it.clone())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--save")
    ap.add_argument("--ref")
    ap.add_argument("--cfg4-cells", type=int, default=256)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("CRN_LIB", "libcrn.so")))
    a = ap.parse_args()
    out, res = {"lib": a.tag}, {}
    b4 = bmod.build(wlmod.make_workload(4, seed=0, cells=range(a.cfg4_cells), device="cuda"))
    ms, res["cfg4"] = timed(crn.Plan(b4.desc), b4, 8, False, 5)
    out["cfg4_ms"] = round(ms, 4)
    out["cfg4_frac"] = round(crn.counted_ops(b4.K, 8, None) / (ms * 1e-3) / 74.44992e12, 4)
    del b4
    b3 = bmod.build(wlmod.make_workload(3, seed=0, device="cuda"))
    ms, res["cfg3"] = timed(crn.Plan(b3.desc), b3, 8, True, 20)
    its = res["cfg3"][2][:b3.n_cb].cpu().numpy()
    out["cfg3_ms"] = round(ms, 4)
    out["cfg3_frac"] = round(crn.counted_ops(b3.K, 8, its) / (ms * 1e-3) / 74.44992e12, 4)
    lat = []
    for t in range(20):
        b5 = bmod.build(wlmod.make_workload(5, seed=0, cells=range(20 * t, 20 * t + 20), device="cuda"))
        ms, r = timed(crn.Plan(b5.desc), b5, 8, True, 5)
        lat.append(ms * 1e3)
        res[f"cfg5_{t}"] = r
    out["cfg5_us_med"] = round(statistics.median(lat), 1)
    out["cfg5_us_max"] = round(max(lat), 1)
    b1 = bmod.build(wlmod.make_workload(1, seed=0, device="cuda"))
    ms, res["cfg1"] = timed(crn.Plan(b1.desc), b1, 6, False, 20)
    out["cfg1_us"] = round(ms * 1e3, 1)
    if a.save:
        torch.save({k: [x.cpu() for x in v] for k, v in res.items()}, a.save)
    if a.ref and os.path.exists(a.ref):
        ref = torch.load(a.ref)
        out["same_as_ref"] = all(torch.equal(x.cpu(), y) for k in ref for x, y in zip(res[k], ref[k]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
