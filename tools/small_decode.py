"""One small-batch decode (BASELINE cfg1: 32 CBs K=1056, 6 fixed iterations, or
cfg2 with --cfg 2) for latency profiling under ncu.  usage: python tools/small_decode.py [cfg]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import batch as bmod  # noqa: E402
from paper_1905_01141_b200 import build as B  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402
from paper_1905_01141_b200 import workload as wlmod  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    B.build()
    wl = wlmod.make_workload(cfg, seed=0, device="cuda")
    b = bmod.build(wl)
    plan = crn.Plan(b.desc)
    bits, ok, it, _ = bmod.outputs(b, want_ext=False)
    for _ in range(4):
        plan.decode(*b.llr, wl.max_iters, wl.early_term, bits, ok, it)
    torch.cuda.synchronize()
    print("ok", int(ok[:b.n_cb].sum()), b.n_cb)


if __name__ == "__main__":
    main()
