"""End-to-end (pinned host LLRs -> bits + crc_ok in host memory) time of the cfg4
batch through crn_plan_decode_host vs the number of chunks.  Prints JSON."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import batch as bmod  # noqa: E402
from paper_1905_01141_b200 import build as B  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402
from paper_1905_01141_b200 import workload as wlmod  # noqa: E402


def main():
    B.build()
    b = bmod.build(wlmod.make_workload(4, seed=0, device="cuda"))
    host = [x.cpu().pin_memory() for x in b.llr]
    bits, ok, _, _ = bmod.outputs(b, want_ext=False)
    hb = torch.empty(bits.numel(), dtype=bits.dtype).pin_memory()
    hok = torch.empty(ok.numel(), dtype=ok.dtype).pin_memory()
    st = torch.cuda.current_stream()
    out = {}
    for nc in (8, 16, 24, 32, 48, 64):
        plan = crn.Plan(b.desc)
        for _ in range(2):
            plan.decode_host(*host, 8, False, hb, hok, None, n_chunks=nc, stream=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            plan.decode_host(*host, 8, False, hb, hok, None, n_chunks=nc, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        out[nc] = round(e0.elapsed_time(e1) / 3, 3)
        plan.close()
    print(json.dumps({"ms_per_step_by_chunks": out, "upload_bytes": 3 * 2 * b.n_llr}))


if __name__ == "__main__":
    main()
