"""Device time of the DL kernels, byte and packed-bit forms, on n_cells cells of
cfg4 (256 CBs of K=6144 each): CRC24B attach + turbo encode, rate matching to
E = 3(K+4) at rv 0, and de-matching of E int16 values.  CUDA events around each call on the launching stream, after
warm-up; median of 10 (the host-side descriptor staging of a call is inside, as
for any caller of the C ABI).  usage: python tools/dl_time.py [n_cells]"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import batch as bmod  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402
from paper_1905_01141_b200 import workload as wlmod  # noqa: E402


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    b = bmod.build(wlmod.make_workload(4, seed=0, cells=range(cells), device="cuda"))
    d = b.desc
    st = torch.cuda.current_stream()
    coded = tuple(torch.empty_like(x) for x in b.coded)
    rm = np.zeros(d.size, crn.RM_DTYPE)
    rm["K"], rm["E"], rm["rv"] = d["K"], 3 * (d["K"] + 4), 0
    rm["e_off"], rm["llr_off"] = d["llr_off"] * 3, d["llr_off"]
    e = torch.empty(int((rm["e_off"] + rm["E"]).max()), dtype=torch.uint8, device="cuda")
    h = b.info.cpu().numpy()
    info_w = torch.from_numpy(np.packbits(np.concatenate([h, np.zeros((-h.size) % 32, np.uint8)]),
                                          bitorder="little").view(np.int32).copy()).cuda()
    coded_w = tuple(torch.zeros((b.coded[0].numel() + 31) // 32, dtype=torch.int32, device="cuda") for _ in range(3))
    e_w = torch.zeros((e.numel() + 31) // 32, dtype=torch.int32, device="cuda")
    soft = torch.zeros(e.numel(), dtype=torch.int16, device="cuda")
    hs = tuple(torch.empty_like(x) for x in b.llr)
    calls = {"encode_byte": lambda: crn.encode_batch(d, b.info, True, *coded, stream=st),
             "rate_match_byte": lambda: crn.rate_match_batch(rm, *coded, e, stream=st),
             "encode_packed": lambda: crn.encode_batch_packed(d, info_w, True, *coded_w, stream=st),
             "rate_match_packed": lambda: crn.rate_match_batch_packed(rm, *coded_w, e_w, stream=st),
             "rate_dematch": lambda: crn.rate_dematch_batch(rm, soft, False, *hs, stream=st)}
    out = {"n_cb": int(d.size)}
    for name, fn in calls.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name + "_ms"] = round(statistics.median(ts), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
