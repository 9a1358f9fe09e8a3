"""Host-side cost per call of the one-shot batch entry points (descriptor
validation + pinned staging + launch), for a cfg4-sized batch (65,536 CBs of
K=6144).  Prints one JSON line.  usage: python tools/host_overhead.py"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import build as crn_build  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402


def main():
    crn_build.build()
    n, K = 65536, 6144
    d = np.zeros(n, crn.DESC_DTYPE)
    d["K"], d["crc_kind"] = K, crn.CRC24B
    d["ext_off"] = np.arange(n) * K
    d["llr_off"] = np.arange(n) * (K + 4)
    d["bit_off"] = np.arange(n) * (K // 32)
    info = torch.zeros(n * K, dtype=torch.uint8, device="cuda")
    coded = [torch.empty(n * (K + 4), dtype=torch.uint8, device="cuda") for _ in range(3)]
    rm = np.zeros(n, crn.RM_DTYPE)
    rm["K"], rm["E"], rm["rv"] = K, 3 * (K + 4), 0
    rm["e_off"], rm["llr_off"] = d["llr_off"] * 3, d["llr_off"]
    e = torch.empty(n * 3 * (K + 4), dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("encode_batch", lambda: crn.encode_batch(d, info, True, *coded)),
                     ("rate_match_batch", lambda: crn.rate_match_batch(rm, *coded, e))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e3)
        torch.cuda.synchronize()
        out[name + "_host_ms"] = float(np.median(ts))
    # the bare C call (arguments prepared once), every repetition
    L = crn.lib()
    args = (d.ctypes.data, n, info.data_ptr(), 1, coded[0].data_ptr(), coded[1].data_ptr(), coded[2].data_ptr(),
            torch.cuda.current_stream().cuda_stream)
    reps = []
    for _ in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.crn_encode_batch(*args)
        reps.append(round((time.perf_counter() - t0) * 1e3, 3))
    torch.cuda.synchronize()
    out["encode_c_call_ms"] = reps
    bad = d.copy()
    bad["K"][-1] = 7                       # rejected after the full validation pass
    t0 = time.perf_counter()
    L.crn_encode_batch(bad.ctypes.data, n, *args[2:])
    out["encode_validate_only_ms"] = (time.perf_counter() - t0) * 1e3
    v = np.zeros(n, np.int64)
    t0 = time.perf_counter()
    for _ in range(5):
        np.ascontiguousarray(d, crn.DESC_DTYPE)
    out["ascontiguous_ms"] = (time.perf_counter() - t0) / 5 * 1e3
    t0 = time.perf_counter()
    for _ in range(5):
        v[:] = d["K"]
    out["numpy_field_copy_ms"] = (time.perf_counter() - t0) / 5 * 1e3
    out["desc_bytes"] = int(d.nbytes)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
