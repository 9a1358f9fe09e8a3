"""Breakdown of the cfg5 streaming latency (crn_stream_run): host submission time
(release -> all groups enqueued), device span, completion; both runner modes.
usage: python tools/lat_breakdown.py [n_tti]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402


class A:
    lat_distinct = 50
    lat_ttis = int(sys.argv[1]) if len(sys.argv) > 1 else 300


def main():
    import torch
    from paper_1905_01141_b200 import build as crn_build
    crn_build.build()
    torch.cuda.set_device(0)
    out = {}
    # reuse bench's generator by calling run_latency once (it builds the group buffers)
    r = bench.run_latency(A(), seed=0)
    out["bench_latency"] = {k: r[k] for k in r if k.endswith("_us") or k == "stages_p50_us"}
    os.environ["CRN_LAT_ZEROCOPY"] = "1"
    r = bench.run_latency(A(), seed=0)
    out["zerocopy"] = {k: r[k] for k in r if k.endswith("_us") or k == "stages_p50_us"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
