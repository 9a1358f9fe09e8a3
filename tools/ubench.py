"""Run the int16x2 ALU microbenchmark and print JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_01141_b200 import build as crn_build  # noqa: E402
from paper_1905_01141_b200 import crn  # noqa: E402

crn_build.build()
dev = crn.device_info()
names = ["VIADD.16x2", "VIMNMX.S16x2", "VIMNMX3.S16x2", "VIADDMNMX.S16x2"]
ops_per_lane = [2, 2, 4, 4]
res = {"device": dev, "ops": {}}
for op in range(4):
    r = crn.ubench_int16x2(op)
    lanes_per_clk_sm = r["lane_instr"] / (dev["num_sms"] * r["max_block_cycles"])
    eff_mhz = r["max_block_cycles"] / (r["ms"] * 1e3)
    res["ops"][names[op]] = dict(r, lanes_per_clk_per_sm=lanes_per_clk_sm, clock_mhz_est=eff_mhz,
                                 int16_ops_per_clk_per_sm=lanes_per_clk_sm * ops_per_lane[op],
                                 tops=r["lane_instr"] * ops_per_lane[op] / (r["ms"] * 1e-3) / 1e12)
print(json.dumps(res, indent=1))
