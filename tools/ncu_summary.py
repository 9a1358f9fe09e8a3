"""Summarise an ncu report: key metrics (raw page) + opcode histogram (source page).
usage: python tools/ncu_summary.py report.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct"]
STALL = "smsp__average_warps_issue_stalled_"

rep = sys.argv[1]
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
out = {k: f"{d[k]} {u[k]}".strip() for k in KEYS if k in d}
_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
try:   # roofline "traffic": DRAM bytes of the captured launch (read + write)
    out["dram_bytes_per_launch"] = int(sum(float(d[k].replace(",", "")) * _SCALE[u[k]]
                                           for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")))
    out["report"] = rep
except (KeyError, ValueError):
    pass
st = {k[len(STALL):].replace("_per_issue_active.ratio", ""): float(d[k]) for k in hdr
      if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")}
out["stalls_per_issue"] = dict(sorted(((k, round(v, 3)) for k, v in st.items() if v > 0.01), key=lambda x: -x[1]))
src = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                              stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
iS, iE = h.index("Source"), h.index("Instructions Executed")
from collections import Counter
ex = Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iE or not r[iS].strip():
        continue
    toks = r[iS].split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    key = op if op.startswith(("VI", "LD", "ST")) else op.split(".")[0]
    n = float(r[iE] or 0)
    ex[key] += n
    tot += n
out["warp_instructions"] = tot
out["opcode_share_pct"] = {k: round(100 * v / tot, 2) for k, v in ex.most_common(20)}
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
