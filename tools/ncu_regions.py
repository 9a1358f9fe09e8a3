"""Attribute ncu warp-stall samples of decode_kernel to source statements of the
hot functions (siso_split / build_chunk / run_task_fast / decode_kernel), using
the inline chains of a local nvdisasm -gi of the same build.
usage: python tools/ncu_regions.py report.ncu-rep [N]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1905_01141_b200 import build as B  # noqa: E402

SRC = os.path.join(B.CSRC, "crn_decode.cu")
KEYS = ["build_chunk", "siso_split", "run_task_fast", "decode_kernel", "run_task_generic", "siso_generic",
        "decide", "finish_iteration"]


def func_ranges():
    lines = open(SRC).read().split("\n")
    starts = []
    for i, l in enumerate(lines, 1):
        m = re.match(r"^(?:__device__|__global__|template).*?\b(\w+)\(", l)
        if m:
            starts.append((i, m.group(1)))
        elif re.match(r"^(\w+)\(const crn_cb_desc", l):
            starts.append((i, "decode_kernel"))
    rng = []
    for k, (s, name) in enumerate(starts):
        e = starts[k + 1][0] - 1 if k + 1 < len(starts) else len(lines)
        rng.append((s, e, name))
    return rng, lines


def local_chains():
    cub = "/tmp/crn_decode_regions.cubin"
    defs = [f"-D{d}" for d in os.environ.get("CRN_DEFINES", "").split()]   # the variant's -D flags
    subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, *defs, "-cubin", "-o", cub, SRC])
    out = subprocess.check_output(["nvdisasm", "-gi", "-fun", "", cub], stderr=subprocess.DEVNULL).decode() \
        if False else subprocess.check_output(["nvdisasm", "-gi", cub]).decode()
    chains, cur, in_kernel, pending = {}, [], False, []
    for l in out.split("\n"):
        if re.match(r"\s*\.text\.", l) or "Function :" in l:
            in_kernel = os.environ.get("CRN_KERNEL", "decode_kernelILb0ELb0ELi0E") in l
        m = re.search(r'//## File ".*?crn_decode.cu", line (\d+)(?: inlined at ".*?", line (\d+))?', l)
        if m:
            pending.append(int(m.group(1)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m and in_kernel:
            if pending:
                cur = pending
                pending = []
            chains[int(m.group(1), 16)] = cur
    return chains


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                  stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    recs = [r for r in rows[2:] if len(r) >= len(hdr)]
    base = int(recs[0][ix["Address"]], 16)
    chains = local_chains()
    rng, lines = func_ranges()

    def region(chain):
        for ln in chain:
            for s, e, name in rng:
                if s <= ln <= e and name in KEYS:
                    return f"{name}:{ln}"
        return f"?:{chain[0] if chain else -1}"

    agg = collections.defaultdict(lambda: collections.Counter())
    tot = 0.0
    for r in recs:
        off = int(r[ix["Address"]], 16) - base
        reg = region(chains.get(off, []))
        for h in stall_cols:
            v = float(r[ix[h]] or 0)
            agg[reg][h[6:]] += v
            tot += v
        agg[reg]["_inst"] += float(r[ix["Instructions Executed"]] or 0)
    items = sorted(agg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_inst"))
    print(f"total samples {tot:.0f}; mismatched-address check: {sum(1 for r in recs if int(r[ix['Address']], 16) - base not in chains)} of {len(recs)}")
    for reg, c in items[:n]:
        s = sum(v for k, v in c.items() if k != "_inst")
        top = sorted(((k, v) for k, v in c.items() if k != "_inst" and v), key=lambda x: -x[1])[:4]
        ln = int(reg.split(":")[1])
        src = lines[ln - 1].strip()[:55] if ln > 0 else ""
        print(f"{100 * s / tot:5.1f}% {reg:24s} {src:55s} " + " ".join(f"{k}={100 * v / s:.0f}%" for k, v in top))


if __name__ == "__main__":
    main()
