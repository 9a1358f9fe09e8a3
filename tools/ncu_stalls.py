"""Top SASS instructions by warp-stall samples from an ncu report (source page).
usage: python tools/ncu_stalls.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                              stderr=subprocess.DEVNULL).decode()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
tot = {h: 0 for h in stall_cols}
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    s = {h: float(r[ix[h]] or 0) for h in stall_cols}
    for h in stall_cols:
        tot[h] += s[h]
    recs.append((sum(s.values()), r[ix["Address"]], r[ix["Source"]], s))
T = sum(tot.values())
print("total samples", T)
print({k[6:]: round(100 * v / T, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
recs.sort(key=lambda x: -x[0])
for tot_s, addr, src, s in recs[:n]:
    top = sorted(((k[6:], v) for k, v in s.items() if v), key=lambda x: -x[1])[:3]
    print(f"{addr:>8} {100 * tot_s / T:5.2f}%  {src[:60]:60s} {top}")
