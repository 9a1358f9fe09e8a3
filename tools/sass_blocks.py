"""Hot SASS basic blocks (equal execution count runs) of one ncu report.
usage: python tools/sass_blocks.py rep.ncu-rep [N] [x: print the SASS]"""
import csv,subprocess,sys
out=subprocess.run(['ncu','-i',sys.argv[1],'--page','source','--print-source','sass','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))[2:]
tot=sum(int(r[5]) for r in rows)
blocks=[]
for r in rows:
    n=int(r[5])
    if blocks and blocks[-1][1]==n: blocks[-1][2].append(r[1].strip())
    else: blocks.append([r[0][-5:],n,[r[1].strip()]])
print("total", tot)
for b in sorted(blocks,key=lambda b:-b[1]*len(b[2]))[:int(sys.argv[2]) if len(sys.argv)>2 else 12]:
    print(f"{b[0]} n={b[1]:>10} len={len(b[2]):3d} share={b[1]*len(b[2])/tot*100:5.1f}%")
    if len(sys.argv)>3: print("    "+"\n    ".join(b[2]))
