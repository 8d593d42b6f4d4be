"""Basic-block summary of an ncu --set full capture's SASS source page:
executed instructions, stall samples and opcode mix per block (runs of equal
execution count), largest first.  usage: k6_blocks.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
src = hdr.index("Source")
pi = hdr.index("Avg. Predicated-On Threads Executed")
runs, cur = [], None
for i, r in enumerate(data):
    e = int(r[ei])
    toks = r[src].split()
    op = (toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else ""))
    if cur and cur["e"] == e:
        cur["n"] += 1
        cur["s"] += int(r[si])
        cur["ops"].append(op)
        cur["th"].append(float(r[pi] or 0))
    else:
        cur = {"e": e, "n": 1, "s": int(r[si]), "start": i, "ops": [op], "th": [float(r[pi] or 0)]}
        runs.append(cur)
tot = sum(int(r[si]) for r in data)
totI = sum(int(r[ei]) for r in data)
print(f"total warp instructions {totI}, stall samples {tot}")
for c in sorted(runs, key=lambda c: -c["e"] * c["n"])[:top]:
    oc = Counter(o.split(".")[0] for o in c["ops"])
    print(f"[{c['start']}+{c['n']}] exec {c['e']} instr {100 * c['e'] * c['n'] / totI:.1f}% "
          f"samples {100 * c['s'] / tot:.1f}% thr {sum(c['th']) / len(c['th']):.1f}",
          dict(oc.most_common(8)))
