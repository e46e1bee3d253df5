"""Stall-reason samples per opcode of one kernel in an .ncu-rep (SASS source page).

    python tools/ncu_stall_by_op.py gpurun_out/prof.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
isrc = hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tab = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in body:
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    for h in reasons:
        v = int(r[hdr.index(h)] or 0)
        tab[op][h] += v
        tot[h] += v
T = sum(tot.values())
print("all:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tot.most_common(10)))
for op in sorted(tab, key=lambda o: -sum(tab[o].values()))[:8]:
    s = sum(tab[op].values())
    print(f"{op:8s} {100 * s / T:5.1f}%:", ", ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in tab[op].most_common(5)))
