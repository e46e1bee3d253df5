"""Per-instruction stall samples of one kernel in an .ncu-rep (SASS source page): the hottest
instructions and the samples per opcode and per stall reason.

    python tools/ncu_sass_hot.py gpurun_out/prof.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") or "Stall" in h and h not in hdr[isamp:isamp + 2]]
tot = sum(int(r[isamp] or 0) for r in body)
print(f"total samples {tot}, instructions {len(body)}")
by_op = collections.Counter()
for r in body:
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    by_op[op.split(".")[0]] += int(r[isamp] or 0)
for op, n in by_op.most_common(15):
    print(f"  {op:12s} {n:8d} {100 * n / tot:5.1f}%")
print("hottest:")
for r in sorted(body, key=lambda r: -int(r[isamp] or 0))[:top]:
    print(f"  {r[ia][-5:]} {int(r[isamp]):7d} {r[isrc].strip()[:90]}")
