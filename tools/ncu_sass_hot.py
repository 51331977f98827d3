"""Per-SASS-instruction execution counts and stall samples of the first kernel in an ncu report."""
import csv
import io
import subprocess
import sys
from collections import Counter

path = sys.argv[1]
kid = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", path, "--page", "source", "--csv"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
blk = blocks[1 if kid is None else int(kid) + 1]
lines = blk.split("\n", 1)[1]
rows = list(csv.DictReader(io.StringIO(lines)))
tot = sum(int(r["Instructions Executed"] or 0) for r in rows)
samp = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print("total warp instructions", tot, "samples", samp)
op = Counter()
stall = Counter()
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    o = r["Source"].split()
    o = [t for t in o if not t.startswith("@")]
    op[o[0].split(".")[0] if o else "?"] += n
    for k, v in r.items():
        if k and k.startswith("stall_") and "Not Issued" not in k and v:
            stall[k] += int(v)
print("opcode mix (warp instr):")
for k, v in op.most_common(25):
    print(f"  {k:12s} {v:12d} {100*v/tot:5.1f}%")
print("stall reasons (samples):")
for k, v in stall.most_common(10):
    print(f"  {k:28s} {v:8d} {100*v/max(samp,1):5.1f}%")
top = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:25]
print("hottest instructions:")
for r in top:
    print(f"  {r['Warp Stall Sampling (All Samples)']:>6s} {r['Instructions Executed']:>10s}  {r['Source'].strip()[:80]}")
