"""Opcode mix, stall reasons and hottest SASS lines of ONE kernel launch of an ncu report:
    python tools/ncu_opmix.py REPORT KERNEL_REGEX SKIP
(the SKIP-th launch matching KERNEL_REGEX, as ncu's --launch-skip counts them)."""
import csv
import io
import subprocess
import sys
from collections import Counter

path, rx, skip = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{rx}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
lines = out.splitlines()
name = lines[0]
hdr = next(l for l in lines if l.startswith('"Address"'))
body = "\n".join([hdr] + [l for l in lines if l.startswith('"0x')])
rows, seen = [], set()
for r in csv.DictReader(io.StringIO(body)):  # the export may list a function's SASS twice
    if r["Address"] not in seen:
        seen.add(r["Address"])
        rows.append(r)
tot = sum(int(r["Instructions Executed"] or 0) for r in rows)
samp = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(name[:200])
print("total warp instructions", tot, "stall samples", samp)
op, stall = Counter(), Counter()
for r in rows:
    o = [t for t in r["Source"].split() if not t.startswith("@")]
    op[o[0].split(".")[0] if o else "?"] += int(r["Instructions Executed"] or 0)
    for k, v in r.items():
        if k and k.startswith("stall_") and "Not Issued" not in k and v:
            stall[k] += int(v)
print("opcode mix (warp instructions):")
for k, v in op.most_common(24):
    print(f"  {k:14s} {v:12d} {100 * v / max(tot, 1):5.1f}%")
print("stall reasons (samples):")
for k, v in stall.most_common(10):
    print(f"  {k:30s} {v:8d} {100 * v / max(sum(stall.values()), 1):5.1f}%")
print("hottest instructions (samples, executions, SASS):")
for r in sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:12]:
    print(f"  {r['Warp Stall Sampling (All Samples)']:>6s} {r['Instructions Executed']:>10s}  {r['Source'].strip()[:90]}")
