"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    if name.startswith("at::") or "elementwise" in name:
        continue
    tot[name] += float(r["Metric Value"]) / 1e3
    cnt[name] += 1
all_us = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k]/cnt[k]:9.2f} {100*tot[k]/all_us:5.1f}%")
print(f"(ncu per-launch times are cold-cache and serialised: compare shares, not absolutes)")
