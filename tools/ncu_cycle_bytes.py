"""B_meas of SURVEY §8(d): DRAM bytes of one cycle + norm, every kernel, from two ncu metric lists
of tools/prof_solve.py CFG with 1 and 2 cycles (host loop; the difference is one pipelined cycle:
the tail of cycle k + the head of cycle k+1 with its norm):
    python tools/ncu_cycle_bytes.py CFG run1.csv run2.csv   -> profiles/ncu_cycle_bytes.json[CFG]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9,
        "second": 1.0}


def totals(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hi]
    mn, mu, mv = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    b = t = 0.0
    n = 0
    for r in rows[hi + 1:]:
        if len(r) <= mv:
            continue
        v = float(r[mv].replace(",", "")) * UNIT.get(r[mu], 1.0)
        if r[mn].startswith("dram__bytes"):
            b += v
        elif r[mn] == "gpu__time_duration.sum":
            t += v
            n += 1
    return b, t, n


def main(cfg, p1, p2):
    b1, t1, n1 = totals(p1)
    b2, t2, n2 = totals(p2)
    rec = {"bytes": b2 - b1, "kernels": n2 - n1, "serialised_kernel_seconds": t2 - t1,
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum, "
                     f"tools/prof_solve.py {cfg} 2 minus 1 cycles ({os.path.basename(p2)}, {os.path.basename(p1)})"}
    p = os.path.join(ROOT, "profiles", "ncu_cycle_bytes.json")
    data = json.load(open(p)) if os.path.exists(p) else {}
    data[cfg] = rec
    json.dump(data, open(p, "w"), indent=1)
    print(cfg, rec)


if __name__ == "__main__":
    main(*sys.argv[1:4])
