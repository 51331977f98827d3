"""Summarise an ncu report: key metrics per captured kernel (reads `ncu -i --page details --csv`)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "No Eligible", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "Executed Instructions", "Dynamic Shared Memory Per Block", "Block Limit Shared Mem",
        "Block Limit Registers", "Elapsed Cycles"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(out)))
    seen = {}
    for r in rows:
        kid = r["ID"]
        if kid not in seen:
            seen[kid] = True
            print(f"== [{kid}] {r['Kernel Name'][:90]} grid={r['Grid Size']} block={r['Block Size']}")
        if r["Metric Name"] in KEYS and r["Metric Value"]:
            print(f"   {r['Metric Name']:40s} {r['Metric Unit']:12s} {r['Metric Value']}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hdr, units = rr[0], rr[1]
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum"]
        idx = [hdr.index(w) for w in want if w in hdr]
        for row in rr[2:]:
            print("   raw:", row[hdr.index("Kernel Name")][:40] if "Kernel Name" in hdr else "",
                  {hdr[i]: (row[i], units[i]) for i in idx})


if __name__ == "__main__":
    main(sys.argv[1])
