"""profiles/ncu_traffic.json entries from an ncu --set full summary of the level-0 3D kernels
(tools/round.sh full:CFG): DRAM bytes (read + write) per launch of each bench kernel name.

    python tools/ncu_traffic.py CFG profiles/<round>/CFG_full_summary.txt

Level 0 = the largest grid of a kernel family in the capture; bench names: k_sweep3d_rows NM 0 / 3
-> rbgs_fused, NM 1 / 2 -> sweep+norm, CORR -> prolong+sweep, k_resid_restrict3d_rows ->
resid_restrict, k_prolong3d_flat -> prolong_correct (kernels_pm.cu template order
<T, MODE, ZERO, NM, RPT, CORR>)."""
import ast
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench_name(sig):
    m = re.search(r"k_sweep3d_rows<\w+, (\d), (\d), (\d), \d, (\d)>", sig)
    if m:
        mode, zero, nm, corr = map(int, m.groups())
        if corr:
            return "prolong+sweep"
        if mode == 2:
            return "norm_partial"
        if zero:
            return None
        return "sweep+norm" if nm in (1, 2) else "rbgs_fused" if mode == 1 else "jacobi_pm"
    if "k_resid_restrict3d_rows" in sig:
        return "resid_restrict"
    if "k_prolong3d_flat" in sig:
        return "prolong_correct"
    return None


def main(cfg, path):
    heads, raws = [], []
    for line in open(path):
        if line.startswith("== ["):
            g = re.search(r"grid=\((\d+)", line)
            heads.append((line, int(g.group(1)) if g else 0))
        elif line.strip().startswith("raw:"):
            d = ast.literal_eval(line[line.index("{"):].strip())
            unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
            b = sum(float(d[k][0]) * unit[d[k][1]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            raws.append(b)
    biggest = {}
    for (line, grid), b in zip(heads, raws):
        name = bench_name(line)
        if name is None:
            continue
        fam = "rr" if name == "resid_restrict" else "prolong" if name == "prolong_correct" else "sweep"
        biggest[fam] = max(biggest.get(fam, 0), grid)
    out = {}
    for (line, grid), b in zip(heads, raws):
        name = bench_name(line)
        if name is None:
            continue
        fam = "rr" if name == "resid_restrict" else "prolong" if name == "prolong_correct" else "sweep"
        if grid == biggest[fam]:
            out.setdefault(f"{cfg}:{name}@L0", []).append(b)
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(p)) if os.path.exists(p) else {}
    for k, v in out.items():
        data[k] = sum(v) / len(v)
        print(k, "%.4e" % data[k], f"({len(v)} launches)")
    src = data.get("_source", "")
    note = f"{cfg}: {os.path.relpath(path, ROOT)}"
    if note not in src:
        data["_source"] = (src + "; " if src else "") + note
    json.dump(data, open(p, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
