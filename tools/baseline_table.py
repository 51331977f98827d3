"""Regenerate BASELINE.md §4's table (and the oracle paragraph) from profiles/r1e_bench/*.json
(the bench_all.sh lines): python tools/baseline_table.py [profiles subdir, default r1f_bench]"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "profiles", sys.argv[1] if len(sys.argv) > 1 else "r1f_bench")


def L(c):
    d = None
    for line in open(os.path.join(B, f"{c}.json")):
        line = line.strip()
        if line.startswith("{"):
            d = json.loads(line)
    return d


ROWS = [
    ("C3-f64", "**C3** 513³ RBGS V(2,2) FP64 (bench line)", "RBGS sweep L0", "—", True),
    ("C3-f32", "C3 513³ FP32", "RBGS sweep L0", "—", False),
    ("C5", "C5 1025³ RBGS FP64", "RBGS sweep L0", "—", False),
    ("C2", "C2 129³ RBGS FP64", None, "—", False),
    ("C4", "C4 8193² Jacobi V(3,3) FP32 (2D warp-marching, 3 sweeps per pass, level 0 two HBM passes per cycle)",
     "head: norm + 3 Jacobi sweeps + residual/restriction L0 (issue-bound)", "2D 4095² Jacobi FP32: 60 ms", False),
    ("C1", "C1 65² Jacobi V(2,2) FP64 (the whole solve in one launch)", None, "—", False),
    ("C2-lex", "C2-lex 129³ lexicographic GS V(2,2) FP64 (one launch per hyperplane)", None, "—", False),
    ("CD2-f32", "CD2 complex diffusion 4096² cells, Jacobi FAS V(2,2), complex FP32", "CD Jacobi L0 (warp-marching)",
     "**275 ms** generated (P:558), 37 ms hand-tuned (P:581)", True),
    ("CD2-gs-f32", "CD2 … RBGS, complex FP32", "CD RBGS colour L0", "2D GS FP32: 457 ms (P:560)", False),
    ("CD2-f64", "CD2 … Jacobi, complex FP64", "CD Jacobi L0 (warp-marching)", "2D Jacobi FP64: 385 ms (P:558)", False),
    ("CD3-f32", "CD3 complex diffusion 256³ cells, Jacobi, complex FP32", "CD Jacobi L0 (plane-marching, issue-bound)",
     "3D Jacobi FP32: 224 ms (P:562)", False),
    ("CD3-gs-f32", "CD3 … RBGS, complex FP32", "CD RBGS colour L0", "3D GS FP32: 374 ms (P:564)", False),
]


def fmt(x):
    return re.sub(r"e\+0?(\d)", r"e\1", f"{x:.2e}")


def main():
    out = []
    for c, name, dom, paper, bold in ROWS:
        d = L(c)
        ms, v, r = d["ms_per_step"], d["value"], d["roofline"]
        b = (lambda x: f"**{x}**") if bold else (lambda x: x)
        msf = f"{ms:.3f}" if ms < 1 else f"{ms:.2f}" if ms < 10 else f"{ms:.1f}"
        if dom is None:
            domc = ("(latency-bound: %d launches per cycle)" % round(d["gpu_launches_per_step"]) if c == "C2-lex" else
                    "(L2-resident, latency-bound; L2 traffic: `profiles/r1e_C2_l2_traffic.txt`)" if c == "C2" else
                    "(latency-bound)")
            bw = "—"
        else:
            domc, bw = dom, f"{r['achieved']:.0f} GB/s ({b(format(r['frac'], '.3f'))})"
        out.append(f"| {name} | {b(msf)} | {b(fmt(v))} | {domc} | {bw} | {fmt(d['e2e']['value'])} | {paper} |")
        nk = os.path.join(B, "C4-nokfuse.json")
        if c == "C4" and os.path.exists(nk):
            k = json.loads(open(nk).read().strip().splitlines()[-1])
            kr = k["roofline"]
            out.append(f"| C4 one sweep per pass (`bench.py --no-kfuse`, MG_FLAG_NO_KFUSE) | {k['ms_per_step']:.2f} | "
                       f"{fmt(k['value'])} | Jacobi L0 | {kr['achieved']:.0f} GB/s ({kr['frac']:.3f}) | — | — |")
    p = os.path.join(ROOT, "BASELINE.md")
    s = open(p).read()
    a = s.index("| Config | ms / step | unknowns/s |")
    a = s.index("\n", s.index("|---|", a)) + 1
    s = s[:a] + "\n".join(out) + s[s.index("\n\n", a):]
    c3, c5 = L("C3-f64"), L("C5")
    ref = json.loads(open(os.path.join(B, "reference_C3-f64.json")).read().strip().splitlines()[-1])
    # the clocks sentence: configs whose timed region ran below the max clock, and throttle flags
    low, flagged = [], []
    for c, *_ in ROWS:
        try:
            d = L(c)
        except FileNotFoundError:
            continue
        ck = d.get("clocks", {})
        if ck.get("sm_mhz") and ck.get("sm_max_mhz") and ck["sm_mhz"] < ck["sm_max_mhz"]:
            low.append(f"{c} ({ck['sm_mhz']} MHz)")
        if ck.get("reasons"):
            flagged.append(f"{c} ({', '.join('`%s`' % r for r in ck['reasons'])})")
    sent = ("SM clock median at its maximum in every timed region" if not low else
            "SM clock median at its maximum in every timed region except " + ", ".join(low))
    if flagged:
        sent += "; throttle reasons sampled during " + ", ".join(flagged)
    a2 = s.index("SM clock ")
    b2 = s.index("\n", s.index(").", a2))  # end of the sentence's line
    s = s[:a2] + sent + " (`clocks` in each bench line; `sw_power_cap` moves a run by a few %)." + s[b2:]
    s = re.sub(r"CPU oracle \(plain C, the `--impl reference` arm\): [0-9.]+ s per 513³ cycle \+ norm on 16 threads\n"
               r"= [0-9.e]+ unknowns/s",
               f"CPU oracle (plain C, the `--impl reference` arm): {ref['ms_per_step'] / 1000:.2f} s per 513³ cycle + "
               f"norm on 16 threads\n= {fmt(ref['value'])} unknowns/s", s)
    s = re.sub(r"The C3 FP64 GPU step is [0-9]+x the Poisson oracle \(e2e with host buffers: [0-9]+x\)",
               f"The C3 FP64 GPU step is {c3['value'] / ref['value']:.0f}x the Poisson oracle (e2e with host buffers: "
               f"{c3['e2e']['value'] / ref['value']:.0f}x)", s)
    s = re.sub(r"it moves [0-9.]+ TB/s averaged over the\nwhole step \([0-9]+% of the measured copy bandwidth\)",
               f"it moves {c3['model_GBps'] / 1000:.1f} TB/s averaged over the\nwhole step "
               f"({c3['model_GBps'] / 6453.1 * 100:.0f}% of the measured copy bandwidth)", s)
    open(p, "w").write(s)
    print("\n".join(out))


if __name__ == "__main__":
    main()
