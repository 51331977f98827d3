#!/usr/bin/env python
"""Benchmark of the B200 V-cycle (the driver's contract).

One STEP = one pass of the whole hot path over the workload: one V(2,2)-cycle
(pre-smoothing, residual, full-weighting restriction, coarse solve,
prolongation + correction, post-smoothing on every level) plus the residual
norm that the paper's driver loop evaluates after every cycle.

Workload (N=1): BASELINE.json configs[2], the north_star's headline case:
3D Poisson 7-point, 513^3 nodes, red-black Gauss-Seidel V(2,2), FP64,
W1 = the paper's f = 0 / random initial guess, seed 42, generated
on the device by the same SplitMix64 counter generator the oracle side uses.
Each array is 1.08 GB, far larger than the 126 MB L2, so no L2 flush is
needed between steps.

Metric: unknowns/s = 511^3 interior unknowns per step / step time (all ranks'
unknowns / max-over-ranks time for N>1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mg|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dim, nodes, smoother, nu1, nu2, dtype, levels, omega)
    "C3-f64": (3, 513, "rbgs", 2, 2, "f64", 0, 1.0),
    "C3-f32": (3, 513, "rbgs", 2, 2, "f32", 0, 1.0),
    "C2": (3, 129, "rbgs", 2, 2, "f64", 0, 1.0),
    "C4": (2, 8193, "jacobi", 3, 3, "f32", 0, 0.8),
    "C5": (3, 1025, "rbgs", 2, 2, "f64", 0, 1.0),
    "C1": (2, 65, "jacobi", 2, 2, "f64", 5, 0.8),
    # smoother variant: lexicographic omega-GS, one launch per hyperplane
    "C2-lex": (3, 129, "gs_lex", 2, 2, "f64", 0, 1.0),
}
WORKLOAD_DESC = {
    "C3-f64": "3D Poisson 7-point 513^3 nodes, RBGS V(2,2), FP64, W1 (f=0, u0~U[0,1) seed 42)",
    "C3-f32": "3D Poisson 7-point 513^3 nodes, RBGS V(2,2), FP32, W1 (f=0, u0~U[0,1) seed 42)",
    "C2": "3D Poisson 7-point 129^3 nodes, RBGS V(2,2), FP64, W1 seed 42",
    "C4": "2D Poisson 5-point 8193^2 nodes, Jacobi(0.8) V(3,3), FP32, W1 seed 42",
    "C5": "3D Poisson 7-point 1025^3 nodes, RBGS V(2,2), FP64, W1 seed 42",
    "C1": "2D Poisson 5-point 65^2 nodes, 5 levels, Jacobi(0.8) V(2,2), FP64, W1 seed 42",
    "C2-lex": "3D Poisson 7-point 129^3 nodes, lexicographic GS V(2,2), FP64, W1 seed 42",
}
# complex diffusion, FAS on cell-centred grids (the paper's Table 2
# "Complex Diff." rows: N = 4096^2 cells in 2D, 256^3 in 3D)
# name: (dim, cells, smoother, nu1, nu2, dtype, omega)
CD_CONFIGS = {
    "CD2-f32": (2, 4096, "jacobi", 2, 2, "f32", 0.8),
    "CD2-gs-f32": (2, 4096, "rbgs", 2, 2, "f32", 1.0),
    "CD2-f64": (2, 4096, "jacobi", 2, 2, "f64", 0.8),
    "CD2-gs-f64": (2, 4096, "rbgs", 2, 2, "f64", 1.0),
    "CD3-f32": (3, 256, "jacobi", 2, 2, "f32", 0.8),
    "CD3-gs-f32": (3, 256, "rbgs", 2, 2, "f32", 1.0),
}
for _k, (_d, _n, _sm, _a, _b, _dt, _om) in CD_CONFIGS.items():
    WORKLOAD_DESC[_k] = (f"{_d}D complex diffusion (one implicit-Euler step, tau=0.1, theta=pi/30, k=2), "
                         f"{_n}^{_d} cells, Neumann, FAS V({_a},{_b}) "
                         f"{'Jacobi(0.8)' if _sm == 'jacobi' else 'RBGS'}, complex {_dt.upper()}, "
                         f"W5 (noise image u^n ~ U[0,1) seed 42, f = u^n)")
METRIC = "V(2,2)-cycle unknowns/s (one cycle + residual norm per step)"


def is_cd(name):
    return name in CD_CONFIGS


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def interior_unknowns(dim, nodes):
    return (nodes - 2) ** dim


def model_bytes_per_step(S, esz):
    """B_alg of SURVEY §8(a) for this hierarchy (fused schedule model) + the norm pass."""
    total = 0.0
    nu = S.cfg.nu1 + S.cfg.nu2
    for l in range(S.levels - 1):
        n = 1
        for c in S.level_cells(l):
            n *= c + 1
        total += n * (3 * nu + 2 * 2.0 ** -S.dim) * esz
    n0 = 1
    for c in S.level_cells(0):
        n0 *= c + 1
    return total + 2 * n0 * esz


def unfused_bytes_per_step(dim, nodes, levels, smoother, nu1, nu2, esz):
    """B_unfused of SURVEY §8(a): Alg. 1 op by op (the oracle's schedule; two-pass RBGS, w = 6) + the
    norm pass, for the full-size workload."""
    w = 6 if smoother == "rbgs" else 3
    q = 2.0 ** -dim
    total = 0.0
    for l in range(levels - 1):
        total += ((nodes - 1) // 2 ** l + 1) ** dim * (w * (nu1 + nu2) + 3 + (1 + q) + q + (2 + q)) * esz
    return total + 2 * nodes ** dim * esz


def ncu_cycle_bytes(config):
    """Measured DRAM bytes of one cycle + norm (all kernels, ncu; profiles/ncu_cycle_bytes.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_cycle_bytes.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(config)


def l2_note(array_bytes):
    if array_bytes > 126e6:
        return f"inputs larger than L2 ({array_bytes / 1e9:.3f} GB per array), no flush needed"
    return (f"inputs L2-resident ({array_bytes / 1e6:.1f} MB per array < 126 MB L2): no flush; this config "
            "measures the L2-resident regime")


def cd_model_bytes_per_step(S, esz):
    """Complex diffusion, op-by-op FAS schedule (kernels_cd.cu), complex words s = 2 esz per cell:
    per level l < L-1: g field 2, Jacobi sweep 4 (read u, g, f; write u) x (nu1+nu2) [RBGS: 2 colour
    passes of 2.5 each], u^ = R u 1 + 2/2^d, coarse g 2/2^d, FAS rhs 3 + 3/2^d, prolongation 2 + 2/2^d;
    coarsest: g 2 + ncoarse sweeps; + the norm pass (2 words of level 0)."""
    s = 2 * esz
    sweep = 4.0 if S.cfg.smoother == 0 else 5.0
    nu = S.cfg.nu1 + S.cfg.nu2
    q = 2.0 ** -S.dim
    total = 0.0
    for l in range(S.levels):
        n = 1
        for c in S.level_cells(l):
            n *= c
        if l < S.levels - 1:
            total += n * s * (2 + sweep * nu + (1 + 2 * q) + 2 * q + (3 + 3 * q) + (2 + 2 * q))
        else:
            total += n * s * (2 + sweep * S.cfg.ncoarse)
    n0 = 1
    for c in S.level_cells(0):
        n0 *= c
    return total + 2 * n0 * s


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index):
        self.ok = False
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs"), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write bytes)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` in bench config `config` from one committed ncu --set full
    capture (profiles/ncu_traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{config}:{kernel}")


# --------------------------------------------------------------------- oracle (CPU) legs
def _host_threads_for_oracle():
    """torchrun exports OMP_NUM_THREADS=1 to every rank; the oracle leg runs on rank 0 alone and
    is meant to use the host's cores (as at N=1), so lift that default before the oracle's
    OpenMP runtime is first loaded (it reads the variable once, at load time)."""
    if os.environ.get("TORCHELASTIC_RUN_ID") is not None and os.environ.get("OMP_NUM_THREADS") == "1":
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)


def oracle_step_time(cfgname, max_seconds=30.0):
    """Time the CPU oracle, as it stands, on one V-cycle + norm of the workload.
    Returns (seconds per step, unknowns per step, sample description, threads)."""
    import numpy as np

    _host_threads_for_oracle()
    import oracle as orc
    from paper_1406_5369_b200 import workloads as wl
    if is_cd(cfgname):
        return cd_oracle_step_time(cfgname, max_seconds)
    dim, nodes, sm, nu1, nu2, dt, levels, omega = CONFIGS[cfgname]
    cells = (nodes - 1,) * dim
    # full size when it fits the budget, else the largest power-of-two grid that does
    npdt = np.float64 if dt == "f64" else np.float32
    # untimed warm-up on a small grid: the OpenMP runtime starts its thread pool on the first
    # parallel region (≈ 1 s on this host), which must not be charged to the timed cycle
    wc = orc.Config(dim=dim, cells=(8,) * dim)
    Ow = orc.Oracle(wc, npdt)
    uw, fw = wl.workload("W1", dim, (8,) * dim, seed=1, dtype=npdt)
    Ow.vcycle_inplace(uw, fw)
    for n in [nodes - 1, (nodes - 1) // 2, (nodes - 1) // 4]:
        cells = (n,) * dim
        c = orc.Config(dim=dim, cells=cells, levels=levels if n == nodes - 1 else 0,
                       smoother={"rbgs": orc.RBGS, "gs_lex": orc.GS_LEX}.get(sm, orc.JACOBI), omega=omega, nu1=nu1, nu2=nu2)
        O = orc.Oracle(c, npdt)
        u, f = wl.workload("W1", dim, cells, seed=42, dtype=npdt)
        t0 = time.perf_counter()
        O.vcycle_inplace(u, f)
        O.norm(0, u, f)
        t = time.perf_counter() - t0
        if t <= max_seconds or n == (nodes - 1) // 4:
            desc = (f"one V({nu1},{nu2})-cycle + residual norm of the CPU oracle (plain C, -O2 "
                    f"-ffp-contract=off, OpenMP over planes) on {'x'.join(str(c + 1) for c in cells)} nodes, W1 seed 42"
                    + ("" if n == nodes - 1 else f" (reduced from {nodes}^{dim} to fit the CPU time budget)"))
            return t, interior_unknowns(dim, n + 1), desc, orc.num_threads(npdt), (O, u, f)
    raise RuntimeError("unreachable")


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_leg(cfgname):
    """--cpu-baseline-leg: the oracle timed on one step, all host threads, then one thread
    (OMP_NUM_THREADS=1 in a grandchild: OpenMP reads it at load time); prints one JSON object."""
    import subprocess
    t, cunk, desc, threads, _ = oracle_step_time(cfgname, max_seconds=30.0)
    out = {"value": cunk / t, "unit": "unknowns/s", "cores": threads, "kind": "oracle", "sample": desc,
           "cpu_model": _cpu_model(), "host_threads": os.cpu_count()}
    if not is_cd(cfgname):  # the oracle's effective bandwidth over B_unfused (its schedule)
        dim, nodes, sm, nu1, nu2, dt, levels, omega = CONFIGS[cfgname]
        ns = int(round(cunk ** (1.0 / dim))) + 2
        lv = levels if ns == nodes else int(ns - 1).bit_length() - 1
        b = unfused_bytes_per_step(dim, ns, lv, sm, nu1, nu2, 8 if dt == "f64" else 4)
        out["unfused_bytes_per_step"] = b
        out["effective_GBps"] = b / t / 1e9
    if os.environ.get("MG_BENCH_ONE_THREAD") is None:
        env = dict(os.environ, OMP_NUM_THREADS="1", MG_BENCH_ONE_THREAD="1")
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-baseline-leg", "--config", cfgname],
                           env=env, capture_output=True, text=True, timeout=600)
        try:
            one = json.loads(r.stdout.strip().splitlines()[-1])
            out["one_thread"] = {"value": one["value"], "unit": "unknowns/s", "cores": one["cores"],
                                 "sample": one["sample"]}
        except Exception as e:  # reported, not fatal
            out["one_thread"] = {"error": f"{e}: {r.stderr[-300:]}"}
    print(json.dumps(out), flush=True)
    return 0


def cpu_baseline_subprocess(cfgname):
    import subprocess
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-baseline-leg", "--config", cfgname],
                       capture_output=True, text=True, timeout=1200)
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:
        return {"error": f"cpu baseline leg failed: {e}: {r.stderr[-300:]}"}


class _CdStepper:
    """Adapter so the reference arm can step the complex-diffusion oracle like the Poisson one."""

    def __init__(self, O):
        self.O = O

    def vcycle_inplace(self, u, f):
        u[...] = self.O.cycle(u, f)

    def norm(self, l, u, f):
        return self.O.norm(l, u, f)


def cd_oracle_step_time(cfgname, max_seconds):
    import numpy as np

    from oracle.cd import CDConfig, CDOracle, JACOBI, RBGS
    from paper_1406_5369_b200 import workloads as wl
    dim, n0, sm, nu1, nu2, dt, omega = CD_CONFIGS[cfgname]
    cdt = np.complex128 if dt == "f64" else np.complex64
    for n in [n0, n0 // 2, n0 // 4, n0 // 8]:
        cells = (n,) * dim
        O = CDOracle(CDConfig(dim=dim, cells=cells, smoother=RBGS if sm == "rbgs" else JACOBI, omega=omega,
                              nu1=nu1, nu2=nu2), cdt)
        u, f = wl.cd_workload(dim, cells, 42, cdt)
        t0 = time.perf_counter()
        u = O.cycle(u, f)
        O.norm(0, u, f)
        t = time.perf_counter() - t0
        if t <= max_seconds or n == n0 // 8:
            desc = (f"one FAS V({nu1},{nu2})-cycle + nonlinear residual norm of the CPU oracle (plain C, -O2 "
                    f"-ffp-contract=off, one thread) on {'x'.join(str(c) for c in cells)} cells, W5 seed 42"
                    + ("" if n == n0 else f" (reduced from {n0}^{dim} to fit the CPU time budget)"))
            return t, n ** dim, desc, 1, (_CdStepper(O), u, f)
    raise RuntimeError("unreachable")


def workload_levels(cfgname):
    """Levels of the full-size workload: explicit, else the paper's rule (DESIGN reading 2/20)."""
    if is_cd(cfgname):
        return int(CD_CONFIGS[cfgname][1]).bit_length() - 1
    levels, n = CONFIGS[cfgname][6], CONFIGS[cfgname][1]
    return levels or int(n - 1).bit_length() - 1


def workload_config(cfgname):
    """The `config` object of the JSON line: the workload only, identical in both arms."""
    levels = workload_levels(cfgname)
    if is_cd(cfgname):
        dim, n, *_ = CD_CONFIGS[cfgname]
        esz = 16 if CD_CONFIGS[cfgname][5] == "f64" else 8
        key, nodes = "grid_cells", n
        arr = n ** dim * esz
    else:
        dim, n, *_ = CONFIGS[cfgname]
        esz = 8 if CONFIGS[cfgname][5] == "f64" else 4
        key, nodes = "grid_nodes", n
        arr = n ** dim * esz
    return {"workload": WORKLOAD_DESC[cfgname], key: nodes, "dim": dim, "levels": levels, "l2": l2_note(arr)}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0  # the reference arm runs on rank 0 only
    t_first, unk, desc, threads, (O, u, f) = oracle_step_time(args.config, max_seconds=20.0)
    # warm-up steps beyond the first, then exactly K timed steps
    for _ in range(max(args.warmup - 1, 0)):
        O.vcycle_inplace(u, f)
        O.norm(0, u, f)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.vcycle_inplace(u, f)
        O.norm(0, u, f)
    dt = (time.perf_counter() - t0) / args.steps
    val = unk / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "unknowns/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": (("c" if is_cd(args.config) else "") + (CD_CONFIGS[args.config][5] if is_cd(args.config)
                                                          else CONFIGS[args.config][5])),
        "data": "synthetic",
        "config": workload_config(args.config),
        "parallelism": "cpu-oracle (OpenMP over planes)" if threads > 1 else "cpu-oracle (one thread)",
        "cpu_baseline": {"value": val, "unit": "unknowns/s", "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": val, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- GPU arm
def single_gpu_point(cfgname, dev, stream, steps=8, warmup=3):
    """Step time of `cfgname` on this GPU alone (device loop, the same step as the main line):
    the N = 1 point of the scaling workload, reported next to the N = 1 metric line."""
    import torch

    import paper_1406_5369_b200 as mgb
    dim, nodes, sm, nu1, nu2, dt, levels, omega = CONFIGS[cfgname]
    S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt, device=dev)
    u, f = S.empty(), S.empty()
    with torch.cuda.stream(stream):
        S.workload_fill(u, 42, stream=stream)
    torch.cuda.synchronize()
    S.solve(u, f, -1.0, warmup, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    k, _ = S.solve(u, f, -1.0, steps, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    S.close()
    return {"workload": WORKLOAD_DESC[cfgname], "steps": steps, "warmup": warmup, "ms_per_step": ms,
            "value": interior_unknowns(dim, nodes) / (ms * 1e-3), "unit": "unknowns/s",
            "note": "bench.py --gpus N > 1 defaults to this workload (z-slab decomposition of the same grid)"}


def run_mg(args):
    import torch

    import paper_1406_5369_b200 as mgb
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cd = is_cd(args.config)
    if cd:  # complex diffusion: `nodes` are cells, FAS with ncoarse sweeps on the coarsest level
        dim, nodes, sm, nu1, nu2, dt, omega = CD_CONFIGS[args.config]
        levels = 0
    else:
        dim, nodes, sm, nu1, nu2, dt, levels, omega = CONFIGS[args.config]
    esz = 8 if dt == "f64" else 4
    kw = dict(levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt, device=dev,
              flags=(mgb.FLAG_HOST_LOOP if args.host_loop else 0) | (mgb.FLAG_SEPARATE_PROLONG if args.separate_prolong else 0)
              | (mgb.FLAG_NO_KFUSE if args.no_kfuse else 0))
    if cd:
        kw.update(problem="complex_diffusion", coarse="sweeps")
    # mg_solve runs its loop on the device (one CUDA graph, conditional WHILE node) unless
    # --host-loop or the slab run spans several ranks (NCCL cannot run in a conditional body)
    slab = world > 1 and args.decomp == "slab" and not cd
    device_loop = not args.host_loop and not slab
    if slab:  # z-slab decomposition of ONE global grid over the ranks (strong scaling), NCCL halos
        S = mgb.distributed_solver(dim, nodes, **kw)
    else:     # N independent replicas (weak scaling)
        S = mgb.Solver(dim, nodes, **kw)
    stream = torch.cuda.Stream(device=dev)
    u = S.empty()
    f = S.empty()
    with torch.cuda.stream(stream):
        S.workload_fill(u, 42, stream=stream)
        if cd:  # W5: f = u^n = the initial iterate
            S.workload_fill(f, 42, stream=stream)
    torch.cuda.synchronize()
    unk = nodes ** dim if cd else interior_unknowns(dim, nodes)
    assert S.levels == workload_levels(args.config), (S.levels, workload_levels(args.config))

    # K steps = the library's driver loop mg_solve(rtol=0, max_cycles=K): K V-cycles, each
    # followed by the residual norm (pipelined into the next cycle's first sweep; the
    # call also computes the initial norm: K+1 norms, counted against us)
    def steps(k):
        # rtol < 0: exactly k cycles — W1 (f = 0) decays ~10x per cycle and would reach an
        # exact zero (an rtol = 0 stop) after a few hundred cycles
        cycles, hist = S.solve(u, f, -1.0, k, stream=stream)
        assert cycles == k
        return hist

    r0 = S.residual_norm(u, f, stream=stream)
    unk_total = unk if slab else unk * world  # unknowns processed per step by all ranks
    steps(args.warmup)
    sampler = ClockSampler(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    hist = steps(args.steps)
    ev1.record(stream)
    rk = hist[-1]
    torch.cuda.synchronize()
    sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    # ---- per-kernel CUDA-event timing (separate instrumented pass, eager launches)
    S.profile_enable(True)
    nprof = max(3, min(args.steps, 10))
    steps(nprof)
    recs = S.profile_read()
    S.profile_enable(False)
    ours = [r for r in recs if not (r["name"].startswith("memset") or r["name"].startswith("nccl"))]
    launches = sum(r["count"] for r in ours) / nprof  # our kernels per step (incl. the norm pipeline)
    if device_loop and not any(r["name"].startswith("coarse_tail_solve") for r in ours):
        # the loop's check kernel (k_loop_check) per cycle (the profile pass is eager); a
        # whole-cycle tail grid runs the whole solve in one launch
        launches += 1
    tot = sum(r["ms"] for r in recs)
    dom = max(recs, key=lambda r: r["ms"])  # the dominant kernel of the step
    dom_avg_ms = dom["ms"] / dom["count"]
    peak, peak_src = measured_peaks()
    achieved = dom["bytes"] / (dom_avg_ms * 1e-3) / 1e9
    roofline = {
        "bound": "hbm", "kernel": dom["name"], "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": ncu_traffic(args.config, dom["name"]), "peak_source": peak_src,
        "frac_of_nominal_8TBps": achieved / 8000.0,
        "alg_bytes_per_launch": dom["bytes"], "avg_launch_ms": dom_avg_ms,
        "share_of_step": dom["ms"] / tot if tot else None,
        "timing": ("per-kernel CUDA events on the solver stream, separate instrumented eager pass of the same "
                   "kernels (the timed region replays a CUDA graph)"),
    }
    array_bytes = S.shape[0] * S.shape[1] * S.shape[2] * esz * (2 if cd else 1)
    if array_bytes * 3 < 126e6:  # L2-resident sizes
        roofline["note"] = ("L2-resident grid (three arrays < 126 MB L2): the HBM fraction is not meaningful; "
                            "the step is bound by launch and barrier latency. L2 traffic per kernel "
                            "(lts__t_bytes, ncu): profiles/r1e_C2_l2_traffic.txt")
    B = cd_model_bytes_per_step(S, esz) if cd else model_bytes_per_step(S, esz)
    breakdown = sorted(({"kernel": r["name"], "ms_per_step": r["ms"] / nprof, "launches_per_step": r["count"] / nprof,
                         "GBps": (r["bytes"] * r["count"] / (r["ms"] * 1e-3) / 1e9) if r["ms"] else None}
                        for r in recs), key=lambda d: -d["ms_per_step"])[:8]

    # ---- end to end through the C ABI with host buffers: every step is one problem whose
    # inputs u, f are copied from pinned host memory, cycled once + normed, and whose u is
    # copied back; mg_vcycle_host_batch pipelines H2D(k+1) / cycle(k) / D2H(k-1) over two
    # staging sets and two copy streams (PCIe is full duplex)
    e2e = None
    if not args.no_e2e:
        hu = torch.empty(S.shape, dtype=S.torch_dtype).pin_memory()
        hf = torch.empty(S.shape, dtype=S.torch_dtype).pin_memory()
        ho = torch.empty(S.shape, dtype=S.torch_dtype).pin_memory()
        hu.copy_(u.cpu())
        hf.copy_(f.cpu())
        S.vcycle_host_batch([hu] * 2, [ho] * 2, [hf] * 2, stream=stream)  # warm-up (allocates staging)
        ne = max(4, min(args.steps, 8))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        S.vcycle_host_batch([hu] * ne, [ho] * ne, [hf] * ne, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / ne
        nbytes = hu.numel() * hu.element_size()
        if world > 1:
            t = torch.tensor([ems], device=f"cuda:{dev}", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": unk_total / (ems * 1e-3), "unit": "unknowns/s", "ms_per_step": ems,
               "h2d_bytes_per_step": 2 * nbytes, "d2h_bytes_per_step": nbytes,
               "path": (f"mg_vcycle_host_batch over {ne} problems (pinned host u, f -> device, 1 cycle + norm, "
                        "u -> host; H2D / compute / D2H pipelined)")}

    # ---- for the rtol configs also the whole solve to 1e-10 (time and cycle count)
    solve = None
    if world == 1 and not cd and args.config in ("C3-f64", "C3-f32", "C2", "C5"):
        with torch.cuda.stream(stream):
            S.workload_fill(u, 42, stream=stream)
            f.zero_()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        kc, sh = S.solve(u, f, 1e-10, 40, stream=stream)
        s1.record(stream)
        torch.cuda.synchronize()
        solve = {"rtol": 1e-10, "cycles": kc, "ms": s0.elapsed_time(s1), "final_reduction": sh[-1] / sh[0],
                 "note": "mg_solve from the W1 start (device loop): initial norm + cycles until ||r|| <= 1e-10 ||r0||"}

    # ---- the N>1 default workload (C5, 1025^3) on this one GPU: the 1-GPU point of the scaling curve
    c5 = None
    if world == 1 and args.config == "C3-f64" and not args.no_c5:
        S.close()
        del u, f
        torch.cuda.empty_cache()
        c5 = single_gpu_point("C5", dev, stream)

    # ---- CPU oracle baseline (rank 0, N=1 only), in a child process so that this (product)
    # process never maps the oracle's library
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_subprocess(args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": unk_total / (ms * 1e-3), "unit": "unknowns/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if (world > 1 and not slab) else "strong", "vs_baseline": None,
            "dtype": ("c" if cd else "") + dt,
            "data": "synthetic",
            "config": workload_config(args.config),
            "parallelism": (f"z-slab x{world} (NCCL halos, agglomeration below 8 planes/rank)" if slab
                            else ("replicas" if world > 1 else "single-gpu")),
            "driver": "device loop (CUDA graph WHILE node)" if device_loop else "host loop",
            "residual_reduction_per_step": (rk / r0) ** (1.0 / (args.steps + args.warmup)) if r0 else None,
            "model_bytes_per_step": B, "model_GBps": B / (ms * 1e-3) / 1e9,
            "roofline": roofline, "kernels": breakdown, "cpu_baseline": cpu, "e2e": e2e,
            "single_gpu_C5": c5, "solve_to_1e-10": solve,
            "measured_bytes_per_step": ncu_cycle_bytes(args.config),
            "gpu_launches": int(round(launches * args.steps)), "gpu_launches_per_step": launches,
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def check_world(args):
    """--gpus N must match the launch: under torchrun WORLD_SIZE == N; without torchrun and N > 1,
    re-launch this command under torch.distributed.run with N ranks (never time fewer GPUs than
    asked for).  Returns an exit code to stop with, or None to go on."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if os.environ.get("WORLD_SIZE") is not None:
        if world != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            return 2
        return None
    if args.gpus == 1:
        return None
    if args.gpus < 1:
        print("bench.py: --gpus must be >= 1", file=sys.stderr)
        return 2
    if args.impl == "mg":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {n} CUDA device(s) visible", file=sys.stderr)
            return 2
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    import subprocess
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mg", choices=["mg", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS) + sorted(CD_CONFIGS),
                    help="default: C3-f64 (the metric's workload) at N=1, C5 (the north star's scaling "
                         "workload, 1025^3) at N>1")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--host-loop", action="store_true", help="mg_solve with MG_FLAG_HOST_LOOP (per-cycle sync)")
    ap.add_argument("--separate-prolong", action="store_true",
                    help="MG_FLAG_SEPARATE_PROLONG (prolongation as its own pass, not in the first post-sweep)")
    ap.add_argument("--decomp", default="slab", choices=["slab", "replicas"],
                    help="N>1: z-slab decomposition of one grid (default) or independent replicas")
    ap.add_argument("--no-c5", action="store_true", help="N=1 C3-f64: skip the single-GPU C5 point")
    ap.add_argument("--no-kfuse", action="store_true", help="MG_FLAG_NO_KFUSE (2D Jacobi: one sweep per pass)")
    ap.add_argument("--cpu-baseline-leg", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.config is None:
        args.config = "C5" if args.gpus > 1 else "C3-f64"
    if args.cpu_baseline_leg:
        return cpu_baseline_leg(args.config)
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    rc = check_world(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_mg(args)


if __name__ == "__main__":
    sys.exit(main())
