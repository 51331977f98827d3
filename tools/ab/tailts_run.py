import sys, ctypes, os
sys.path.insert(0, ".")
import numpy as np, torch, bench
import paper_1406_5369_b200 as mgb
lib = mgb.load_library()
f = lib.mg_exp_tail_ts; f.restype = ctypes.c_int
for cfg in sys.argv[1:]:
    dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
    S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt, flags=mgb.FLAG_HOST_LOOP | mgb.FLAG_NO_GRAPH)
    u, fr = S.empty(), S.empty(); S.workload_fill(u, 42)
    S.solve(u, fr, 0.0, 3); torch.cuda.synchronize()
    ts = (ctypes.c_longlong * 1024)(); tg = (ctypes.c_int * 1024)()
    f(ts, tg, 1024)
    S.solve(u, fr, 0.0, 1); torch.cuda.synchronize()
    n = f(ts, tg, 1024)
    ts2 = (ctypes.c_longlong * 1024)(); tg2 = (ctypes.c_int * 1024)()
    import ctypes as C
    S.workload_fill(u, 42); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True); a.record(); S.solve(u, fr, -1.0, 200); b.record(); torch.cuda.synchronize()
    print(cfg, "device-loop ms/cycle %.4f" % (a.elapsed_time(b) / 200))
    t = np.array(ts[:n]); g = list(tg[:n])
    print(cfg, "kernel globaltimer ns", ts[1000])
    print(cfg, "stamps", n, "total cycles", t[-1] - t[0], "= %.1f us @1.965GHz" % ((t[-1] - t[0]) / 1965.0))
    for i in range(1, n):
        print("  %5d -> %5d : %7d cyc %6.2f us" % (g[i-1], g[i], t[i] - t[i-1], (t[i] - t[i-1]) / 1965.0))
    S.close()
