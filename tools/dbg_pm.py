"""Debug helper: run one op_smooth of the plane-marching path for a config in isolation."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1406_5369_b200 as mgb
import oracle as orc

dim, n, dt, sm, lvl = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], int(sys.argv[5])
S = mgb.Solver(dim, n + 1, smoother=sm, dtype=dt, omega=1.0 if sm == "rbgs" else 0.8)
O = orc.Oracle(orc.Config(dim=dim, cells=(n,) * dim, levels=S.levels, smoother=orc.RBGS if sm == "rbgs" else orc.JACOBI,
                          omega=1.0 if sm == "rbgs" else 0.8), S.np_dtype)
shp = O.shape(lvl)
rng = np.random.default_rng(1)
u = rng.uniform(-1, 1, shp).astype(S.np_dtype)
f = rng.uniform(-1, 1, shp).astype(S.np_dtype)
for a in (u, f):
    a[0] = 0; a[-1] = 0; a[:, 0] = 0; a[:, -1] = 0; a[:, :, 0] = 0; a[:, :, -1] = 0
du, df = S.from_numpy(u, lvl), S.from_numpy(f, lvl)
out = S.empty(lvl)
S.op_smooth(lvl, du, df, out)
import torch
torch.cuda.synchronize()
got = S.to_numpy(out, lvl)
ref = O.smooth(lvl, u, f)
print(dim, n, dt, sm, lvl, "maxdiff", np.abs(got - ref).max())
