import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1604_02153_b200 import api, slab, synth
ctx = api.Context(0)
for n, nt, G, sc in [(256, 4, 1, 0.5), (256, 4, 1, 1.0), (1024, 8, 1, 1.0), (1024, 8, 2, 0.5)]:
    mT = synth.smoothed_noise(n, n, 1000); v1, v2 = synth.smooth_velocity(n, n, 2000)
    F = ctx.field
    v = (F(sc * v1), F(sc * v2))
    H = api.HessianOperator(ctx, v, F(mT), F(mT), 2, 1e-3, 0, nt)
    S = slab.SlabHessian.from_operator(ctx, slab.LocalComm(G), H, 2, 1e-3)
    ref = api.Solver(ctx, v, nt).solve_state(F(mT)).cpu().numpy()  # (nt+1, n, n)
    L = n // G
    cur = [F(mT)[i*L:(i+1)*L].contiguous() for i in range(G)]
    S._prefilter(cur, S.win)
    errs = []
    outs = [[ctx.empty(L, n) for _ in range(G)] for _ in range(nt)]
    for j in range(1, nt + 1):
        if j > 1:
            S._windows_from_rows()
        for i in range(G):
            S._step(i, slab.KIND_STATE, S.win[i], S.parts[i]["Xf"], [outs[j-1][i]], 1.0/nt, 0.0, S.rows[i], S.partials[i][j], None)
        got = np.concatenate([o.cpu().numpy() for o in outs[j-1]], axis=0)
        errs.append(np.abs(got - ref[j]).max() / np.abs(ref[j]).max())
    print(n, nt, G, sc, "D", S.geo.D, ["%.1e" % e for e in errs], flush=True)
