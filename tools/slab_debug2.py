import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1604_02153_b200 import api, slab, synth
ctx = api.Context(0)
for n, nt, G in [(256, 4, 1), (512, 8, 1), (1024, 8, 1), (1024, 8, 2)]:
    mT = synth.smoothed_noise(n, n, 1000); v1, v2 = synth.smooth_velocity(n, n, 2000)
    F = ctx.field
    H = api.HessianOperator(ctx, (F(v1), F(v2)), F(mT), F(mT), 2, 1e-3, 0, nt)
    S = slab.SlabHessian.from_operator(ctx, slab.LocalComm(G), H, 2, 1e-3)
    u = F(mT)
    c = api.prefilter(ctx, u).cpu().numpy()
    L = n // G
    us = [u[i*L:(i+1)*L].contiguous() for i in range(G)]
    S._prefilter(us, S.win)
    g = S.geo
    errw = []
    for i in range(G):
        w = S.win[i].cpu().numpy()
        rows = [(g.win_base(i) + r) % n for r in range(g.win_rows)]
        ref = c[rows]
        errw.append(np.abs(w[:, 1:n+1] - ref).max() / np.abs(ref).max())
        # periodic column padding
        errw.append(np.abs(w[:, 0] - ref[:, n-1]).max() + np.abs(w[:, n+1] - ref[:, 0]).max())
    # store gather vs api.evaluate at Xf
    X = [p["Xf"] for p in S.parts]
    Xfull = torch.cat(X, dim=1)
    ev = api.evaluate(ctx, F(c), Xfull[0].contiguous(), Xfull[1].contiguous()).cpu().numpy()
    outs = []
    for i in range(G):
        o = ctx.empty(L, n)
        S._step(i, slab.KIND_STORE, S.win[i], S.parts[i]["Xf"], [o], 1.0/nt, 0.0, S.scr[i], S.partials[i][0], None)
        outs.append(o.cpu().numpy())
    got = np.concatenate(outs, axis=0)
    fl = [f.cpu().numpy().tolist() for f in S.flags]
    print(n, nt, G, "D", g.D, "win", g.win_rows, "window err", ["%.2e" % e for e in errw], "gather err %.3e" % (np.abs(got - ev).max() / np.abs(ev).max()), "flags", fl, flush=True)
