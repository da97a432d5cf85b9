import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1604_02153_b200 import api, slab, synth
ctx = api.Context(0)
for n, nt, G, beta, sc in [(1024, 8, 1, 1e-3, 1.0), (1024, 16, 4, 1e-3, 1.0), (2048, 8, 2, 1e-4, 1.0), (4096, 32, 8, 1e-4, 1.0)]:
    mT = synth.smoothed_noise(n, n, 1000); v1, v2 = synth.smooth_velocity(n, n, 2000); vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    F = ctx.field
    H = api.HessianOperator(ctx, (F(sc * v1), F(sc * v2)), F(mT), F(mT), 2, beta, 0, nt)
    try:
        d = H.apply_data_term((F(vt1), F(vt2))); dd = np.stack([d[0].cpu().numpy(), d[1].cpu().numpy()]); err = None
    except Exception as e:
        dd = None; err = repr(e)
    S = slab.SlabHessian.from_operator(ctx, slab.LocalComm(G), H, 2, beta)
    L = n // G
    vts = [F(np.stack([vt1[i*L:(i+1)*L], vt2[i*L:(i+1)*L]])) for i in range(G)]
    try:
        o = S.apply(vts, data_term_only=True); got = np.concatenate([x.cpu().numpy() for x in o], axis=1); serr = None
    except Exception as e:
        got = None; serr = repr(e)
    mx = [p.amax(dim=1).cpu().numpy() for p in S.partials]
    print(n, nt, G, beta, sc, "single:", err, "slab:", serr, "D", S.geo.D, "rel", None if (dd is None or got is None) else np.abs(got-dd).max()/np.abs(dd).max(), "stepmax", np.max(mx, axis=0)[[0, 1, nt-1, nt]], flush=True)
    del H, S
    torch.cuda.empty_cache()
