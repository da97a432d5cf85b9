"""Diagnostic: fused band data term vs plain 3-kernel data term (same inputs)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_02153_b200 import api, synth
ctx = api.Context(0)
cases = [(256, 1), (256, 2), (512, 4)] if len(sys.argv) < 2 else [(int(sys.argv[1]), int(sys.argv[2]))]
for n, nt in cases:
    mT = synth.smoothed_noise(n, n, 1000); v1, v2 = synth.smooth_velocity(n, n, 2000); w1, w2 = synth.smooth_velocity(n, n, 3000)
    F = ctx.field
    out = {}
    for f in ("0", "1", "1b", "0b"):
        os.environ["VRG_FUSED_BANDS"] = f[0]
        H = api.HessianOperator(ctx, (F(0.5*v1), F(0.5*v2)), F(mT), F(mT), 2, 1e-3, 0, nt)
        d1, d2 = H.apply_data_term((F(w1), F(w2)))
        out[f] = d1.cpu().numpy()
        del H
    s = np.abs(out["0"]).max()
    print(n, nt, "fused-plain", np.abs(out["0"] - out["1"]).max() / s, "fused-fused", np.abs(out["1"] - out["1b"]).max() / s,
          "plain-plain", np.abs(out["0"] - out["0b"]).max() / s, flush=True)
