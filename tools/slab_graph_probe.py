"""Slab matvec (LocalComm, G virtual slabs on one GPU) eager vs CUDA-graph replay: the Python
orchestration cost per matvec that the capture removes.  python tools/slab_graph_probe.py [n] [nt]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1604_02153_b200 import api, slab, synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = api.Context(0)
F = ctx.field
mT = synth.smoothed_noise(n, n, 1000)
v1, v2 = synth.smooth_velocity(n, n, 2000)
vt1, vt2 = synth.smooth_velocity(n, n, 3000)
H = api.HessianOperator(ctx, (F(0.5 * v1), F(0.5 * v2)), F(mT), F(mT), 2, 1e-3, api.COMPRESSIBLE, nt)
out = {}
for G in (1, 2, 4, 8):
    S = slab.SlabHessian.from_operator(ctx, slab.LocalComm(G), H, 2, 1e-3)
    L = n // G
    vts = [F(np.stack([vt1[i * L:(i + 1) * L], vt2[i * L:(i + 1) * L]])) for i in range(G)]
    outs = [ctx.empty(2, L, n) for _ in range(G)]
    res = {}
    for mode in ("eager", "graph"):
        S.graphs = mode == "graph"
        for _ in range(S.capture_after + 2):  # eager uses, then the capture
            S.apply(vts, outs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 10
        for _ in range(reps):
            S.apply(vts, outs)
        torch.cuda.synchronize()
        res[mode] = (time.perf_counter() - t0) / reps * 1e3
    out[f"G{G}"] = {k: round(v, 3) for k, v in res.items()}
    print(G, out[f"G{G}"], flush=True)
print(json.dumps({"n": n, "nt": nt, "ms_per_matvec": out}))
