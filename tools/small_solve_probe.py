"""Config 1 (64^2, nt=4, H2 1e-2, 2L-PCG) and config 2 registrations: wall time per solve,
library launches per solve (host-side count) and, under ncu, the device time (launch list).
  python tools/small_solve_probe.py [config1|config2] [reps]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1604_02153_b200 import api

name = sys.argv[1] if len(sys.argv) > 1 else "config1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = next(v for k, v in bench.TTS_RUNS.items() if k.startswith(name))
ctx = api.Context(0)
mT, v1, v2 = bench.tts_problem(cfg)
mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), cfg["nt"]).solve_state_final(ctx.field(mT)).cpu().numpy()
kw = dict(nt=cfg["nt"], kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB if cfg["cheb"] else api.COARSE_PCG,
          cheb_iters=10, tol_rel=1e-2)
import torch
for r in range(reps):
    l0 = bench.ctypes_launches(ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, recs, summ = api.newton_solve(ctx, mR, mT, cfg["norm"], cfg["beta"], cfg.get("deformation", 0), **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(name, "wall_ms", round(dt * 1e3, 2), "launches", bench.ctypes_launches(ctx) - l0, "iters", summ["iterations"],
          flush=True)
