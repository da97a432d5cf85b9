"""Newton time-to-solution of one config with the per-phase trace (VRG_TRACE=1)."""
import os, sys, time
os.environ.setdefault("VRG_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import torch
from paper_1604_02153_b200 import api
ctx = api.Context(0)
name = sys.argv[1] if len(sys.argv) > 1 else "config2_256_nt8_H1_1e-3_2L-cheb10"
cfg = bench.TTS_RUNS[name]
mT, v1, v2 = bench.tts_problem(cfg)
mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), cfg["nt"]).solve_state_final(ctx.field(mT)).cpu().numpy()
kw = dict(nt=cfg["nt"], kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB if cfg["cheb"] else api.COARSE_PCG,
          cheb_iters=10, tol_rel=1e-2)
for rep in range(2):
    print("=== run", rep, file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    _, _, recs, summ = api.newton_solve(ctx, mR, mT, cfg["norm"], cfg["beta"], api.COMPRESSIBLE, **kw)
    torch.cuda.synchronize()
    print("total", time.perf_counter() - t0, summ, file=sys.stderr, flush=True)
