"""Time one coarse split matvec (precond::CoarseOperator::applySplitHessian) of a config's
coarse grid at v = 0, fixed buffers (graph replay), and one with a fresh input buffer each call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1604_02153_b200 import api

ctx = api.Context(0)
for name in sys.argv[1:] or ["config2_256_nt8_H1_1e-3_2L-cheb10", "config1_64_nt4_H2_1e-2_2L-pcg"]:
    cfg = bench.TTS_RUNS[name]
    mT, v1, v2 = bench.tts_problem(cfg)
    mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), cfg["nt"]).solve_state_final(ctx.field(mT))
    Cop = api.CoarseOperator(ctx, None, mR, ctx.field(mT), cfg["norm"], cfg["beta"], api.COMPRESSIBLE)
    s = (ctx.empty(*Cop.shape).normal_(), ctx.empty(*Cop.shape).normal_())
    o = ctx.empty(2, *Cop.shape)
    lib = ctx.lib
    def call():
        ctx.check(lib.vrg_coarse_apply_split(Cop.h, api._p(s[0]), api._p(s[1]), api._p(o[0]), api._p(o[1])))
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        call()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    l0 = ctx.lib and None
    print(f"{name}: coarse {Cop.shape} nt={Cop.nt}: {dt*1e6:.1f} us per split matvec (replay)", flush=True)
