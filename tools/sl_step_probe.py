"""SL state step (config 4 unit ii, 1024^2) pieces timed back to back: band kernel + column pass
(9), band kernel alone (12), column pass alone (4), plain prefilter + gather (10)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1604_02153_b200 import api

n = int(os.environ.get("N", "1024"))
bench.N_GRID = n
ctx = api.Context(0)
mT, v, vtA, vtB = bench.make_problem(0)
F = 8 * n * n
T = ctx.field
H = api.HessianOperator(ctx, (T(v[0]), T(v[1])), T(mT), T(mT), 2, 1e-3, 0, 16)
H.apply((T(vtA[0]), T(vtA[1])))
reps = int(os.environ.get("REPS", "50"))
for kid in [int(k) for k in (sys.argv[1:] or ["9", "12", "4", "10"])]:
    ms = ctypes.c_double()
    ctx.check(ctx.lib.vrg_hess_bench_kernel(H.h, kid, reps, ctypes.byref(ms)))
    us = ms.value * 1e3
    print(n, kid, round(us, 2), "us", "(unit 9/10: 4F ->", round(4 * F / us / 1e3, 1), "GB/s)", flush=True)
