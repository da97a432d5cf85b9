"""SL state step (config 4 unit ii, 1024^2) pieces timed back to back: band kernel + column pass
(9), band kernel alone (12), column pass alone (4), plain prefilter + gather (10)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1604_02153_b200 import api

ctx = api.Context(0)
mT, v, vtA, vtB = bench.make_problem(0)
T = ctx.field
H = api.HessianOperator(ctx, (T(v[0]), T(v[1])), T(mT), T(mT), 2, 1e-3, 0, 16)
H.apply((T(vtA[0]), T(vtA[1])))
reps = int(os.environ.get("REPS", "50"))
for kid in [int(k) for k in (sys.argv[1:] or ["9", "12", "4", "10"])]:
    ms = ctypes.c_double()
    ctx.check(ctx.lib.vrg_hess_bench_kernel(H.h, kid, reps, ctypes.byref(ms)))
    print(kid, round(ms.value * 1e3, 2), "us", flush=True)
