"""Shape of the captured matvec graph at 1024^2 nt=16: nodes, edges and programmatic (PDL)
edges (vrg_hess_graph_info), and the graph replay vs direct-launch time of one matvec."""
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
vt = (T(vtA[0]), T(vtA[1]))
for _ in range(3):
    H.apply(vt)
info = (ctypes.c_int * 3)()
ctx.check(ctx.lib.vrg_hess_graph_info(H.h, info))
print("graph nodes", info[0], "edges", info[1], "programmatic", info[2], flush=True)
for kid in (13, 14):
    ms = ctypes.c_double()
    ctx.check(ctx.lib.vrg_hess_bench_kernel(H.h, kid, 30, ctypes.byref(ms)))
    print("kernel id", kid, round(ms.value * 1e3, 1), "us", flush=True)
