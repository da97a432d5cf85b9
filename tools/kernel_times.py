import sys, ctypes
sys.path.insert(0, '/root/repo')
import bench
from paper_1604_02153_b200 import api
ctx = api.Context(0)
mT, v, vtA, vtB = bench.make_problem(0)
T = ctx.field
H = api.HessianOperator(ctx, (T(v[0]), T(v[1])), T(mT), T(mT), 2, 1e-3, 0, 16)
H.apply((T(vtA[0]), T(vtA[1])))
for kid in (7, 11, 8, 4, 9):
    ms = ctypes.c_double()
    ctx.check(ctx.lib.vrg_hess_bench_kernel(H.h, kid, 50, ctypes.byref(ms)))
    print(kid, round(ms.value * 1e3, 2), "us")
