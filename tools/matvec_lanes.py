"""Experiment: L independent GN matvec streams on one GPU (each lane its own context, stream
and HessianOperator at the same iterate; host threads, ctypes releases the GIL).  Prints the
aggregate matvecs/s per L (config 4)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1604_02153_b200 import api

K = int(os.environ.get("K", "40"))
mT, v, vtA, vtB = bench.make_problem(0)
ctx0 = api.Context(0)
T = ctx0.field
mT_d, v_d = T(mT), (T(v[0]), T(v[1]))
mR_d = api.Solver(ctx0, v_d, bench.NT).solve_state_final(mT_d)
for L in [int(x) for x in (sys.argv[1:] or ["1", "2", "3"])]:
    lanes = []
    for k in range(L):
        c = ctx0 if k == 0 else api.Context(0, stream=torch.cuda.Stream(0))
        H = api.HessianOperator(c, v_d, mR_d, mT_d, bench.NORM, bench.BETA, api.COMPRESSIBLE, bench.NT)
        vts = [c.empty(2, bench.N_GRID, bench.N_GRID) for _ in range(2)]
        vts[0].copy_(torch.stack([T(vtA[0]), T(vtA[1])])); vts[1].copy_(torch.stack([T(vtB[0]), T(vtB[1])]))
        out = c.empty(2, bench.N_GRID, bench.N_GRID)
        lanes.append((c, H, vts, out))
    torch.cuda.synchronize()

    def run(lane, n):
        c, H, vts, out = lane
        for i in range(n):
            H.apply((vts[i & 1][0], vts[i & 1][1]), out=out)

    for lane in lanes:  # graph priming
        run(lane, 4)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=run, args=(lane, K)) for lane in lanes]
    for t in th: t.start()
    for t in th: t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"lanes={L}: {L*K/dt:.1f} matvec/s ({dt/K*1e3:.3f} ms per lane-matvec)", flush=True)
    del lanes
