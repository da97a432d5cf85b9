"""Times the pieces of the GN HessianOperator constructor at a large grid (device events)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1604_02153_b200 import api, synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ctx = api.Context(0)
F = ctx.field
mT = F(synth.smoothed_noise(n, n, 1000))
v1, v2 = synth.smooth_velocity(n, n, 2000)
v = (F(0.1 * v1), F(0.1 * v2))
S = api.Solver(ctx, v, nt)
state = S.solve_state(mT)


def timed(name, fn, reps=3):
    fn()
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    ctx.sync()
    print(f"{name:40s} {(time.perf_counter() - t0) / reps * 1e3:9.3f} ms", flush=True)


timed("HessianOperator ctor (state given)", lambda: api.HessianOperator(ctx, v, mT, mT, 2, 1e-4, 0, nt, state=state))
timed("HessianOperator ctor (state solved)", lambda: api.HessianOperator(ctx, v, mT, mT, 2, 1e-4, 0, nt))
timed(f"gradient x{nt + 1}", lambda: [api.gradient(ctx, state[j]) for j in range(nt + 1)])
timed(f"prefilter x{2 * nt}", lambda: [api.prefilter(ctx, state[j % (nt + 1)]) for j in range(2 * nt)])
c = api.prefilter(ctx, state[0])
X = S.departure(api.FORWARD)
timed(f"evaluate x{2 * nt}", lambda: [api.evaluate(ctx, c, X[0], X[1]) for j in range(2 * nt)])
timed("Solver + departure fwd/bwd", lambda: (lambda s: (s.departure(api.FORWARD), s.departure(api.BACKWARD)))(api.Solver(ctx, v, nt)))
timed("solve_state", lambda: S.solve_state(mT))
timed("evaluate_gradient", lambda: api.evaluate_gradient(ctx, v, mT, mT, 2, 1e-4, 0, nt))
