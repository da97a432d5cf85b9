"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck): the band-path matvec
(gather + epilogue + row pass, column pass), the plain path, the prefilter segment kernels, the
Lanczos cluster kernel and a state / adjoint solve, on 256^2 and 64 x 48 grids.
    compute-sanitizer --tool racecheck python tools/sanitize_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_02153_b200 import api, synth  # noqa: E402

ctx = api.Context(0)
F = ctx.field
for (n1, n2, nt) in [(256, 256, 3), (64, 48, 2)]:
    mT = synth.smoothed_noise(n1, n2, 1000)
    v1, v2 = synth.smooth_velocity(n1, n2, 2000)
    vt1, vt2 = synth.smooth_velocity(n1, n2, 3000)
    H = api.HessianOperator(ctx, (F(0.5 * v1), F(0.5 * v2)), F(mT), F(mT), 2, 1e-3, 0, nt)
    H.apply((F(vt1), F(vt2)))
    H.apply_split((F(vt1), F(vt2)))
    S = api.Solver(ctx, (F(v1), F(v2)), nt)
    traj = S.solve_state(F(mT))
    S.solve_adjoint(traj[nt])
    api.prefilter(ctx, F(mT))
m = F(synth.config12_fields(64)[0])
api.estimate_eigs(ctx, m, m, 2, 1e-2, 0)  # Lanczos: the k_lanczos_orth cluster kernel
ctx.sync()
print("sanitize probe done")
