"""State solve (slState, nt steps) with alternating-direction fused steps vs the band path:
device time per solve and per step (CUDA events on the library stream), 1024^2 by default."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1604_02153_b200 import api, synth

n = int(os.environ.get("N", "1024"))
nt = int(os.environ.get("NT", "16"))
ctx = api.Context(0)
m0 = ctx.field(synth.smoothed_noise(n, n, 1000))
v1, v2 = synth.smooth_velocity(n, n, 2000)
v = (ctx.field(v1), ctx.field(v2))
for mode in ("band", "adi", "band", "adi"):
    if mode == "adi":
        os.environ["VRG_ADI"] = "1"
    else:
        os.environ.pop("VRG_ADI", None)
    S = api.Solver(ctx, v, nt)
    S.solve_state(m0)  # warm: departure points, plan
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        S.solve_state(m0)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{mode:5s} n={n} nt={nt}: {ms * 1e3:8.1f} us per solve, {ms * 1e3 / nt:6.2f} us per step "
          f"({4 * 8 * n * n / (ms / nt * 1e-3) / 1e9:7.1f} GB/s on 4F)", flush=True)
