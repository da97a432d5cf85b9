"""Small driver for ncu captures of the matvec (profiling range = K matvecs after warm-up).

  ncu --profile-from-start off ... python tools/ncu_matvec.py [--n 1024] [--nt 16] [--steps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1604_02153_b200 import api, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--nt", type=int, default=16)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--what", default="matvec", choices=["matvec", "state"])
    a = ap.parse_args()
    ctx = api.Context(0)
    n = a.n
    mT = ctx.field(synth.smoothed_noise(n, n, 1000))
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    v = (ctx.field(v1), ctx.field(v2))
    w1, w2 = synth.smooth_velocity(n, n, 3000)
    vt = (ctx.field(w1), ctx.field(w2))
    if a.what == "matvec":
        H = api.HessianOperator(ctx, v, mT, mT, 2, 1e-3, 0, a.nt)
        out = ctx.empty(2, n, n)
        for _ in range(2):
            H.apply(vt, out=out)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(a.steps):
            H.apply(vt, out=out)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    else:
        s = api.Solver(ctx, v, a.nt)
        s.solve_state_final(mT)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for _ in range(a.steps):
            s.solve_state_final(mT)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    print("ok")


if __name__ == "__main__":
    main()
