import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1604_02153_b200 import api, slab, synth
ctx = api.Context(0)
n, nt, G = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 2, 1
mT = synth.smoothed_noise(n, n, 1000); v1, v2 = synth.smooth_velocity(n, n, 2000)
F = ctx.field
H = api.HessianOperator(ctx, (F(0.5*v1), F(0.5*v2)), F(mT), F(mT), 2, 1e-3, 0, nt)
S = slab.SlabHessian.from_operator(ctx, slab.LocalComm(G), H, 2, 1e-3)
p = S.parts[0]
ht = 1.0 / nt
rnd = lambda s: F(np.random.default_rng(s).standard_normal((n, n)))
vt = [rnd(1), rnd(2)]; vtD = [rnd(3), rnd(4)]
def rowfilt(u):
    o = ctx.empty(n, n); ctx.check(ctx.lib.vrg_prefilter_rows(ctx.h, n, n, api._p(u), api._p(o), None)); return o
def rel(a, b): return float((a - b).abs().max() / b.abs().max())
# INC0
rows = ctx.empty(n, n)
ops = [vtD[0], vtD[1], p["GD"][1][0], p["GD"][1][1], vt[0], vt[1], p["G"][2][0], p["G"][2][1]]
S._step(0, slab.KIND_INC0, S.win[0], p["Xf"], ops, ht, 0.0, rows, S.partials[0][0], None)
torch.cuda.synchronize()
s = 0.5 * ht * (-(vtD[0] * p["GD"][1][0] + vtD[1] * p["GD"][1][1]) - (vt[0] * p["G"][2][0] + vt[1] * p["G"][2][1]))
print("INC0", rel(rows, rowfilt(s)), flush=True)
# INC with a window of a random field
u = rnd(5)
S._prefilter([u], S.win)
c = api.prefilter(ctx, u)
ev = api.evaluate(ctx, c, p["Xf"][0].contiguous(), p["Xf"][1].contiguous())
S._step(0, slab.KIND_INC, S.win[0], p["Xf"], ops, ht, 0.0, rows, S.partials[0][0], None)
torch.cuda.synchronize()
print("INC", rel(rows, rowfilt(ev + s)), flush=True)
# STATE with the same window
o = ctx.empty(n, n)
S._step(0, slab.KIND_STATE, S.win[0], p["Xf"], [o], ht, 0.0, rows, S.partials[0][0], None)
print("STATE", rel(o, ev), rel(rows, rowfilt(ev)), flush=True)
# SEED (gather): returns l = -(ev + s) row-filtered; b = w l G(nt)
b = [ctx.empty(n, n), ctx.empty(n, n)]
w = 0.25
S._step(0, slab.KIND_SEED, S.win[0], p["Xf"], ops + [b[0], b[1]], ht, w, rows, S.partials[0][nt], S.flags[0][nt:nt+1])
torch.cuda.synchronize()
l = -1.0 * (ev + s)
print("SEED rows", rel(rows, rowfilt(l)), "b", rel(b[0], w * (l * p["G"][2][0])), rel(b[1], w * (l * p["G"][2][1])), flush=True)
# ADJ with the backward departure points
evb = api.evaluate(ctx, c, p["Xb"][0].contiguous(), p["Xb"][1].contiguous())
b0 = [rnd(7), rnd(8)]
bb = [b0[0].clone(), b0[1].clone()]
opsA = [p["dvd"], p["dv"], p["G"][1][0], p["G"][1][1], bb[0], bb[1]]
S._step(0, slab.KIND_ADJ, S.win[0], p["Xb"], opsA, ht, w, rows, S.partials[0][1], S.flags[0][1:2])
torch.cuda.synchronize()
uD = evb
f0 = uD * p["dvd"]
pred = uD + ht * f0
o = uD + 0.5 * ht * (f0 + pred * p["dv"])
print("ADJ rows", rel(rows, rowfilt(o)), "b", rel(bb[0], b0[0] + w * (o * p["G"][1][0])), rel(bb[1], b0[1] + w * (o * p["G"][1][1])), flush=True)
