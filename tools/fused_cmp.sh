# fused band path vs plain path, and parity of both
VRG_FUSED_BANDS=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_precond.py -m gpu -q -x 2>&1 | tail -2
VRG_FUSED_BANDS=0 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
python - <<'PY'
import os, time, json, torch
from paper_1604_02153_b200 import api, synth
ctx = api.Context(0)
res = {}
for n, nt in [(1024, 16), (2048, 16), (4096, 32)]:
    mT = ctx.field(synth.smoothed_noise(n, n, 1000)); v1, v2 = synth.smooth_velocity(n, n, 2000)
    v = (ctx.field(v1), ctx.field(v2)); w1, w2 = synth.smooth_velocity(n, n, 3000); vt = (ctx.field(w1), ctx.field(w2))
    for fused in ("0", "1"):
        os.environ["VRG_FUSED_BANDS"] = fused
        H = api.HessianOperator(ctx, v, mT, mT, 2, 1e-3, 0, nt)
        out = ctx.empty(2, n, n)
        for _ in range(3): H.apply(vt, out=out)
        torch.cuda.synchronize(); t = time.perf_counter(); k = 10 if n < 4096 else 4
        for _ in range(k): H.apply(vt, out=out)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / k
        res[f"{n}_{nt}_fused{fused}"] = dt * 1e3
        del H
print(json.dumps(res))
PY
