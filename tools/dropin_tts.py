"""Time to solution of the drop-in: the reference's own newtonSolve (dropin_newton, linked with
the unmodified reference objects and the device pImpls over libvrg) on configs 1 and 2, the
second solve of the process (DROPIN_REPEAT=2: the first pays the CUDA context and module
start-up), next to vrg_newton_solve (the library's own host driver) on the same inputs."""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402  (the inputs: m_R by the compiled reference's SL solve)
from paper_1604_02153_b200 import api, synth, vrf  # noqa: E402

BIN = os.path.join(ROOT, "paper_1604_02153_b200", "dropin", "_build", "dropin_newton")
CFGS = {"config1": dict(n=64, nt=4, norm=2, beta=1e-2, cheb=False),
        "config2": dict(n=256, nt=8, norm=1, beta=1e-3, cheb=True)}
out = {}
ctx = api.Context(0)
with tempfile.TemporaryDirectory() as d:
    for name, c in CFGS.items():
        mT, (v1, v2) = synth.config12_fields(c["n"])
        mR = ref.solve_state_final(v1, v2, c["nt"], mT)
        vrf.write_field(os.path.join(d, "mR.vrf"), mR)
        vrf.write_field(os.path.join(d, "mT.vrf"), mT)
        runs = []
        for _ in range(3):
            t0 = time.perf_counter()
            r = subprocess.run(["env", "DROPIN_REPEAT=2", BIN, os.path.join(d, "mR.vrf"), os.path.join(d, "mT.vrf"), str(c["norm"]),
                                repr(float(c["beta"])), "0", str(c["nt"]), "2l", "cheb" if c["cheb"] else "pcg", "10",
                                "1e-2"], capture_output=True, text=True, timeout=600)
            wall = time.perf_counter() - t0
            lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
            runs.append((lines[-1].get("totalTimeSec"), wall))
        kw = dict(nt=c["nt"], kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB if c["cheb"] else api.COARSE_PCG,
                  cheb_iters=10, tol_rel=1e-2)
        api.newton_solve(ctx, mR, mT, c["norm"], c["beta"], 0, **kw)
        t0 = time.perf_counter()
        api.newton_solve(ctx, mR, mT, c["norm"], c["beta"], 0, **kw)
        lib = time.perf_counter() - t0
        out[name] = {"dropin_newtonSolve_s": min(t for t, _ in runs),
                     "dropin_process_wall_s_two_solves": min(w for _, w in runs),
                     "vrg_newton_solve_s": lib}
        print(name, out[name], flush=True)
print(json.dumps(out))
