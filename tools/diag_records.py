"""Per-iteration comparison of the library's newton_solve records with a golden reference record
set (tests/golden/newton_default.npz / newton_cfg3_5b.npz / newton.npz): prints the relative
differences of the objective and of ||g||_inf / ||g_0||_inf per outer iteration."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref  # noqa: E402
from paper_1604_02153_b200 import api, synth  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def run(name, fixed_nt=None):
    d = dict(np.load(os.path.join(G, "newton_default.npz")))
    n, norm, beta, two_level, cheb = d[name + "_meta"]
    n, norm = int(n), int(norm)
    mT, (v1, v2) = synth.config12_fields(n)
    mR = ref.solve_state_final(v1, v2, {64: 4, 256: 8}[n], mT)
    ctx = api.Context(0)
    kind = api.PC_TWO_LEVEL if two_level else api.PC_REG
    _, _, recs, summ = api.newton_solve(ctx, mR, mT, norm, float(beta), 0, nt=fixed_nt or 0, kind=kind,
                                        coarse_solver=api.COARSE_CHEB if cheb else api.COARSE_PCG, cheb_iters=10,
                                        tol_rel=1e-2)
    rr = d[name + "_records"]
    g0 = rr[0][1]
    print(name, "iters", summ["iterations"], int(d[name + "_summary"][1]))
    for r, q in zip(recs, rr):
        print(f"  it {int(q[0])} inner {int(r['innerIterations'])}/{int(q[5])} ls {int(r['lineSearchSteps'])}/{int(q[6])}"
              f" dJ/J {abs(r['objective'] - q[3]) / abs(q[3]):.2e} dg/g0 {abs(r['gradNormInf'] - q[1]) / g0:.2e}"
              f" J {q[3]:.6e} ffts {int(r['ffts'])}/{int(q[8])} interps {int(r['interps'])}/{int(q[9])}")


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["cfg1_reg", "cfg1_2lpcg", "cfg2_2lcheb", "cfg2_reg"]:
        run(nm)
