"""One config-5b registration (256^2, nt=16, H2 1e-3, 2L-Cheb(10)) for a kernel launch list:
  ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/solve_profile.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_02153_b200 import api, batch

ctx = api.Context(0)
mR, mT = batch.make_images(ctx, 256, 0, 16)
_, _, recs, summ = api.newton_solve(ctx, mR, mT, api.H2SEMI, 1e-3, api.COMPRESSIBLE, nt=16, kind=api.PC_TWO_LEVEL,
                                    coarse_solver=api.COARSE_CHEB, cheb_iters=10, tol_rel=1e-2)
print(summ, file=sys.stderr)
