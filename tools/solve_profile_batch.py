"""One batched config-5b solve (8 pairs at 256^2, nt=16, H2 1e-3, 2L-Cheb(10)) for a kernel launch list:
  ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/solve_profile_batch.py [pairs]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1604_02153_b200 import api, batch

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = api.Context(0)
imgs = [batch.make_images(ctx, 256, p, 16) for p in range(P)]
out = api.newton_solve_batch(ctx, np.stack([a for a, _ in imgs]), np.stack([b for _, b in imgs]), api.H2SEMI, 1e-3,
                             api.COMPRESSIBLE, nt=16, kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB,
                             cheb_iters=10, tol_rel=1e-2)
print([o[3]["iterations"] for o in out], file=sys.stderr)
