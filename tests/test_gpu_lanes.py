"""GPU: concurrent registrations on one device (batch.py lanes: own context + stream per host
thread) give the same solves as the same pairs run one after another: identical Newton and
Krylov iteration counts and the same velocities."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1604_02153_b200 import batch

pytestmark = pytest.mark.gpu


def _make_runner(n, nt):
    from paper_1604_02153_b200 import api

    def make(lane):
        ctx = api.Context(0, stream=torch.cuda.Stream(0)) if lane >= 0 else api.Context(0)

        def run(p):
            mT, (v1, v2) = batch.pair_inputs(n, p, nt)
            mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), nt).solve_state_final(ctx.field(mT)).cpu().numpy()
            w1, w2, recs, summ = api.newton_solve(ctx, mR, mT, api.H2SEMI, 1e-3, api.COMPRESSIBLE, nt=nt,
                                                  kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB,
                                                  cheb_iters=10, tol_rel=1e-2)
            return {"iters": summ["iterations"], "inner": [r["innerIterations"] for r in recs],
                    "v": np.stack([np.asarray(w1), np.asarray(w2)])}
        return run
    return make


def test_lanes_match_sequential():
    n, nt, pairs = 128, 8, 6
    make = _make_runner(n, nt)
    seq = batch.run_lanes(list(range(pairs)), lambda k: make(-1), 1)
    par = batch.run_lanes(list(range(pairs)), make, 3)
    assert len({r["lane"] for r in par}) > 1
    for a, b in zip(seq, par):
        assert a["iters"] == b["iters"] and a["inner"] == b["inner"], a["item"]
        err = np.abs(a["v"] - b["v"]).max() / np.abs(a["v"]).max()
        assert err <= 1e-12, (a["item"], err)
