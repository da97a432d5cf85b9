"""GPU: inexact GN-Krylov registration whose fine Hessian data term is the slab-decomposed
operator (slab.SlabFineOperator through the C ABI hook vrg_set_fine_operator, config 5a's
path) against the library's own single-device solve on the same images: identical Newton,
Krylov and line-search iteration counts, step lengths and op counters; objective, gradient norm
within 1e-8 (the gradient norm on the scale of |g0|) and velocity within 1e-8 of max|v|.  G virtual slabs run on one device (LocalComm)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1604_02153_b200 import batch, slab

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1604_02153_b200 import api as A

    return A


def _pair(ctx, api, n, nt):
    mT, (v1, v2) = batch.pair_inputs(n, 0, nt)
    mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), nt).solve_state_final(ctx.field(mT)).cpu().numpy()
    return mR, mT


KW = dict(kind=1, coarse_solver=1, cheb_iters=10, tol_rel=1e-2)


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("n,nt,G,full", [(256, 8, 1, False), (256, 8, 2, False), (256, 16, 4, False),
                                         (512, 8, 8, False), (256, 8, 2, True), (512, 8, 1, True),
                                         (512, 16, 2, True), (512, 8, 4, True), (512, 8, 8, True)])
def test_slab_newton_matches_single_device(ctx, api, n, nt, G, full):
    """full: the gradient and every line-search objective are slab solves too (vrg_set_external_ops),
    so the driver runs no whole-grid transport; else only the fine matvec is decomposed."""
    mR, mT = _pair(ctx, api, n, nt)
    kw = dict(KW, kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB, nt=nt)
    w1, w2, recs, summ = api.newton_solve(ctx, mR, mT, 2, 1e-3, api.COMPRESSIBLE, **kw)
    fo = slab.SlabFineOperator(ctx, slab.LocalComm(G), mT, 2, 1e-3, mR=mR if full else None)
    s1, s2, srecs, ssumm = api.newton_solve(ctx, mR, mT, 2, 1e-3, api.COMPRESSIBLE, fine_operator=fo, **kw)
    assert ssumm["status"] == summ["status"] and ssumm["iterations"] == summ["iterations"]
    assert summ["iterations"] >= 2
    for a, b in zip(srecs, recs):
        for k in ("innerIterations", "lineSearchSteps", "stepLength", "ffts", "interps"):
            assert a[k] == b[k], (k, a["iter"], a[k], b[k])
        assert rel(a["objective"], b["objective"]) < 1e-8
        # |g|/|g0|: rounding-level operator differences move the Krylov iterates by ~cond*eps,
        # so the gradient norm is compared on the scale of |g0|
        assert abs(a["gradNormRel"] - b["gradNormRel"]) < 1e-8
    assert abs(ssumm["finalGradNormRel"] - summ["finalGradNormRel"]) < 1e-8
    v, sv = np.stack([w1, w2]), np.stack([s1, s2])
    assert np.abs(sv - v).max() <= 1e-8 * np.abs(v).max()
    # one slab build per Hessian (every iteration but a converged last one), one gather per matvec
    assert fo.builds == sum(1 for r in recs if r["innerIterations"] > 0)
    assert fo.matvecs >= sum(r["innerIterations"] for r in recs)
    if full:  # one slab gradient per outer iteration, one slab objective per line-search trial,
        # one slab coarse operator per KKT solve and a two-level application per PCG step (+1)
        assert fo.gradients == len(recs)
        assert fo.objectives == sum(r["lineSearchSteps"] for r in recs)
        if fo.coarse_slabs:  # n = 512: the half grid's 256-sample rows fit the slab step
            assert fo.coarse_builds == fo.builds
            assert fo.precond_applies >= sum(r["innerIterations"] + 1 for r in recs if r["innerIterations"] > 0)


class _Failing:
    def __init__(self, api, exc):
        self.error = None
        self._exc = exc
        self._b = api.FINE_BUILD_FN(self._build)
        self._d = api.FINE_DATA_TERM_FN(lambda u, a, b: 1)

    def callbacks(self):
        return self._b, self._d

    def _build(self, _u, _v, _nt):
        self.error = self._exc
        return 1


def test_fine_operator_errors(ctx, api):
    n, nt = 64, 4
    mR, mT = _pair(ctx, api, n, nt)
    kw = dict(KW, kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB, nt=nt)
    with pytest.raises(api.BlowupError, match="boom"):
        api.newton_solve(ctx, mR, mT, 2, 1e-3, api.COMPRESSIBLE, fine_operator=_Failing(api, api.BlowupError("boom")),
                         **kw)
    fo = slab.SlabFineOperator(ctx, slab.LocalComm(2), mT, 2, 1e-3)
    with pytest.raises(api.NotSupported):
        api.newton_solve(ctx, mR, mT, 2, 1e-3, api.INCOMPRESSIBLE, fine_operator=fo, **kw)
    with pytest.raises(api.NotSupported):
        api.newton_solve(ctx, mR, mT, 2, 1e-3, api.COMPRESSIBLE, fine_operator=fo, hessian_mode=api.FULL_NEWTON, **kw)
    # the hook is cleared after a failed solve: a plain solve on the same context still works
    _, _, recs, summ = api.newton_solve(ctx, mR, mT, 2, 1e-3, api.COMPRESSIBLE, **kw)
    assert summ["iterations"] >= 1
    with pytest.raises(api.InvalidArgument):
        slab.SlabFineOperator(ctx, slab.LocalComm(3), mT, 2, 1e-3)


def test_slab_newton_over_nccl_world1(ctx, api):
    """The same registration through DistComm on a one-rank NCCL group (the torchrun path of
    tools/slab_newton.py): identical iteration counts to the single-device solve."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    n, nt = 256, 8
    mR, mT = _pair(ctx, api, n, nt)
    kw = dict(KW, kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB, nt=nt)
    _, _, recs, summ = api.newton_solve(ctx, mR, mT, 2, 1e-3, api.COMPRESSIBLE, **kw)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        fo = slab.SlabFineOperator(ctx, slab.DistComm(), mT, 2, 1e-3)
        _, _, srecs, ssumm = api.newton_solve(ctx, mR, mT, 2, 1e-3, api.COMPRESSIBLE, fine_operator=fo, **kw)
    finally:
        dist.destroy_process_group()
    assert ssumm["iterations"] == summ["iterations"]
    assert [r["innerIterations"] for r in srecs] == [r["innerIterations"] for r in recs]
    assert abs(ssumm["finalGradNormRel"] - summ["finalGradNormRel"]) < 1e-8
