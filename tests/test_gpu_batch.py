"""GPU: batched registration (C ABI vrg_newton_solve_batch, csrc/batch.cu) — P image pairs solved in
lockstep in the same kernel launches must give each pair exactly its own newtonSolve: identical
Newton / Krylov / line-search counts, step lengths and op counters, and the same iterates; and on
the config-5b pairs the reference's own records (tests/golden/newton_cfg3_5b.npz)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from paper_1604_02153_b200 import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))


@pytest.fixture(scope="module")
def api():
    from paper_1604_02153_b200 import api as A

    return A


def _pairs(ctx, api, n, nt, seeds, vmax=0.3):
    out = []
    for p in seeds:
        mT = synth.smoothed_noise(n, n, 1000 + p)
        v1, v2 = synth.smooth_velocity(n, n, 2000 + p, vmax)
        mR = api.Solver(ctx, (ctx.field(v1), ctx.field(v2)), nt).solve_state_final(ctx.field(mT)).cpu().numpy()
        out.append((mR, mT))
    return out


def _same(single, batched, exact):
    v1, v2, recs, summ = single
    w1, w2, brecs, bsumm = batched
    assert bsumm["error"] == 0
    assert summ["status"] == bsumm["status"] and summ["iterations"] == bsumm["iterations"]
    for r, b in zip(recs, brecs):
        for key in ("iter", "innerIterations", "lineSearchSteps", "stepLength", "ffts", "interps"):
            assert r[key] == b[key], (key, r, b)
        for key in ("objective", "mismatch", "gradNormInf", "gradNormRel", "searchDirDivRatio"):
            if exact:
                assert r[key] == b[key], (key, r[key], b[key])
            else:
                assert abs(r[key] - b[key]) <= 1e-12 * max(abs(r[key]), 1e-300), (key, r[key], b[key])
    for key in ("finalGradNormRel", "finalResidualRel", "jacMin", "jacMax"):
        assert abs(summ[key] - bsumm[key]) <= 1e-12 * max(abs(summ[key]), 1e-300), key
    err = max(np.abs(v1 - w1).max(), np.abs(v2 - w2).max()) / max(np.abs(v1).max(), np.abs(v2).max())
    assert err <= (0.0 if exact else 1e-12), err


@pytest.mark.parametrize("n,nt,P", [(128, 4, 3), (256, 8, 2), (64, 3, 5)])
def test_batched_hessian_equals_single(ctx, api, n, nt, P):
    """A HessianOperator of P stacked pairs (vrg_hess_create_batch): its state solve, per-iterate
    invariants and data term / full / split matvecs give every pair its own operator's result,
    bit for bit."""
    import ctypes as C

    from paper_1604_02153_b200.api import _p

    vs, ms, ts = [], [], []
    for p in range(P):
        v1, v2 = synth.smooth_velocity(n, n, 2000 + p)
        vs.append((0.5 * v1, 0.5 * v2))
        ms.append(synth.smoothed_noise(n, n, 1000 + p))
        ts.append(synth.smooth_velocity(n, n, 3000 + p))
    F = ctx.field
    V1, V2 = F(np.stack([v[0] for v in vs])), F(np.stack([v[1] for v in vs]))
    MT = F(np.stack(ms))
    MR = F(np.stack([np.roll(m, 3, axis=1) for m in ms]))
    T1, T2 = F(np.stack([t[0] for t in ts])), F(np.stack([t[1] for t in ts]))
    h = C.c_void_p()
    ctx.check(ctx.lib.vrg_hess_create_batch(ctx.h, n, n, P, _p(V1), _p(V2), _p(MR), _p(MT), 2, 1e-3, 0, nt,
                                            C.byref(h)))
    outs = {}
    try:
        for name, fn in (("data", ctx.lib.vrg_hess_apply_data), ("apply", ctx.lib.vrg_hess_apply),
                         ("split", ctx.lib.vrg_hess_apply_split)):
            for rep in range(2):  # direct launch, then graph replay
                o1, o2 = ctx.empty(P, n, n), ctx.empty(P, n, n)
                ctx.check(fn(h, _p(T1), _p(T2), _p(o1), _p(o2)))
                outs[name, rep] = (o1.cpu().numpy(), o2.cpu().numpy())
    finally:
        ctx.lib.vrg_hess_destroy(h)
    for p in range(P):
        H = api.HessianOperator(ctx, (F(vs[p][0]), F(vs[p][1])), F(np.roll(ms[p], 3, axis=1)), F(ms[p]), 2, 1e-3,
                                api.COMPRESSIBLE, nt)
        vt = (F(ts[p][0]), F(ts[p][1]))
        single = {"data": H.apply_data_term(vt), "apply": H.apply(vt), "split": H.apply_split(vt)}
        for name, (s1, s2) in single.items():
            for rep in range(2):
                b1, b2 = outs[name, rep]
                assert np.array_equal(b1[p], s1.cpu().numpy()) and np.array_equal(b2[p], s2.cpu().numpy()), (name, p)


@pytest.mark.parametrize("kind,n,nt,P", [("2l", 128, 8, 5), ("reg", 64, 4, 3), ("2l", 256, 16, 2)])
def test_batch_equals_single_pair_solves(ctx, api, kind, n, nt, P):
    """Each pair of a batch takes its own solve's decisions and arithmetic: the batch's records
    and velocities equal the per-pair newton_solve's, bit for bit (reductions per pair with the
    single-field partition, masked per-pair updates, coarse groups per coarse step count)."""
    imgs = _pairs(ctx, api, n, nt, range(P))
    pc = dict(kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB, cheb_iters=10) if kind == "2l" else \
        dict(kind=api.PC_REG)
    single = [api.newton_solve(ctx, mR, mT, api.H2SEMI, 1e-3, api.COMPRESSIBLE, nt=nt, tol_rel=1e-2, **pc)
              for mR, mT in imgs]
    mR = np.stack([a for a, _ in imgs])
    mT = np.stack([b for _, b in imgs])
    batched = api.newton_solve_batch(ctx, mR, mT, api.H2SEMI, 1e-3, api.COMPRESSIBLE, nt=nt, tol_rel=1e-2, **pc)
    assert len(batched) == P
    for s, b in zip(single, batched):
        _same(s, b, exact=True)


def test_batch_of_one_and_pair_order(ctx, api):
    """A batch of one pair is the single solve; permuting the pairs of a batch permutes the
    results (no cross-pair coupling)."""
    n, nt = 128, 8
    imgs = _pairs(ctx, api, n, nt, range(3))
    mR = np.stack([a for a, _ in imgs])
    mT = np.stack([b for _, b in imgs])
    kw = dict(nt=nt, tol_rel=1e-2, kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB, cheb_iters=10)
    one = api.newton_solve_batch(ctx, mR[:1], mT[:1], api.H2SEMI, 1e-3, api.COMPRESSIBLE, **kw)[0]
    single = api.newton_solve(ctx, mR[0], mT[0], api.H2SEMI, 1e-3, api.COMPRESSIBLE, **kw)
    _same(single, one, exact=True)
    fwd = api.newton_solve_batch(ctx, mR, mT, api.H2SEMI, 1e-3, api.COMPRESSIBLE, **kw)
    rev = api.newton_solve_batch(ctx, mR[::-1].copy(), mT[::-1].copy(), api.H2SEMI, 1e-3, api.COMPRESSIBLE, **kw)
    for a, b in zip(fwd, rev[::-1]):
        _same(a, b, exact=True)


def test_batch_config5b_vs_reference(ctx, api, ref):
    """Config 5b pairs 0-3 (256^2, nt=16, H2 beta=1e-3, 2L + CHEB(10)) in one batch against the
    reference's newtonSolve records of each pair (identical counts, objectives within 1e-8)."""
    from test_gpu_headline_parity import _check_records, gold

    d = gold("newton_cfg3_5b")
    names = ["cfg5b_p0", "cfg5b_p1", "cfg5b_p2", "cfg5b_p3"]
    mRs, mTs = [], []
    for p, name in enumerate(names):
        meta = d[name + "_meta"]
        n, nt, beta = int(meta[0]), int(meta[2]), float(meta[4])
        mT = synth.smoothed_noise(n, n, 1000 + p)
        v1, v2 = synth.smooth_velocity(n, n, 2000 + p)
        mRs.append(ref.solve_state_final(v1, v2, nt, mT))
        mTs.append(mT)
    out = api.newton_solve_batch(ctx, np.stack(mRs), np.stack(mTs), 2, beta, api.COMPRESSIBLE, nt=nt,
                                 kind=api.PC_TWO_LEVEL, coarse_solver=api.COARSE_CHEB, cheb_iters=10, tol_rel=1e-2)
    for (w1, w2, recs, summ), name in zip(out, names):
        assert summ["error"] == 0
        _check_records(recs, summ, d[name + "_records"], d[name + "_summary"])
