"""GPU: the host-buffer entry points of the Hessian (the drop-in call a host-side caller of
HessianOperator::apply makes, inverse.hpp:83): vrg_hess_apply_host and the pipelined
vrg_hess_apply_host_batch give bit-identical results to the device apply, and the batch
reports the reference's error at the matvec that raised it; the queued device batch
(vrg_hess_apply_batch) likewise."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1604_02153_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1604_02153_b200 import api as A

    return A


def _operator(ctx, api, n, nt, deformation):
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    F = ctx.field
    return api.HessianOperator(ctx, (F(0.5 * v1), F(0.5 * v2)), F(mT), F(mT), api.H2SEMI, 1e-3, deformation, nt)


def _pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.copy_(torch.from_numpy(a))
    return t


@pytest.mark.parametrize("n,nt,deformation,pinned", [(256, 4, 0, True), (128, 3, 1, False), (512, 8, 0, True)])
def test_apply_host_batch_matches_device_apply(ctx, api, n, nt, deformation, pinned):
    H = _operator(ctx, api, n, nt, deformation)
    k = 5
    vts = [synth.smooth_velocity(n, n, 3000 + i) for i in range(k)]
    want = []
    for a, b in vts:
        o = H.apply((ctx.field(a), ctx.field(b)))
        want.append(np.stack([o[0].cpu().numpy(), o[1].cpu().numpy()]))
    conv = _pinned if pinned else (lambda a: np.ascontiguousarray(a.copy()))
    hin = [(conv(a), conv(b)) for a, b in vts]
    hout = [(conv(np.zeros((n, n))), conv(np.zeros((n, n)))) for _ in range(k)]
    for rep in range(3):  # direct, graph capture, replay of both device slots
        for o in hout:
            o[0].fill(np.nan) if not pinned else o[0].fill_(float("nan"))
        H.apply_host_batch(hin, hout)
        for i in range(k):
            got = np.stack([np.asarray(hout[i][0]), np.asarray(hout[i][1])])
            assert np.array_equal(got, want[i]), (rep, i)
    # the single-call host entry point
    o1, o2 = conv(np.zeros((n, n))), conv(np.zeros((n, n)))
    H.apply_host(hin[2][0], hin[2][1], o1, o2)
    assert np.array_equal(np.stack([np.asarray(o1), np.asarray(o2)]), want[2])
    H.apply_host_batch([], [])  # k = 0 is a no-op


def test_apply_host_batch_error_at_the_failing_matvec(ctx, api):
    n = 128
    H = _operator(ctx, api, n, 4, 0)
    good = [synth.smooth_velocity(n, n, 5000 + i) for i in range(4)]
    bad = (good[2][0].copy(), good[2][1].copy())
    bad[0][7, 9] = np.nan
    hin = [good[0], good[1], bad, good[3]]
    hout = [(np.full((n, n), -1.0), np.full((n, n), -1.0)) for _ in range(4)]
    with pytest.raises(api.InvalidArgument, match="non-finite"):
        H.apply_host_batch(hin, hout)
    ref0 = H.apply((ctx.field(good[0][0]), ctx.field(good[0][1])))
    assert np.array_equal(hout[0][0], ref0[0].cpu().numpy())  # matvecs before the failing one delivered
    assert np.all(hout[3][0] == -1.0)  # nothing after it ran
    # the operator is still usable after the error
    H.apply_host_batch(hin[:2], hout[:2])
    assert np.array_equal(hout[0][0], ref0[0].cpu().numpy())


@pytest.mark.parametrize("n,nt,deformation", [(256, 4, 0), (128, 3, 1), (1024, 4, 0)])
def test_apply_batch_matches_device_apply(ctx, api, n, nt, deformation):
    """Queued device matvecs (each guard checked while the next matvec runs) give the same bits
    as apply() one call at a time, through direct launches, the capture and graph replays."""
    H = _operator(ctx, api, n, nt, deformation)
    k = 5
    vts = [tuple(ctx.field(x) for x in synth.smooth_velocity(n, n, 3000 + i)) for i in range(k)]
    want = [[t.cpu().numpy() for t in H.apply(vt)] for vt in vts]
    outs = [(ctx.empty(n, n), ctx.empty(n, n)) for _ in range(k)]
    for rep in range(3):
        for o in outs:
            o[0].fill_(float("nan"))
            o[1].fill_(float("nan"))
        H.apply_batch(vts, outs)
        for i in range(k):
            assert np.array_equal(outs[i][0].cpu().numpy(), want[i][0]), (rep, i)
            assert np.array_equal(outs[i][1].cpu().numpy(), want[i][1]), (rep, i)
    # alternating inputs into one output (the bench's timed loop): the last input's result
    H.apply_batch([vts[i & 1] for i in range(6)], [outs[0]] * 6)
    assert np.array_equal(outs[0][0].cpu().numpy(), want[1][0])
    H.apply_batch([], [])


def test_apply_batch_error_at_the_failing_matvec(ctx, api):
    n = 128
    H = _operator(ctx, api, n, 4, 0)
    good = [synth.smooth_velocity(n, n, 5000 + i) for i in range(4)]
    bad = (good[2][0].copy(), good[2][1].copy())
    bad[0][7, 9] = np.nan
    vts = [tuple(ctx.field(x) for x in p) for p in (good[0], good[1], bad, good[3])]
    outs = [(ctx.field(np.full((n, n), -1.0)), ctx.field(np.full((n, n), -1.0))) for _ in range(4)]
    with pytest.raises(api.InvalidArgument, match="non-finite"):
        H.apply_batch(vts, outs)
    ref0 = H.apply(vts[0])
    ref1 = H.apply(vts[1])
    assert np.array_equal(outs[0][0].cpu().numpy(), ref0[0].cpu().numpy())  # before the failing one: final
    assert np.array_equal(outs[1][1].cpu().numpy(), ref1[1].cpu().numpy())
    # the operator is still usable after the error
    H.apply_batch(vts[:2], outs[:2])
    assert np.array_equal(outs[1][0].cpu().numpy(), ref1[0].cpu().numpy())


@pytest.mark.parametrize("mode,scheme", [(1, 0), (0, 1)])
def test_apply_batch_on_operators_checked_per_call(ctx, api, mode, scheme):
    """Full-Newton (mode 1) and RK2 (scheme 1) operators check their guards their own way: the
    queued batch falls back to one checked apply per matvec, with the same results."""
    n, nt = 128, 4
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    F = ctx.field
    ctx.set_scheme(scheme)
    try:
        H = api.HessianOperator(ctx, (F(0.5 * v1), F(0.5 * v2)), F(mT), F(mT), api.H2SEMI, 1e-3, 0, nt, mode=mode)
        vts = [tuple(F(x) for x in synth.smooth_velocity(n, n, 3000 + i)) for i in range(3)]
        want = [[t.cpu().numpy() for t in H.apply(vt)] for vt in vts]
        outs = [(ctx.empty(n, n), ctx.empty(n, n)) for _ in range(3)]
        for _ in range(2):
            H.apply_batch(vts, outs)
            for i in range(3):
                assert np.array_equal(outs[i][0].cpu().numpy(), want[i][0])
                assert np.array_equal(outs[i][1].cpu().numpy(), want[i][1])
    finally:
        ctx.set_scheme(0)
