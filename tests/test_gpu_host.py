"""GPU: the host-buffer entry points of the Hessian (the drop-in call a host-side caller of
HessianOperator::apply makes, inverse.hpp:83): vrg_hess_apply_host and the pipelined
vrg_hess_apply_host_batch give bit-identical results to the device apply, and the batch
reports the reference's error at the matvec that raised it."""
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
