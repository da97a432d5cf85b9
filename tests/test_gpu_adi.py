"""GPU: alternating-direction fused SL steps (adi.cuh: one kernel per step, the prefilter fused,
taps from shared memory) against the band path on the same inputs.  The two differ only in
the order of the two commuting 1-D prefilter passes, i.e. at rounding level."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1604_02153_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_1604_02153_b200 import api as A

    return A


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _solve_state(ctx, api, monkeypatch, adi, v, m0, nt):
    if adi:
        monkeypatch.setenv("VRG_ADI", "1")
    else:
        monkeypatch.delenv("VRG_ADI", raising=False)
    S = api.Solver(ctx, v, nt)
    return S.solve_state(m0).cpu().numpy()


@pytest.mark.parametrize("n1,n2,nt,scale", [(256, 256, 4, 1.0), (512, 512, 8, 1.0), (1024, 1024, 16, 1.0),
                                            (256, 512, 3, 1.0), (96, 1280, 2, 0.5), (160, 256, 2, 2.0),
                                            (1024, 1024, 2, 3.0)])
def test_adi_state_vs_band(ctx, api, monkeypatch, n1, n2, nt, scale):
    m0 = ctx.field(synth.smoothed_noise(n1, n2, 1000))
    v1, v2 = synth.smooth_velocity(n1, n2, 2000)
    v = (ctx.field(scale * v1), ctx.field(scale * v2))
    a = _solve_state(ctx, api, monkeypatch, True, v, m0, nt)
    b = _solve_state(ctx, api, monkeypatch, False, v, m0, nt)
    assert rel(a, b) <= 1e-13


def test_adi_identity_and_guard(ctx, api, monkeypatch):
    n, nt = 256, 4
    m0 = synth.smoothed_noise(n, n, 7)
    z = ctx.field(np.zeros((n, n)))
    tr = _solve_state(ctx, api, monkeypatch, True, (z, z), ctx.field(m0), nt)
    assert rel(tr[-1], m0) < 1e-14  # v = 0: every step reproduces the field
    bad = m0.copy()
    bad[3, 5] = np.nan
    monkeypatch.setenv("VRG_ADI", "1")
    with pytest.raises(api.InvalidArgument, match="prefilter: non-finite value"):
        api.Solver(ctx, (z, z), nt).solve_state(ctx.field(bad))
