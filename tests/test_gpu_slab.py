"""GPU: slab-decomposed GN Hessian matvec against the single-device
operator on the same inputs, with G virtual slabs on one device (LocalComm: every slab's work
runs in turn, exchanges are copies; no kernels of different slabs wait on one another).  The
multi-process NCCL path uses the same code with DistComm (tests/test_slab_cpu.py covers its
host logic over gloo)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1604_02153_b200 import slab, synth

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def api():
    from paper_1604_02153_b200 import api as A

    return A


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def apply_floor(n, p, beta, vmax, outmax):
    kmax2 = 2.0 * (n // 2) ** 2
    return 4 * 2.2e-16 * beta * kmax2 ** p * vmax / outmax


@pytest.mark.parametrize("n,nt,G", [(256, 4, 1), (256, 4, 2), (256, 8, 4), (512, 8, 4), (256, 4, 8)])
def test_slab_matvec_vs_single_device(ctx, api, n, nt, G):
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    F = ctx.field
    w = (F(0.5 * v1), F(0.5 * v2))
    H = api.HessianOperator(ctx, w, F(mT), F(mT), 2, 1e-3, api.COMPRESSIBLE, nt)
    vt = (F(vt1), F(vt2))
    d1, d2 = H.apply_data_term(vt)
    h1, h2 = H.apply(vt)
    comm = slab.LocalComm(G)
    S = slab.SlabHessian.from_operator(ctx, comm, H, 2, 1e-3)
    L = n // G
    vts = [ctx.field(np.stack([vt1[i * L:(i + 1) * L], vt2[i * L:(i + 1) * L]])) for i in range(G)]
    dt = S.apply(vts, data_term_only=True)
    got = np.concatenate([o.cpu().numpy() for o in dt], axis=1)
    assert rel(got[0], d1.cpu().numpy()) < TOL and rel(got[1], d2.cpu().numpy()) < TOL
    full = S.apply(vts)
    got = np.concatenate([o.cpu().numpy() for o in full], axis=1)
    e1 = h1.cpu().numpy()
    tol = max(TOL, apply_floor(n, 2, 1e-3, max(np.abs(vt1).max(), np.abs(vt2).max()), np.abs(e1).max()))
    assert rel(got[0], e1) < tol and rel(got[1], h2.cpu().numpy()) < tol


def test_slab_window_too_small_is_detected(ctx, api):
    n, nt, G = 256, 4, 2
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    F = ctx.field
    H = api.HessianOperator(ctx, (F(v1), F(v2)), F(mT), F(mT), 2, 1e-3, api.COMPRESSIBLE, nt)
    S = slab.SlabHessian.from_operator(ctx, slab.LocalComm(G), H, 2, 1e-3)
    S.geo = slab.SlabGeometry(n, n, G, 0)  # pretend the departure points stay in their rows
    S._alloc_windows()
    L = n // G
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    vts = [ctx.field(np.stack([vt1[i * L:(i + 1) * L], vt2[i * L:(i + 1) * L]])) for i in range(G)]
    with pytest.raises(api.VrgError, match="window too small"):
        S.apply(vts)


@pytest.mark.parametrize("n,nt,G", [(256, 4, 2), (512, 8, 4)])
def test_slab_distributed_setup_vs_single_device(ctx, api, n, nt, G):
    """SlabHessian.build: departure points, state, gradients, (grad m)_D, div v, (div v)_D and
    the matvec computed on the slabs, against the single-device operator."""
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    F = ctx.field
    H = api.HessianOperator(ctx, (F(v1), F(v2)), F(mT), F(mT), 2, 1e-3, api.COMPRESSIBLE, nt)
    ref = slab.SlabHessian.from_operator(ctx, slab.LocalComm(G), H, 2, 1e-3)
    L = n // G
    comm = slab.LocalComm(G)
    vs = [F(np.stack([v1[i * L:(i + 1) * L], v2[i * L:(i + 1) * L]])) for i in range(G)]
    mTs = [F(mT[i * L:(i + 1) * L]) for i in range(G)]
    S = slab.SlabHessian.build(ctx, comm, vs, mTs, n, nt, 2, 1e-3)
    for key in ("Xf", "Xb", "G", "GD", "dv", "dvd"):
        got = np.concatenate([p[key].cpu().numpy() for p in S.parts], axis=-2)
        exp = np.concatenate([p[key].cpu().numpy() for p in ref.parts], axis=-2)
        assert rel(got, exp) < TOL, key
    state = np.concatenate([p["m"].cpu().numpy() for p in S.parts], axis=-2)
    assert rel(state, H.state().cpu().numpy()) < TOL
    vts = [F(np.stack([vt1[i * L:(i + 1) * L], vt2[i * L:(i + 1) * L]])) for i in range(G)]
    d1, d2 = H.apply_data_term((F(vt1), F(vt2)))
    got = np.concatenate([o.cpu().numpy() for o in S.apply(vts, data_term_only=True)], axis=1)
    assert rel(got[0], d1.cpu().numpy()) < TOL and rel(got[1], d2.cpu().numpy()) < TOL


def test_slab_state_guard(ctx, api):
    """The slab state solve raises the reference's blow-up error (amplifying velocity)."""
    n, nt, G = 64, 4, 2
    x = np.linspace(-np.pi, np.pi, n, endpoint=False)
    X1, X2 = np.meshgrid(x, x, indexing="ij")
    v1, v2 = 30 * np.sin(X1), 30 * np.sin(X2)  # compressive: the transported field blows up
    mT = np.cos(X1) + np.cos(X2)
    F = ctx.field
    L = n // G
    vs = [F(np.stack([v1[i * L:(i + 1) * L], v2[i * L:(i + 1) * L]])) for i in range(G)]
    mTs = [F(mT[i * L:(i + 1) * L]) for i in range(G)]
    with pytest.raises((api.BlowupError, api.VrgError)):
        slab.SlabHessian.build(ctx, slab.LocalComm(G), vs, mTs, n, nt, 2, 1e-3)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_slab_matvec_graph_replay_bit_identical(ctx, api, G):
    """The slab matvec's per-step orchestration captured into one CUDA graph (SlabHessian.apply:
    eager on the first uses of a pointer set, then captured, replayed afterwards) gives the
    eager bits, for the full matvec and the data term."""
    n, nt = 256, 4
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    F = ctx.field
    H = api.HessianOperator(ctx, (F(0.5 * v1), F(0.5 * v2)), F(mT), F(mT), 2, 1e-3, api.COMPRESSIBLE, nt)
    comm = slab.LocalComm(G)
    S = slab.SlabHessian.from_operator(ctx, comm, H, 2, 1e-3)
    L = n // G
    vts = [ctx.field(np.stack([vt1[i * L:(i + 1) * L], vt2[i * L:(i + 1) * L]])) for i in range(G)]
    outs = [ctx.empty(2, L, n) for _ in range(G)]
    for data_only in (False, True):
        runs = []
        for _ in range(S.capture_after + 3):  # eager runs, capture (+ replay), replays
            for o in outs:
                o.fill_(float("nan"))
            S.apply(vts, outs, data_term_only=data_only)
            runs.append(np.concatenate([o.cpu().numpy() for o in outs], axis=1))
        assert S._capturable(vts)
        for r in runs[1:]:
            assert np.array_equal(r, runs[0])
    assert sum(1 for e in S._graph_cache.values() if not isinstance(e, int)) == 2
