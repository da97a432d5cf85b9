"""GPU: the RK2 / RK2A spectral transport schemes (transport.cpp:129-195,
267-309, 345-377, 426-485; inverse.cpp:30-88) against the compiled reference, selected with
vrg_set_scheme / ref.set_scheme: every Solver entry point, the GN and full-Newton Hessian
(matvec, data term, counters), gradient/objective and a Newton registration.

The schemes take every derivative spectrally, so FFT rounding (cuFFT vs the reference's FFT) is
amplified by |k| per derivative: transport solves agree to ~1e-13, matvecs within the
conditioning floor of beta A (apply_floor) and 1e-10 for the data term."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1604_02153_b200 import synth

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def api():
    from paper_1604_02153_b200 import api as A

    return A


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def apply_floor(n, p, beta, vmax, outmax):
    kmax2 = 2.0 * (n // 2) ** 2
    return 4 * 2.2e-16 * beta * kmax2 ** p * vmax / outmax


@pytest.fixture(params=[1, 2], ids=["RK2", "RK2A"])
def scheme(request, ctx, ref):
    ctx.set_scheme(request.param)
    ref.set_scheme(request.param)
    yield request.param
    ctx.set_scheme(0)
    ref.set_scheme(0)


def _problem(n=48):
    mT, (v1, v2) = synth.config12_fields(n)
    return mT, 0.6 * v1, 0.6 * v2


def test_solver_entry_points(ctx, api, ref, scheme):
    n, nt = 48, 8
    mT, v1, v2 = _problem(n)
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    lt1 = synth.smoothed_noise(n, n, 1000) - 0.5
    F = ctx.field
    S = api.Solver(ctx, (F(v1), F(v2)), nt)
    st = ref.solve_state(v1, v2, nt, mT)
    assert rel(S.solve_state(F(mT)), st) < TOL
    assert rel(S.solve_state_final(F(mT)), ref.solve_state_final(v1, v2, nt, mT)) < TOL
    adj = ref.solve_adjoint(v1, v2, nt, lt1)
    assert rel(S.solve_adjoint(F(lt1)), adj) < TOL
    assert rel(S.solve_adjoint_final(F(lt1)), ref.solve_adjoint_final(v1, v2, nt, lt1)) < TOL
    inc = ref.solve_incstate(v1, v2, nt, mT, vt1, vt2)
    assert rel(S.solve_inc_state((F(vt1), F(vt2)), F(st)), inc) < TOL
    assert rel(S.solve_inc_adjoint((F(vt1), F(vt2)), F(lt1)), ref.solve_incadjoint_gn(v1, v2, nt, lt1)) < TOL
    fn = ref.solve_incadjoint_fn(v1, v2, nt, vt1, vt2, lt1, lt1)
    assert rel(S.solve_inc_adjoint((F(vt1), F(vt2)), F(lt1), adjoint=F(adj), mode=api.FULL_NEWTON), fn) < TOL
    assert rel(S.jacobian_determinant(), ref.jacobian_det(v1, v2, nt)) < TOL


@pytest.mark.parametrize("mode,deform", [(0, 0), (1, 0), (0, 1)])
def test_hessian_vs_reference(ctx, api, ref, scheme, mode, deform):
    n, nt = 48, 8
    mT, v1, v2 = _problem(n)
    mR = ref.solve_state_final(v1 / 0.6, v2 / 0.6, nt, mT)
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    F = ctx.field
    ref.counters_reset()
    R = ref.Hessian(v1, v2, mR, mT, 2, 1e-2, deform, nt, mode=mode)
    rc = ref.counters()
    ctx.reset_counters()
    H = api.HessianOperator(ctx, (F(v1), F(v2)), F(mR), F(mT), api.H2SEMI, 1e-2, deform, nt, mode=mode)
    assert ctx.counters() == rc
    vt = (F(vt1), F(vt2))
    for _ in range(2):
        ref.counters_reset()
        e1, e2 = R.apply(vt1, vt2)
        rc = ref.counters()
        ctx.reset_counters()
        h1, h2 = H.apply(vt)
        assert ctx.counters() == rc
        tol = max(TOL, apply_floor(n, 2, 1e-2, max(np.abs(vt1).max(), np.abs(vt2).max()), np.abs(e1).max()))
        assert rel(h1, e1) < tol and rel(h2, e2) < tol
    d1, d2 = R.apply(vt1, vt2, data_only=True)
    g1, g2 = H.apply_data_term(vt)
    assert rel(g1, d1) < TOL and rel(g2, d2) < TOL


def test_gradient_objective_vs_reference(ctx, api, ref, scheme):
    n, nt = 48, 8
    mT, v1, v2 = _problem(n)
    mR = ref.solve_state_final(v1 / 0.6, v2 / 0.6, nt, mT)
    F = ctx.field
    (g1, g2), sc = api.evaluate_gradient(ctx, (F(v1), F(v2)), F(mR), F(mT), api.H2SEMI, 1e-2, 0, nt)
    r1, r2, rsc = ref.evaluate_gradient(v1, v2, mR, mT, 2, 1e-2, 0, nt)
    tol = max(TOL, apply_floor(n, 2, 1e-2, max(np.abs(v1).max(), np.abs(v2).max()), np.abs(r1).max()))
    assert rel(g1, r1) < tol and rel(g2, r2) < tol
    assert abs(sc[0] - rsc[0]) <= 1e-12 * abs(rsc[0])
    osc = api.evaluate_objective(ctx, (F(v1), F(v2)), F(mR), F(mT), api.H2SEMI, 1e-2, 0, nt)
    assert abs(osc[0] - ref.evaluate_objective(v1, v2, mR, mT, 2, 1e-2, 0, nt)[0]) <= 1e-12 * abs(rsc[0])


def test_newton_vs_reference(ctx, api, ref, scheme):
    n, nt = 64, 8
    mT, (v1, v2) = synth.config12_fields(n)
    mR = ref.solve_state_final(v1, v2, nt, mT)
    _, _, rrep, rs = ref.newton_solve(mR, mT, 2, 1e-2, 0, nt=nt, two_level=True, cheb=False, tol_rel=1e-2)
    _, _, recs, summ = api.newton_solve(ctx, mR, mT, 2, 1e-2, 0, nt=nt, kind=api.PC_TWO_LEVEL,
                                        coarse_solver=api.COARSE_PCG, tol_rel=1e-2)
    assert summ["iterations"] == int(rs[1]) and summ["status"] == int(rs[0])
    g0 = rrep[0][1]
    for r, q in zip(recs, rrep):
        assert r["innerIterations"] == int(q[5]) and r["lineSearchSteps"] == int(q[6])
        assert abs(r["objective"] - q[3]) <= 1e-8 * abs(q[3])
        assert abs(r["gradNormInf"] - q[1]) <= 1e-7 * g0
