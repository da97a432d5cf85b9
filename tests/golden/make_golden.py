"""Generates the committed golden vectors tests/golden/*.npz from the UNMODIFIED reference
compiled in oracle/_ref (run in the build container, where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

The reference ships no fixture files, so these vectors are produced by
running its own public API on seeded synthetic inputs (paper_1604_02153_b200/synth.py).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_1604_02153_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def case_cfg1():
    """Config 1 problem (64^2, nt=4, H2, beta=1e-2): transport, matvec, gradient."""
    n, nt, beta = 64, 4, 1e-2
    mT, (v1, v2) = synth.config12_fields(n)
    mR = ref.solve_state_final(v1, v2, nt, mT)
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    lam1 = synth.smooth_scalar(n, n, 77)
    # iterate away from the truth so the residual and adjoint are non-trivial
    w1, w2 = 0.6 * v1, 0.6 * v2
    d = {"mT": mT, "v1": v1, "v2": v2, "mR": mR, "vt1": vt1, "vt2": vt2, "lam1": lam1, "w1": w1, "w2": w2}
    d["state"] = ref.solve_state(w1, w2, nt, mT)
    d["adjoint"] = ref.solve_adjoint(w1, w2, nt, lam1)
    d["incstate"] = ref.solve_incstate(w1, w2, nt, mT, vt1, vt2)
    d["xf1"], d["xf2"] = ref.trace(w1, w2, 1.0 / nt)
    d["xb1"], d["xb2"] = ref.trace(w1, w2, 1.0 / nt, True)
    H = ref.Hessian(w1, w2, mR, mT, 2, beta, 0, nt)
    d["hv1"], d["hv2"] = H.apply(vt1, vt2)
    d["dt1"], d["dt2"] = H.apply(vt1, vt2, data_only=True)
    g1, g2, sc = ref.evaluate_gradient(w1, w2, mR, mT, 2, beta, 0, nt)
    d["g1"], d["g2"], d["gscalars"] = g1, g2, sc
    d["oscalars"] = ref.evaluate_objective(w1, w2, mR, mT, 2, beta, 0, nt)
    ref.counters_reset()
    ref.solve_state(w1, w2, nt, mT)
    d["count_state"] = np.array(ref.counters())
    ref.counters_reset()
    ref.solve_adjoint(w1, w2, nt, lam1)
    d["count_adjoint"] = np.array(ref.counters())
    d["meta"] = np.array([n, nt, beta])
    return d


def case_incompressible():
    """Config 2 flavour at 64^2: H1, beta=1e-3, Leray-projected, nt=8."""
    n, nt, beta = 64, 8, 1e-3
    mT, (v1, v2) = synth.config12_fields(n)
    mR = ref.solve_state_final(v1, v2, nt, mT)
    vt1, vt2 = synth.smooth_velocity(n, n, 3001)
    w1, w2 = 0.5 * v1, 0.5 * v2
    H = ref.Hessian(w1, w2, mR, mT, 1, beta, 1, nt)
    d = {"mT": mT, "mR": mR, "vt1": vt1, "vt2": vt2, "w1": w1, "w2": w2}
    d["hv1"], d["hv2"] = H.apply(vt1, vt2)
    g1, g2, sc = ref.evaluate_gradient(w1, w2, mR, mT, 1, beta, 1, nt)
    d["g1"], d["g2"], d["gscalars"] = g1, g2, sc
    d["meta"] = np.array([n, nt, beta])
    return d


def case_interp_spectral():
    """Non-square, non-power-of-two grid 48 x 32: interp + spectral operators."""
    n1, n2 = 48, 32
    u = ref.random_bandlimited_field(n1, n2, 3)
    a1, a2 = synth.smooth_velocity(n1, n2, 11)
    rng = np.random.default_rng(5)
    x1 = rng.uniform(-10.0, 10.0, (n1, n2))
    x2 = rng.uniform(-10.0, 10.0, (n1, n2))
    d = {"u": u, "a1": a1, "a2": a2, "x1": x1, "x2": x2}
    c = ref.prefilter(u)
    d["coef"] = c
    d["eval"] = ref.evaluate(c, x1, x2)
    d["grad1"], d["grad2"] = ref.gradient(u)
    d["div"] = ref.divergence(a1, a2)
    d["reg1"], d["reg2"] = ref.apply_reg(a1, a2, 2, 1e-2)
    d["ireg1"], d["ireg2"] = ref.apply_inv_reg(a1, a2, 2, 1e-2, -0.5)
    d["leray1"], d["leray2"] = ref.project_div_free(a1, a2)
    d["restrict"] = ref.resample(u, 24, 16)
    d["prolong"] = ref.resample(d["restrict"], 48, 32)
    d["low"] = ref.cutoff(u, False)
    d["high"] = ref.cutoff(u, True)
    d["rbl_seed3"] = u
    return d


NEWTON_RUNS = {
    # name: (n, nt, norm, beta, deformation, chebyshev coarse solver)
    "cfg1": (64, 4, 2, 1e-2, 0, False),          # config 1: 2L + nested PCG (eps 0.1)
    "cfg2": (256, 8, 1, 1e-3, 0, True),          # config 2: 2L + CHEB(10)
    "cfg2_incomp": (256, 8, 1, 1e-3, 1, True),   # config 2, div v = 0
}


def case_newton():
    """Full inexact GN-Krylov registrations (newtonSolve) of configs 1 and 2, tolRelGrad 1e-2."""
    d = {}
    for name, (n, nt, norm, beta, deform, cheb) in NEWTON_RUNS.items():
        mT, (v1, v2) = synth.config12_fields(n)
        mR = ref.solve_state_final(v1, v2, nt, mT)
        a, b, rep, s = ref.newton_solve(mR, mT, norm, beta, deform, nt=nt, two_level=True, cheb=cheb,
                                        cheb_iters=10, tol_rel=1e-2)
        d[name + "_records"] = rep
        d[name + "_summary"] = s
        d[name + "_v1"] = a
        d[name + "_v2"] = b
        d[name + "_meta"] = np.array([n, nt, norm, beta, deform, int(cheb)])
    return d


def case_precond():
    """Two-level preconditioner and Lanczos estimate at 64^2 (config 1 problem, iterate 0.6 v*)."""
    n, nt, beta = 64, 4, 1e-2
    mT, (v1, v2) = synth.config12_fields(n)
    mR = ref.solve_state_final(v1, v2, nt, mT)
    w1, w2 = 0.6 * v1, 0.6 * v2
    r1, r2 = synth.smooth_velocity(n, n, 3002)
    c = ref.Coarse(w1, w2, mR, mT, 2, beta, 0)
    emin, emax = ref.estimate_eigs(mR, mT, 2, beta, 0)
    d = {"mR": mR, "mT": mT, "w1": w1, "w2": w2, "r1": r1, "r2": r2, "eig": np.array([emin, emax])}
    d["cheb1"], d["cheb2"] = c.two_level(r1, r2, 1, 10, 0.1, 0.5, emin, emax)
    d["pcg1"], d["pcg2"] = c.two_level(r1, r2, 0, 10, 0.1, 0.5, emin, emax)
    s1, s2 = ref.random_bandlimited_velocity(n // 2, n // 2, 5)
    d["s1"], d["s2"] = s1, s2
    d["split1"], d["split2"] = c.split_apply(s1, s2)
    d["rbl_coarse_0x5eed"] = ref.random_bandlimited_field(n // 2, n // 2, 0x5EED)
    return d


def main():
    for name, fn in [("cfg1_64", case_cfg1), ("incomp_64", case_incompressible), ("interp_48x32", case_interp_spectral),
                     ("precond_64", case_precond), ("newton", case_newton)]:
        d = fn()
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
        print(name, sorted(d))


if __name__ == "__main__":
    main()
