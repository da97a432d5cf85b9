"""Round-2 golden records of the configs the bench numbers are quoted on, produced by the
UNMODIFIED reference compiled in oracle/_ref (build container only, where /root/reference
exists):

    make -C oracle && python tests/golden/make_golden_r2.py [case ...]
    VRG_REF_LIB=libveloreg_ref_altfft.so python tests/golden/make_golden_r2.py newton_default_altfft

cases (each writes tests/golden/<case>.npz):
  newton_cfg3_5b  the reference's newtonSolve records of config 3 pair 0 (512^2) and config 5b
                  pairs 0..3 (256^2): nt=16, H2 beta=1e-3, 2L + CHEB(10), tolRelGrad 1e-2;
                  m_R = the reference's SL transport of m_T by v* (nt=16).  No fields are
                  stored: the GPU test regenerates the inputs (synth.py, seeded) and m_R
                  (oracle/_ref on the GPU box's host) and compares records.
  newton_default  the reference's default path: no ntOverride (the CFL ratchet of
                  newton.cpp:49-52, gradScheme cfl 1.0) with PrecondKind::Reg (the library
                  default, precond.hpp:17, precond.cpp:315-317) and with 2L + PCG / CHEB, on
                  the config 1 and config 2 problems.
  cfg5a_digest    config 5a (4096^2, nt=32, H2 beta=1e-4): one SL state solve of the
                  smoothed-noise template at the iterate w = v*/2, and one GN data term
                  (HessianOperator::applyDataTerm, inverse.cpp:235-237) at w along a smooth
                  random direction.  A 4096^2 trajectory is 4.2 GB, so the digest holds the
                  values at 16384 seeded sample nodes of frames 1, 16, 32 and of both data
                  term components, plus every frame's L2 norm and both components' norms.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_1604_02153_b200 import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, n, pair): the batched-pairs configs, recipe of SURVEY §8d (nt=16, H2 1e-3, 2L-CHEB(10))
PAIR_RUNS = [("cfg3_p0", 512, 0), ("cfg5b_p0", 256, 0), ("cfg5b_p1", 256, 1), ("cfg5b_p2", 256, 2),
             ("cfg5b_p3", 256, 3)]
PAIR_NT, PAIR_BETA = 16, 1e-3

# name: (problem n, norm, beta, two_level, cheb); all with nt=0 (CFL ratchet, cfl 1.0)
DEFAULT_RUNS = {
    "cfg1_reg": (64, 2, 1e-2, False, False),
    "cfg1_2lpcg": (64, 2, 1e-2, True, False),
    "cfg2_2lcheb": (256, 1, 1e-3, True, True),
    "cfg2_reg": (256, 1, 1e-3, False, False),
}
DEFAULT_MR_NT = {64: 4, 256: 8}  # the m_R of configs 1/2 is made with their own nt

CFG5A = dict(n=4096, nt=32, beta=1e-4, samples=16384, sample_seed=4242, frames=(1, 16, 32))


def pair_images(n: int, p: int):
    """m_T (seed 1000+p), v* (2000+p), m_R = reference SL transport of m_T by v* (nt=16)."""
    mT = synth.smoothed_noise(n, n, 1000 + p)
    v1, v2 = synth.smooth_velocity(n, n, 2000 + p)
    return ref.solve_state_final(v1, v2, PAIR_NT, mT), mT


def sample_nodes(n: int, count: int, seed: int) -> np.ndarray:
    return (synth.splitmix64(seed, count) % np.uint64(n * n)).astype(np.int64)


def case_newton_cfg3_5b():
    d = {}
    for name, n, p in PAIR_RUNS:
        t0 = time.perf_counter()
        mR, mT = pair_images(n, p)
        _, _, rep, s = ref.newton_solve(mR, mT, 2, PAIR_BETA, 0, nt=PAIR_NT, two_level=True, cheb=True,
                                        cheb_iters=10, tol_rel=1e-2)
        d[name + "_records"], d[name + "_summary"] = rep, s
        d[name + "_meta"] = np.array([n, p, PAIR_NT, 2, PAIR_BETA])
        print(name, f"{time.perf_counter() - t0:.1f}s", int(s[1]), "iterations", flush=True)
    return d


def case_newton_default():
    d = {}
    for name, (n, norm, beta, two_level, cheb) in DEFAULT_RUNS.items():
        t0 = time.perf_counter()
        mT, (v1, v2) = synth.config12_fields(n)
        mR = ref.solve_state_final(v1, v2, DEFAULT_MR_NT[n], mT)
        _, _, rep, s = ref.newton_solve(mR, mT, norm, beta, 0, nt=0, two_level=two_level, cheb=cheb,
                                        cheb_iters=10, tol_rel=1e-2)
        d[name + "_records"], d[name + "_summary"] = rep, s
        d[name + "_meta"] = np.array([n, norm, beta, int(two_level), int(cheb)])
        print(name, f"{time.perf_counter() - t0:.1f}s", int(s[1]), "iterations", flush=True)
    return d


def case_cfg5a_digest():
    c = CFG5A
    n, nt, beta = c["n"], c["nt"], c["beta"]
    t0 = time.perf_counter()
    mT = synth.smoothed_noise(n, n, 1000)
    v1, v2 = synth.smooth_velocity(n, n, 2000)
    w1, w2 = 0.5 * v1, 0.5 * v2
    vt1, vt2 = synth.smooth_velocity(n, n, 3000)
    idx = sample_nodes(n, c["samples"], c["sample_seed"])
    d = {"idx": idx, "meta": np.array([n, nt, beta, c["samples"], c["sample_seed"]])}
    traj = ref.solve_state(w1, w2, nt, mT)
    d["state_norms"] = np.sqrt((traj.reshape(nt + 1, -1) ** 2).sum(axis=1))
    d["state_frames"] = np.array(c["frames"])
    d["state_samples"] = np.stack([traj[j].reshape(-1)[idx] for j in c["frames"]])
    del traj
    print("cfg5a state", f"{time.perf_counter() - t0:.1f}s", flush=True)
    H = ref.Hessian(w1, w2, mT, mT, 2, beta, 0, nt)
    o1, o2 = H.apply(vt1, vt2, data_only=True)
    del H
    d["data_norms"] = np.array([np.sqrt((o1 ** 2).sum()), np.sqrt((o2 ** 2).sum())])
    d["data_samples"] = np.stack([o1.reshape(-1)[idx], o2.reshape(-1)[idx]])
    print("cfg5a data term", f"{time.perf_counter() - t0:.1f}s", flush=True)
    return d


def case_newton_default_altfft():
    """The newton_default runs on the reference rebuilt over a differently-rounded correct FFT
    (oracle/_ref/libveloreg_ref_altfft.so: the shim's recursive mixed-radix path for every
    length).  Its distance from newton_default is the reference-vs-reference floor of each
    record: a Newton iterate whose Krylov solve sits near the preconditioner's breakdown test
    (2L-CHEB, precond.cpp:338-347) or needs many PCG steps amplifies FFT rounding far beyond
    1e-8, for the reference itself.  Run with VRG_REF_LIB=libveloreg_ref_altfft.so."""
    if os.environ.get("VRG_REF_LIB") != "libveloreg_ref_altfft.so":
        raise SystemExit("run newton_default_altfft with VRG_REF_LIB=libveloreg_ref_altfft.so")
    return case_newton_default()


CASES = {"newton_cfg3_5b": case_newton_cfg3_5b, "newton_default": case_newton_default,
         "newton_default_altfft": case_newton_default_altfft, "cfg5a_digest": case_cfg5a_digest}


def main(argv):
    for name in argv or list(CASES):
        d = CASES[name]()
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
        print(name, sorted(d), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
