"""ctypes binding of oracle/_ref/libveloreg_ref.so — the UNMODIFIED reference C++ library
(/root/reference/proj/core) compiled by oracle/Makefile with the FFTW3-API shim.

TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline): imported by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference legs.  Nothing in
the product package imports this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# VRG_REF_LIB=libveloreg_ref_altfft.so selects the same reference over the alternative-rounding
# FFT shim (the reference-vs-reference floor, oracle/Makefile)
LIB_PATH = os.path.join(_HERE, "_ref", os.environ.get("VRG_REF_LIB", "libveloreg_ref.so"))

_D = C.POINTER(C.c_double)
_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code  # 1 invalid_argument, 2 BlowupError, 3 other


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        for name in ("ref_hess_create", "ref_hess_create_mode", "ref_coarse_create"):
            getattr(_lib, name).restype = C.c_void_p
        _lib.ref_hess_apply.argtypes = [C.c_void_p, _D, _D, C.c_int, _D, _D]
        _lib.ref_hess_destroy.argtypes = [C.c_void_p]
        _lib.ref_coarse_split_apply.argtypes = [C.c_void_p, _D, _D, _D, _D]
        _lib.ref_coarse_destroy.argtypes = [C.c_void_p]
        _lib.ref_two_level_apply.argtypes = [C.c_void_p, C.c_int, C.c_int, _D, _D, C.c_int, C.c_int,
                                             C.c_double, C.c_double, C.c_double, C.c_double, _D, _D]
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(code: int):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def set_scheme(scheme):
    """0 SL, 1 RK2, 2 RK2A for the solvers/operators/gradients/Newton built afterwards."""
    lib().ref_set_scheme(int(scheme))


def set_penalty_weight(beta_w):
    lib().ref_set_penalty_weight(C.c_double(beta_w))


def counters_reset():
    lib().ref_counters_reset()


def counters():
    f, i = C.c_longlong(), C.c_longlong()
    lib().ref_counters(C.byref(f), C.byref(i))
    return f.value, i.value


def prefilter(u):
    u = _c(u)
    out = np.empty_like(u)
    _check(lib().ref_prefilter(u.shape[0], u.shape[1], _p(u), _p(out)))
    return out


def evaluate(c, x1, x2):
    c, x1, x2 = _c(c), _c(x1), _c(x2)
    out = np.empty_like(c)
    _check(lib().ref_evaluate(c.shape[0], c.shape[1], _p(c), _p(x1), _p(x2), _p(out)))
    return out


def derive_steps(v1, v2, cfl):
    v1, v2 = _c(v1), _c(v2)
    nt = C.c_int()
    _check(lib().ref_derive_steps(v1.shape[0], v1.shape[1], _p(v1), _p(v2), C.c_double(cfl), C.byref(nt)))
    return nt.value


def trace(v1, v2, ht, backward=False):
    v1, v2 = _c(v1), _c(v2)
    x1, x2 = np.empty_like(v1), np.empty_like(v1)
    _check(lib().ref_trace(v1.shape[0], v1.shape[1], _p(v1), _p(v2), C.c_double(ht), int(backward), _p(x1), _p(x2)))
    return x1, x2


def _traj_call(fn, v1, v2, nt, *fields):
    v1, v2 = _c(v1), _c(v2)
    n1, n2 = v1.shape
    out = np.empty((nt + 1, n1, n2))
    args = [_p(_c(f)) for f in fields]
    _check(fn(n1, n2, _p(v1), _p(v2), nt, *args, _p(out)))
    return out


def solve_state(v1, v2, nt, m0):
    return _traj_call(lib().ref_solve_state, v1, v2, nt, m0)


def solve_adjoint(v1, v2, nt, lam1):
    return _traj_call(lib().ref_solve_adjoint, v1, v2, nt, lam1)


def solve_incstate(v1, v2, nt, m0, vt1, vt2):
    return _traj_call(lib().ref_solve_incstate, v1, v2, nt, m0, vt1, vt2)


def solve_incadjoint_gn(v1, v2, nt, lt1):
    return _traj_call(lib().ref_solve_incadjoint_gn, v1, v2, nt, lt1)


def solve_incadjoint_fn(v1, v2, nt, vt1, vt2, lt1, adj_seed):
    """full-Newton incremental adjoint, the adjoint solved from adj_seed (lambda(1)) inside."""
    v1, v2 = _c(v1), _c(v2)
    n1, n2 = v1.shape
    out = np.empty((nt + 1, n1, n2))
    vt1, vt2, lt1, seed = map(_c, (vt1, vt2, lt1, adj_seed))
    _check(lib().ref_solve_incadjoint_fn(n1, n2, _p(v1), _p(v2), nt, _p(vt1), _p(vt2), _p(lt1), _p(seed),
                                         _p(out)))
    return out


def solve_state_final(v1, v2, nt, m0):
    v1, v2, m0 = _c(v1), _c(v2), _c(m0)
    out = np.empty_like(m0)
    _check(lib().ref_solve_state_final(v1.shape[0], v1.shape[1], _p(v1), _p(v2), nt, _p(m0), _p(out)))
    return out


def solve_adjoint_final(v1, v2, nt, lam1):
    v1, v2, lam1 = _c(v1), _c(v2), _c(lam1)
    out = np.empty_like(lam1)
    _check(lib().ref_solve_adjoint_final(v1.shape[0], v1.shape[1], _p(v1), _p(v2), nt, _p(lam1), _p(out)))
    return out


def jacobian_det(v1, v2, nt=0, cfl=0.2):
    v1, v2 = _c(v1), _c(v2)
    out = np.empty_like(v1)
    _check(lib().ref_jacobian_det(v1.shape[0], v1.shape[1], _p(v1), _p(v2), nt, C.c_double(cfl), _p(out)))
    return out


def gradient(u):
    u = _c(u)
    g1, g2 = np.empty_like(u), np.empty_like(u)
    _check(lib().ref_gradient(u.shape[0], u.shape[1], _p(u), _p(g1), _p(g2)))
    return g1, g2


def divergence(v1, v2):
    v1, v2 = _c(v1), _c(v2)
    out = np.empty_like(v1)
    _check(lib().ref_divergence(v1.shape[0], v1.shape[1], _p(v1), _p(v2), _p(out)))
    return out


def apply_reg(v1, v2, norm, beta):
    v1, v2 = _c(v1), _c(v2)
    o1, o2 = np.empty_like(v1), np.empty_like(v1)
    _check(lib().ref_apply_reg(v1.shape[0], v1.shape[1], norm, C.c_double(beta), _p(v1), _p(v2), _p(o1), _p(o2)))
    return o1, o2


def apply_inv_reg(v1, v2, norm, beta, power):
    v1, v2 = _c(v1), _c(v2)
    o1, o2 = np.empty_like(v1), np.empty_like(v1)
    _check(lib().ref_apply_inv_reg(v1.shape[0], v1.shape[1], norm, C.c_double(beta), C.c_double(power),
                                   _p(v1), _p(v2), _p(o1), _p(o2)))
    return o1, o2


def project_div_free(v1, v2):
    v1, v2 = _c(v1), _c(v2)
    o1, o2 = np.empty_like(v1), np.empty_like(v1)
    _check(lib().ref_project_div_free(v1.shape[0], v1.shape[1], _p(v1), _p(v2), _p(o1), _p(o2)))
    return o1, o2


def resample(u, t1, t2):
    u = _c(u)
    out = np.empty((t1, t2))
    _check(lib().ref_resample(u.shape[0], u.shape[1], _p(u), t1, t2, _p(out)))
    return out


def cutoff(u, high):
    u = _c(u)
    out = np.empty_like(u)
    _check(lib().ref_cutoff(u.shape[0], u.shape[1], _p(u), int(high), _p(out)))
    return out


def apply_helmholtz(u):
    u = _c(u)
    out = np.empty_like(u)
    _check(lib().ref_apply_helmholtz(u.shape[0], u.shape[1], _p(u), _p(out)))
    return out


def gaussian_smooth(u, sigma):
    u = _c(u)
    out = np.empty_like(u)
    _check(lib().ref_gaussian_smooth(u.shape[0], u.shape[1], _p(u), C.c_double(sigma), _p(out)))
    return out


def random_bandlimited_field(n1, n2, seed):
    out = np.empty((n1, n2))
    _check(lib().ref_random_bandlimited_field(n1, n2, C.c_ulonglong(seed), _p(out)))
    return out


def random_bandlimited_velocity(n1, n2, seed):
    return (random_bandlimited_field(n1, n2, seed),
            random_bandlimited_field(n1, n2, seed ^ 0x9E3779B97F4A7C15))


class Hessian:
    """inverse::HessianOperator (GN, SL, fixed nt) held open for steady-state applies."""

    def __init__(self, v1, v2, mR, mT, norm, beta, deform, nt, mode=0):
        v1, v2, mR, mT = map(_c, (v1, v2, mR, mT))
        self.shape = v1.shape
        st = C.c_int()
        self.h = lib().ref_hess_create_mode(v1.shape[0], v1.shape[1], _p(v1), _p(v2), _p(mR), _p(mT), norm,
                                            C.c_double(beta), deform, nt, int(mode), C.byref(st))
        _check(st.value)

    def apply(self, vt1, vt2, data_only=False):
        vt1, vt2 = _c(vt1), _c(vt2)
        o1, o2 = np.empty_like(vt1), np.empty_like(vt1)
        _check(lib().ref_hess_apply(C.c_void_p(self.h), _p(vt1), _p(vt2), int(data_only), _p(o1), _p(o2)))
        return o1, o2

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_hess_destroy(C.c_void_p(self.h))
            self.h = None


class Coarse:
    """precond::CoarseOperator at fine velocity v (SL, CFL-derived coarse nt)."""

    def __init__(self, v1, v2, mR, mT, norm, beta, deform, coarse_cfl=5.0):
        v1, v2, mR, mT = map(_c, (v1, v2, mR, mT))
        st = C.c_int()
        self.h = lib().ref_coarse_create(v1.shape[0], v1.shape[1], _p(v1), _p(v2), _p(mR), _p(mT), norm,
                                         C.c_double(beta), deform, C.c_double(coarse_cfl), C.byref(st))
        _check(st.value)
        self.shape = (v1.shape[0] // 2, v1.shape[1] // 2)

    def split_apply(self, s1, s2):
        s1, s2 = _c(s1), _c(s2)
        o1, o2 = np.empty_like(s1), np.empty_like(s1)
        _check(lib().ref_coarse_split_apply(C.c_void_p(self.h), _p(s1), _p(s2), _p(o1), _p(o2)))
        return o1, o2

    def two_level(self, r1, r2, cheb, cheb_iters, eps_scale, outer_tol, emin, emax):
        r1, r2 = _c(r1), _c(r2)
        o1, o2 = np.empty_like(r1), np.empty_like(r1)
        _check(lib().ref_two_level_apply(C.c_void_p(self.h), r1.shape[0], r1.shape[1], _p(r1), _p(r2), int(cheb),
                                         cheb_iters, C.c_double(eps_scale), C.c_double(outer_tol), C.c_double(emin),
                                         C.c_double(emax), _p(o1), _p(o2)))
        return o1, o2

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_coarse_destroy(C.c_void_p(self.h))
            self.h = None


def evaluate_gradient(v1, v2, mR, mT, norm, beta, deform, nt):
    v1, v2, mR, mT = map(_c, (v1, v2, mR, mT))
    g1, g2 = np.empty_like(v1), np.empty_like(v1)
    sc = np.zeros(3)
    _check(lib().ref_evaluate_gradient(v1.shape[0], v1.shape[1], _p(v1), _p(v2), _p(mR), _p(mT), norm,
                                       C.c_double(beta), deform, nt, _p(g1), _p(g2), _p(sc)))
    return g1, g2, sc


def evaluate_objective(v1, v2, mR, mT, norm, beta, deform, nt):
    v1, v2, mR, mT = map(_c, (v1, v2, mR, mT))
    sc = np.zeros(3)
    _check(lib().ref_evaluate_objective(v1.shape[0], v1.shape[1], _p(v1), _p(v2), _p(mR), _p(mT), norm,
                                        C.c_double(beta), deform, nt, _p(sc)))
    return sc


def estimate_eigs(mR, mT, norm, beta, deform):
    mR, mT = _c(mR), _c(mT)
    a, b = C.c_double(), C.c_double()
    _check(lib().ref_estimate_eigs(mR.shape[0], mR.shape[1], _p(mR), _p(mT), norm, C.c_double(beta), deform,
                                   C.byref(a), C.byref(b)))
    return a.value, b.value


def newton_solve(mR, mT, norm, beta, deform, *, max_outer=50, max_inner=500, nt=0, grad_cfl=1.0,
                 two_level=True, cheb=True, cheb_iters=10, tol_rel=1e-2, tol_abs=1e-5, eps_scale=0.1, mode=0):
    mR, mT = _c(mR), _c(mT)
    n1, n2 = mR.shape
    cfg_i = np.array([max_outer, max_inner, nt, int(two_level), int(cheb), cheb_iters, int(mode)], dtype=np.int32)
    cfg_d = np.array([tol_rel, tol_abs, grad_cfl, eps_scale])
    v1, v2 = np.empty_like(mR), np.empty_like(mR)
    rep = np.zeros((max_outer + 1, 10))
    summ = np.zeros(6)
    _check(lib().ref_newton_solve(n1, n2, _p(mR), _p(mT), norm, C.c_double(beta), deform,
                                  cfg_i.ctypes.data_as(C.POINTER(C.c_int)), _p(cfg_d), _p(v1), _p(v2), _p(rep),
                                  max_outer + 1, _p(summ)))
    k = int(summ[1])
    return v1, v2, rep[:k], summ
