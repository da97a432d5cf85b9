"""Python host mirror of the reference's operator/solver API over the C ABI (include/vrg.h).

Names, argument meaning and error behaviour follow veloreg:: (include/veloreg/*.hpp):
``interp.prefilter/evaluate``, ``transport.Solver``, ``spectral.*``,
``inverse.HessianOperator``, ``evaluateGradient/evaluateObjective``.  Fields are float64
CUDA tensors of shape (n1, n2) on the context's device; vector fields are pairs of tensors.
Exceptions: InvalidArgument (std::invalid_argument), BlowupError (transport::BlowupError),
NotSupported.  Every call runs the sm_100a kernels in libvrg.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi

H1SEMI, H2SEMI, H3SEMI = 1, 2, 3
COMPRESSIBLE, INCOMPRESSIBLE, NEAR_INCOMPRESSIBLE = 0, 1, 2
FORWARD, BACKWARD = 0, 1
GAUSS_NEWTON, FULL_NEWTON = 0, 1
BAND_LOW, BAND_HIGH = 0, 1
SL, RK2, RK2A = 0, 1, 2


class VrgError(RuntimeError):
    code = _capi.VRG_RUNTIME_ERROR


class InvalidArgument(VrgError, ValueError):
    code = _capi.VRG_INVALID_ARGUMENT


class BlowupError(VrgError):
    code = _capi.VRG_BLOWUP


class NotSupported(VrgError, NotImplementedError):
    code = _capi.VRG_NOT_SUPPORTED


_ERRORS = {1: InvalidArgument, 2: BlowupError, 3: VrgError, 4: NotSupported}


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


_STREAMS = {}


class Context:
    """One device + stream (the library's vrg_ctx_t).  By default the first context of a device
    creates the library's non-blocking stream and makes it torch's current stream of that
    device (torch.cuda.ExternalStream), and later contexts share it: torch ops and library calls
    are then stream-ordered.  (torch's own default stream is the legacy NULL stream, on which
    CUDA graphs cannot be captured.)"""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise VrgError("libvrg needs a CUDA device (no CPU fallback)")
        self.lib = _capi.load()
        self.device = torch.device("cuda", device)
        if stream is None or stream.cuda_stream == 0:
            stream = _STREAMS.get(device)
        handle = stream.cuda_stream if stream is not None else 0
        h = C.c_void_p()
        code = self.lib.vrg_ctx_create(device, C.c_void_p(handle), C.byref(h))
        if code:
            raise _ERRORS.get(code, VrgError)(self.lib.vrg_last_error(None).decode())
        self.h = h
        self._owner = stream is None
        if stream is None:  # the library created its stream: adopt it for torch
            stream = torch.cuda.ExternalStream(self.lib.vrg_ctx_stream(h), device=self.device)
            _STREAMS[device] = stream
        self.stream = stream
        with torch.cuda.device(self.device):
            if torch.cuda.current_stream(self.device) != stream:
                torch.cuda.set_stream(stream)

    def set_scheme(self, scheme: int):
        """Transport scheme (SL, RK2, RK2A) of solvers/operators/gradients created on this context."""
        self.check(self.lib.vrg_set_scheme(self.h, int(scheme)))

    def set_penalty_weight(self, beta_w: float):
        """Model::betaW of the near-incompressible model for calls on this context."""
        self.check(self.lib.vrg_set_penalty_weight(self.h, float(beta_w)))

    def check(self, code: int):
        if code:
            raise _ERRORS.get(code, VrgError)(self.lib.vrg_last_error(self.h).decode())

    def counters(self):
        f, i = C.c_longlong(), C.c_longlong()
        self.lib.vrg_counters(self.h, C.byref(f), C.byref(i))
        return f.value, i.value

    def reset_counters(self):
        self.lib.vrg_counters_reset(self.h)

    def sync(self):
        self.check(self.lib.vrg_sync(self.h))

    def field(self, a) -> torch.Tensor:
        """A float64 contiguous device tensor holding `a` (numpy array or tensor)."""
        t = torch.as_tensor(a, dtype=torch.float64)
        return t.to(self.device).contiguous()

    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(*shape, dtype=torch.float64, device=self.device)

    def close(self):
        if getattr(self, "_owner", False):
            return  # owns the device's shared stream (torch's current stream): kept for the process
        if getattr(self, "h", None):
            self.lib.vrg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _shape(u):
    n1, n2 = u.shape[-2], u.shape[-1]
    return int(n1), int(n2)


# ---------------------------------------------------------------- field BLAS-1 (field.hpp:62-80)
def dot(ctx, a, b):
    """h1*h2*sum(a*b) for scalar fields, sum over components for pairs (field.cpp:47-54)."""
    out = C.c_double()
    if isinstance(a, tuple):
        n1, n2 = _shape(a[0])
        ctx.check(ctx.lib.vrg_dot(ctx.h, n1, n2, _p(a[0]), _p(a[1]), _p(b[0]), _p(b[1]), C.byref(out)))
    else:
        n1, n2 = _shape(a)
        ctx.check(ctx.lib.vrg_dot(ctx.h, n1, n2, _p(a), None, _p(b), None, C.byref(out)))
    return out.value


def norm_linf(ctx, a):
    out = C.c_double()
    if isinstance(a, tuple):
        n1, n2 = _shape(a[0])
        ctx.check(ctx.lib.vrg_norm_linf(ctx.h, n1, n2, _p(a[0]), _p(a[1]), C.byref(out)))
    else:
        n1, n2 = _shape(a)
        ctx.check(ctx.lib.vrg_norm_linf(ctx.h, n1, n2, _p(a), None, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- interp (interp.hpp:27-34)
def prefilter(ctx, u):
    n1, n2 = _shape(u)
    c = ctx.empty(n1, n2)
    ctx.check(ctx.lib.vrg_prefilter(ctx.h, n1, n2, _p(u), _p(c)))
    return c


def evaluate(ctx, c, x1, x2):
    n1, n2 = _shape(c)
    if tuple(x1.shape) != (n1, n2) or tuple(x2.shape) != (n1, n2):
        raise InvalidArgument("evaluate: point set does not match coefficient grid")
    out = ctx.empty(n1, n2)
    ctx.check(ctx.lib.vrg_evaluate(ctx.h, n1, n2, _p(c), _p(x1), _p(x2), _p(out)))
    return out


# ---------------------------------------------------------------- spectral (spectral.hpp:27-56)
def gradient(ctx, u):
    n1, n2 = _shape(u)
    g = ctx.empty(2, n1, n2)
    ctx.check(ctx.lib.vrg_gradient(ctx.h, n1, n2, _p(u), _p(g[0]), _p(g[1])))
    return g[0], g[1]


def apply_helmholtz(ctx, u):
    """spectral::applyHelmholtz (spectral.cpp:214-223): (1 - Laplacian) u."""
    n1, n2 = _shape(u)
    out = ctx.empty(n1, n2)
    ctx.check(ctx.lib.vrg_apply_helmholtz(ctx.h, n1, n2, _p(u), _p(out)))
    return out


def body_force(ctx, state, adjoint):
    """assembleBodyForce, SL (inverse.cpp:50-65): trajectories (nt+1, n1, n2) -> (b1, b2)."""
    if tuple(state.shape) != tuple(adjoint.shape):
        raise InvalidArgument("assembleBodyForce: trajectory length mismatch")
    nt = int(state.shape[0]) - 1
    n1, n2 = _shape(state)
    b = ctx.empty(2, n1, n2)
    ctx.check(ctx.lib.vrg_body_force(ctx.h, n1, n2, nt, _p(state.contiguous()), _p(adjoint.contiguous()), _p(b[0]),
                                     _p(b[1])))
    return b[0], b[1]


def divergence(ctx, v):
    n1, n2 = _shape(v[0])
    out = ctx.empty(n1, n2)
    ctx.check(ctx.lib.vrg_divergence(ctx.h, n1, n2, _p(v[0]), _p(v[1]), _p(out)))
    return out


def apply_reg(ctx, v, norm, beta):
    n1, n2 = _shape(v[0])
    o = ctx.empty(2, n1, n2)
    ctx.check(ctx.lib.vrg_apply_reg(ctx.h, n1, n2, norm, beta, _p(v[0]), _p(v[1]), _p(o[0]), _p(o[1])))
    return o[0], o[1]


def apply_inv_reg(ctx, v, norm, beta, power):
    n1, n2 = _shape(v[0])
    o = ctx.empty(2, n1, n2)
    ctx.check(ctx.lib.vrg_apply_inv_reg(ctx.h, n1, n2, norm, beta, power, _p(v[0]), _p(v[1]), _p(o[0]), _p(o[1])))
    return o[0], o[1]


def project_div_free(ctx, b):
    n1, n2 = _shape(b[0])
    o = ctx.empty(2, n1, n2)
    ctx.check(ctx.lib.vrg_project_div_free(ctx.h, n1, n2, _p(b[0]), _p(b[1]), _p(o[0]), _p(o[1])))
    return o[0], o[1]


def resample(ctx, u, target):
    n1, n2 = _shape(u)
    out = ctx.empty(*target)
    ctx.check(ctx.lib.vrg_resample(ctx.h, n1, n2, _p(u), int(target[0]), int(target[1]), _p(out)))
    return out


def cutoff_filter(ctx, u, band):
    n1, n2 = _shape(u)
    out = ctx.empty(n1, n2)
    ctx.check(ctx.lib.vrg_cutoff(ctx.h, n1, n2, _p(u), band, _p(out)))
    return out


def gaussian_smooth(ctx, u, sigma):
    n1, n2 = _shape(u)
    out = ctx.empty(n1, n2)
    ctx.check(ctx.lib.vrg_gaussian_smooth(ctx.h, n1, n2, _p(u), sigma, _p(out)))
    return out


# ---------------------------------------------------------------- transport (transport.hpp)
def derive_steps(ctx, v, cfl):
    n1, n2 = _shape(v[0])
    nt = C.c_int()
    ctx.check(ctx.lib.vrg_derive_steps(ctx.h, n1, n2, _p(v[0]), _p(v[1]), cfl, C.byref(nt)))
    return nt.value


def trace_characteristics(ctx, v, ht, direction=FORWARD):
    n1, n2 = _shape(v[0])
    x = ctx.empty(2, n1, n2)
    ctx.check(ctx.lib.vrg_trace(ctx.h, n1, n2, _p(v[0]), _p(v[1]), ht, direction, _p(x[0]), _p(x[1])))
    return x[0], x[1]


class Solver:
    """transport::Solver with scheme SL (transport.hpp:71-100)."""

    def __init__(self, ctx, v, nt):
        self.ctx = ctx
        self.shape = _shape(v[0])
        self.nt = int(nt)
        h = C.c_void_p()
        ctx.check(ctx.lib.vrg_solver_create(ctx.h, *self.shape, _p(v[0]), _p(v[1]), self.nt, C.byref(h)))
        self.h = h

    def _traj(self):
        return self.ctx.empty(self.nt + 1, *self.shape)

    def solve_state(self, m0):
        t = self._traj()
        self.ctx.check(self.ctx.lib.vrg_solver_state(self.h, _p(m0), _p(t)))
        return t

    def solve_adjoint(self, lam1):
        t = self._traj()
        self.ctx.check(self.ctx.lib.vrg_solver_adjoint(self.h, _p(lam1), _p(t)))
        return t

    def solve_state_final(self, m0):
        o = self.ctx.empty(*self.shape)
        self.ctx.check(self.ctx.lib.vrg_solver_state_final(self.h, _p(m0), _p(o)))
        return o

    def solve_adjoint_final(self, lam1):
        o = self.ctx.empty(*self.shape)
        self.ctx.check(self.ctx.lib.vrg_solver_adjoint_final(self.h, _p(lam1), _p(o)))
        return o

    def solve_inc_state(self, vt, state):
        t = self._traj()
        self.ctx.check(self.ctx.lib.vrg_solver_incstate(self.h, _p(vt[0]), _p(vt[1]), _p(state), _p(t)))
        return t

    def solve_inc_adjoint(self, vt, lt1, adjoint=None, mode=GAUSS_NEWTON):
        t = self._traj()
        self.ctx.check(self.ctx.lib.vrg_solver_incadjoint(self.h, _p(vt[0]), _p(vt[1]), _p(lt1), _p(adjoint), mode,
                                                          _p(t)))
        return t

    def jacobian_determinant(self):
        o = self.ctx.empty(*self.shape)
        self.ctx.check(self.ctx.lib.vrg_solver_jacobian(self.h, _p(o)))
        return o

    def departure(self, direction=FORWARD):
        x = self.ctx.empty(2, *self.shape)
        self.ctx.check(self.ctx.lib.vrg_solver_departure(self.h, direction, _p(x[0]), _p(x[1])))
        return x[0], x[1]

    def __del__(self):
        if getattr(self, "h", None):
            self.ctx.lib.vrg_solver_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------- inverse (inverse.hpp)
class HessianOperator:
    """inverse::HessianOperator, GN mode, SL scheme with fixed nt (inverse.hpp:74-97)."""

    def __init__(self, ctx, v, mR, mT, norm, beta, deformation, nt, mode=GAUSS_NEWTON, state=None):
        self.ctx = ctx
        self.shape = _shape(v[0])
        self.nt = int(nt)
        h = C.c_void_p()
        ctx.check(ctx.lib.vrg_hess_create(ctx.h, *self.shape, _p(v[0]), _p(v[1]), _p(mR), _p(mT), norm, beta,
                                          deformation, self.nt, mode, _p(state), C.byref(h)))
        self.h = h

    def _out(self, out):
        return out if out is not None else self.ctx.empty(2, *self.shape)

    def apply(self, vt, out=None):
        o = self._out(out)
        self.ctx.check(self.ctx.lib.vrg_hess_apply(self.h, _p(vt[0]), _p(vt[1]), _p(o[0]), _p(o[1])))
        return o[0], o[1]

    def apply_data_term(self, vt, out=None):
        o = self._out(out)
        self.ctx.check(self.ctx.lib.vrg_hess_apply_data(self.h, _p(vt[0]), _p(vt[1]), _p(o[0]), _p(o[1])))
        return o[0], o[1]

    def apply_split(self, s, out=None):
        o = self._out(out)
        self.ctx.check(self.ctx.lib.vrg_hess_apply_split(self.h, _p(s[0]), _p(s[1]), _p(o[0]), _p(o[1])))
        return o[0], o[1]

    def apply_host(self, vt1, vt2, o1, o2):
        """apply() on host (numpy or pinned torch) buffers: H2D + matvec + D2H."""
        def hp(a):
            return C.c_void_p(a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr())
        self.ctx.check(self.ctx.lib.vrg_hess_apply_host(self.h, hp(vt1), hp(vt2), hp(o1), hp(o2)))

    def apply_host_batch(self, vts, outs):
        """apply_host over k independent inputs vts[i] = (vt1, vt2) -> outs[i] = (o1, o2), host
        buffers (pinned for overlap); neighbouring matvecs' copies overlap the compute."""
        k = len(vts)
        if len(outs) != k:
            raise ValueError("apply_host_batch: as many outputs as inputs")

        def hp(a):
            return a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr()
        arr = [(C.c_void_p * max(k, 1))(*[hp(x[j]) for x in seq]) for seq, j in
               ((vts, 0), (vts, 1), (outs, 0), (outs, 1))]
        self.ctx.check(self.ctx.lib.vrg_hess_apply_host_batch(self.h, k, *[C.cast(a, C.c_void_p) for a in arr]))

    def apply_batch(self, vts, outs):
        """apply() over k device inputs vts[i] = (vt1, vt2) -> outs[i] = (o1, o2), queued back to
        back: matvec i's guard is checked on the host while matvec i+1 runs (vrg_hess_apply_batch)."""
        k = len(vts)
        if len(outs) != k:
            raise ValueError("apply_batch: as many outputs as inputs")
        arr = [(C.c_void_p * max(k, 1))(*[_p(x[j]).value for x in seq]) for seq, j in
               ((vts, 0), (vts, 1), (outs, 0), (outs, 1))]
        self.ctx.check(self.ctx.lib.vrg_hess_apply_batch(self.h, k, *[C.cast(a, C.c_void_p) for a in arr]))

    @property
    def band_path(self):
        """True when the matvec runs the fused band kernels (evalband.cuh), False on the 3-kernel step."""
        b = C.c_int()
        self.ctx.check(self.ctx.lib.vrg_hess_band_path(self.h, C.byref(b)))
        return bool(b.value)

    def state(self):
        t = self.ctx.empty(self.nt + 1, *self.shape)
        self.ctx.check(self.ctx.lib.vrg_hess_state(self.h, _p(t)))
        return t

    def __del__(self):
        if getattr(self, "h", None):
            self.ctx.lib.vrg_hess_destroy(self.h)
            self.h = None


def evaluate_gradient(ctx, v, mR, mT, norm, beta, deformation, nt):
    n1, n2 = _shape(v[0])
    g = ctx.empty(2, n1, n2)
    sc = (C.c_double * 3)()
    ctx.check(ctx.lib.vrg_evaluate_gradient(ctx.h, n1, n2, _p(v[0]), _p(v[1]), _p(mR), _p(mT), norm, beta,
                                            deformation, nt, _p(g[0]), _p(g[1]), C.cast(sc, C.c_void_p)))
    return (g[0], g[1]), tuple(sc)


def evaluate_objective(ctx, v, mR, mT, norm, beta, deformation, nt):
    n1, n2 = _shape(v[0])
    sc = (C.c_double * 3)()
    ctx.check(ctx.lib.vrg_evaluate_objective(ctx.h, n1, n2, _p(v[0]), _p(v[1]), _p(mR), _p(mT), norm, beta,
                                             deformation, nt, C.cast(sc, C.c_void_p)))
    return tuple(sc)


# ---------------------------------------------------------------- precond (precond.hpp)
PC_REG, PC_TWO_LEVEL = 0, 1
COARSE_PCG, COARSE_CHEB = 0, 1
COARSE_CFL = 5.0  # kCoarseScheme, newton.cpp:16


def random_bandlimited_field(ctx, shape, seed):
    out = ctx.empty(*shape)
    ctx.check(ctx.lib.vrg_random_bandlimited_field(ctx.h, int(shape[0]), int(shape[1]), C.c_ulonglong(seed), _p(out)))
    return out


def random_bandlimited_velocity(ctx, shape, seed):
    return (random_bandlimited_field(ctx, shape, seed),
            random_bandlimited_field(ctx, shape, seed ^ 0x9E3779B97F4A7C15))


class CoarseOperator:
    """precond::CoarseOperator: half-grid split GN Hessian at the restricted velocity (v=None: 0)."""

    def __init__(self, ctx, v, mR, mT, norm, beta, deformation, coarse_cfl=COARSE_CFL):
        self.ctx = ctx
        self.fine = _shape(mR)
        h = C.c_void_p()
        v1, v2 = (v[0], v[1]) if v is not None else (None, None)
        ctx.check(ctx.lib.vrg_coarse_create(ctx.h, *self.fine, _p(v1), _p(v2), _p(mR), _p(mT), norm, beta,
                                            deformation, coarse_cfl, C.byref(h)))
        self.h = h
        a, b, nt = C.c_int(), C.c_int(), C.c_int()
        ctx.lib.vrg_coarse_info(h, C.byref(a), C.byref(b), C.byref(nt))
        self.shape, self.nt = (a.value, b.value), nt.value

    def apply_split(self, s):
        o = self.ctx.empty(2, *self.shape)
        self.ctx.check(self.ctx.lib.vrg_coarse_apply_split(self.h, _p(s[0]), _p(s[1]), _p(o[0]), _p(o[1])))
        return o[0], o[1]

    def two_level(self, r, coarse_solver, cheb_iters, eps_scale, outer_tol, emin, emax):
        o = self.ctx.empty(2, *self.fine)
        fb = C.c_int()
        self.ctx.check(self.ctx.lib.vrg_two_level_apply(self.h, _p(r[0]), _p(r[1]), coarse_solver, cheb_iters,
                                                        eps_scale, outer_tol, emin, emax, _p(o[0]), _p(o[1]),
                                                        C.byref(fb)))
        return (o[0], o[1]), bool(fb.value)

    def __del__(self):
        if getattr(self, "h", None):
            self.ctx.lib.vrg_coarse_destroy(self.h)
            self.h = None


def estimate_eigs(ctx, mR, mT, norm, beta, deformation, v=None, coarse_cfl=COARSE_CFL, seed=0x5EED):
    n1, n2 = _shape(mR)
    a, b = C.c_double(), C.c_double()
    v1, v2 = (v[0], v[1]) if v is not None else (None, None)
    ctx.check(ctx.lib.vrg_estimate_eigs(ctx.h, n1, n2, _p(v1), _p(v2), _p(mR), _p(mT), norm, beta, deformation,
                                        coarse_cfl, C.c_ulonglong(seed), C.byref(a), C.byref(b)))
    return a.value, b.value


def _pc_arrays(kind, coarse_solver, cheb_iters, eps_scale, eig):
    pi = (C.c_int * 4)(kind, coarse_solver, cheb_iters, 1 if eig else 0)
    pd = (C.c_double * 3)(eps_scale, eig[0] if eig else 1.0, eig[1] if eig else 10.0)
    return pi, pd


def solve_kkt(hess, rhs, tol, max_iter, mR, mT, v, *, kind=PC_TWO_LEVEL, coarse_solver=COARSE_CHEB, cheb_iters=10,
              eps_scale=0.1, eig=None, coarse_cfl=COARSE_CFL):
    """precond::solveKkt; returns (delta_v, dict(iterations, converged, negative_curvature, rel_residual, ...))."""
    ctx = hess.ctx
    pi, pd = _pc_arrays(kind, coarse_solver, cheb_iters, eps_scale, eig)
    sol = ctx.empty(2, *hess.shape)
    res = (C.c_double * 6)()
    ctx.check(ctx.lib.vrg_solve_kkt(hess.h, _p(rhs[0]), _p(rhs[1]), tol, max_iter, C.cast(pi, C.c_void_p),
                                    C.cast(pd, C.c_void_p), _p(mR), _p(mT), _p(v[0]), _p(v[1]), coarse_cfl,
                                    _p(sol[0]), _p(sol[1]), C.cast(res, C.c_void_p)))
    return (sol[0], sol[1]), dict(iterations=int(res[0]), converged=bool(res[1]), negative_curvature=bool(res[2]),
                                  rel_residual=res[3], total_s=res[4], precond_s=res[5])


RECORD_FIELDS = ("iter", "gradNormInf", "gradNormRel", "objective", "mismatch", "innerIterations",
                 "lineSearchSteps", "stepLength", "searchDirDivRatio", "wallTimeSec", "ffts", "interps")


FINE_BUILD_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int)
FINE_DATA_TERM_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
# the external operators of include/vrg.h (vrg_external_ops)
GRADIENT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
OBJECTIVE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p)
COARSE_BUILD_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int))
TWO_LEVEL_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double)
COARSE_EMAX_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int))
SPLIT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
EXTERNAL_OPS_FIELDS = ("build", "data_term", "gradient", "objective", "coarse_build", "two_level", "coarse_emax",
                       "split")


class ExternalOps(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in EXTERNAL_OPS_FIELDS] + [("user", C.c_void_p)]


def newton_solve_batch(ctx, mR, mT, norm, beta, deformation, *, max_outer=50, max_inner=500, nt=16,
                       ls_max_steps=20, tol_rel=1e-2, tol_abs=1e-5, forcing_cap=0.5, ls_c1=1e-4, ls_shrink=0.5,
                       grad_cfl=1.0, kind=PC_TWO_LEVEL, coarse_solver=COARSE_CHEB, cheb_iters=10, eps_scale=0.1,
                       eig=None):
    """newtonSolve of P independent image pairs in lockstep (C ABI vrg_newton_solve_batch): mR, mT
    are (P, n1, n2) host arrays; returns one (v1, v2, records, summary) per pair, each identical to
    that pair's own newton_solve.  A pair whose solve raised gets summary['error'] = the status
    code (the message goes to stderr); the others are unaffected."""
    import numpy as np

    mR = np.ascontiguousarray(mR, dtype=np.float64)
    mT = np.ascontiguousarray(mT, dtype=np.float64)
    P, n1, n2 = mR.shape
    ci = (C.c_int * 5)(max_outer, max_inner, nt, ls_max_steps, GAUSS_NEWTON)
    cd = (C.c_double * 6)(tol_rel, tol_abs, forcing_cap, ls_c1, ls_shrink, grad_cfl)
    pi, pd = _pc_arrays(kind, coarse_solver, cheb_iters, eps_scale, eig)
    v1, v2 = np.empty_like(mR), np.empty_like(mR)
    rec = np.zeros((P, max_outer + 1, 12))
    summ = np.zeros((P, 7))
    st = np.zeros(P, dtype=np.int32)
    hp = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    ctx.check(ctx.lib.vrg_newton_solve_batch(ctx.h, n1, n2, P, hp(mR), hp(mT), norm, beta, deformation,
                                             C.cast(ci, C.c_void_p), C.cast(cd, C.c_void_p), C.cast(pi, C.c_void_p),
                                             C.cast(pd, C.c_void_p), hp(v1), hp(v2), hp(rec), max_outer + 1,
                                             hp(summ), hp(st)))
    out = []
    for k in range(P):
        n = int(summ[k, 1])
        records = [dict(zip(RECORD_FIELDS, row)) for row in rec[k, :n]]
        summary = dict(status=int(summ[k, 0]), iterations=n, finalGradNormRel=summ[k, 2],
                       finalResidualRel=summ[k, 3], jacMin=summ[k, 4], jacMax=summ[k, 5], totalTimeSec=summ[k, 6],
                       error=int(st[k]))
        out.append((v1[k], v2[k], records, summary))
    return out


def newton_solve(ctx, mR, mT, norm, beta, deformation, *, max_outer=50, max_inner=500, nt=0, ls_max_steps=20,
                 tol_rel=1e-2, tol_abs=1e-5, forcing_cap=0.5, ls_c1=1e-4, ls_shrink=0.5, grad_cfl=1.0,
                 kind=PC_TWO_LEVEL, coarse_solver=COARSE_CHEB, cheb_iters=10, eps_scale=0.1, eig=None,
                 hessian_mode=GAUSS_NEWTON, fine_operator=None):
    """inverse::newtonSolve on host images (numpy); returns (v1, v2, records, summary).

    fine_operator: an object with `callbacks()` -> (build, data_term) ctypes callbacks, or
    (build, data_term, gradient, objective), and an `error` attribute (e.g.
    slab.SlabFineOperator); the solve then takes its fine GN data term (and its gradient and
    line-search objective) from it (C ABI vrg_set_fine_operator / vrg_set_external_ops) and
    re-raises the callback's exception."""
    import numpy as np

    mR = np.ascontiguousarray(mR, dtype=np.float64)
    mT = np.ascontiguousarray(mT, dtype=np.float64)
    n1, n2 = mR.shape
    ci = (C.c_int * 5)(max_outer, max_inner, nt, ls_max_steps, hessian_mode)
    cd = (C.c_double * 6)(tol_rel, tol_abs, forcing_cap, ls_c1, ls_shrink, grad_cfl)
    pi, pd = _pc_arrays(kind, coarse_solver, cheb_iters, eps_scale, eig)
    v1, v2 = np.empty_like(mR), np.empty_like(mR)
    rec = np.zeros((max_outer + 1, 12))
    summ = np.zeros(7)
    hp = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    if fine_operator is not None:
        cbs = fine_operator.callbacks()
        if not isinstance(cbs, dict):
            cbs = dict(zip(EXTERNAL_OPS_FIELDS, cbs))
        ops = ExternalOps(**{k: C.cast(cb, C.c_void_p) for k, cb in cbs.items() if cb is not None})
        fine_operator.error = None
        ctx.check(ctx.lib.vrg_set_external_ops(ctx.h, C.c_void_p(C.addressof(ops))))
    try:
        code = ctx.lib.vrg_newton_solve(ctx.h, n1, n2, hp(mR), hp(mT), norm, beta, deformation,
                                        C.cast(ci, C.c_void_p), C.cast(cd, C.c_void_p), C.cast(pi, C.c_void_p),
                                        C.cast(pd, C.c_void_p), hp(v1), hp(v2), hp(rec), max_outer + 1, hp(summ))
    finally:
        if fine_operator is not None:
            ctx.lib.vrg_set_external_ops(ctx.h, None)
    if fine_operator is not None and code and fine_operator.error is not None:
        raise fine_operator.error
    ctx.check(code)
    k = int(summ[1])
    records = [dict(zip(RECORD_FIELDS, row)) for row in rec[:k]]
    summary = dict(status=int(summ[0]), iterations=k, finalGradNormRel=summ[2], finalResidualRel=summ[3],
                   jacMin=summ[4], jacMax=summ[5], totalTimeSec=summ[6])
    return v1, v2, records, summary
