"""CPU restatement (numpy) of the reference's GN Hessian-matvec path — TEST INFRASTRUCTURE.

This module is the parity oracle: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg import it, and only as the checker.  It is itself pinned against the
UNMODIFIED reference compiled in oracle/_ref (tests/test_oracle_pins.py) and against the
reference's own analytic pins (test_interp.cpp / test_spectral.cpp / test_transport.cpp).

Each function cites the reference file:line it restates (paths relative to
/root/reference/proj/core).  Fields are numpy (n1, n2) float64 arrays, row-major, axis 1
fastest, node (i1, i2) at (-pi + i1*h1, -pi + i2*h2) (include/veloreg/field.hpp:13-24).
FFT: numpy's pocketfft rfft2/irfft2 — forward unnormalised, inverse carrying 1/N, the same
n1 x (n2/2+1) half spectrum as src/fft.cpp:57-78.
"""
from __future__ import annotations

import math

import numpy as np

PI = math.pi
TWO_PI = 2.0 * math.pi
BLOWUP_FACTOR = 1e3           # src/transport.cpp:14
EMAX_INFLATION = 1.05         # src/precond.cpp:18


class BlowupError(RuntimeError):
    """transport::BlowupError (include/veloreg/transport.hpp:35-38)."""


# ----------------------------------------------------------------------------- grid / BLAS-1
def spacing(shape):
    return (TWO_PI / shape[0], TWO_PI / shape[1])


def coords(shape):
    """Grid::coord (field.hpp:24): node a of axis i at -pi + a*h_i."""
    h1, h2 = spacing(shape)
    x1 = -PI + h1 * np.arange(shape[0])
    x2 = -PI + h2 * np.arange(shape[1])
    return np.meshgrid(x1, x2, indexing="ij")


def dot(u, w):
    """field.cpp:47-54: midpoint rule h1*h2*sum(u*w); vector fields sum components."""
    h1, h2 = spacing(u[0].shape if isinstance(u, tuple) else u.shape)
    if isinstance(u, tuple):
        return float(h1 * h2 * np.sum(u[0] * w[0])) + float(h1 * h2 * np.sum(u[1] * w[1]))
    return float(h1 * h2 * np.sum(u * w))


def norm_l2(u):
    return math.sqrt(dot(u, u))


def norm_linf(u):
    """field.cpp:59-65 (std::max ignores a NaN right operand)."""
    if isinstance(u, tuple):
        return max(norm_linf(u[0]), norm_linf(u[1]))
    a = np.abs(u)
    a = a[~np.isnan(a)]
    return float(a.max()) if a.size else 0.0


# ----------------------------------------------------------------------------- B-spline interp
def _cyclic_solve(f, axis):
    """CyclicSpline1D (src/interp.cpp:16-57): periodic (c_{i-1}+4c_i+c_{i+1})/6 = f_i by the
    Thomas algorithm on the modified diagonal plus a Sherman-Morrison rank-one correction,
    vectorised over the other axis."""
    f = np.moveaxis(np.array(f, dtype=np.float64), axis, 0)
    n = f.shape[0]
    a, b = 1.0 / 6.0, 2.0 / 3.0
    gamma = -b
    diag = np.full(n, b)
    diag[0] = b - gamma
    diag[n - 1] = b - a * a / gamma

    def thomas(rhs):
        out = np.empty_like(rhs)
        cp = np.empty(n)
        beta = diag[0]
        out[0] = rhs[0] / beta
        for i in range(1, n):
            cp[i] = a / beta
            beta = diag[i] - a * cp[i]
            out[i] = (rhs[i] - a * out[i - 1]) / beta
        for i in range(n - 2, -1, -1):
            out[i] -= cp[i + 1] * out[i + 1]
        return out

    u = np.zeros(n)
    u[0] = gamma
    u[n - 1] = a
    q = thomas(u)
    w = thomas(f)
    vy = w[0] + (a / gamma) * w[n - 1]
    vq = q[0] + (a / gamma) * q[n - 1]
    fact = vy / (1.0 + vq)
    out = w - fact * (q.reshape((n,) + (1,) * (w.ndim - 1)))
    return np.moveaxis(out, 0, axis)


def prefilter(u):
    """interp::prefilter (src/interp.cpp:75-85): rows (axis 1) then columns (axis 0)."""
    if not np.all(np.isfinite(u)):
        raise ValueError("prefilter: non-finite value")
    return _cyclic_solve(_cyclic_solve(u, 1), 0)


def _bspline_weights(f):
    """bsplineWeights (src/interp.cpp:59-65)."""
    f2 = f * f
    f3 = f2 * f
    return ((1.0 - 3.0 * f + 3.0 * f2 - f3) / 6.0, (3.0 * f3 - 6.0 * f2 + 4.0) / 6.0,
            (-3.0 * f3 + 3.0 * f2 + 3.0 * f + 1.0) / 6.0, f3 / 6.0)


def evaluate(c, x1, x2):
    """interp::evaluate (src/interp.cpp:87-127): wrap into [-pi,pi), s=(x+pi)/h, floor, 4x4
    tensor-product B-spline weights over b-1..b+2 with periodic index wrap."""
    if not (np.all(np.isfinite(x1)) and np.all(np.isfinite(x2))):
        raise ValueError("evaluate: non-finite point coordinate")
    n1, n2 = c.shape
    h1, h2 = spacing(c.shape)
    x1 = x1 - TWO_PI * np.floor((x1 + PI) / TWO_PI)
    x2 = x2 - TWO_PI * np.floor((x2 + PI) / TWO_PI)
    s1 = (x1 + PI) / h1
    s2 = (x2 + PI) / h2
    b1 = np.floor(s1)
    b2 = np.floor(s2)
    w1 = _bspline_weights(s1 - b1)
    w2 = _bspline_weights(s2 - b2)
    b1 = b1.astype(np.int64)
    b2 = b2.astype(np.int64)
    acc = np.zeros(c.shape)
    for a in range(4):
        i1 = np.mod(b1 - 1 + a, n1)
        row = np.zeros(c.shape)
        for b in range(4):
            i2 = np.mod(b2 - 1 + b, n2)
            row += w2[b] * c[i1, i2]
        acc += w1[a] * row
    return acc


def interp(u, x1, x2):
    return evaluate(prefilter(u), x1, x2)


# ----------------------------------------------------------------------------- spectral
def _wave(n):
    """fft::wavenumber (src/fft.cpp:80)."""
    k = np.arange(n)
    return np.where(k <= n // 2, k, k - n).astype(np.float64)


def _wave_nyq0(n):
    """nyquistZeroedWave (src/spectral.cpp:31-33)."""
    k = _wave(n)
    k[n // 2] = 0.0
    return k


def _half_waves(shape, nyq0):
    n1, n2 = shape
    f = _wave_nyq0 if nyq0 else _wave
    k1 = f(n1)[:, None]
    k2 = f(n2)[: n2 // 2 + 1][None, :]
    return k1, k2


def fft_forward(u):
    return np.fft.rfft2(u)


def fft_inverse(s, shape):
    return np.fft.irfft2(s, s=shape)


def gradient(u):
    """spectral::gradient (src/spectral.cpp:68-87): i*k per axis, Nyquist zeroed."""
    s = fft_forward(u)
    k1, k2 = _half_waves(u.shape, True)
    return fft_inverse(1j * k1 * s, u.shape), fft_inverse(1j * k2 * s, u.shape)


def divergence(v1, v2):
    """spectral::divergence (src/spectral.cpp:89-107)."""
    k1, k2 = _half_waves(v1.shape, True)
    return fft_inverse(1j * k1 * fft_forward(v1) + 1j * k2 * fft_forward(v2), v1.shape)


def norm_order(norm):
    return {1: 1, 2: 2, 3: 3}[norm]


def weights(shape, norm):
    """SpectralWeights::make (src/spectral.cpp:46-66) restricted to the half spectrum:
    gamma = (k1^2+k2^2)^p, gammaRegularized = gamma with 0 -> 1."""
    k1, k2 = _half_waves(shape, False)
    ksq = k1 * k1 + k2 * k2
    val = np.ones_like(ksq)
    for _ in range(norm_order(norm)):
        val = val * ksq
    return val, np.where(val == 0.0, 1.0, val)


def apply_reg(v1, v2, norm, beta):
    """spectral::applyReg (src/spectral.cpp:109-119): beta*gamma per mode."""
    if beta <= 0.0:
        raise ValueError("applyReg: beta must be positive")
    g, _ = weights(v1.shape, norm)
    return tuple(fft_inverse(fft_forward(v) * (beta * g), v1.shape) for v in (v1, v2))


def apply_inv_reg(v1, v2, norm, beta, power):
    """spectral::applyInvReg (src/spectral.cpp:121-131): (beta*gammaReg)^power (std::pow)."""
    if beta <= 0.0:
        raise ValueError("applyInvReg: beta must be positive")
    _, gr = weights(v1.shape, norm)
    sym = np.power(beta * gr, power)
    return tuple(fft_inverse(fft_forward(v) * sym, v1.shape) for v in (v1, v2))


def project_div_free(b1, b2):
    """spectral::projectDivFree (src/spectral.cpp:133-155): Leray on Nyquist-zeroed k;
    |k|^2 = 0 modes pass through."""
    s1, s2 = fft_forward(b1), fft_forward(b2)
    k1, k2 = _half_waves(b1.shape, True)
    k1 = np.broadcast_to(k1, s1.shape)
    k2 = np.broadcast_to(k2, s1.shape)
    ksq = k1 * k1 + k2 * k2
    m = ksq != 0.0
    kdotb = k1 * s1 + k2 * s2
    s1 = np.where(m, s1 - np.where(m, k1 * kdotb / np.where(m, ksq, 1.0), 0.0), s1)
    s2 = np.where(m, s2 - np.where(m, k2 * kdotb / np.where(m, ksq, 1.0), 0.0), s2)
    return fft_inverse(s1, b1.shape), fft_inverse(s2, b1.shape)


def resample(u, target):
    """spectral::resample (src/spectral.cpp:157-186): keep |k_i| < min(n_s,n_t)/2, amplitude
    N_t/N_s."""
    if tuple(u.shape) == tuple(target):
        return u.copy()
    s = fft_forward(u)
    t1, t2 = target
    tc = t2 // 2 + 1
    t = np.zeros((t1, tc), dtype=np.complex128)
    band1 = min(u.shape[0], t1) // 2
    band2 = min(u.shape[1], t2) // 2
    amp = float(t1 * t2) / float(u.shape[0] * u.shape[1])
    k1 = _wave(t1).astype(np.int64)
    k2 = _wave(t2).astype(np.int64)[:tc]
    for rt in range(t1):
        if abs(k1[rt]) >= band1:
            continue
        rs = k1[rt] if k1[rt] >= 0 else k1[rt] + u.shape[0]
        cols = np.nonzero(np.abs(k2) < band2)[0]
        t[rt, cols] = amp * s[rs, cols]
    return fft_inverse(t, (t1, t2))


def cutoff(u, high):
    """spectral::cutoffFilter (src/spectral.cpp:188-203): low = |k1|<n1/4 and |k2|<n2/4."""
    k1, k2 = _half_waves(u.shape, False)
    low = (np.abs(k1) < u.shape[0] // 4) & (np.abs(k2) < u.shape[1] // 4)
    keep = ~low if high else low
    return fft_inverse(fft_forward(u) * keep, u.shape)


def gaussian_smooth(u, sigma):
    """spectral::gaussianSmooth (src/spectral.cpp:205-212)."""
    h1, h2 = spacing(u.shape)
    s1, s2 = sigma * h1, sigma * h2
    k1, k2 = _half_waves(u.shape, False)
    return fft_inverse(fft_forward(u) * np.exp(-0.5 * (k1 * k1 * s1 * s1 + k2 * k2 * s2 * s2)), u.shape)


# ----------------------------------------------------------------------------- transport (SL)
def derive_steps(v1, v2, cfl):
    """transport::deriveSteps (src/transport.cpp:44-50)."""
    if not (cfl > 0.0) or cfl > 20.0:
        raise ValueError("cfl must lie in (0, 20]")
    h1, h2 = spacing(v1.shape)
    ratio = max(norm_linf(v1) / (cfl * h1), norm_linf(v2) / (cfl * h2))
    return max(2, int(math.ceil(ratio)))


def trace(v1, v2, ht, backward=False):
    """traceCharacteristics (src/transport.cpp:60-89): Heun, sgn=+1 forward / -1 backward."""
    if not ht > 0.0:
        raise ValueError("traceCharacteristics: ht must be positive")
    sgn = -1.0 if backward else 1.0
    c1, c2 = prefilter(v1), prefilter(v2)
    X1, X2 = coords(v1.shape)
    s1 = X1 - sgn * ht * v1
    s2 = X2 - sgn * ht * v2
    v1s = evaluate(c1, s1, s2)
    v2s = evaluate(c2, s1, s2)
    return X1 - sgn * 0.5 * ht * (v1 + v1s), X2 - sgn * 0.5 * ht * (v2 + v2s)


class Solver:
    """transport::Solver, SL branches (src/transport.cpp:91-454) with the lazy per-velocity
    caches of src/transport.cpp:107-127."""

    def __init__(self, v1, v2, nt):
        if not (np.all(np.isfinite(v1)) and np.all(np.isfinite(v2))):
            raise ValueError("transport velocity: non-finite value")
        self.v1, self.v2 = v1, v2
        self.nt = nt
        self.ht = 1.0 / nt
        self._char = {}
        self._divv = None
        self._dvdep = {}

    def characteristics(self, backward):
        if backward not in self._char:
            self._char[backward] = trace(self.v1, self.v2, self.ht, backward)
        return self._char[backward]

    def div_velocity(self):
        if self._divv is None:
            self._divv = divergence(self.v1, self.v2)
        return self._divv

    def div_velocity_at_departure(self, backward):
        if backward not in self._dvdep:
            self._dvdep[backward] = interp(self.div_velocity(), *self.characteristics(backward))
        return self._dvdep[backward]

    def continuity_step(self, u, backward=True):
        """slContinuityStep (src/transport.cpp:200-212)."""
        X = self.characteristics(backward)
        dv = self.div_velocity()
        dvd = self.div_velocity_at_departure(backward)
        uD = interp(u, *X)
        f0 = uD * dvd
        pred = uD + self.ht * f0
        return uD + 0.5 * self.ht * (f0 + pred * dv)

    def solve_state(self, m0, guard=True):
        """slState (src/transport.cpp:214-227)."""
        X = self.characteristics(False)
        thr = BLOWUP_FACTOR * norm_linf(m0)
        frames = [m0.copy()]
        m = m0
        for j in range(1, self.nt + 1):
            m = interp(m, *X)
            if guard and norm_linf(m) > thr:
                raise BlowupError(f"state solve exceeded the blow-up guard at step {j}")
            frames.append(m)
        return np.stack(frames)

    def solve_adjoint(self, lam1, guard=True):
        """slAdjoint (src/transport.cpp:229-241)."""
        thr = BLOWUP_FACTOR * norm_linf(lam1)
        frames = [None] * (self.nt + 1)
        frames[self.nt] = lam1.copy()
        lam = lam1
        for j in range(self.nt, 0, -1):
            lam = self.continuity_step(lam, True)
            if guard and norm_linf(lam) > thr:
                raise BlowupError(f"adjoint solve exceeded the blow-up guard at step {j}")
            frames[j - 1] = lam
        return np.stack(frames)

    def solve_incstate(self, vt1, vt2, state):
        """solveIncState, SL branch (src/transport.cpp:322-342)."""
        X = self.characteristics(False)
        vt1D = interp(vt1, *X)
        vt2D = interp(vt2, *X)
        gp1, gp2 = gradient(state[0])
        mt = np.zeros_like(vt1)
        frames = [mt.copy()]
        for j in range(1, self.nt + 1):
            g1D = interp(gp1, *X)
            g2D = interp(gp2, *X)
            gc1, gc2 = gradient(state[j])
            mtD = interp(mt, *X)
            s_prev = -(vt1D * g1D + vt2D * g2D)
            s_cur = -(vt1 * gc1 + vt2 * gc2)
            mt = mtD + 0.5 * self.ht * (s_prev + s_cur)
            gp1, gp2 = gc1, gc2
            frames.append(mt)
        return np.stack(frames)

    def jacobian_det(self):
        """Solver::jacobianDeterminant, SL (src/transport.cpp:456-464)."""
        jac = np.ones_like(self.v1)
        for _ in range(self.nt):
            jac = self.continuity_step(jac, False)
        return jac


def body_force(state, adjoint, ht):
    """assembleBodyForce, SL trapezoid (src/inverse.cpp:58-64)."""
    nt = state.shape[0] - 1
    b1 = np.zeros_like(state[0])
    b2 = np.zeros_like(state[0])
    for j in range(nt + 1):
        w = ht * (0.5 if j in (0, nt) else 1.0)
        g1, g2 = gradient(state[j])
        b1 += w * (adjoint[j] * g1)
        b2 += w * (adjoint[j] * g2)
    return b1, b2


# ----------------------------------------------------------------------------- reduced operators
COMPRESSIBLE, INCOMPRESSIBLE = 0, 1


def _projection(b1, b2, deform):
    """applyProjection (src/inverse.cpp:90-92)."""
    return project_div_free(b1, b2) if deform == INCOMPRESSIBLE else (b1, b2)


class Hessian:
    """inverse::HessianOperator, GN + SL (src/inverse.cpp:150-233)."""

    def __init__(self, v1, v2, mR, mT, norm, beta, deform, nt, state=None):
        self.solver = Solver(v1, v2, nt)
        self.norm, self.beta, self.deform = norm, beta, deform
        self.state = state if state is not None else self.solver.solve_state(mT)

    def data_term(self, vt1, vt2):
        """HessianOperator::Impl::dataTerm, GN (src/inverse.cpp:177-187, 213)."""
        mt = self.solver.solve_incstate(vt1, vt2, self.state)
        adj = self.solver.solve_adjoint(-1.0 * mt[-1], guard=True)
        b = body_force(self.state, adj, self.solver.ht)
        return _projection(*b, self.deform)

    def apply(self, vt1, vt2):
        """HessianOperator::apply (src/inverse.cpp:229-233): beta A vt + data term."""
        r1, r2 = apply_reg(vt1, vt2, self.norm, self.beta)
        d1, d2 = self.data_term(vt1, vt2)
        return r1 + d1, r2 + d2

    def split_apply(self, s1, s2):
        """applySplitHessianOf (src/precond.cpp:20-26)."""
        t = apply_inv_reg(s1, s2, self.norm, self.beta, -0.5)
        q = self.data_term(*t)
        o = apply_inv_reg(*q, self.norm, self.beta, -0.5)
        return o[0] + s1, o[1] + s2


def evaluate_objective(v1, v2, mR, mT, norm, beta, deform, nt):
    """evaluateObjective (src/inverse.cpp:96-114), compressible/incompressible."""
    st = Solver(v1, v2, nt).solve_state(mT)
    resid = st[-1] - mR
    mismatch = 0.5 * dot(resid, resid)
    reg = 0.5 * dot(apply_reg(v1, v2, norm, beta), (v1, v2))
    return mismatch + reg, mismatch, reg, st


def evaluate_gradient(v1, v2, mR, mT, norm, beta, deform, nt):
    """evaluateGradient (src/inverse.cpp:116-148)."""
    s = Solver(v1, v2, nt)
    st = s.solve_state(mT)
    resid = st[-1] - mR
    mismatch = 0.5 * dot(resid, resid)
    adj = s.solve_adjoint(-1.0 * resid)
    b = body_force(st, adj, s.ht)
    g1, g2 = apply_reg(v1, v2, norm, beta)
    reg = 0.5 * dot((g1, g2), (v1, v2))
    p1, p2 = _projection(*b, deform)
    return (g1 + p1, g2 + p2), mismatch + reg, mismatch, reg, st, adj


# ----------------------------------------------------------------------------- Krylov / PC
def chebyshev(op, r1, r2, k, emin, emax):
    """chebyshevSolve (src/precond.cpp:180-205)."""
    if not (emax > emin) or not (emin > 0.0):
        raise ValueError("chebyshevSolve: need eMax > eMin > 0")
    x1, x2 = np.zeros_like(r1), np.zeros_like(r2)
    if k <= 0:
        return x1, x2
    theta = 0.5 * (emax + emin)
    delta = 0.5 * (emax - emin)
    sigma = theta / delta
    rho = 1.0 / sigma
    r1, r2 = r1.copy(), r2.copy()
    d1, d2 = (1.0 / theta) * r1, (1.0 / theta) * r2
    for it in range(1, k + 1):
        if it > 1:
            rho_new = 1.0 / (2.0 * sigma - rho)
            d1 = (rho_new * rho) * d1 + (2.0 * rho_new / delta) * r1
            d2 = (rho_new * rho) * d2 + (2.0 * rho_new / delta) * r2
            rho = rho_new
        x1 = x1 + d1
        x2 = x2 + d2
        a1, a2 = op(d1, d2)
        r1 = r1 - a1
        r2 = r2 - a2
    return x1, x2


def pcg(A, b, M, tol, max_iter):
    """pcg (src/precond.cpp:38-85), residual in the preconditioned norm sqrt(r'Mr).
    Returns (x, iterations, converged, negCurv, indefinite, relResidual)."""
    x = (np.zeros_like(b[0]), np.zeros_like(b[1]))
    r = (b[0].copy(), b[1].copy())
    z = M(*r) if M else r
    rz = dot(r, z)
    if rz < 0.0 or not math.isfinite(rz):
        return x, 0, False, False, True, 0.0
    norm0 = math.sqrt(max(rz, 0.0))
    if not norm0 > 0.0:
        return x, 0, True, False, False, 0.0
    p = z
    its, rel = 0, 0.0
    for it in range(max_iter):
        Ap = A(*p)
        pAp = dot(p, Ap)
        if not pAp > 0.0:
            return x, its, False, True, False, math.sqrt(max(rz, 0.0)) / norm0
        alpha = rz / pAp
        x = (x[0] + alpha * p[0], x[1] + alpha * p[1])
        r = (r[0] - alpha * Ap[0], r[1] - alpha * Ap[1])
        z = M(*r) if M else r
        rz_new = dot(r, z)
        its = it + 1
        if rz_new < 0.0 or not math.isfinite(rz_new):
            return x, its, False, False, True, rel
        rel = math.sqrt(rz_new) / norm0
        if rel <= tol:
            return x, its, True, False, False, rel
        beta = rz_new / rz
        rz = rz_new
        p = (beta * p[0] + z[0], beta * p[1] + z[1])
    return x, its, False, False, False, rel


def tridiag_max_eig(alpha, beta):
    """tridiagMaxEig (src/precond.cpp:88-117): Sturm bisection, 100 iterations."""
    m = len(alpha)
    if m == 1:
        return alpha[0]
    lo = hi = alpha[0]
    for i in range(m):
        off = (abs(beta[i - 1]) if i > 0 else 0.0) + (abs(beta[i]) if i < m - 1 else 0.0)
        lo = min(lo, alpha[i] - off)
        hi = max(hi, alpha[i] + off)

    def count_below(x):
        cnt, d = 0, 1.0
        for i in range(m):
            offsq = beta[i - 1] * beta[i - 1] if i > 0 else 0.0
            d = alpha[i] - x - offsq / d
            if d == 0.0:
                d = -1e-300
            if d < 0.0:
                cnt += 1
        return cnt

    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if count_below(mid) >= m:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def lanczos_emax(op, q0, steps=30):
    """lanczosEmax (src/precond.cpp:134-161) from a given probe q0 (the reference draws it
    with randomBandLimitedVelocity(seed 0x5eed), src/problems.cpp:87-118)."""
    nq = norm_l2(q0)
    if not nq > 0.0:
        return 1.0
    basis = [(q0[0] / nq, q0[1] / nq)]
    alpha, beta = [], []
    for j in range(steps):
        w = op(*basis[j])
        if j > 0:
            w = (w[0] - beta[j - 1] * basis[j - 1][0], w[1] - beta[j - 1] * basis[j - 1][1])
        a = dot(w, basis[j])
        alpha.append(a)
        w = (w[0] - a * basis[j][0], w[1] - a * basis[j][1])
        for qi in basis:
            d = dot(w, qi)
            w = (w[0] - d * qi[0], w[1] - d * qi[1])
        b = norm_l2(w)
        if not math.isfinite(b):
            raise RuntimeError("lanczos breakdown (power-iteration fallback not restated)")
        if b < 1e-12:
            break
        beta.append(b)
        basis.append((w[0] / b, w[1] / b))
    beta = beta[: len(alpha) - 1]
    return tridiag_max_eig(alpha, beta)


class Coarse:
    """precond::CoarseOperator (src/precond.cpp:207-240): restricted problem, coarse nt from
    CFL (default SL CFL 5, src/newton.cpp:16)."""

    def __init__(self, v1, v2, mR, mT, norm, beta, deform, coarse_cfl=5.0):
        n1, n2 = v1.shape
        self.shape = (n1 // 2, n2 // 2)
        mRc = resample(mR, self.shape)
        mTc = resample(mT, self.shape)
        vc1, vc2 = resample(v1, self.shape), resample(v2, self.shape)
        self.nt = derive_steps(vc1, vc2, coarse_cfl)
        self.hess = Hessian(vc1, vc2, mRc, mTc, norm, beta, deform, self.nt)

    def split_apply(self, s1, s2):
        return self.hess.split_apply(s1, s2)


def two_level(r1, r2, coarse, cheb, cheb_iters, eps_scale, outer_tol, emin, emax):
    """applyTwoLevel (src/precond.cpp:264-289)."""
    lo = (cutoff(r1, False), cutoff(r2, False))
    hi = (cutoff(r1, True), cutoff(r2, True))
    rc = (resample(lo[0], coarse.shape), resample(lo[1], coarse.shape))
    if cheb:
        sc = chebyshev(coarse.split_apply, *rc, cheb_iters, emin, EMAX_INFLATION * emax)
    else:
        sc = pcg(coarse.split_apply, rc, None, eps_scale * outer_tol, 500)[0]
    if not (np.all(np.isfinite(sc[0])) and np.all(np.isfinite(sc[1]))):
        return r1, r2
    shape = r1.shape
    return resample(sc[0], shape) + hi[0], resample(sc[1], shape) + hi[1]
