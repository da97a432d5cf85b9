#include <functional>
// Device-resident two-level preconditioner, Chebyshev / PCG / Lanczos and the inexact
// Gauss-Newton-Krylov driver.  Host control flow mirrors src/precond.cpp and src/newton.cpp
// line for line (same decisions, same comparisons); all vectors and operator applications
// stay on the device.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <random>

#include <cooperative_groups.h>

#include "heun.cuh"
#include "precond.cuh"

namespace vrg {

namespace {

constexpr double kEmaxInflation = 1.05;  // precond.cpp:18

__device__ __forceinline__ int waveOfP(int idx, int n) { return idx <= n / 2 ? idx : idx - n; }

// problems.cpp:94-105: zero the top third of the spectrum (|k_i| >= n_i/3), with the 1/N of
// the inverse transform folded in.
__global__ void k_bandlimit(double2* s, int n1, int n2, double scale) {
    const int nc = n2 / 2 + 1;
    const std::size_t n = static_cast<std::size_t>(n1) * nc;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = static_cast<int>(i / nc), c = static_cast<int>(i - static_cast<std::size_t>(r) * nc);
    const bool cut = abs(waveOfP(r, n1)) >= n1 / 3 || abs(waveOfP(c, n2)) >= n2 / 3;
    s[i] = cut ? make_double2(0.0, 0.0) : make_double2(s[i].x * scale, s[i].y * scale);
}

// Two-level restriction (cutoffFilter Low + resample to the half grid, precond.cpp:266-268):
// coarse spectrum = amp * fine spectrum on |k_i| < n_i^c / 2, times 1/N_c.
// `sets` spectra one after another (pairs x components of a batch).
__global__ void k_restrict_low(const double2* __restrict__ f, int n1f, int n2f, double2* __restrict__ c, int n1c,
                               int n2c, int sets, double amp, double scale) {
    const int ncc = n2c / 2 + 1, ncf = n2f / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1c) * ncc;
    const std::size_t n = nPer * sets;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t set = i / nPer, li = i - set * nPer;
    f += set * static_cast<std::size_t>(n1f) * ncf;
    const int rt = static_cast<int>(li / ncc), col = static_cast<int>(li - static_cast<std::size_t>(rt) * ncc);
    const int k1 = waveOfP(rt, n1c), k2 = waveOfP(col, n2c);
    double2 v = make_double2(0.0, 0.0);
    // low band of the fine cut-off (|k_i| < n_i^f/4) intersected with the resample band
    if (abs(k1) < n1c / 2 && abs(k2) < n2c / 2 && abs(k1) < n1f / 4 && abs(k2) < n2f / 4) {
        const int rs = k1 >= 0 ? k1 : k1 + n1f;
        const double2 s = f[static_cast<std::size_t>(rs) * ncf + col];
        v = make_double2(s.x * amp, s.y * amp);
    }
    c[i] = make_double2(v.x * scale, v.y * scale);
}

// out^ = (prolong(sc^) * amp + highpass(r^)) * scale on the fine half spectrum
// (resample(sc, fine) + cutoffFilter(r, High), precond.cpp:267, 286-287).
// rf and out may alias (in-place update, one element per thread)
__global__ void k_prolong_add_high(const double2* __restrict__ sc, int n1c, int n2c, const double2* rf, double2* out,
                                   int n1f, int n2f, int sets, double amp, double scale) {
    const int ncc = n2c / 2 + 1, ncf = n2f / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1f) * ncf;
    const std::size_t n = nPer * sets;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t set = i / nPer, li = i - set * nPer;
    sc += set * static_cast<std::size_t>(n1c) * ncc;
    const int rt = static_cast<int>(li / ncf), col = static_cast<int>(li - static_cast<std::size_t>(rt) * ncf);
    const int k1 = waveOfP(rt, n1f), k2 = waveOfP(col, n2f);
    double2 v = make_double2(0.0, 0.0);
    if (abs(k1) < n1c / 2 && abs(k2) < n2c / 2) {
        const int rs = k1 >= 0 ? k1 : k1 + n1c;
        const double2 s = sc[static_cast<std::size_t>(rs) * ncc + col];
        v = make_double2(s.x * amp, s.y * amp);
    }
    const bool low = abs(k1) < n1f / 4 && abs(k2) < n2f / 4;
    if (!low) {
        v.x += rf[i].x;
        v.y += rf[i].y;
    }
    out[i] = make_double2(v.x * scale, v.y * scale);
}

unsigned specBlocks(const GridDims& g) { return static_cast<unsigned>((g.specPoints() + 255) / 256); }

double secondsSince(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}


// Unpreconditioned PCG step with the scalars on the device: alpha = rz / pAp, x += alpha p,
// r -= alpha ap (the arithmetic of axpby(alpha, p, 1, x) and axpby(-alpha, ap, 1, r)); no
// update when !(pAp > 0), where pcg() returns with negative curvature and x as it was.
__global__ void k_pcg_update(std::size_t n, const double* __restrict__ rz, const double* __restrict__ pAp,
                             const double* __restrict__ p, const double* __restrict__ ap, double* x, double* r) {
    const double d = *pAp;
    if (!(d > 0.0)) return;
    const double alpha = *rz / d, na = -alpha;
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        x[i] = x[i] + alpha * p[i];
        r[i] = r[i] + na * ap[i];
    }
}

// ------------------------------------------------------------------------------ Lanczos step
// One Lanczos step's orthogonalisation in one launch: w -= beta_{j-1} q_{j-1}; alpha_j = <w,q_j>;
// w -= alpha_j q_j; modified Gram-Schmidt against q_0..q_{nb-1}; |w|^2.  One thread-block
// cluster of kLzCtas CTAs holds w in registers (kPer elements per thread); each inner product is
// a warp / block / cluster (DSMEM) reduction in a fixed order, identical in every CTA, so the
// coefficients never leave the device.  Replaces 3(nb+2) launches and nb+2 host reads per step
// on small coarse grids (2 N <= kLzCtas * 1024 * 8), where launch latency dominates.
constexpr int kLzCtas = 8;
constexpr int kLzThreads = 1024;

struct LzRed {
    double warp[32];
    double part[2];  // this CTA's partial, double-buffered by call parity
    double total[2];
};

__device__ __forceinline__ double lzClusterSum(double v, LzRed& red, int& parity) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red.warp[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double x = red.warp[lane];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) red.part[parity] = x;
    }
    cluster.sync();  // every CTA's partial of this call is visible cluster-wide
    if (wid == 0) {
        double x = 0.0;
        if (lane < kLzCtas) x = *cluster.map_shared_rank(&red.part[parity], lane);
        for (int o = 4; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) red.total[parity] = x;
    }
    __syncthreads();
    const double t = red.total[parity];
    parity ^= 1;
    return t;
}

// beta_{j-1} of every pair of a batch (kernel parameter)
constexpr int kLzMaxPairs = 64;
struct LzBeta {
    double v[kLzMaxPairs];
};

// Batches of stacked pairs (GridDims::pairs): one cluster per pair (blockIdx.x / kLzCtas), the
// pair's vector being its slots of the two components (nPer values each, component stride
// nTot); with one pair this is the contiguous vector of length n = 2 nPer.  betaPrev, alphaOut
// and bsqOut are per pair (alphaOut at stride alphaStride).
template <int kPer, bool kBatch>
__global__ void __cluster_dims__(kLzCtas, 1, 1) __launch_bounds__(kLzThreads, 1)
    k_lanczos_orth(double* __restrict__ w, const double* __restrict__ Q, std::size_t nPer, std::size_t nTot, int j,
                   int nb, LzBeta betaPrev, double hh, double* __restrict__ alphaOut,
                   int alphaStride, double* __restrict__ bsqOut) {
    __shared__ LzRed red;
    int parity = 0;
    const int pair = blockIdx.x / kLzCtas;
    const std::size_t n = 2 * nPer;  // elements of one pair's vector
    const std::size_t base = static_cast<std::size_t>(blockIdx.x % kLzCtas) * kLzThreads + threadIdx.x;
    const std::size_t qStride = 2 * nTot;  // one basis vector of the batch
    constexpr std::size_t kStride = static_cast<std::size_t>(kLzCtas) * kLzThreads;
    // batch offset of element e of this pair's vector
    auto at = [&](std::size_t e) {
        if constexpr (kBatch)
            return e < nPer ? pair * nPer + e : nTot + pair * nPer + (e - nPer);
        else
            return e;
    };
    const bool lead = blockIdx.x % kLzCtas == 0 && threadIdx.x == 0;
    double x[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const std::size_t e = base + k * kStride;
        x[k] = e < n ? w[at(e)] : 0.0;
    }
    auto qv = [&](int i, double (&q)[kPer]) {
        const double* qi = Q + static_cast<std::size_t>(i) * qStride;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const std::size_t e = base + k * kStride;
            q[k] = e < n ? qi[at(e)] : 0.0;
        }
    };
    // kPer = 8 re-reads q_i (L1/L2 hits) after the cluster sum instead of holding it across
    // the sum: 64 registers at 1024 threads cannot hold x, q and the addresses without spills
    constexpr bool kReload = kPer >= 8;
    auto project = [&](int i, bool storeAlpha) {
        double q[kReload ? 1 : kPer];
        const double* qi = Q + static_cast<std::size_t>(i) * qStride;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const std::size_t e = base + k * kStride;
            const double qk = e < n ? qi[at(e)] : 0.0;
            if constexpr (!kReload) q[k] = qk;
            s += x[k] * qk;
        }
        const double c = hh * lzClusterSum(s, red, parity);
        if (storeAlpha && lead) alphaOut[static_cast<std::size_t>(pair) * alphaStride] = c;
        const double a = -c;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            if constexpr (kReload) {
                const std::size_t e = base + k * kStride;
                x[k] = x[k] + a * (e < n ? qi[at(e)] : 0.0);
            } else {
                x[k] = x[k] + a * q[k];
            }
        }
    };
    if (j > 0) {
        double q[kPer];
        qv(j - 1, q);
        const double a = -betaPrev.v[pair];
#pragma unroll
        for (int k = 0; k < kPer; ++k) x[k] = x[k] + a * q[k];
    }
    project(j, true);
    for (int i = 0; i < nb; ++i) project(i, false);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) s += x[k] * x[k];
    const double bsq = hh * lzClusterSum(s, red, parity);
    if (lead) bsqOut[pair] = bsq;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const std::size_t e = base + k * kStride;
        if (e < n) w[at(e)] = x[k];
    }
}

// One pair or a batch of `pairs` (alphaOut / bsqOut per pair on the device).
bool launchLanczosOrth(Ctx& ctx, double* w, const double* Q, std::size_t nPer, int pairs, int j, int nb,
                       const LzBeta& betaPrev, double hh, double* alphaOut, int alphaStride, double* bsqOut) {
    if (pairs > kLzMaxPairs) return false;
    const std::size_t per = (2 * nPer + kLzCtas * kLzThreads - 1) / (kLzCtas * kLzThreads);
    LaunchScope ls_(ctx, "k_lanczos_orth");
    const dim3 grid(kLzCtas * pairs), block(kLzThreads);
    const std::size_t nTot = nPer * pairs;
#define VRG_LZ(P, B) \
    k_lanczos_orth<P, B><<<grid, block, 0, ctx.stream>>>(w, Q, nPer, nTot, j, nb, betaPrev, hh, alphaOut, alphaStride, bsqOut)
    if (pairs == 1) {
        if (per <= 1) VRG_LZ(1, false);
        else if (per <= 2) VRG_LZ(2, false);
        else if (per <= 4) VRG_LZ(4, false);
        else if (per <= 8) VRG_LZ(8, false);
        else return false;
    } else {  // a batch: one cluster per pair, up to 4 values per thread (coarse grids up to 128^2)
        if (per <= 1) VRG_LZ(1, true);
        else if (per <= 2) VRG_LZ(2, true);
        else if (per <= 4) VRG_LZ(4, true);
        else return false;
    }
#undef VRG_LZ
    VRG_LAUNCH_CHECK();
    return true;
}
}  // namespace

// ------------------------------------------------------------------------------ vector BLAS
double vdot(Ctx& ctx, const GridDims& g, const double* a, const double* b) {
    const std::size_t N = g.points();
    return dot(ctx, g, a, a + N, b, b + N);
}

double vnormL2(Ctx& ctx, const GridDims& g, const double* a) { return std::sqrt(vdot(ctx, g, a, a)); }

double vnormLinf(Ctx& ctx, const GridDims& g, const double* a) {
    const std::size_t N = g.points();
    return normLinf(ctx, N, a, a + N);
}

// ------------------------------------------------------------------------------ random probes
void randomBandLimitedField(Ctx& ctx, const GridDims& g, std::uint64_t seed, double* out) {
    const std::size_t N = g.points();
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::vector<double> noise(N);
    for (double& x : noise) x = gauss(rng);
    VRG_CUDA(cudaMemcpyAsync(out, noise.data(), sizeof(double) * N, cudaMemcpyHostToDevice, ctx.stream));
    cplx* s = specScratch(ctx, g, 4, 1);
    fftForward(ctx, g, out, s, 1);
    {
        LaunchScope ls_(ctx, "k_bandlimit");
        k_bandlimit<<<specBlocks(g), 256, 0, ctx.stream>>>(s, g.n1, g.n2, 1.0 / N);
    }
    VRG_LAUNCH_CHECK();
    fftInverse(ctx, g, s, out, 1);
    ctx.ffts += 2;
    const double m = normLinf(ctx, N, out);  // synchronises: `noise` may go out of scope
    if (m > 0.0) axpby(ctx, N, 0.0, out, 1.0 / m, out);
}

void randomBandLimitedVelocity(Ctx& ctx, const GridDims& g, std::uint64_t seed, double* out) {
    randomBandLimitedField(ctx, g, seed, out);
    randomBandLimitedField(ctx, g, seed ^ 0x9e3779b97f4a7c15ull, out + g.points());
}

// ------------------------------------------------------------------------------ coarse operator
CoarseOperator::CoarseOperator(Ctx& c, const GridDims& fg, const double* v, const double* mR, const double* mT,
                               const Model& model, double coarseCfl)
    : ctx(c), fine(fg), gc(fg.n1 / 2, fg.n2 / 2, fg.pairs) {
    checkGrid(gc.n1, gc.n2);
    // a batch of stacked pairs shares one coarse step count: only at v = 0 (every pair nt = 2)
    if (fg.pairs > 1 && v) throw NotSupported("CoarseOperator: a batch of pairs at v = 0 only");
    const std::size_t Nc = gc.points(), Nf = fine.points();
    mRc.alloc(sizeof(double) * Nc);
    mTc.alloc(sizeof(double) * Nc);
    vc.alloc(sizeof(double) * 2 * Nc);
    resample(ctx, fine, mR, gc, mRc.d());
    resample(ctx, fine, mT, gc, mTc.d());
    if (v) {
        resample(ctx, fine, v, gc, vc.d());
        resample(ctx, fine, v + Nf, gc, vc.d() + Nc);
    } else {
        fill(ctx, 2 * Nc, 0.0, vc.d());
        ctx.ffts += 4;  // the reference resamples the zero velocity too
    }
    nt = deriveSteps(ctx, gc, vc.d(), vc.d() + Nc, coarseCfl);
    Model coarseModel = model;
    coarseModel.scheme = kSchemeSL;  // the coarse problem is SL(5) whatever the fine scheme (kCoarseScheme)
    hess = std::make_unique<Hessian>(ctx, gc, vc.d(), vc.d() + Nc, mRc.d(), mTc.d(), coarseModel, nt, nullptr);
}

// ------------------------------------------------------------------------------ Chebyshev / PCG
namespace {
// The vector updates of chebyshevSolve fused per iteration, with the rounding of the separate
// BLAS kernels they replace (k_lincomb: fma(x, a, b*y); k_axpby with b = 1: fma(x, a, y)), so
// the iterates are bit-identical:
//   init:  r = rhs, d = (1/theta) r + 0 r, x = 0 + d
//   step:  r -= A d, d = c1 d + c2 r, x += d   (the last iteration's r -= A d is dead)
__global__ void k_cheb_init(std::size_t n, const double* __restrict__ rhs, double* __restrict__ r,
                            double* __restrict__ d, double* __restrict__ x, double invTheta) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double ri = rhs[i];
        r[i] = ri;
        const double di = __fma_rn(ri, invTheta, __dmul_rn(ri, 0.0));
        d[i] = di;
        x[i] = __fma_rn(di, 1.0, 0.0);
    }
}

__global__ void k_cheb_step(std::size_t n, const double* __restrict__ ad, double* __restrict__ r,
                            double* __restrict__ d, double* __restrict__ x, double c1, double c2) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double ri = __fma_rn(ad[i], -1.0, r[i]);
        r[i] = ri;
        const double di = __fma_rn(d[i], c1, __dmul_rn(ri, c2));
        d[i] = di;
        x[i] = __fma_rn(di, 1.0, x[i]);
    }
}
}  // namespace

void chebyshevSolve(Ctx& ctx, const GridDims& g, const LinOpDev& op, const double* rhs, int k, double eMin,
                    double eMax, double* x) {
    if (!(eMax > eMin) || !(eMin > 0.0)) throw InvalidArgument("chebyshevSolve: need eMax > eMin > 0");
    const std::size_t n = 2 * g.points();
    if (k <= 0) {
        fill(ctx, n, 0.0, x);
        return;
    }
    const double theta = 0.5 * (eMax + eMin);
    const double delta = 0.5 * (eMax - eMin);
    const double sigma = theta / delta;
    double rho = 1.0 / sigma;
    double* r = ctx.scratchBuf(120, sizeof(double) * n);
    double* d = ctx.scratchBuf(121, sizeof(double) * n);
    double* ad = ctx.scratchBuf(122, sizeof(double) * n);
    {
        LaunchScope ls_(ctx, "k_cheb_init");
        k_cheb_init<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, rhs, r, d, x, 1.0 / theta);
    }
    VRG_LAUNCH_CHECK();
    for (int it = 1; it <= k; ++it) {
        op(d, ad);
        if (it == k) break;
        const double rhoNew = 1.0 / (2.0 * sigma - rho);
        const double c1 = rhoNew * rho, c2 = 2.0 * rhoNew / delta;
        rho = rhoNew;
        {
            LaunchScope ls_(ctx, "k_cheb_step");
            k_cheb_step<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, ad, r, d, x, c1, c2);
        }
        VRG_LAUNCH_CHECK();
    }
}

// The M = null branch of pcg() (the coarse solve of the two-level preconditioner) with one host
// read per iteration: pAp and rzNew land in adjacent device scalars (k_pcg_update applies the
// step only when pAp > 0) and come back together.  Same decisions and arithmetic as the loop
// in pcg().
// VRG_TRACE=1: per-phase host wall times of newtonSolve and the PCG exits on stderr
// (diagnostics only).
static bool traceOn() {
    static const bool on = [] {
        const char* e = std::getenv("VRG_TRACE");
        return e && e[0] == '1';
    }();
    return on;
}

static PcgOut pcgUnpreconditioned(Ctx& ctx, const GridDims& g, const LinOpDev& A, double rz, double norm0, int maxIter,
                           double tol, double* x, double* r, double* p, double* ap) {
    PcgOut out;
    const std::size_t N = g.points(), n = 2 * N;
    const double hh = g.h1() * g.h2();
    double* sc = ctx.reduce.d() + 2 * kReduceBlocks + 40;  // [rz, pAp, rzNew]
    fill(ctx, 1, rz, sc);
    for (int it = 0; it < maxIter; ++it) {
        A(p, ap);
        launchDotInto(ctx, N, p, ap, p + N, ap + N, hh, sc + 1);
        {
            LaunchScope ls_(ctx, "k_pcg_update");
            k_pcg_update<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, sc, sc + 1, p, ap, x, r);
        }
        VRG_LAUNCH_CHECK();
        launchDotInto(ctx, N, r, r, r + N, r + N, hh, sc + 2);
        VRG_CUDA(cudaMemcpyAsync(ctx.hostScalars, sc + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        const double pAp = ctx.hostScalars[0], rzNew = ctx.hostScalars[1];
        if (!(pAp > 0.0)) {
            out.negativeCurvature = true;
            out.relResidual = std::sqrt(std::max(rz, 0.0)) / norm0;
            return out;
        }
        out.iterations = it + 1;
        if (rzNew < 0.0 || !std::isfinite(rzNew)) {
            out.indefinitePreconditioner = true;
            return out;
        }
        out.relResidual = std::sqrt(rzNew) / norm0;
        if (out.relResidual <= tol) {
            out.converged = true;
            if (traceOn())
                std::fprintf(stderr, "[trace] coarse pcg converged it=%d rel=%.17g tol=%.17g\n", out.iterations,
                             out.relResidual, tol);
            return out;
        }
        if (traceOn())
            std::fprintf(stderr, "[trace] coarse pcg it=%d rel=%.17g tol=%.17g\n", out.iterations, out.relResidual, tol);
        const double beta = rzNew / rz;
        rz = rzNew;
        VRG_CUDA(cudaMemcpyAsync(sc, sc + 2, sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
        lincomb(ctx, n, beta, p, 1.0, r, p);
    }
    return out;
}

PcgOut pcg(Ctx& ctx, const GridDims& g, const LinOpDev& A, const double* b, const LinOpDev* M, double tol,
           int maxIter, double* x) {
    PcgOut out;
    const std::size_t n = 2 * g.points();
    const int base = M ? 100 : 110;  // fine (preconditioned) and coarse PCG use separate buffers
    double* r = ctx.scratchBuf(base + 0, sizeof(double) * n);
    double* z = M ? ctx.scratchBuf(base + 1, sizeof(double) * n) : r;
    double* p = ctx.scratchBuf(base + 2, sizeof(double) * n);
    double* ap = ctx.scratchBuf(base + 3, sizeof(double) * n);
    fill(ctx, n, 0.0, x);
    copy(ctx, n, b, r);
    if (M) (*M)(r, z);
    double rz = vdot(ctx, g, r, z);
    if (rz < 0.0 || !std::isfinite(rz)) {
        out.indefinitePreconditioner = true;
        return out;
    }
    const double norm0 = std::sqrt(std::max(rz, 0.0));
    if (!(norm0 > 0.0)) {
        out.converged = true;
        return out;
    }
    copy(ctx, n, z, p);
    if (!M) return pcgUnpreconditioned(ctx, g, A, rz, norm0, maxIter, tol, x, r, p, ap);
    for (int it = 0; it < maxIter; ++it) {
        A(p, ap);
        const double pAp = vdot(ctx, g, p, ap);
        if (!(pAp > 0.0)) {
            out.negativeCurvature = true;
            out.relResidual = std::sqrt(std::max(rz, 0.0)) / norm0;
            return out;
        }
        const double alpha = rz / pAp;
        axpby(ctx, n, alpha, p, 1.0, x);
        axpby(ctx, n, -alpha, ap, 1.0, r);
        if (M) (*M)(r, z);
        const double rzNew = vdot(ctx, g, r, z);
        out.iterations = it + 1;
        if (rzNew < 0.0 || !std::isfinite(rzNew)) {
            out.indefinitePreconditioner = true;
            return out;
        }
        out.relResidual = std::sqrt(rzNew) / norm0;
        if (out.relResidual <= tol) {
            out.converged = true;
            return out;
        }
        const double beta = rzNew / rz;
        rz = rzNew;
        lincomb(ctx, n, beta, p, 1.0, z, p);
    }
    return out;
}

// ------------------------------------------------------------------------------ Lanczos
double tridiagMaxEig(const std::vector<double>& alpha, const std::vector<double>& beta) {
    const int m = static_cast<int>(alpha.size());
    if (m == 1) return alpha[0];
    double lo = alpha[0], hi = alpha[0];
    for (int i = 0; i < m; ++i) {
        const double off = (i > 0 ? std::abs(beta[i - 1]) : 0.0) + (i < m - 1 ? std::abs(beta[i]) : 0.0);
        lo = std::min(lo, alpha[i] - off);
        hi = std::max(hi, alpha[i] + off);
    }
    auto countBelow = [&](double x) {
        int count = 0;
        double d = 1.0;
        for (int i = 0; i < m; ++i) {
            const double offsq = i > 0 ? beta[i - 1] * beta[i - 1] : 0.0;
            d = alpha[i] - x - offsq / d;
            if (d == 0.0) d = -1e-300;
            if (d < 0.0) ++count;
        }
        return count;
    };
    for (int it = 0; it < 100; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (countBelow(mid) >= m)
            hi = mid;
        else
            lo = mid;
    }
    return 0.5 * (lo + hi);
}

static double powerIterationEmax(Ctx& ctx, const GridDims& g, const LinOpDev& op, std::uint64_t seed) {
    const std::size_t n = 2 * g.points();
    DBuf qb(sizeof(double) * n), wb(sizeof(double) * n);
    double* q = qb.d();
    double* w = wb.d();
    randomBandLimitedVelocity(ctx, g, seed, q);
    double lambda = 1.0;
    const double nq = vnormL2(ctx, g, q);
    axpby(ctx, n, 0.0, q, 1.0 / nq, q);
    for (int it = 0; it < 50; ++it) {
        op(q, w);
        lambda = vdot(ctx, g, q, w);
        const double nw = vnormL2(ctx, g, w);
        if (!(nw > 0.0)) break;
        axpby(ctx, n, 0.0, w, 1.0 / nw, w);
        std::swap(q, w);
    }
    return lambda;
}

struct PhaseTimer {
    Ctx& ctx;
    const char* what;
    std::chrono::steady_clock::time_point t0;
    NvtxRange nv_;
    PhaseTimer(Ctx& c, const char* w) : ctx(c), what(w), t0(std::chrono::steady_clock::now()), nv_(w) {}
    ~PhaseTimer() {
        if (!traceOn()) return;
        ctx.sync();
        std::fprintf(stderr, "trace %-22s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

double lanczosEmax(Ctx& ctx, const GridDims& g, const LinOpDev& op, int steps, std::uint64_t seed) {
    // The alpha and Gram-Schmidt coefficients stay on the device, so a step costs two host
    // syncs (the operator's guard and beta) instead of 3 + j: on small grids one cluster
    // launch per step (k_lanczos_orth), else launchDotInto + axpyNegDevCoef per basis vector
    // (the same arithmetic as vdot + axpby).
    const std::size_t N = g.points(), n = 2 * N;
    const double hh = g.h1() * g.h2();
    DBuf basisBuf(sizeof(double) * n * (steps + 1));
    DBuf wBuf(sizeof(double) * 2 * n);
    DBuf coefBuf(sizeof(double) * (steps + 1));
    auto Q = [&](int j) { return basisBuf.d() + static_cast<std::size_t>(j) * n; };
    double* w = wBuf.d();
    double* qIn = w + n;  // fixed operator input: the operator's CUDA graph replays from step 2
    double* alphaDev = coefBuf.d();   // alpha_j
    double* cDev = alphaDev + steps;  // reorthogonalisation coefficient
    auto dotInto = [&](const double* a, const double* b, double* out) {
        launchDotInto(ctx, N, a, b, a + N, b + N, hh, out);
    };
    std::vector<double> beta;
    int nAlpha = 0;
    randomBandLimitedVelocity(ctx, g, seed, Q(0));
    const double nq = vnormL2(ctx, g, Q(0));
    if (!(nq > 0.0)) return 1.0;
    axpby(ctx, n, 0.0, Q(0), 1.0 / nq, Q(0));
    int nb = 1;
    for (int j = 0; j < steps; ++j) {
        copy(ctx, n, Q(j), qIn);
        op(qIn, w);
        double b;
        LzBeta bp{};
        bp.v[0] = j > 0 ? beta[j - 1] : 0.0;
        if (launchLanczosOrth(ctx, w, Q(0), N, 1, j, nb, bp, hh, alphaDev + j, 1, cDev)) {
            ++nAlpha;
            b = std::sqrt(readScalar(ctx, cDev));  // cDev = |w|^2
        } else {
            if (j > 0) axpby(ctx, n, -beta[j - 1], Q(j - 1), 1.0, w);
            dotInto(w, Q(j), alphaDev + j);
            ++nAlpha;
            axpyNegDevCoef(ctx, n, alphaDev + j, Q(j), w);
            for (int i = 0; i < nb; ++i) {  // full reorthogonalisation (modified Gram-Schmidt)
                dotInto(w, Q(i), cDev);
                axpyNegDevCoef(ctx, n, cDev, Q(i), w);
            }
            b = vnormL2(ctx, g, w);
        }
        if (!std::isfinite(b)) return powerIterationEmax(ctx, g, op, seed ^ 0x1234567);
        if (b < 1e-12) break;
        beta.push_back(b);
        lincomb(ctx, n, 1.0 / b, w, 0.0, w, Q(nb));
        ++nb;
    }
    if (nAlpha == 0) return powerIterationEmax(ctx, g, op, seed ^ 0x1234567);
    std::vector<double> alpha(nAlpha);
    VRG_CUDA(cudaMemcpyAsync(alpha.data(), alphaDev, sizeof(double) * nAlpha, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    beta.resize(alpha.size() - 1);
    return tridiagMaxEig(alpha, beta);
}

// Lanczos on the coarse split operator with its guard checks deferred: a step then needs one
// host read (beta) instead of two; the first guard violation is thrown at the end, in order.
double coarseLanczosEmax(Ctx& ctx, CoarseOperator& coarse, int steps, std::uint64_t seed) {
    LinOpDev op = [&](const double* s, double* o) { coarse.applySplit(s, o); };
    coarse.hess->beginDeferredGuards(steps + 1);
    double e;
    try {
        e = lanczosEmax(ctx, coarse.gc, op, steps, seed);
    } catch (...) {
        coarse.hess->endDeferredGuards();
        throw;
    }
    coarse.hess->endDeferredGuards();
    return e;
}

namespace {
__global__ void k_scale_pairs(std::size_t n, std::size_t nPer, int P, LzBeta a, const double* __restrict__ w,
                              double* __restrict__ out) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double c = a.v[(i / nPer) % static_cast<std::size_t>(P)];
        out[i] = c == 0.0 ? 0.0 : w[i] * c;  // lincomb(1/b, w, 0, w) of the single-pair path; 0 retires a pair
    }
}
}  // namespace

bool lanczosEmaxPairs(Ctx& ctx, const GridDims& g, const LinOpDev& op, int steps, std::uint64_t seed,
                      std::vector<double>& emax, std::vector<char>& fallback,
                      const std::function<void(const std::vector<char>&)>& counted) {
    const int P = g.pairs;
    const std::size_t nPer = g.pointsPer(), N = g.points(), n = 2 * N;
    if (P > kLzMaxPairs || 2 * nPer > static_cast<std::size_t>(4) * kLzCtas * kLzThreads) return false;
    const double hh = g.h1() * g.h2();
    emax.assign(P, 1.0);
    fallback.assign(P, 0);
    DBuf basisBuf(sizeof(double) * n * (steps + 1));
    DBuf wBuf(sizeof(double) * 2 * n);
    DBuf coefBuf(sizeof(double) * (static_cast<std::size_t>(steps) * P + P));
    auto Q = [&](int j) { return basisBuf.d() + static_cast<std::size_t>(j) * n; };
    double* w = wBuf.d();
    double* qIn = w + n;
    double* alphaDev = coefBuf.d();  // pair k, step j at k * steps + j
    double* bsqDev = alphaDev + static_cast<std::size_t>(steps) * P;
    // the seeded start vector of lanczosEmax, the same in every pair's slots
    const GridDims one = g.one();
    const std::size_t n1v = 2 * nPer;
    double* q0 = ctx.scratchBuf(162, sizeof(double) * n1v);
    randomBandLimitedVelocity(ctx, one, seed, q0);
    const double nq = vnormL2(ctx, one, q0);
    if (!(nq > 0.0)) return true;  // every pair: eMax 1 (lanczosEmax's early return)
    axpby(ctx, n1v, 0.0, q0, 1.0 / nq, q0);
    for (int k = 0; k < P; ++k)
        for (int c = 0; c < 2; ++c)
            VRG_CUDA(cudaMemcpyAsync(Q(0) + c * N + k * nPer, q0 + c * nPer, sizeof(double) * nPer,
                                     cudaMemcpyDeviceToDevice, ctx.stream));
    std::vector<std::vector<double>> beta(P);
    std::vector<int> nAlpha(P, 0);
    std::vector<char> on(P, 1);
    std::vector<double> bsq(P);
    int nb = 1;
    for (int j = 0; j < steps; ++j) {
        copy(ctx, n, Q(j), qIn);
        op(qIn, w);
        counted(on);
        LzBeta bp{};
        for (int k = 0; k < P; ++k) bp.v[k] = (j > 0 && on[k]) ? beta[k][j - 1] : 0.0;
        if (!launchLanczosOrth(ctx, w, Q(0), nPer, P, j, nb, bp, hh, alphaDev + j, steps, bsqDev)) return false;
        readPairs(ctx, bsqDev, P, bsq.data());
        LzBeta inv{};
        bool any = false;
        for (int k = 0; k < P; ++k) {
            if (!on[k]) continue;
            ++nAlpha[k];
            const double b = std::sqrt(bsq[k]);
            if (!std::isfinite(b)) {
                fallback[k] = 1;  // lanczosEmax: power iteration
                on[k] = 0;
            } else if (b < 1e-12) {
                on[k] = 0;
            } else {
                beta[k].push_back(b);
                inv.v[k] = 1.0 / b;
                any = true;
            }
        }
        {
            LaunchScope ls_(ctx, "k_scale_pairs");
            k_scale_pairs<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, nPer, P, inv, w, Q(nb));
        }
        VRG_LAUNCH_CHECK();
        ++nb;
        if (!any) break;
    }
    std::vector<double> alpha(static_cast<std::size_t>(steps) * P);
    VRG_CUDA(cudaMemcpyAsync(alpha.data(), alphaDev, sizeof(double) * alpha.size(), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    for (int k = 0; k < P; ++k) {
        if (fallback[k]) continue;
        if (nAlpha[k] == 0) {
            fallback[k] = 1;
            continue;
        }
        std::vector<double> a(alpha.begin() + static_cast<std::ptrdiff_t>(k) * steps,
                              alpha.begin() + static_cast<std::ptrdiff_t>(k) * steps + nAlpha[k]);
        std::vector<double> b = beta[k];
        b.resize(a.size() - 1);
        emax[k] = tridiagMaxEig(a, b);
    }
    return true;
}

std::pair<double, double> estimateEigsAt(Ctx& ctx, const GridDims& g, const double* v, const double* mR,
                                         const double* mT, const Model& model, double coarseCfl, std::uint64_t seed) {
    std::unique_ptr<PhaseTimer> pt(new PhaseTimer(ctx, "eigs: coarse setup"));
    CoarseOperator coarse(ctx, g, v, mR, mT, model, coarseCfl);
    pt.reset(new PhaseTimer(ctx, "eigs: lanczos(30)"));
    return {1.0, coarseLanczosEmax(ctx, coarse, 30, seed)};
}

// ------------------------------------------------------------------------------ two-level
// restriction of a (batched) vector field r on g to rc on gc: R, C spectra scratch of the two
// components; the components of all pairs are 2 * pairs spectra in a row
void restrictLow(Ctx& ctx, const GridDims& g, const GridDims& gc, const double* r, cplx* R, cplx* C, double* rc,
                 double ampDown) {
    fftForward(ctx, g, r, R, 2);
    {
        LaunchScope ls_(ctx, "k_restrict_low");
        k_restrict_low<<<static_cast<unsigned>((2 * gc.specPoints() + 255) / 256), 256, 0, ctx.stream>>>(
            R, g.n1, g.n2, C, gc.n1, gc.n2, 2 * gc.pairs, ampDown, 1.0 / gc.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    fftInverse(ctx, gc, C, rc, 2);
}

// out = prolong(sc) + high band of r (R holds r's spectra from restrictLow)
void prolongAddHigh(Ctx& ctx, const GridDims& g, const GridDims& gc, const double* sc, cplx* C, cplx* R, double* out,
                    double ampUp) {
    fftForward(ctx, gc, sc, C, 2);
    {
        LaunchScope ls_(ctx, "k_prolong_add_high");
        k_prolong_add_high<<<static_cast<unsigned>((2 * g.specPoints() + 255) / 256), 256, 0, ctx.stream>>>(
            C, gc.n1, gc.n2, R, R, g.n1, g.n2, 2 * g.pairs, ampUp, 1.0 / g.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    fftInverse(ctx, g, R, out, 2);
}

bool applyTwoLevel(Ctx& ctx, const GridDims& g, const double* r, CoarseOperator& coarse, const PrecondChoice& choice,
                   double outerTol, double eMin, double eMax, double* out) {
    NvtxRange nv_("applyTwoLevel");
    const GridDims& gc = coarse.gc;
    const std::size_t N = g.points(), Nc = gc.points(), NS = g.specPoints(), NSc = gc.specPoints();
    cplx* R = specScratch(ctx, g, 5, 2);    // fine spectra of r (both components)
    cplx* C = specScratch(ctx, gc, 6, 2);   // coarse spectra
    double* rc = ctx.scratchBuf(130, sizeof(double) * 2 * Nc);
    double* sc = ctx.scratchBuf(131, sizeof(double) * 2 * Nc);
    const double ampDown = static_cast<double>(Nc) / static_cast<double>(N);
    // both components (and every pair of a batch) in one transform chain
    restrictLow(ctx, g, gc, r, R, C, rc, ampDown);
    LinOpDev op = [&](const double* s, double* o) { coarse.applySplit(s, o); };
    if (choice.coarseSolver == kCoarseCheb) {
        // the Chebyshev loop has no host decisions: its coarse matvecs run back to back on the
        // stream and their guards are checked once at the end, in order
        coarse.hess->beginDeferredGuards(choice.chebIters);
        try {
            chebyshevSolve(ctx, gc, op, rc, choice.chebIters, eMin, kEmaxInflation * eMax, sc);
        } catch (...) {
            coarse.hess->endDeferredGuards();
            throw;
        }
        coarse.hess->endDeferredGuards();
    } else {
        // the coarse PCG reads its scalars once per iteration; the matvecs' guard checks ride
        // on those reads instead of adding a sync each (checked in order at the end)
        coarse.hess->beginDeferredGuards(500);
        try {
            pcg(ctx, gc, op, rc, nullptr, choice.epsScale * outerTol, 500, sc);
        } catch (...) {
            coarse.hess->endDeferredGuards();
            throw;
        }
        coarse.hess->endDeferredGuards();
    }
    // reference counting: cutoff Low/High (8 FFTs) + restrict (4); prolong (4) below
    ctx.ffts += 12;
    if (anyNonFinite(ctx, 2 * Nc, sc)) {
        std::fprintf(stderr, "precond: coarse solve diverged, falling back to identity\n");
        copy(ctx, 2 * N, r, out);
        return false;
    }
    const double ampUp = static_cast<double>(N) / static_cast<double>(Nc);
    prolongAddHigh(ctx, g, gc, sc, C, R, out, ampUp);
    ctx.ffts += 4;
    (void)NS;
    (void)NSc;
    return true;
}

// ------------------------------------------------------------------------------ KKT
KktResult solveKkt(Ctx& ctx, Hessian& hess, const double* rhs, double tol, int maxIter, const PrecondChoice& choice,
                   const double* mR, const double* mT, const double* v, double coarseCfl, double* solution) {
    if (choice.kind == kPcTwoLevel) {
        if (choice.coarseSolver == kCoarsePcg && !(choice.epsScale > 0.0 && choice.epsScale < 1.0))
            throw InvalidArgument("solveKkt: epsScale must lie in (0,1)");
        if (choice.coarseSolver == kCoarseCheb && choice.chebIters < 1)
            throw InvalidArgument("solveKkt: chebIters must be >= 1");
        if (choice.hasEig && !(choice.eMax > choice.eMin && choice.eMin > 0.0))
            throw InvalidArgument("solveKkt: need eMax > eMin > 0");
    }
    const std::size_t N = hess.g.points();
    LinOpDev A = [&](const double* s, double* o) { hess.applySplit(s, s + N, o, o + N); };
    return solveKktOp(ctx, hess.g, hess.model, hess.weights, A, rhs, tol, maxIter, choice, mR, mT, v, coarseCfl,
                      solution);
}

KktResult solveKktOp(Ctx& ctx, const GridDims& g, const Model& model, Weights& weights, const LinOpDev& A,
                     const double* rhs, double tol, int maxIter, const PrecondChoice& choice, const double* mR,
                     const double* mT, const double* v, double coarseCfl, double* solution) {
    NvtxRange nv_("solveKkt");
    const std::size_t N = g.points();
    const auto t0 = std::chrono::steady_clock::now();
    double precondTime = 0.0;
    const double* invHalf = weights.invRegSymbol(model.betaV, -0.5);
    double* rhsSplit = ctx.scratchBuf(140, sizeof(double) * 2 * N);
    double* x = ctx.scratchBuf(141, sizeof(double) * 2 * N);
    applyRealSymbol(ctx, g, rhs, rhs + N, rhsSplit, rhsSplit + N, invHalf);

    std::unique_ptr<CoarseOperator> coarse;
    double eMin = 1.0, eMax = 10.0;
    LinOpDev M;
    // an external (slab-decomposed) coarse level: built per solve like the CoarseOperator, the
    // two-level application and the re-estimate by the hooks; logical counts as the library's
    const bool extCoarse = ctx.fine.coarseBuild && choice.kind == kPcTwoLevel && choice.coarseSolver == kCoarseCheb;
    int ntc = 0;
    bool lazyCoarse = true;  // the coarse operator's lazy caches are counted by its first matvec
    auto countCoarseMatvecs = [&](long long k) {
        if (k <= 0) return;
        ctx.ffts += k * (8 + (3 + 3LL * ntc) + 3LL * (ntc + 1)) + (lazyCoarse ? 3 : 0);
        ctx.interps += k * (4LL * ntc + 2) + (lazyCoarse ? 3 : 0);
        lazyCoarse = false;
    };
    if (choice.kind == kPcTwoLevel) {
        if (extCoarse) {
            if (ctx.fine.coarseBuild(ctx.fine.user, v, &ntc) != 0)
                throw std::runtime_error("external coarse operator: build callback failed");
            ctx.ffts += 8;         // restrictProblem + the coarse velocity: 4 resamples (precond.cpp:166-167,221)
            ctx.interps += 2 + ntc;  // the coarse GN Hessian's state solve
        } else {
            coarse = std::make_unique<CoarseOperator>(ctx, g, v, mR, mT, model, coarseCfl);
        }
        if (choice.coarseSolver == kCoarseCheb) {
            if (choice.hasEig) {
                eMin = choice.eMin;
                eMax = choice.eMax;
            } else {
                std::tie(eMin, eMax) = estimateEigsAt(ctx, g, nullptr, mR, mT, model, coarseCfl);
            }
        }
        M = [&](const double* r, double* z) {
            const auto tp = std::chrono::steady_clock::now();
            if (extCoarse) {
                const int rc = ctx.fine.twoLevel(ctx.fine.user, r, z, choice.chebIters, eMin, kEmaxInflation * eMax);
                if (rc == 3)
                    std::fprintf(stderr, "precond: coarse solve diverged, falling back to identity\n");
                else if (rc != 0)
                    throw std::runtime_error("external coarse operator: two-level callback failed");
                ctx.ffts += 16;  // cutoff low / high, restrict, prolong (precond.cpp:265-287)
                countCoarseMatvecs(choice.chebIters);
            } else {
                applyTwoLevel(ctx, g, r, *coarse, choice, tol, eMin, eMax, z);
            }
            precondTime += secondsSince(tp);
        };
    }
    PcgOut out = pcg(ctx, g, A, rhsSplit, M ? &M : nullptr, tol, maxIter, x);
    if (out.indefinitePreconditioner && choice.kind == kPcTwoLevel && choice.coarseSolver == kCoarseCheb) {
        if (extCoarse) {
            int applied = 0;
            if (ctx.fine.coarseEmax(ctx.fine.user, &eMax, &applied) != 0)
                throw std::runtime_error("external coarse operator: re-estimate callback failed");
            ctx.ffts += 4;  // the seeded random probe (randomBandLimitedVelocity: 2 fields x 2 FFTs)
            countCoarseMatvecs(applied);
        } else {
            eMax = coarseLanczosEmax(ctx, *coarse, 30, 0x5eed);
        }
        std::fprintf(stderr, "precond: re-estimated Chebyshev bound eMax=%.6g after breakdown\n", eMax);
        out = pcg(ctx, g, A, rhsSplit, &M, tol, maxIter, x);
    }
    applyRealSymbol(ctx, g, x, x + N, solution, solution + N, invHalf);
    KktResult res;
    res.iterations = out.iterations;
    res.negativeCurvature = out.negativeCurvature;
    res.converged = out.converged;
    res.relResidual = out.relResidual;
    res.totalTimeSec = secondsSince(t0);
    res.precondTimeSec = precondTime;
    return res;
}

// ------------------------------------------------------------------------------ external fine operator
ExternalFineOperator::ExternalFineOperator(Ctx& ctx, const GridDims& g, const double* v, const Model& model, int nt,
                                           Weights& weights)
    : ctx_(ctx), g_(g), model_(model), nt_(nt), weights_(weights) {
    if (model.scheme != kSchemeSL || model.deformation != kCompressible)
        throw NotSupported("external fine operator: compressible Gauss-Newton SL model only");
    if (ctx.fine.build(ctx.fine.user, v, nt) != 0) throw std::runtime_error("external fine operator: build callback failed");
    for (int batch = 1; batch <= 2; ++batch) {
        ctx.plan(g, CUFFT_D2Z, batch);
        ctx.plan(g, CUFFT_Z2D, batch);
    }
}

// Hessian::launchSplit with the data term of the hook: t = M^{-1/2} s, b = Q t, o = M^{-1/2} b + s.
void ExternalFineOperator::applySplit(const double* s, double* o) {
    if (ctx_.fine.split) {
        if (ctx_.fine.split(ctx_.fine.user, s, o) != 0)
            throw std::runtime_error("external fine operator: split callback failed");
        ctx_.ffts += 8 + (3 + 3LL * nt_) + 3LL * (nt_ + 1) + lazyFfts_;
        ctx_.interps += 4LL * nt_ + 2 + lazyInterps_;
        lazyInterps_ = 0;
        lazyFfts_ = 0;
        return;
    }
    const std::size_t N = g_.points(), NS = g_.specPoints();
    cplx* S = reinterpret_cast<cplx*>(ctx_.scratchBuf(150, sizeof(cplx) * 4 * NS));
    cplx* T = S + 2 * NS;
    double* t = ctx_.scratchBuf(151, sizeof(double) * 2 * N);
    double* b = ctx_.scratchBuf(152, sizeof(double) * 2 * N);
    const double* inv = weights_.invRegSymbol(model_.betaV, -0.5);
    fftForward(ctx_, g_, s, S, 2);
    specCombine(ctx_, g_, S, S + NS, nullptr, nullptr, inv, false, 1.0 / g_.pointsPer(), T, T + NS);
    fftInverse(ctx_, g_, T, t, 2);
    if (ctx_.fine.dataTerm(ctx_.fine.user, t, b) != 0)
        throw std::runtime_error("external fine operator: data-term callback failed");
    fftForward(ctx_, g_, b, T, 2);
    specCombine(ctx_, g_, T, T + NS, S, S + NS, inv, false, 1.0 / g_.pointsPer(), T, T + NS);
    fftInverse(ctx_, g_, T, o, 2);
    // counters of one split matvec (Hessian::applySplit + countDataTerm, GN SL compressible)
    ctx_.ffts += 8 + (3 + 3LL * nt_) + 3LL * (nt_ + 1) + lazyFfts_;
    ctx_.interps += 4LL * nt_ + 2 + lazyInterps_;
    lazyInterps_ = 0;
    lazyFfts_ = 0;
}

// ------------------------------------------------------------------------------ Newton
SolverReport newtonSolve(Ctx& ctx, const GridDims& g, const double* mR, const double* mT, const Model& model,
                         const NewtonConfig& cfg, const PrecondChoice& pc, double* vOut) {
    NvtxRange nv_("newtonSolve");
    const std::size_t N = g.points();
    const auto tStart = std::chrono::steady_clock::now();
    const long long f0 = ctx.ffts, i0 = ctx.interps;
    SolverReport report;
    Weights weights(g, model.norm);
    DBuf vBuf(sizeof(double) * 2 * N), trialBuf(sizeof(double) * 2 * N), gBuf(sizeof(double) * 2 * N),
        dvBuf(sizeof(double) * 2 * N), tmpBuf(sizeof(double) * 2 * N);
    double* v = vBuf.d();
    fill(ctx, 2 * N, 0.0, v);  // zero initial guess

    if ((ctx.fine.gradient || ctx.fine.objective) &&
        (model.scheme != kSchemeSL || model.deformation != kCompressible || cfg.hessianMode != 0 || !ctx.fine.build))
        throw NotSupported("external gradient / objective: compressible Gauss-Newton SL with an external fine operator");
    PrecondChoice choice = pc;
    if (choice.kind == kPcTwoLevel && choice.coarseSolver == kCoarseCheb && !choice.hasEig &&
        !choice.reestimateEachIteration) {
        PhaseTimer pt(ctx, "estimateEigs");
        std::tie(choice.eMin, choice.eMax) = estimateEigsAt(ctx, g, nullptr, mR, mT, model, kCoarseCfl);
        choice.hasEig = true;
    }

    double g0inf = 0.0;
    int ntRatchet = 0;
    int carriedNt = -1;
    DBuf carried, state, adjoint, grads;
    DBuf finalDeformed(sizeof(double) * N);
    copy(ctx, N, mT, finalDeformed.d());
    double scal[4];

    for (int iter = 0; iter < cfg.maxOuterIter; ++iter) {
        const auto tIter = std::chrono::steady_clock::now();
        ntRatchet = std::max(ntRatchet, cfg.ntOverride > 0 ? cfg.ntOverride
                                                          : deriveSteps(ctx, g, v, v + N, cfg.gradCfl));
        const int nt = ntRatchet;
        state.alloc(sizeof(double) * (nt + 1) * N);
        adjoint.alloc(sizeof(double) * (nt + 1) * N);
        // grad m_j of the gradient's state, reused by the GN SL Hessian of this iterate
        const bool keepGrads = model.scheme == kSchemeSL && cfg.hessianMode == 0 && !ctx.fine.build;
        if (keepGrads) grads.alloc(sizeof(double) * (nt + 1) * 2 * N);
        const bool reuse = carriedNt == nt;
        if (ctx.fine.gradient) {
            // external (e.g. slab-decomposed) evaluateGradient; logical counts as the reference's
            // (inverse.cpp:119-148: state unless reused, adjoint with the lazy backward
            // characteristics / div v / (div v)_D, body force, applyReg)
            PhaseTimer pt(ctx, "evaluateGradient (external)");
            if (ctx.fine.gradient(ctx.fine.user, v, nt, reuse ? 1 : 0, gBuf.d(), finalDeformed.d(), scal) != 0)
                throw std::runtime_error("external fine operator: gradient callback failed");
            ctx.interps += (reuse ? 0 : 2LL + nt) + 3 + nt;
            ctx.ffts += 3 + 3LL * (nt + 1) + 4;
        } else {
            PhaseTimer pt(ctx, "evaluateGradient");
            evaluateGradient(ctx, g, v, v + N, mR, mT, model, nt, gBuf.d(), gBuf.d() + N, scal, state.d(),
                             adjoint.d(), reuse ? carried.d() : nullptr, keepGrads ? grads.d() : nullptr);
            copy(ctx, N, state.d() + static_cast<std::size_t>(nt) * N, finalDeformed.d());
        }
        const double objective = scal[0], mismatch = scal[1];

        const double ginf = vnormLinf(ctx, g, gBuf.d());
        if (iter == 0) g0inf = std::max(ginf, 1e-300);
        const double grel = ginf / g0inf;

        IterationRecord rec;
        rec.iter = iter;
        rec.gradNormInf = ginf;
        rec.gradNormRel = grel;
        rec.objective = objective;
        rec.mismatch = mismatch;
        rec.ffts = ctx.ffts - f0;
        rec.interps = ctx.interps - i0;

        report.finalGradNormRel = grel;
        if (grel <= cfg.tolRelGrad || ginf <= cfg.tolAbsGrad) {
            rec.wallTimeSec = secondsSince(tIter);
            report.iterations.push_back(rec);
            report.status = kConverged;
            break;
        }

        const double eta = std::min(cfg.forcingCap, std::sqrt(grel));
        std::unique_ptr<PhaseTimer> ptH(new PhaseTimer(ctx, "Hessian ctor"));
        // the fine operator: this library's Hessian, or the external (e.g. slab-decomposed) one
        std::unique_ptr<Hessian> hess;
        std::unique_ptr<ExternalFineOperator> ext;
        if (ctx.fine.build) {
            if (cfg.hessianMode != 0) throw NotSupported("external fine operator: Gauss-Newton mode only");
            ext = std::make_unique<ExternalFineOperator>(ctx, g, v, model, nt, weights);
        } else {
            // NewtonConfig::hessianScheme (newton.cpp:83-92): the gradient's discretization
            // unless hessScheme is set; the state (and adjoint) are reused only when both
            // the step count and the scheme agree
            Model hmodel = model;
            int hnt = nt;
            if (cfg.hasHessScheme) {
                hmodel.scheme = cfg.hessScheme;
                hnt = cfg.hessNtOverride > 0 ? cfg.hessNtOverride : deriveSteps(ctx, g, v, v + N, cfg.hessCfl);
            }
            const bool same = hnt == nt && hmodel.scheme == model.scheme;
            hess = std::make_unique<Hessian>(ctx, g, v, v + N, mR, mT, hmodel, hnt, same ? state.d() : nullptr,
                                             cfg.hessianMode, (same && cfg.hessianMode == 1) ? adjoint.d() : nullptr,
                                             (same && keepGrads) ? grads.d() : nullptr);
        }
        ptH.reset();
        // rhs = -g
        lincomb(ctx, 2 * N, -1.0, gBuf.d(), 0.0, gBuf.d(), tmpBuf.d());
        std::unique_ptr<PhaseTimer> ptK(new PhaseTimer(ctx, "solveKkt"));
        KktResult kkt;
        if (ext) {
            LinOpDev A = [&](const double* s, double* o) { ext->applySplit(s, o); };
            kkt = solveKktOp(ctx, g, model, weights, A, tmpBuf.d(), eta, cfg.maxInnerIter, choice, mR, mT, v,
                             kCoarseCfl, dvBuf.d());
        } else {
            kkt = solveKkt(ctx, *hess, tmpBuf.d(), eta, cfg.maxInnerIter, choice, mR, mT, v, kCoarseCfl, dvBuf.d());
        }
        ptK.reset();
        rec.innerIterations = kkt.iterations;
        double* dv = dvBuf.d();

        double gdotd = vdot(ctx, g, gBuf.d(), dv);
        if (!std::isfinite(gdotd) || gdotd >= 0.0) {
            // inner solve broke down: Sobolev-gradient fallback direction
            applyRealSymbol(ctx, g, gBuf.d(), gBuf.d() + N, dv, dv + N, weights.invRegSymbol(model.betaV, -1.0));
            axpby(ctx, 2 * N, 0.0, dv, -1.0, dv);
            gdotd = vdot(ctx, g, gBuf.d(), dv);
        }
        divergence(ctx, g, dv, dv + N, tmpBuf.d());
        rec.searchDirDivRatio = normLinf(ctx, N, tmpBuf.d()) / std::max(vnormLinf(ctx, g, dv), 1e-300);

        // Armijo backtracking on the objective at this iteration's time grid
        double alpha = 1.0;
        bool accepted = false;
        int lsSteps = 0;
        if (!carried || carried.bytes() < sizeof(double) * (nt + 1) * N) carried.alloc(sizeof(double) * (nt + 1) * N);
        PhaseTimer ptLs(ctx, "line search");
        for (; lsSteps < cfg.lsMaxSteps; ++lsSteps) {
            lincomb(ctx, 2 * N, 1.0, v, alpha, dv, trialBuf.d());
            bool blewUp = false;
            double ob[4] = {0, 0, 0, 0};
            double* trialM1 = tmpBuf.d();
            if (ctx.fine.objective) {
                const int rc = ctx.fine.objective(ctx.fine.user, trialBuf.d(), nt, trialM1, ob);
                if (rc == 2) {
                    blewUp = true;
                } else if (rc != 0) {
                    throw std::runtime_error("external fine operator: objective callback failed");
                }
                ctx.interps += 2LL + nt;  // evaluateObjective: solveState (inverse.cpp:101-103), applyReg
                ctx.ffts += 4;
            } else {
                try {
                    evaluateObjective(ctx, g, trialBuf.d(), trialBuf.d() + N, mR, mT, model, nt, ob, carried.d());
                } catch (const BlowupError&) {
                    blewUp = true;
                }
                copy(ctx, N, carried.d() + static_cast<std::size_t>(nt) * N, trialM1);
            }
            if (!blewUp && ob[0] <= objective + cfg.lsC1 * alpha * gdotd) {
                copy(ctx, 2 * N, trialBuf.d(), v);
                carriedNt = nt;
                copy(ctx, N, trialM1, finalDeformed.d());
                accepted = true;
                break;
            }
            alpha *= cfg.lsShrink;
        }
        if (!accepted) carriedNt = -1;
        rec.lineSearchSteps = lsSteps + (accepted ? 1 : 0);
        rec.stepLength = accepted ? alpha : 0.0;
        rec.wallTimeSec = secondsSince(tIter);
        rec.ffts = ctx.ffts - f0;
        rec.interps = ctx.interps - i0;
        report.iterations.push_back(rec);
        if (!accepted) {
            report.status = kLineSearchFailure;
            break;
        }
        if (iter + 1 == cfg.maxOuterIter) report.status = kIterationLimit;
    }

    // final diagnostics (newton.cpp:147-157)
    lincomb(ctx, N, 1.0, mT, -1.0, mR, tmpBuf.d());
    const double residDenom = std::sqrt(dot(ctx, g, tmpBuf.d(), nullptr, tmpBuf.d(), nullptr));
    lincomb(ctx, N, 1.0, finalDeformed.d(), -1.0, mR, tmpBuf.d());
    const double residNum = std::sqrt(dot(ctx, g, tmpBuf.d(), nullptr, tmpBuf.d(), nullptr));
    report.finalResidualRel = residDenom > 0.0 ? residNum / residDenom : 0.0;
    {
        const int ntJ = deriveSteps(ctx, g, v, v + N, 0.2);
        Solver js(ctx, g, v, v + N, ntJ);
        js.jacobian(tmpBuf.d());
        std::vector<double> jac(N);
        VRG_CUDA(cudaMemcpyAsync(jac.data(), tmpBuf.d(), sizeof(double) * N, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        report.jacMin = *std::min_element(jac.begin(), jac.end());
        report.jacMax = *std::max_element(jac.begin(), jac.end());
    }
    copy(ctx, 2 * N, v, vOut);
    ctx.sync();
    report.totalTimeSec = secondsSince(tStart);
    return report;
}

}  // namespace vrg
