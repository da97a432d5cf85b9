// RK2 / RK2A spectral transport (heun.cuh).
#include "heun.cuh"

namespace vrg {

namespace {

constexpr int kB = 256;

// y + a x without contraction (axpy, field.cpp:33-36)
__device__ __forceinline__ double axpyRn(double y, double a, double x) { return __dadd_rn(y, __dmul_rn(a, x)); }

// out = v0 g0 + 1.0 (v1 g1)   (advectBy)
__global__ void k_advect(std::size_t N, const double* __restrict__ v1, const double* __restrict__ v2,
                         const double* __restrict__ g1, const double* __restrict__ g2, double* __restrict__ out) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    out[p] = axpyRn(__dmul_rn(v1[p], g1[p]), 1.0, __dmul_rn(v2[p], g2[p]));
}

// o_i = m v_i   (the products of divOfProduct)
__global__ void k_prod(std::size_t N, const double* __restrict__ m, const double* __restrict__ v1,
                       const double* __restrict__ v2, double* o1, double* o2) {  // o1 == o2 allowed
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    o1[p] = __dmul_rn(m[p], v1[p]);
    o2[p] = __dmul_rn(m[p], v2[p]);
}

// out = ((a + c1 b) + c2 (m d)) * s, with b / m d optional (null); out may alias an input
__global__ void k_comb(std::size_t N, const double* a, double c1, const double* b, double c2, const double* m,
                       const double* d, double s, double* out) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    double r = a[p];
    if (b) r = axpyRn(r, c1, b[p]);
    if (m) r = axpyRn(r, c2, __dmul_rn(m[p], d[p]));
    out[p] = __dmul_rn(r, s);
}

// k += 1.0 src (optional); pred = y + ht k
__global__ void k_stage1(std::size_t N, double* __restrict__ k, const double* __restrict__ src,
                         const double* __restrict__ y, double ht, double* __restrict__ pred) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    double kk = k[p];
    if (src) kk = axpyRn(kk, 1.0, src[p]);
    k[p] = kk;
    pred[p] = axpyRn(y[p], ht, kk);
}

// k2 += 1.0 src (optional); yNext = (y + h/2 k1) + h/2 k2
__global__ void k_stage2(std::size_t N, const double* __restrict__ k1, double* __restrict__ k2,
                         const double* __restrict__ src, const double* y, double hh, double* yNext) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    double kk = k2[p];
    if (src) kk = axpyRn(kk, 1.0, src[p]);
    yNext[p] = axpyRn(axpyRn(y[p], hh, k1[p]), hh, kk);
}

// S(m)^T mu components: ((mu gm_i + (-1) m gmu_i) + 1.0 gprod_i) * 0.5
__global__ void k_antisym(std::size_t N, const double* __restrict__ m, const double* __restrict__ mu,
                          const double* __restrict__ gm, const double* __restrict__ gmu, const double* __restrict__ gp,
                          double* __restrict__ o1, double* __restrict__ o2) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    for (int i = 0; i < 2; ++i) {
        const std::size_t q = p + i * N;
        double r = __dmul_rn(mu[p], gm[q]);
        r = axpyRn(r, -1.0, __dmul_rn(m[p], gmu[q]));
        r = axpyRn(r, 1.0, gp[q]);
        (i ? o2 : o1)[p] = __dmul_rn(r, 0.5);
    }
}

// b_i += a (x term_i) per component, term = lam * g (hadamard) or a precomputed vector field
__global__ void k_axpy_had(std::size_t N, double a, const double* __restrict__ lam, const double* __restrict__ g1,
                           const double* __restrict__ g2, double* __restrict__ b1, double* __restrict__ b2) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const double l = lam ? lam[p] : 1.0;
    b1[p] = axpyRn(b1[p], a, lam ? __dmul_rn(l, g1[p]) : g1[p]);
    b2[p] = axpyRn(b2[p], a, lam ? __dmul_rn(l, g2[p]) : g2[p]);
}

dim3 grid(const GridDims& g) { return grid1d(g.points(), kB); }

}  // namespace

void advectBy(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* m, double* out) {
    const std::size_t N = g.points();
    double* gm = ctx.scratchBuf(50, sizeof(double) * 2 * N);
    gradient(ctx, g, m, gm, gm + N);
    LaunchScope ls_(ctx, "k_advect");
    k_advect<<<grid(g), kB, 0, ctx.stream>>>(N, v1, v2, gm, gm + N, out);
    VRG_LAUNCH_CHECK();
}

void divOfProduct(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* m, double* out) {
    const std::size_t N = g.points();
    double* pr = ctx.scratchBuf(51, sizeof(double) * 2 * N);
    {
        LaunchScope ls_(ctx, "k_prod");
        k_prod<<<grid(g), kB, 0, ctx.stream>>>(N, m, v1, v2, pr, pr + N);
    }
    VRG_LAUNCH_CHECK();
    divergence(ctx, g, pr, pr + N, out);
}

void antisymmetricForceTerm(Ctx& ctx, const GridDims& g, const double* m, const double* mu, double* o1, double* o2) {
    const std::size_t N = g.points();
    double* s = ctx.scratchBuf(52, sizeof(double) * 7 * N);  // gm (2N), gmu (2N), prod (N), gprod (2N)
    double* gm = s;
    double* gmu = s + 2 * N;
    double* prod = s + 4 * N;
    double* gp = s + 5 * N;
    gradient(ctx, g, m, gm, gm + N);
    gradient(ctx, g, mu, gmu, gmu + N);
    {  // hadamard(mu, m)
        LaunchScope ls_(ctx, "k_prod");
        k_prod<<<grid(g), kB, 0, ctx.stream>>>(N, mu, m, m, prod, prod);
    }
    VRG_LAUNCH_CHECK();
    gradient(ctx, g, prod, gp, gp + N);
    LaunchScope ls_(ctx, "k_antisym");
    k_antisym<<<grid(g), kB, 0, ctx.stream>>>(N, m, mu, gm, gmu, gp, o1, o2);
    VRG_LAUNCH_CHECK();
}

void bodyForceHeun(Ctx& ctx, const GridDims& g, int nt, bool anti, const double* stNodes, const double* stStages,
                   const double* adNodes, const double* adStages, double* b1, double* b2) {
    const std::size_t N = g.points();
    const double hh = 0.5 * (1.0 / nt);  // 0.5 * ht
    double* t = ctx.scratchBuf(53, sizeof(double) * 4 * N);
    fill(ctx, N, 0.0, b1);
    fill(ctx, N, 0.0, b2);
    for (int j = 1; j <= nt; ++j) {
        const double* mPrev = stNodes + static_cast<std::size_t>(j - 1) * N;
        const double* mStage = stStages + static_cast<std::size_t>(j - 1) * N;
        const double* lamNode = adNodes + static_cast<std::size_t>(j) * N;
        const double* lamStage = adStages + static_cast<std::size_t>(j - 1) * N;
        if (anti) {
            antisymmetricForceTerm(ctx, g, mPrev, lamStage, t, t + N);
            {
                LaunchScope ls_(ctx, "k_axpy_had");
                k_axpy_had<<<grid(g), kB, 0, ctx.stream>>>(N, hh, nullptr, t, t + N, b1, b2);
            }
            antisymmetricForceTerm(ctx, g, mStage, lamNode, t, t + N);
            LaunchScope ls_(ctx, "k_axpy_had");
            k_axpy_had<<<grid(g), kB, 0, ctx.stream>>>(N, hh, nullptr, t, t + N, b1, b2);
        } else {
            gradient(ctx, g, mPrev, t, t + N);
            gradient(ctx, g, mStage, t + 2 * N, t + 3 * N);
            {
                LaunchScope ls_(ctx, "k_axpy_had");
                k_axpy_had<<<grid(g), kB, 0, ctx.stream>>>(N, hh, lamStage, t, t + N, b1, b2);
            }
            LaunchScope ls_(ctx, "k_axpy_had");
            k_axpy_had<<<grid(g), kB, 0, ctx.stream>>>(N, hh, lamNode, t + 2 * N, t + 3 * N, b1, b2);
        }
        VRG_LAUNCH_CHECK();
    }
}

// ------------------------------------------------------------------------------ transport
HeunTransport::HeunTransport(Ctx& c, const GridDims& gd, const double* v1, const double* v2, int steps,
                             bool antisymmetric)
    : ctx(c), g(gd), nt(steps), ht(1.0 / steps), anti(antisymmetric) {
    checkGrid(g.n1, g.n2);
    if (steps < 1) throw InvalidArgument("TimeGrid: nt must be >= 1");
    const std::size_t N = g.points();
    v.alloc(sizeof(double) * 2 * N);
    copy(ctx, N, v1, v.d());
    copy(ctx, N, v2, v.d() + N);
    if (anyNonFinite(ctx, 2 * N, v.d())) throw InvalidArgument("transport velocity: non-finite value");
    work_.alloc(sizeof(double) * 8 * N);
    log.ensure(nt + 1, g);
}

const double* HeunTransport::divVelocity() {
    if (!haveDivv_) {
        divv_.alloc(sizeof(double) * g.points());
        divergence(ctx, g, v.d(), v.d() + g.points(), divv_.d());
        haveDivv_ = true;
    }
    return divv_.d();
}

void HeunTransport::forwardRhs(const double* m, double* out) {
    const std::size_t N = g.points();
    const double* v1 = v.d();
    const double* v2 = v1 + N;
    double* a = w(6);
    advectBy(ctx, g, v1, v2, m, a);
    if (!anti) {
        LaunchScope ls_(ctx, "k_comb");
        k_comb<<<grid(g), kB, 0, ctx.stream>>>(N, a, 0.0, nullptr, 0.0, nullptr, nullptr, -1.0, out);
        VRG_LAUNCH_CHECK();
        return;
    }
    double* dp = w(7);
    divOfProduct(ctx, g, v1, v2, m, dp);
    const double* dv = divVelocity();
    LaunchScope ls_(ctx, "k_comb");
    k_comb<<<grid(g), kB, 0, ctx.stream>>>(N, a, 1.0, dp, -1.0, m, dv, -0.5, out);
    VRG_LAUNCH_CHECK();
}

void HeunTransport::backwardRhs(const double* lam, double* out) {
    const std::size_t N = g.points();
    const double* v1 = v.d();
    const double* v2 = v1 + N;
    if (!anti) {
        divOfProduct(ctx, g, v1, v2, lam, out);
        return;
    }
    double* dp = w(6);
    double* a = w(7);
    divOfProduct(ctx, g, v1, v2, lam, dp);
    advectBy(ctx, g, v1, v2, lam, a);
    const double* dv = divVelocity();
    LaunchScope ls_(ctx, "k_comb");
    k_comb<<<grid(g), kB, 0, ctx.stream>>>(N, dp, 1.0, a, 1.0, lam, dv, 0.5, out);
    VRG_LAUNCH_CHECK();
}

// one Heun step y -> yNext (pred receives the predictor), with optional sources added to k1/k2
void HeunTransport::heunStep(const double* y, double* yNext, double* pred, bool fwd, const double* src1,
                             const double* src2) {
    const std::size_t N = g.points();
    double* k1 = w(0);
    double* k2 = w(1);
    if (fwd)
        forwardRhs(y, k1);
    else
        backwardRhs(y, k1);
    {
        LaunchScope ls_(ctx, "k_stage1");
        k_stage1<<<grid(g), kB, 0, ctx.stream>>>(N, k1, src1, y, ht, pred);
    }
    VRG_LAUNCH_CHECK();
    if (fwd)
        forwardRhs(pred, k2);
    else
        backwardRhs(pred, k2);
    LaunchScope ls_(ctx, "k_stage2");
    k_stage2<<<grid(g), kB, 0, ctx.stream>>>(N, k1, k2, src2, y, 0.5 * ht, yNext);
    VRG_LAUNCH_CHECK();
}

void HeunTransport::forward(const double* m0, double* nodes, double* stages, bool guard) {
    const std::size_t N = g.points();
    log.reset(ctx);
    if (nodes != m0) copy(ctx, N, m0, nodes);
    launchFieldMax(ctx, g, nodes, log.partial(0));
    for (int j = 1; j <= nt; ++j) {
        heunStep(nodes + (j - 1) * N, nodes + j * N, stages + (j - 1) * N, true, nullptr, nullptr);
        launchFieldMax(ctx, g, nodes + j * N, log.partial(j));
    }
    log.check(ctx, "state", nt, true, guard, 0);
}

void HeunTransport::backward(const double* lam1, double* nodes, double* stages, bool guard) {
    const std::size_t N = g.points();
    log.reset(ctx);
    if (nodes + nt * N != lam1) copy(ctx, N, lam1, nodes + nt * N);
    launchFieldMax(ctx, g, nodes + nt * N, log.partial(nt));
    for (int j = nt; j >= 1; --j) {
        heunStep(nodes + j * N, nodes + (j - 1) * N, stages + (j - 1) * N, false, nullptr, nullptr);
        launchFieldMax(ctx, g, nodes + (j - 1) * N, log.partial(j - 1));
    }
    log.check(ctx, "adjoint", nt, false, guard, nt);
}

void HeunTransport::stateFinal(const double* m0, double* out) {
    const std::size_t N = g.points();
    double* a = w(2);
    double* b = w(3);
    double* pred = w(4);
    log.reset(ctx);
    launchFieldMax(ctx, g, m0, log.partial(0));
    const double* cur = m0;
    for (int j = 1; j <= nt; ++j) {
        double* dst = j == nt ? out : (j % 2 ? a : b);
        heunStep(cur, dst, pred, true, nullptr, nullptr);
        launchFieldMax(ctx, g, dst, log.partial(j));
        cur = dst;
    }
    log.check(ctx, "state", nt, true, true, 0);
}

void HeunTransport::adjointFinal(const double* lam1, double* out) {
    const std::size_t N = g.points();
    double* a = w(2);
    double* b = w(3);
    double* pred = w(4);
    log.reset(ctx);
    launchFieldMax(ctx, g, lam1, log.partial(nt));
    const double* cur = lam1;
    for (int j = nt; j >= 1; --j) {
        double* dst = j == 1 ? out : (j % 2 ? a : b);
        heunStep(cur, dst, pred, false, nullptr, nullptr);
        launchFieldMax(ctx, g, dst, log.partial(j - 1));
        cur = dst;
    }
    log.check(ctx, "adjoint", nt, false, true, nt);
}

void HeunTransport::forwardStages(const double* nodes, double* stages) {
    const std::size_t N = g.points();
    for (int j = 1; j <= nt; ++j) {
        double* k1 = w(0);
        forwardRhs(nodes + (j - 1) * N, k1);
        LaunchScope ls_(ctx, "k_stage1");
        k_stage1<<<grid(g), kB, 0, ctx.stream>>>(N, k1, nullptr, nodes + (j - 1) * N, ht, stages + (j - 1) * N);
        VRG_LAUNCH_CHECK();
    }
}

void HeunTransport::backwardStages(const double* nodes, double* stages) {
    const std::size_t N = g.points();
    for (int j = nt; j >= 1; --j) {
        double* k1 = w(0);
        backwardRhs(nodes + j * N, k1);
        LaunchScope ls_(ctx, "k_stage1");
        k_stage1<<<grid(g), kB, 0, ctx.stream>>>(N, k1, nullptr, nodes + j * N, ht, stages + (j - 1) * N);
        VRG_LAUNCH_CHECK();
    }
}

void HeunTransport::incState(const double* vt1, const double* vt2, const double* stNodes, const double* stStages,
                             double* out) {
    const std::size_t N = g.points();
    double* divvt = w(5);
    if (anti) divergence(ctx, g, vt1, vt2, divvt);
    double* s1 = w(2);
    double* s2 = w(3);
    double* pred = w(4);
    auto source = [&](const double* m, double* s) {  // -S(m)[vt]
        double* a = w(6);
        advectBy(ctx, g, vt1, vt2, m, a);
        if (!anti) {
            LaunchScope ls_(ctx, "k_comb");
            k_comb<<<grid(g), kB, 0, ctx.stream>>>(N, a, 0.0, nullptr, 0.0, nullptr, nullptr, -1.0, s);
        } else {
            double* dp = w(7);
            divOfProduct(ctx, g, vt1, vt2, m, dp);
            LaunchScope ls_(ctx, "k_comb");
            k_comb<<<grid(g), kB, 0, ctx.stream>>>(N, a, 1.0, dp, -1.0, m, divvt, -0.5, s);
        }
        VRG_LAUNCH_CHECK();
    };
    fill(ctx, N, 0.0, out);
    for (int j = 1; j <= nt; ++j) {
        // the sources are computed first: the rhs of the step reuses the same work slots
        source(stNodes + (j - 1) * N, s1);
        source(stStages + (j - 1) * N, s2);
        heunStep(out + (j - 1) * N, out + j * N, pred, true, s1, s2);
    }
}

void HeunTransport::incAdjointFullNewton(const double* vt1, const double* vt2, const double* lt1,
                                         const double* adjNodes, const double* adjStages, double* out) {
    const std::size_t N = g.points();
    double* divvt = w(5);
    if (anti) divergence(ctx, g, vt1, vt2, divvt);
    double* s1 = w(2);
    double* s2 = w(3);
    double* pred = w(4);
    auto source = [&](const double* lam, double* q) {
        divOfProduct(ctx, g, vt1, vt2, lam, q);
        if (anti) {
            double* a = w(6);
            advectBy(ctx, g, vt1, vt2, lam, a);
            LaunchScope ls_(ctx, "k_comb");
            k_comb<<<grid(g), kB, 0, ctx.stream>>>(N, q, 1.0, a, 1.0, lam, divvt, 0.5, q);
            VRG_LAUNCH_CHECK();
        }
    };
    if (out + nt * N != lt1) copy(ctx, N, lt1, out + nt * N);
    for (int j = nt; j >= 1; --j) {
        source(adjNodes + j * N, s1);
        source(adjStages + (j - 1) * N, s2);
        heunStep(out + j * N, out + (j - 1) * N, pred, false, s1, s2);
    }
}

void HeunTransport::jacobian(double* out) {
    const std::size_t N = g.points();
    const double* v1 = v.d();
    const double* v2 = v1 + N;
    const double* dv = divVelocity();
    double* k1 = w(0);
    double* k2 = w(1);
    double* pred = w(4);
    double* a = w(6);
    auto rhs = [&](const double* J, double* o) {  // (-v.grad J) + 1.0 (J div v) == -((v.grad J) - J div v)
        advectBy(ctx, g, v1, v2, J, a);
        LaunchScope ls_(ctx, "k_comb");
        k_comb<<<grid(g), kB, 0, ctx.stream>>>(N, a, 0.0, nullptr, -1.0, J, dv, -1.0, o);
        VRG_LAUNCH_CHECK();
    };
    fill(ctx, N, 1.0, out);
    for (int j = 1; j <= nt; ++j) {
        rhs(out, k1);
        {
            LaunchScope ls_(ctx, "k_stage1");
            k_stage1<<<grid(g), kB, 0, ctx.stream>>>(N, k1, nullptr, out, ht, pred);
        }
        VRG_LAUNCH_CHECK();
        rhs(pred, k2);
        LaunchScope ls_(ctx, "k_stage2");
        k_stage2<<<grid(g), kB, 0, ctx.stream>>>(N, k1, k2, nullptr, out, 0.5 * ht, out);
        VRG_LAUNCH_CHECK();
    }
}

}  // namespace vrg
