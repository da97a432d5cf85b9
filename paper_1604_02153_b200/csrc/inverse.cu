// Device GN Hessian matvec: fused SL incremental state (K6), fused SL incremental adjoint +
// trapezoid body force (K5 + K8), spectral regularisation / Leray / split wrapper (K7, K8).
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <vector>

#include "blas.cuh"
#include "epilogues.cuh"
#include "evalband.cuh"
#include "heun.cuh"
#include "inverse.cuh"

namespace vrg {

namespace {

// K5+K8 epilogue: one SL continuity step of the GN incremental adjoint (slContinuityStep,
// src/transport.cpp:206-210) with the trapezoid body force b += w_j lt_j grad m_j
// (assembleBodyForce SL, src/inverse.cpp:58-64) fused in.  On the last step (o1 != null)
// it writes out = reg + b instead of b (HessianOperator::apply, src/inverse.cpp:229-233).
struct EpiAdjointBF {
    static constexpr const char* kName = "evaluate/adjoint_bodyforce";
    static constexpr bool kGuard = true;
    double* guardPartials;
    const double* dvDep;
    const double* dv;
    double ht;
    double* out;
    const double* G1;
    const double* G2;
    double w;
    double* b1;
    double* b2;
    const double* reg1;
    const double* reg2;
    double* o1;
    double* o2;
    struct Pre {
        double dvDep, dv, g1, g2;
    };
    __device__ Pre prefetch(std::size_t p) const {
        return {dvDep[p], dv[p], __ldcs(G1 + p), __ldcs(G2 + p)};  // G_j streamed once per matvec
    }
    __device__ double operator()(std::size_t p, const double* v, const Pre& q) const {
        const double uD = v[0];
        const double f0 = uD * q.dvDep;
        const double pred = uD + ht * f0;
        const double o = uD + 0.5 * ht * (f0 + pred * q.dv);
        const double nb1 = b1[p] + w * (o * q.g1);
        const double nb2 = b2[p] + w * (o * q.g2);
        if (o1) {
            o1[p] = reg1[p] + nb1;
            o2[p] = reg2[p] + nb2;
        } else {
            if (out) out[p] = o;  // null in the fused band path
            b1[p] = nb1;
            b2[p] = nb2;
        }
        return o;
    }
};

// Seed of the incremental adjoint: lt(1) = -m~(1) (inverse.cpp:181), b = w_nt lt(1) grad m_nt.
// Fused band path: `lam` is null and `rowLam` (the row-filtered m~(1)) is negated in place,
// which is the row-filtered lt(1) by linearity; `flag` records a non-finite lt(1).
struct EpiAdjointSeed {
    static constexpr const char* kName = "pointwise/adjoint_seed";
    static constexpr bool kGuard = true;
    double* guardPartials;
    const double* mt;
    double* lam;
    const double* G1;
    const double* G2;
    double w;
    double* b1;
    double* b2;
    double* rowLam = nullptr;
    unsigned* flag = nullptr;
    VRG_NO_PREFETCH
    __device__ double operator()(std::size_t p, const double*, const Pre&) const {
        const double l = -1.0 * mt[p];
        if (lam) lam[p] = l;
        if (rowLam) rowLam[p] = -rowLam[p];
        if (flag && !isfinite(l)) atomicOr(flag, 1u);
        b1[p] = w * (l * G1[p]);
        b2[p] = w * (l * G2[p]);
        return l;
    }
};

// Last incremental-state step with the adjoint seed fused in (GN: lt(1) = -m~(1),
// inverse.cpp:181; b = w_nt lt(1) grad m_nt): returns lt(1), so the row pass that follows
// produces the row-filtered adjoint seed directly (the filter is exactly odd, so this equals
// the band path's in-place negation bit for bit), and writes b with the seed's guard and
// finiteness record (same arithmetic as EpiAdjointSeed).
struct EpiIncSeed {
    static constexpr const char* kName = "evaluate/incstate_seed";
    static constexpr bool kGuard = true;
    double* guardPartials;
    EpiIncState inc;
    double w;
    double* b1;
    double* b2;
    using Pre = EpiIncState::Pre;
    __device__ Pre prefetch(std::size_t p) const { return inc.prefetch(p); }
    __device__ double operator()(std::size_t p, const double* v, const Pre& q) const {
        const double m = inc(p, v, q);
        const double l = -1.0 * m;
        b1[p] = w * (l * inc.g1[p]);
        b2[p] = w * (l * inc.g2[p]);
        return l;
    }
};

}  // namespace
// the last incremental-state step carries the seed's body-force operands too: 64 registers
// spill 8 bytes, so it runs at 3 resident blocks (once per matvec)
template <>
struct BandMinBlocks<EpiIncSeed> {
    static constexpr int value = 3;
};
namespace {


}  // namespace

namespace {
__global__ void k_bf_fn(std::size_t N, double w, const double* __restrict__ lt, const double* __restrict__ g1,
                        const double* __restrict__ g2, const double* __restrict__ lam, const double* __restrict__ t1,
                        const double* __restrict__ t2, double* __restrict__ b1, double* __restrict__ b2) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const double term1 = lt[p] * g1[p] + 1.0 * (lam[p] * t1[p]);
    const double term2 = lt[p] * g2[p] + 1.0 * (lam[p] * t2[p]);
    b1[p] = b1[p] + w * term1;
    b2[p] = b2[p] + w * term2;
}
__global__ void k_add2(std::size_t N, const double* __restrict__ a1, const double* __restrict__ a2,
                       const double* __restrict__ c1, const double* __restrict__ c2, double* __restrict__ o1,
                       double* __restrict__ o2) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    o1[p] = a1[p] + 1.0 * c1[p];
    o2[p] = a2[p] + 1.0 * c2[p];
}
}  // namespace

Hessian::Hessian(Ctx& c, const GridDims& gd, const double* v1, const double* v2, const double* mR, const double* mT,
                 const Model& mdl, int steps, const double* stateTraj, int hmode, const double* adjTraj,
                 const double* gradTraj)
    : ctx(c), g(gd), model(mdl), nt(steps), solver(c, gd, v1, v2, steps), weights(gd, mdl.norm), mode_(hmode) {
    if (!(mdl.betaV > 0.0)) throw InvalidArgument("applyReg: beta must be positive");
    if (g.pairs > 1 && (model.scheme != kSchemeSL || hmode != 0 || model.deformation == kNearIncompressible))
        throw NotSupported("batched pairs: Gauss-Newton SL operators of the compressible / incompressible models only");
    pairStatus.assign(g.pairs, 0);
    pairError.assign(g.pairs, std::string());
    const std::size_t N = g.points();
    state_.alloc(sizeof(double) * (nt + 1) * N);
    if (model.scheme != kSchemeSL) {
        initHeun(mR, mT, stateTraj, adjTraj);
        return;
    }
    if (stateTraj) {
        VRG_CUDA(cudaMemcpyAsync(state_.d(), stateTraj, sizeof(double) * (nt + 1) * N, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
    } else {
        solver.state(mT, state_.d(), true);  // counts 2 + nt interps like solveState in the ctor
        if (g_collectGuards) {
            pairStatus = solver.log.pairStatus;
            pairError = solver.log.pairError;
        }
    }
    // Per-iterate invariants, not counted here: the reference recomputes them inside every
    // matvec and the per-matvec counters below include them.
    const long long f0 = ctx.ffts, i0 = ctx.interps;
    const bool hadFwd = !stateTraj;
    G_.alloc(sizeof(double) * (nt + 1) * 2 * N);
    GD_.alloc(sizeof(double) * nt * 2 * N);
    if (gradTraj && stateTraj) {  // grad m_j of this state, computed by the gradient evaluation (same kernels)
        VRG_CUDA(cudaMemcpyAsync(G_.d(), gradTraj, sizeof(double) * (nt + 1) * 2 * N, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
    } else {
        gradientBatch(ctx, g, state_.d(), nt + 1, G_.d());  // one batched transform chain per chunk
    }
    const double* Xf = solver.departure(kForward);
    // Band path (evalband.cuh) wherever the grid allows it: gather + epilogue + next row pass in
    // one kernel per step, bit-identical to the plain 3-kernel step and 6% faster per matvec at
    // 1024^2 on B200 (0.815 vs 0.867 ms).  The plain step is the generic-grid path.  Its packed
    // departure cells (both directions) exist before any graph capture.
    fused_ = solver.bandPath();
    const Cell* Cf = fused_ ? solver.cells(kForward) : nullptr;
    work_.alloc(sizeof(double) * (11 * N + 2 * paddedTotal(g)));  // + vt coefficients (2 padded)
    // GD_j = (grad m_{j-1})_D, j = 1..nt: the 2nt gradient components prefiltered in one batch
    // (two launches) and evaluated at the forward departure points in one launch per chunk
    {
        const std::size_t P = paddedTotal(g);
        const int total = nt;  // gradient fields G_0 .. G_{nt-1}, two components each
        const std::size_t perField = sizeof(double) * (2 * P + 2 * N);
        const int chunk = static_cast<int>(std::max<std::size_t>(
            1, std::min<std::size_t>(total, (std::size_t(256) << 20) / perField)));
        double* coefs = ctx.scratchBuf(45, sizeof(double) * 2 * chunk * P);
        double* rows = ctx.scratchBuf(46, sizeof(double) * std::max<std::size_t>(2 * chunk * N, 2 * N));
        for (int j0 = 0; j0 < total; j0 += chunk) {
            const int c = std::min(chunk, total - j0);
            launchPrefilterBatch(ctx, g, G_.d() + static_cast<std::size_t>(j0) * 2 * N, N, 2 * c, coefs, P, rows,
                                 nullptr);
            double* gd = GD_.d() + static_cast<std::size_t>(j0) * 2 * N;
            if (fused_)
                launchEvaluateBatch<2>(ctx, g, CoeffSet<2>{{coefs, coefs + P}}, 2 * P, c, Cf, Cf + N,
                                       EpiStore2{nullptr, gd, gd + N}, 2 * N);
            else
                launchEvaluateBatch<2>(ctx, g, CoeffSet<2>{{coefs, coefs + P}}, 2 * P, c, Xf, Xf + N,
                                       EpiStore2{nullptr, gd, gd + N}, 2 * N);
        }
    }
    solver.departure(kBackward);
    solver.divVelocityAtDeparture(kBackward);
    ctx.ffts = f0;
    ctx.interps = i0;
    // lazily-built per-velocity work the reference does on the first apply
    // (charBwd 2 + dvDepBwd 1 interps, divv 3 FFTs; + charFwd 2 if the state was reused)
    lazyInterps_ = 3 + (hadFwd ? 0 : 2);
    if (mode_ == 1) {
        adj_.alloc(sizeof(double) * (nt + 1) * N);
        fn_.alloc(sizeof(double) * (2 * (nt + 1) + 7) * N);
        fnFlag_.alloc(64);
    }
    if (mode_ == 1 && adjTraj) {  // adjoint trajectory reused (inverse.cpp:166-168), copied
        VRG_CUDA(cudaMemcpyAsync(adj_.d(), adjTraj, sizeof(double) * (nt + 1) * N, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
    } else if (mode_ == 1) {
        // full Newton: adjoint seeded with lambda(1) = -(m(1) - mR), guarded (inverse.cpp:169-171);
        // the reference builds the backward characteristics and (div v)_D here, not in the apply
        if (!mR) throw InvalidArgument("HessianOperator: full Newton mode needs the reference image");
        double* lam1 = fn_.d();
        lincomb(ctx, N, 1.0, state_.d() + static_cast<std::size_t>(nt) * N, -1.0, mR, lam1);
        lincomb(ctx, N, -1.0, lam1, 0.0, lam1, lam1);
        solver.adjoint(lam1, adj_.d(), true);  // counted below
        ctx.ffts = f0;
        ctx.interps = i0;
        ctx.interps += nt + 3;  // adjoint + charBwd + dvDep
        ctx.ffts += 3;          // div v
        lazyInterps_ = hadFwd ? 0 : 2;
    }
    if (fused_) solver.cells(kBackward);
    lazyFfts_ = (mode_ == 1 && !adjTraj) ? 0 : 3;
    spec_.alloc(sizeof(cplx) * 4 * g.specPoints());
    for (auto& l : guardLogs_) l.ensure(nt + 1, g);
    weights.regSymbol(model.betaV);
    weights.invRegSymbol(model.betaV, -0.5);
    // every plan a matvec uses exists before any graph capture (plan creation allocates)
    for (int batch = 1; batch <= 2; ++batch) {
        ctx.plan(g, CUFFT_D2Z, batch);
        ctx.plan(g, CUFFT_Z2D, batch);
    }
    ctx.sync();
}


// RK2 / RK2A operator (heun.cuh): state (and, full Newton, adjoint) trajectories with their Heun
// predictors; no graph capture (the Heun solves check their guards on the host).
void Hessian::initHeun(const double* mR, const double* mT, const double* stateTraj, const double* adjTraj) {
    const std::size_t N = g.points();
    const bool anti = model.scheme == kSchemeRK2A;
    heun_ = std::make_unique<HeunTransport>(ctx, g, solver.v1(), solver.v2(), nt, anti);
    stStages_.alloc(sizeof(double) * nt * N);
    if (stateTraj) {
        VRG_CUDA(cudaMemcpyAsync(state_.d(), stateTraj, sizeof(double) * (nt + 1) * N, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
        const long long f0 = ctx.ffts;
        heun_->forwardStages(state_.d(), stStages_.d());  // the reference holds them with the state
        ctx.ffts = f0;
        lazyFfts_ = anti ? 3 : 0;  // div v, built lazily by the first apply in the reference
    } else {
        heun_->forward(mT, state_.d(), stStages_.d(), true);
    }
    if (mode_ == 1) {
        adj_.alloc(sizeof(double) * (nt + 1) * N);
        adjStages_.alloc(sizeof(double) * nt * N);
        if (adjTraj) {
            VRG_CUDA(cudaMemcpyAsync(adj_.d(), adjTraj, sizeof(double) * (nt + 1) * N, cudaMemcpyDeviceToDevice,
                                     ctx.stream));
            const long long f0 = ctx.ffts;
            heun_->backwardStages(adj_.d(), adjStages_.d());
            ctx.ffts = f0;
        } else {
            if (!mR) throw InvalidArgument("HessianOperator: full Newton mode needs the reference image");
            double* lam1 = ctx.scratchBuf(43, sizeof(double) * N);
            lincomb(ctx, N, 1.0, state_.d() + static_cast<std::size_t>(nt) * N, -1.0, mR, lam1);
            lincomb(ctx, N, -1.0, lam1, 0.0, lam1, lam1);
            heun_->backward(lam1, adj_.d(), adjStages_.d(), true);
        }
    }
    work_.alloc(sizeof(double) * (11 * N + paddedPoints(g.n1, g.n2)));
    fn_.alloc(sizeof(double) * (3 * (nt + 1)) * N);  // m~ and lt trajectories, lt predictors
    useGraphs = false;
    lazyInterps_ = 0;
    spec_.alloc(sizeof(cplx) * 4 * g.specPoints());
    for (auto& l : guardLogs_) l.ensure(nt + 1, g);
    weights.regSymbol(model.betaV);
    weights.invRegSymbol(model.betaV, -0.5);
    ctx.sync();
}

namespace {
__global__ void k_bf_terms(std::size_t N, double w, const double* __restrict__ a1, const double* __restrict__ a2,
                           const double* __restrict__ c1, const double* __restrict__ c2, double* __restrict__ b1,
                           double* __restrict__ b2) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    b1[p] = __dadd_rn(b1[p], __dmul_rn(w, __dadd_rn(a1[p], c1[p])));
    b2[p] = __dadd_rn(b2[p], __dmul_rn(w, __dadd_rn(a2[p], c2[p])));
}
}  // namespace

// Data term of the RK2 / RK2A operator (inverse.cpp:176-211 with the Heun solves).
void Hessian::dataTermHeun(const double* vt1, const double* vt2, double* b1, double* b2, const double* reg1,
                           const double* reg2, double* out1, double* out2) {
    const std::size_t N = g.points();
    const double ht = 1.0 / nt;
    const bool anti = model.scheme == kSchemeRK2A;
    double* mt = fn_.d();
    double* lt = mt + static_cast<std::size_t>(nt + 1) * N;
    double* ltS = lt + static_cast<std::size_t>(nt + 1) * N;
    heun_->incState(vt1, vt2, state_.d(), stStages_.d(), mt);
    double* lt1 = lt + static_cast<std::size_t>(nt) * N;
    lincomb(ctx, N, -1.0, mt + static_cast<std::size_t>(nt) * N, 0.0, mt + static_cast<std::size_t>(nt) * N, lt1);
    if (mode_ == 0) {
        heun_->backward(lt1, lt, ltS, true);  // solveAdjoint(-m~(1)), guarded (inverse.cpp:185)
        bodyForceHeun(ctx, g, nt, anti, state_.d(), stStages_.d(), lt, ltS, b1, b2);
    } else {
        heun_->incAdjointFullNewton(vt1, vt2, lt1, adj_.d(), adjStages_.d(), lt);
        double* t = ctx.scratchBuf(44, sizeof(double) * 4 * N);
        fill(ctx, N, 0.0, b1);
        fill(ctx, N, 0.0, b2);
        for (int j = 0; j <= nt; ++j) {
            const double w = ht * ((j == 0 || j == nt) ? 0.5 : 1.0);
            const std::size_t o = static_cast<std::size_t>(j) * N;
            if (anti) {
                antisymmetricForceTerm(ctx, g, state_.d() + o, lt + o, t, t + N);
                antisymmetricForceTerm(ctx, g, mt + o, adj_.d() + o, t + 2 * N, t + 3 * N);
                LaunchScope ls_(ctx, "k_bf_terms");
                k_bf_terms<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, w, t, t + N, t + 2 * N, t + 3 * N, b1, b2);
            } else {
                gradient(ctx, g, state_.d() + o, t, t + N);
                gradient(ctx, g, mt + o, t + 2 * N, t + 3 * N);
                LaunchScope ls_(ctx, "k_bf_fn");
                k_bf_fn<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, w, lt + o, t, t + N, adj_.d() + o, t + 2 * N,
                                                                 t + 3 * N, b1, b2);
            }
            VRG_LAUNCH_CHECK();
        }
    }
    if (out1) {
        waitReg();
        LaunchScope ls_(ctx, "k_add2");
        k_add2<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, reg1, reg2, b1, b2, out1, out2);
        VRG_LAUNCH_CHECK();
    }
}

void Hessian::countDataTerm() {
    if (model.deformation == kNearIncompressible) ctx.ffts += 8;  // penalty gradient of vt
    if (heun_) {  // the Heun solves count as they run (no graph replay); projection and lazy div v
        ctx.ffts += (model.deformation == kIncompressible ? 4 : 0) + lazyFfts_;
        lazyFfts_ = 0;
        return;
    }
    if (mode_ == 1) {
        // incState 2 + 3nt interps, 3 + 3nt FFTs; FN incAdjoint 2nt interps, 3(nt+1) FFTs
        // (div of products); body force 3(nt+1) + 3(nt+1) FFTs (grad m_j, grad m~_j)
        ctx.interps += 5LL * nt + 2 + lazyInterps_;
        ctx.ffts += (3 + 3LL * nt) + 9LL * (nt + 1) + lazyFfts_ + (model.deformation == kIncompressible ? 4 : 0);
        lazyInterps_ = 0;
        lazyFfts_ = 0;
        return;
    }
    ctx.interps += 4LL * nt + 2 + lazyInterps_;
    ctx.ffts += (3 + 3LL * nt) + 3LL * (nt + 1) + lazyFfts_ + (model.deformation == kIncompressible ? 4 : 0);
    lazyInterps_ = 0;
    lazyFfts_ = 0;
}

void Hessian::dataTerm(const double* vt1, const double* vt2, double* b1, double* b2, const double* reg1,
                       const double* reg2, double* out1, double* out2) {
    if (heun_) {
        dataTermHeun(vt1, vt2, b1, b2, reg1, reg2, out1, out2);
        return;
    }
    if (mode_ == 1) {
        dataTermFN(vt1, vt2, b1, b2, reg1, reg2, out1, out2);
        return;
    }
    const std::size_t N = g.points();
    const double ht = solver.ht;
    double* vtD = work_.d();
    double* mt[2] = {vtD + 2 * N, vtD + 3 * N};
    double* lam[2] = {vtD + 4 * N, vtD + 5 * N};
    const double* Xf = solver.departure(kForward);
    const double* Xb = solver.departure(kBackward);
    const Cell* Cf = fused_ ? solver.cells(kForward) : nullptr;
    const Cell* Cb = fused_ ? solver.cells(kBackward) : nullptr;
    const double* dv = solver.divVelocity();
    const double* dvd = solver.divVelocityAtDeparture(kBackward);
    double* coef = solver.coef();
    double* tmp = solver.tmp();
    auto G = [&](int j) { return G_.d() + static_cast<std::size_t>(j) * 2 * N; };
    auto GD = [&](int j) { return GD_.d() + static_cast<std::size_t>(j - 1) * 2 * N; };  // j = 1..nt

    // incremental state (solveIncState SL, transport.cpp:322-342); vt's two components are
    // prefiltered in one batch (two launches) when contiguous
    {
        const std::size_t P = paddedTotal(g);
        double* cv = vtD + 11 * N;
        if (vt2 == vt1 + N) {
            launchPrefilterBatch(ctx, g, vt1, N, 2, cv, P, tmp, nullptr);
        } else {
            launchPrefilter(ctx, g, vt1, cv, tmp, nullptr);
            launchPrefilter(ctx, g, vt2, cv + P, tmp, nullptr);
        }
        if (fused_)
            launchEvaluate<2>(ctx, g, CoeffSet<2>{{cv, cv + P}}, Cf, Cf + N, EpiStore2{nullptr, vtD, vtD + N}, true);
        else
            launchEvaluate<2>(ctx, g, CoeffSet<2>{{cv, cv + P}}, Xf, Xf + N, EpiStore2{nullptr, vtD, vtD + N}, true);
    }
    auto wOf = [&](int j) { return ht * ((j == 0 || j == nt) ? 0.5 : 1.0); };
    if (fused_) {
        // Band path: every step's gather kernel also row-filters its output (evalband.cuh), so
        // each step is [column pass] + [gather + epilogue + row pass].  R[.] ping-pong holds
        // the row-filtered m~_j, then the row-filtered lt_j.
        double* R[2] = {tmp, tmp + N};
        adjLog_->reset(ctx);
        for (int j = 1; j <= nt; ++j) {
            const EpiIncState epi{nullptr, vtD, vtD + N, GD(j), GD(j) + N, vt1, vt2, G(j), G(j) + N, 0.5 * ht, nullptr};
            if (j > 1) launchPrefilterCols(ctx, g, R[(j - 1) & 1], coef);
            const CoeffSet<1> cs{{coef}};
            if (j == nt) {
                // the adjoint seed lt(1) = -m~(1) and b = w lt(1) grad m_nt fused into the last
                // step; its row pass then yields the row-filtered seed directly
                const EpiIncSeed seed{adjLog_->partial(nt), epi, wOf(nt), b1, b2};
                if (j == 1)
                    launchEvalBand<EpiIncSeed, false>(ctx, g, cs, Cf, Cf + N, seed, R[j & 1], adjLog_->flag(nt));
                else
                    launchEvalBand<EpiIncSeed, true>(ctx, g, cs, Cf, Cf + N, seed, R[j & 1], adjLog_->flag(nt));
            } else if (j == 1) {
                launchEvalBand<EpiIncState, false>(ctx, g, cs, Cf, Cf + N, epi, R[j & 1], nullptr);
            } else {
                launchEvalBand<EpiIncState, true>(ctx, g, cs, Cf, Cf + N, epi, R[j & 1], nullptr);
            }
        }
        for (int j = nt; j >= 1; --j) {
            launchPrefilterCols(ctx, g, R[j & 1], coef);
            const bool last = j == 1;
            EpiAdjointBF epi{adjLog_->partial(j - 1), dvd, dv, ht, nullptr, G(j - 1), G(j - 1) + N, wOf(j - 1),
                             b1, b2, reg1, reg2, last ? out1 : nullptr, last ? out2 : nullptr};
            if (last) {
                waitReg();
                launchEvalBand<EpiAdjointBF, true>(ctx, g, CoeffSet<1>{{coef}}, Cb, Cb + N, epi, nullptr, nullptr);
            } else {
                launchEvalBand<EpiAdjointBF, true>(ctx, g, CoeffSet<1>{{coef}}, Cb, Cb + N, epi, R[(j - 1) & 1],
                                                   adjLog_->flag(j - 1));
            }
        }
        return;
    }
    for (int j = 1; j <= nt; ++j) {
        EpiIncState epi{nullptr, vtD, vtD + N, GD(j), GD(j) + N, vt1, vt2, G(j), G(j) + N, 0.5 * ht, mt[j & 1]};
        if (j == 1) {
            launchPointwise(ctx, g, epi);
        } else {
            launchPrefilter(ctx, g, mt[(j - 1) & 1], coef, tmp, nullptr);
            launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xf, Xf + N, epi, true);
        }
    }
    // incremental adjoint (GN: solveAdjoint(-m~(1)), guarded, inverse.cpp:185) + body force
    adjLog_->reset(ctx);
    launchPointwise(ctx, g,
                    EpiAdjointSeed{adjLog_->partial(nt), mt[nt & 1], lam[nt & 1], G(nt), G(nt) + N, wOf(nt), b1, b2});
    for (int j = nt; j >= 1; --j) {
        launchPrefilter(ctx, g, lam[j & 1], coef, tmp, adjLog_->flag(j));
        const bool last = (j == 1) && out1;
        EpiAdjointBF epi{adjLog_->partial(j - 1), dvd, dv, ht, lam[(j - 1) & 1], G(j - 1), G(j - 1) + N, wOf(j - 1),
                         b1, b2, reg1, reg2, last ? out1 : nullptr, last ? out2 : nullptr};
        if (j == 1) waitReg();
        launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xb, Xb + N, epi, true);
    }
}

// Full-Newton data term (HessianOperator::Impl::dataTerm FN branch, inverse.cpp:187-211, SL):
// incremental state trajectory, full-Newton incremental adjoint, and the body force
// b = sum_j w_j (lt_j grad m_j + lambda_j grad m~_j), trapezoid weights, in the reference's
// order (j = 0..nt).


void Hessian::dataTermFN(const double* vt1, const double* vt2, double* b1, double* b2, const double* reg1,
                         const double* reg2, double* out1, double* out2) {
    const std::size_t N = g.points();
    const long long f0 = ctx.ffts, i0 = ctx.interps;  // logical counts come from countDataTerm
    const double ht = solver.ht;
    double* vtD = work_.d();
    double* c2 = vtD + 11 * N;
    double* mt = fn_.d();
    double* lt = mt + static_cast<std::size_t>(nt + 1) * N;
    double* work = lt + static_cast<std::size_t>(nt + 1) * N;  // 5N
    double* gmt = work + 5 * N;                                 // 2N
    unsigned* flag = fnFlag_.as<unsigned>();
    VRG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), ctx.stream));
    const double* Xf = solver.departure(kForward);
    double* coef = solver.coef();
    double* tmp = solver.tmp();
    auto G = [&](int j) { return G_.d() + static_cast<std::size_t>(j) * 2 * N; };
    auto GD = [&](int j) { return GD_.d() + static_cast<std::size_t>(j - 1) * 2 * N; };
    // incremental state trajectory (solveIncState SL)
    launchPrefilter(ctx, g, vt1, coef, tmp, flag);
    launchPrefilter(ctx, g, vt2, c2, tmp, flag);
    launchEvaluate<2>(ctx, g, CoeffSet<2>{{coef, c2}}, Xf, Xf + N, EpiStore2{nullptr, vtD, vtD + N}, true);
    fill(ctx, N, 0.0, mt);
    for (int j = 1; j <= nt; ++j) {
        EpiIncState epi{nullptr, vtD, vtD + N, GD(j), GD(j) + N, vt1, vt2, G(j), G(j) + N, 0.5 * ht,
                        mt + static_cast<std::size_t>(j) * N};
        if (j == 1) {
            launchPointwise(ctx, g, epi);
        } else {
            launchPrefilter(ctx, g, mt + static_cast<std::size_t>(j - 1) * N, coef, tmp, flag);
            launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xf, Xf + N, epi, true);
        }
    }
    // lt(1) = -m~(1), full-Newton incremental adjoint
    double* lt1 = lt + static_cast<std::size_t>(nt) * N;
    lincomb(ctx, N, -1.0, mt + static_cast<std::size_t>(nt) * N, 0.0, mt + static_cast<std::size_t>(nt) * N, lt1);
    solver.incAdjointFullNewton(vt1, vt2, lt1, adj_.d(), lt, work, flag);
    // body force, trapezoid over the nodes
    fill(ctx, 2 * N, 0.0, b1);
    if (b2 != b1 + N) fill(ctx, N, 0.0, b2);
    for (int j = 0; j <= nt; ++j) {
        const double w = ht * ((j == 0 || j == nt) ? 0.5 : 1.0);
        gradient(ctx, g, mt + static_cast<std::size_t>(j) * N, gmt, gmt + N);
        {
            LaunchScope ls_(ctx, "k_bf_fn");
            k_bf_fn<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, w, lt + static_cast<std::size_t>(j) * N, G(j),
                                                             G(j) + N, adj_.d() + static_cast<std::size_t>(j) * N,
                                                             gmt, gmt + N, b1, b2);
        }
        VRG_LAUNCH_CHECK();
    }
    if (out1) {
        waitReg();
        LaunchScope ls_(ctx, "k_add2");
        k_add2<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, reg1, reg2, b1, b2, out1, out2);
        VRG_LAUNCH_CHECK();
    }
    ctx.ffts = f0;
    ctx.interps = i0;
}

void Hessian::waitReg() {
    if (!regPending_) return;
    VRG_CUDA(cudaStreamWaitEvent(ctx.stream, evJoin_, 0));
    regPending_ = false;
}

// b += -betaW grad((1 - Lap) div vt) (inverse.cpp:214-215), without touching the op counters
// (the matvec's logical counts come from countDataTerm; graph replays run no host code)
void Hessian::addPenalty(const double* vt1, const double* vt2, double* b1, double* b2) {
    const std::size_t N = g.points();
    const long long f0 = ctx.ffts;
    double* pen = ctx.scratchBuf(42, sizeof(double) * 2 * N);
    divergencePenaltyGradient(ctx, g, vt1, vt2, model.betaW, pen, pen + N);
    axpby(ctx, N, 1.0, pen, 1.0, b1);
    axpby(ctx, N, 1.0, pen + N, 1.0, b2);
    ctx.ffts = f0;
}

// ------------------------------------------------------------------------------ slabs
// One SL step of a slab-decomposed grid (slab.py): the band kernel over the slab's L rows with
// the coefficients in a window (BandWindow), epilogue by kind (see include/vrg.h).
void slabStep(Ctx& ctx, int kind, int n1, int n2, int L, int winBase, int winRows, const double* coef,
              const double* x1, const double* x2, const double* const* ops, int nops, double ht, double w,
              double* rowOut, double* guardPartials, unsigned* flag, unsigned* winErr) {
    static const int kNeed[] = {1, 8, 8, 10, 10, 6, 10, 1};
    if (kind < 0 || kind > 7) throw InvalidArgument("slab step: unknown kind");
    if (nops < kNeed[kind]) throw InvalidArgument("slab step: too few operand fields");
    if (!bandFusable(GridDims(L, n2)) || n2 % kBandThreads != 0 || L < 1 || n1 < L)
        throw NotSupported("slab step: unsupported row length");
    const BandWindow win{winBase, winRows, winErr};
    const CoeffSet<1> cs{{coef}};
    auto inc = [&] {
        return EpiIncState{nullptr, ops[0], ops[1], ops[2], ops[3], ops[4], ops[5], ops[6], ops[7], 0.5 * ht, nullptr};
    };
    switch (kind) {
        case 0:
            launchEvalBandWindow<EpiStore1, true>(ctx, n1, L, n2, cs, x1, x2, EpiStore1{nullptr, const_cast<double*>(ops[0])},
                                                  rowOut, flag, win);
            break;
        case 1: launchEvalBandWindow<EpiIncState, true>(ctx, n1, L, n2, cs, x1, x2, inc(), rowOut, flag, win); break;
        case 2: launchEvalBandWindow<EpiIncState, false>(ctx, n1, L, n2, cs, x1, x2, inc(), rowOut, flag, win); break;
        case 3:
        case 4: {
            const EpiIncSeed seed{guardPartials, inc(), w, const_cast<double*>(ops[8]), const_cast<double*>(ops[9])};
            if (kind == 3)
                launchEvalBandWindow<EpiIncSeed, true>(ctx, n1, L, n2, cs, x1, x2, seed, rowOut, flag, win);
            else
                launchEvalBandWindow<EpiIncSeed, false>(ctx, n1, L, n2, cs, x1, x2, seed, rowOut, flag, win);
            break;
        }
        case 5:
        case 6: {
            const bool last = kind == 6;
            const EpiAdjointBF epi{guardPartials, ops[0], ops[1], ht, nullptr, ops[2], ops[3], w,
                                   const_cast<double*>(ops[4]), const_cast<double*>(ops[5]), last ? ops[6] : nullptr,
                                   last ? ops[7] : nullptr, last ? const_cast<double*>(ops[8]) : nullptr,
                                   last ? const_cast<double*>(ops[9]) : nullptr};
            launchEvalBandWindow<EpiAdjointBF, true>(ctx, n1, L, n2, cs, x1, x2, epi, rowOut, flag, win);
            break;
        }
        default:
            launchEvalBandWindow<EpiStateStep, true>(ctx, n1, L, n2, cs, x1, x2,
                                                     EpiStateStep{guardPartials, const_cast<double*>(ops[0])}, rowOut,
                                                     flag, win);
            break;
    }
}

void Hessian::beginDeferredGuards(int maxCalls) {
    if (heun_ || mode_ == 1 || maxCalls <= 0) return;  // those paths check as they run / differently
    const std::size_t per = static_cast<std::size_t>(nt + 1) * g.pairs;
    if (maxCalls > deferCap_) {
        deferMax_.alloc(sizeof(double) * per * maxCalls);
        deferFlags_.alloc(sizeof(unsigned) * per * maxCalls);
        deferCap_ = maxCalls;
    }
    deferring_ = true;
    deferCount_ = 0;
}

void Hessian::endDeferredGuards() {
    if (!deferring_) return;
    deferring_ = false;
    const int k = deferCount_;
    if (k == 0) return;
    const int P = g.pairs;
    const std::size_t steps = static_cast<std::size_t>(nt + 1), per = steps * P;
    std::vector<double> mx(per * k);
    std::vector<unsigned> fl(steps * k);
    VRG_CUDA(cudaMemcpyAsync(mx.data(), deferMax_.d(), sizeof(double) * per * k, cudaMemcpyDeviceToHost, ctx.stream));
    VRG_CUDA(cudaMemcpyAsync(fl.data(), deferFlags_.d(), sizeof(unsigned) * steps * k, cudaMemcpyDeviceToHost,
                             ctx.stream));
    ctx.sync();
    if (!g_collectGuards) {
        for (int c = 0; c < k; ++c)
            GuardLog::checkHost(mx.data() + c * per, fl.data() + c * steps, "adjoint", nt, false, true, nt);
        return;
    }
    // a batch: each pair's first error in call order, nothing thrown
    std::vector<double> m1(steps);
    for (int p = 0; p < P; ++p) {
        for (int c = 0; c < k && !pairStatus[p]; ++c) {
            for (std::size_t s = 0; s < steps; ++s) m1[s] = mx[c * per + s * P + p];
            try {
                GuardLog::checkHost(m1.data(), fl.data() + c * steps, "adjoint", nt, false, true, nt);
            } catch (const BlowupError& e) {
                pairStatus[p] = kBlowup;
                pairError[p] = e.what();
            } catch (const InvalidArgument& e) {
                pairStatus[p] = kInvalidArgument;
                pairError[p] = e.what();
            }
        }
    }
}

void Hessian::guardAfterMatvec() {
    if (!deferring_) {
        checkLastGuard();
        return;
    }
    if (deferCount_ >= deferCap_) {  // log full: check what is there, then continue immediately
        endDeferredGuards();
        checkLastGuard();
        return;
    }
    const std::size_t steps = static_cast<std::size_t>(nt + 1), per = steps * g.pairs;
    VRG_CUDA(cudaMemcpyAsync(deferMax_.d() + per * deferCount_, adjLog_->stepMax(), sizeof(double) * per,
                             cudaMemcpyDeviceToDevice, ctx.stream));
    VRG_CUDA(cudaMemcpyAsync(deferFlags_.as<unsigned>() + steps * deferCount_, adjLog_->flags(),
                             sizeof(unsigned) * steps, cudaMemcpyDeviceToDevice, ctx.stream));
    ++deferCount_;
}

void Hessian::checkLastGuard() {
    if (heun_) return;  // the Heun solves checked their guards as they ran
    if (mode_ == 1) {  // full Newton: no guard in the incremental solves, prefilter input checks only
        unsigned h = 0;
        VRG_CUDA(cudaMemcpyAsync(&h, fnFlag_.d(), sizeof h, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        if (h) throw InvalidArgument("prefilter: non-finite value");
        return;
    }
    adjLog_->check(ctx, "adjoint", nt, false, true, nt);
    if (g_collectGuards)
        for (int p = 0; p < g.pairs; ++p)
            if (!pairStatus[p] && adjLog_->pairStatus[p]) {
                pairStatus[p] = adjLog_->pairStatus[p];
                pairError[p] = adjLog_->pairError[p];
            }
}

// Average device time of one launch of a matvec kernel class, `iters` back-to-back launches
// between two events on the context stream, with the operands of a mid-trajectory step
// (steady state after a matvec has run, so the operands are the ones the matvec produced).
double Hessian::benchKernel(int id, int iters) {
    // id + 100: band steps with strip blocks, id + 200: one block per row (evalband.cuh)
    struct MappingScope {
        int old = g_bandMapping.load();
        ~MappingScope() { g_bandMapping = old; }
    } mappingScope_;
    if (id >= 200) {
        g_bandMapping = 1;
        id -= 200;
    } else if (id >= 100) {
        g_bandMapping = 2;
        id -= 100;
    }
    const std::size_t N = g.points();
    const double ht = solver.ht;
    const int j = std::max(2, nt / 2);
    double* vtD = work_.d();
    double* mt = vtD + 2 * N;
    double* lam = vtD + 4 * N;
    double* b = vtD + 6 * N;
    double* c2 = vtD + 11 * N;
    const double* Xf = solver.departure(kForward);
    const double* Xb = solver.departure(kBackward);
    const Cell* Cf = fused_ ? solver.cells(kForward) : nullptr;
    const Cell* Cb = fused_ ? solver.cells(kBackward) : nullptr;
    const double* dv = solver.divVelocity();
    const double* dvd = solver.divVelocityAtDeparture(kBackward);
    double* coef = solver.coef();
    double* tmp = solver.tmp();
    const double* G = G_.d() + static_cast<std::size_t>(j) * 2 * N;
    const double* GD = GD_.d() + static_cast<std::size_t>(j - 1) * 2 * N;
    auto one = [&] {
        switch (id) {
            case 0: {  // incremental-state step (K6)
                EpiIncState epi{nullptr, vtD, vtD + N, GD, GD + N, vtD, vtD + N, G, G + N, 0.5 * ht, mt + N};
                launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xf, Xf + N, epi, true);
                break;
            }
            case 1: {  // incremental-adjoint step + body force (K5+K8); band path: the last step's form
                EpiAdjointBF epi{adjLog_->partial(0), dvd, dv, ht, lam + N, G, G + N, ht, b, b + N,
                                 nullptr, nullptr, nullptr, nullptr};
                if (fused_)
                    launchEvalBand<EpiAdjointBF, true>(ctx, g, CoeffSet<1>{{coef}}, Cb, Cb + N, epi, nullptr, nullptr);
                else
                    launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xb, Xb + N, epi, true);
                break;
            }
            case 2:  // prefilter, both passes (K1)
                launchPrefilter(ctx, g, mt, coef, tmp, nullptr);
                break;
            case 4:  // prefilter column pass only (K1 cols)
                launchPrefilterCols(ctx, g, tmp, coef);
                break;
            case 5:  // reference point: one field copy (F read + F write), cudaMemcpyAsync D2D
                copy(ctx, N, mt, tmp);
                break;
            case 6:  // reference point: one field axpy kernel (2F read + F write)
                axpby(ctx, N, 0.5, mt, 1.0, tmp);
                break;
            case 7: {  // band incremental-state step: gather + epilogue + next row pass
                if (!fused_) throw NotSupported("bench kernel 7: band path not active on this grid");
                EpiIncState epi{nullptr, vtD, vtD + N, GD, GD + N, vtD, vtD + N, G, G + N, 0.5 * ht, nullptr};
                launchEvalBand<EpiIncState, true>(ctx, g, CoeffSet<1>{{coef}}, Cf, Cf + N, epi, tmp, nullptr);
                break;
            }
            case 8: {  // band incremental-adjoint + body-force step
                if (!fused_) throw NotSupported("bench kernel 8: band path not active on this grid");
                EpiAdjointBF epi{adjLog_->partial(0), dvd, dv, ht, nullptr, G, G + N, ht, b, b + N,
                                 nullptr, nullptr, nullptr, nullptr};
                launchEvalBand<EpiAdjointBF, true>(ctx, g, CoeffSet<1>{{coef}}, Cb, Cb + N, epi, tmp + N,
                                                   adjLog_->flag(0));
                break;
            }
            case 11: {  // band incremental-state step without the gather (m~_0 = 0 form): operand traffic only
                if (!fused_) throw NotSupported("bench kernel 11: band path not active on this grid");
                EpiIncState epi{nullptr, vtD, vtD + N, GD, GD + N, vtD, vtD + N, G, G + N, 0.5 * ht, nullptr};
                launchEvalBand<EpiIncState, false>(ctx, g, CoeffSet<1>{{coef}}, Cf, Cf + N, epi, tmp, nullptr);
                break;
            }
            case 9:  // SL state step (config 4 unit ii), band form: gather + m_j + next row pass, column pass
                if (!solver.bandPath()) throw NotSupported("bench kernel 9: band path not active on this grid");
                launchEvalBand<EpiStateStep, true>(ctx, g, CoeffSet<1>{{coef}}, Cf, Cf + N,
                                                   EpiStateStep{adjLog_->partial(0), mt + N}, tmp, nullptr);
                launchPrefilterCols(ctx, g, tmp, coef);
                break;
            case 12:  // the band kernel of the SL state step alone (no column pass)
                if (!solver.bandPath()) throw NotSupported("bench kernel 12: band path not active on this grid");
                launchEvalBand<EpiStateStep, true>(ctx, g, CoeffSet<1>{{coef}}, Cf, Cf + N,
                                                   EpiStateStep{adjLog_->partial(0), mt + N}, tmp, nullptr);
                break;
            case 10:  // SL state step, plain form: prefilter (rows + cols) + gather
                launchPrefilter(ctx, g, mt, coef, tmp, nullptr);
                launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xf, Xf + N, EpiStateStep{adjLog_->partial(0), mt + N}, true);
                break;
            case 13:  // one whole matvec launched directly on the stream (programmatic dependent launch, no graph)
            case 14: {  // the same matvec through its CUDA graph (the apply path's replay)
                double* in = ctx.scratchBuf(160, sizeof(double) * 2 * N);
                double* out = ctx.scratchBuf(161, sizeof(double) * 2 * N);
                VRG_CUDA(cudaMemcpyAsync(in, vtD, sizeof(double) * 2 * N, cudaMemcpyDeviceToDevice, ctx.stream));
                if (id == 13) {
                    launchApply(in, in + N, out, out + N);
                } else {
                    replay(0, in, in + N, out, out + N, [&] { launchApply(in, in + N, out, out + N); });
                }
                break;
            }
            default:  // vtilde at departure (K2, two fields)
                launchEvaluate<2>(ctx, g, CoeffSet<2>{{coef, c2}}, Xf, Xf + N, EpiStore2{nullptr, vtD, vtD + N}, true);
                break;
        }
    };
    one();  // warm
    cudaEvent_t e0, e1;
    VRG_CUDA(cudaEventCreate(&e0));
    VRG_CUDA(cudaEventCreate(&e1));
    VRG_CUDA(cudaEventRecord(e0, ctx.stream));
    for (int i = 0; i < iters; ++i) one();
    VRG_CUDA(cudaEventRecord(e1, ctx.stream));
    VRG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    VRG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms / iters;
}

// The launch sequence of one matvec is fixed for given (kind, in, out) pointers, so it is
// captured once into a CUDA graph and replayed (removes ~100 launch gaps per matvec).  The
// host-side work (counters, guard readback) stays outside the graph.
// With the context profile on, the sequence is launched directly behind a sleeping gate kernel
// (Ctx::profGate), so the whole matvec is queued before the GPU reaches it and the per-kernel
// event pairs time back-to-back execution, as in the graph replay.
template <class F>
void Hessian::replay(int kind, const double* a, const double* b, const double* c, const double* d, F&& launchSeq) {
    if (!useGraphs || ctx.profOn) {
        if (ctx.profOn) ctx.profGate(3000);
        launchSeq();
        return;
    }
    const bool prof = false;
    const GraphKey key{kind, a, b, c, d};
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
        // first use of this (kind, pointers): launch directly; capture on the second use, so an
        // operator applied once or twice (Newton iterations with few Krylov steps) pays no
        // graph instantiation
        launchSeq();
        graphs_.emplace(key, GraphEntry{});
        return;
    }
    if (!it->second.exec) {
        const long long l0 = ctx.launches;
        const std::size_t ev0 = ctx.evNext;
        cudaGraph_t graph = nullptr;
        VRG_CUDA(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal));
        try {
            launchSeq();
        } catch (...) {
            cudaStreamEndCapture(ctx.stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            ctx.launches = l0;
            throw;
        }
        VRG_CUDA(cudaStreamEndCapture(ctx.stream, &graph));
        GraphEntry& e = it->second;
        {  // shape of the captured graph (instrumentation: vrg_hess_graph_info)
            std::size_t nodes = 0, edges = 0;
            VRG_CUDA(cudaGraphGetNodes(graph, nullptr, &nodes));
            VRG_CUDA(cudaGraphGetEdges_v2(graph, nullptr, nullptr, nullptr, &edges));
            std::vector<cudaGraphNode_t> from(edges), to(edges);
            std::vector<cudaGraphEdgeData> data(edges);
            if (edges) VRG_CUDA(cudaGraphGetEdges_v2(graph, from.data(), to.data(), data.data(), &edges));
            int prog = 0;
            for (const auto& d : data) prog += d.type == cudaGraphDependencyTypeProgrammatic;
            graphInfo_[0] = static_cast<int>(nodes);
            graphInfo_[1] = static_cast<int>(edges);
            graphInfo_[2] = prog;
        }
        VRG_CUDA(cudaGraphInstantiate(&e.exec, graph, 0));
        cudaGraphDestroy(graph);
        e.launches = ctx.launches - l0;
        ctx.launches = l0;
        if (prof) {  // the graph takes ownership of the events recorded during capture
            e.recs.swap(ctx.profRecs);
            e.events.assign(ctx.evPool.begin() + ev0, ctx.evPool.begin() + ctx.evNext);
            ctx.evPool.erase(ctx.evPool.begin() + ev0, ctx.evPool.begin() + ctx.evNext);
            ctx.evNext = ev0;
        }
    }
    VRG_CUDA(cudaGraphLaunch(it->second.exec, ctx.stream));
    ctx.launches += it->second.launches;
    if (prof) {
        ctx.sync();
        ctx.profAccumulate(it->second.recs);
    }
}

Hessian::~Hessian() {
    if (aux_) {
        cudaStreamSynchronize(aux_);
        cudaEventDestroy(evFork_);
        cudaEventDestroy(evJoin_);
        cudaStreamDestroy(aux_);
    }
    if (guardStream_) {
        cudaStreamSynchronize(guardStream_);
        for (auto& e : evGuard_) cudaEventDestroy(e);
        for (auto& e : evDone_) cudaEventDestroy(e);
        cudaStreamDestroy(guardStream_);
        cudaFreeHost(hostGuard_);
    }
    for (auto& kv : graphs_) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        for (cudaEvent_t e : kv.second.events) cudaEventDestroy(e);
    }
}

void Hessian::apply(const double* vt1, const double* vt2, double* o1, double* o2) {
    NvtxRange nv_("HessianOperator::apply");
    replay(0, vt1, vt2, o1, o2, [&] { launchApply(vt1, vt2, o1, o2); });
    ctx.ffts += 4;
    countDataTerm();
    checkLastGuard();
}

bool Hessian::queuedGuards() const { return !heun_ && mode_ == 0 && g.pairs == 1 && !g_collectGuards; }

void Hessian::applyQueued(const double* vt1, const double* vt2, double* o1, double* o2, int slot) {
    if (!queuedGuards()) {
        apply(vt1, vt2, o1, o2);
        return;
    }
    NvtxRange nv_("HessianOperator::apply (queued)");
    if (!guardStream_) {
        VRG_CUDA(cudaMallocHost(&hostGuard_, 2 * guardSlotBytes()));
        VRG_CUDA(cudaStreamCreateWithFlags(&guardStream_, cudaStreamNonBlocking));
        for (int s = 0; s < 2; ++s) {
            VRG_CUDA(cudaEventCreateWithFlags(&evGuard_[s], cudaEventDisableTiming));
            VRG_CUDA(cudaEventCreateWithFlags(&evDone_[s], cudaEventDisableTiming));
        }
    }
    // guard log `slot` (the graph of this slot writes it) is free once its previous readback is
    // done; the readback of this matvec runs on the guard stream, off the matvec stream
    VRG_CUDA(cudaStreamWaitEvent(ctx.stream, evGuard_[slot], 0));
    adjLog_ = &guardLogs_[slot];
    try {
        replay(8 * slot, vt1, vt2, o1, o2, [&] { launchApply(vt1, vt2, o1, o2); });
    } catch (...) {
        adjLog_ = &guardLogs_[0];
        throw;
    }
    adjLog_ = &guardLogs_[0];
    ctx.ffts += 4;
    countDataTerm();
    VRG_CUDA(cudaEventRecord(evDone_[slot], ctx.stream));
    VRG_CUDA(cudaStreamWaitEvent(guardStream_, evDone_[slot], 0));
    const GuardLog& L = guardLogs_[slot];
    VRG_CUDA(cudaMemcpyAsync(hostGuardSlot(slot), L.buf.d(), L.bytes(), cudaMemcpyDeviceToHost, guardStream_));
    VRG_CUDA(cudaEventRecord(evGuard_[slot], guardStream_));
}

void Hessian::checkQueued(int slot) {
    if (!queuedGuards()) return;  // applyQueued checked already
    const GuardLog& L = guardLogs_[slot];
    VRG_CUDA(cudaEventSynchronize(evGuard_[slot]));
    const double* host = hostGuardSlot(slot);
    GuardLog::checkHost(host, reinterpret_cast<const unsigned*>(host + static_cast<std::size_t>(L.steps) * L.pairs),
                        "adjoint", nt, false, true, nt);
}

void Hessian::launchApply(const double* vt1, const double* vt2, double* o1, double* o2) {
    const std::size_t N = g.points();
    double* b = work_.d() + 6 * N;
    double* reg = work_.d() + 9 * N;
    cplx* S = spec_.as<cplx>();
    const std::size_t NS = g.specPoints();
    const double* regSym = weights.regSymbol(model.betaV);
    if (model.deformation == kIncompressible) {
        // out = beta A vt + P b, assembled in one spectrum (applyReg + projectDivFree)
        if (vt2 == vt1 + N) {
            fftForward(ctx, g, vt1, S, 2);
        } else {
            fftForward(ctx, g, vt1, S, 1);
            fftForward(ctx, g, vt2, S + NS, 1);
        }
        specScale(ctx, g, S, 2, regSym, 1.0);
        dataTerm(vt1, vt2, b, b + N, nullptr, nullptr, nullptr, nullptr);
        fftForward(ctx, g, b, S + 2 * NS, 2);
        specCombine(ctx, g, S + 2 * NS, S + 3 * NS, S, S + NS, nullptr, true, 1.0 / g.pointsPer(), S + 2 * NS, S + 3 * NS);
        if (o2 == o1 + N) {
            fftInverse(ctx, g, S + 2 * NS, o1, 2);
        } else {
            fftInverse(ctx, g, S + 2 * NS, o1, 1);
            fftInverse(ctx, g, S + 3 * NS, o2, 1);
        }
    } else {
        // reg = beta A vt on the second stream (independent of the data term until its last
        // step), then the last adjoint step writes out = reg + b
        if (!aux_) {
            VRG_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
            VRG_CUDA(cudaEventCreateWithFlags(&evFork_, cudaEventDisableTiming));
            VRG_CUDA(cudaEventCreateWithFlags(&evJoin_, cudaEventDisableTiming));
        }
        if (aux_) {
            VRG_CUDA(cudaEventRecord(evFork_, ctx.stream));
            VRG_CUDA(cudaStreamWaitEvent(aux_, evFork_, 0));
        }
        {
            StreamSwap sw(ctx, aux_ ? aux_ : ctx.stream);
            if (vt2 == vt1 + N) {
                fftForward(ctx, g, vt1, S, 2);
            } else {
                fftForward(ctx, g, vt1, S, 1);
                fftForward(ctx, g, vt2, S + NS, 1);
            }
            specScale(ctx, g, S, 2, regSym, 1.0 / g.pointsPer());
            fftInverse(ctx, g, S, reg, 2);
        }
        if (aux_) {
            VRG_CUDA(cudaEventRecord(evJoin_, aux_));
            regPending_ = true;
        }
        if (model.deformation == kNearIncompressible) {
            // out = beta A vt + (b + penalty gradient) (inverse.cpp:212-233)
            dataTerm(vt1, vt2, b, b + N, nullptr, nullptr, nullptr, nullptr);
            addPenalty(vt1, vt2, b, b + N);
            waitReg();
            LaunchScope ls_(ctx, "k_add2");
            k_add2<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, reg, reg + N, b, b + N, o1, o2);
            VRG_LAUNCH_CHECK();
        } else {
            dataTerm(vt1, vt2, b, b + N, reg, reg + N, o1, o2);
        }
    }
}

void Hessian::applyDataTerm(const double* vt1, const double* vt2, double* o1, double* o2) {
    NvtxRange nv_("HessianOperator::applyDataTerm");
    replay(1, vt1, vt2, o1, o2, [&] {
        const std::size_t N = g.points();
        double* b = work_.d() + 6 * N;
        dataTerm(vt1, vt2, b, b + N, nullptr, nullptr, nullptr, nullptr);
        if (model.deformation == kIncompressible) {
            cplx* T = spec_.as<cplx>() + 2 * g.specPoints();
            fftForward(ctx, g, b, T, 2);
            specCombine(ctx, g, T, T + g.specPoints(), nullptr, nullptr, nullptr, true, 1.0 / g.pointsPer(), T, T + g.specPoints());
            if (o2 == o1 + N) {
                fftInverse(ctx, g, T, o1, 2);
            } else {
                fftInverse(ctx, g, T, o1, 1);
                fftInverse(ctx, g, T + g.specPoints(), o2, 1);
            }
        } else {
            if (model.deformation == kNearIncompressible) addPenalty(vt1, vt2, b, b + N);
            copy(ctx, N, b, o1);
            copy(ctx, N, b + N, o2);
        }
    });
    countDataTerm();
    checkLastGuard();
}

void Hessian::applySplit(const double* s1, const double* s2, double* o1, double* o2) {
    NvtxRange nv_("applySplitHessianOf");
    replay(2, s1, s2, o1, o2, [&] { launchSplit(s1, s2, o1, o2); });
    ctx.ffts += 8;
    countDataTerm();
    guardAfterMatvec();
}

void Hessian::launchSplit(const double* s1, const double* s2, double* o1, double* o2) {
    const std::size_t N = g.points();
    const std::size_t NS = g.specPoints();
    cplx* S = spec_.as<cplx>();      // s^ (kept)
    cplx* T = S + 2 * NS;            // t^ then b^ then out^
    double* t = work_.d() + 9 * N;   // t = M^{-1/2} s
    double* b = work_.d() + 6 * N;
    const double* inv = weights.invRegSymbol(model.betaV, -0.5);
    if (s2 == s1 + N) {
        fftForward(ctx, g, s1, S, 2);
    } else {
        fftForward(ctx, g, s1, S, 1);
        fftForward(ctx, g, s2, S + NS, 1);
    }
    specCombine(ctx, g, S, S + NS, nullptr, nullptr, inv, false, 1.0 / g.pointsPer(), T, T + NS);
    fftInverse(ctx, g, T, t, 2);
    dataTerm(t, t + N, b, b + N, nullptr, nullptr, nullptr, nullptr);
    if (model.deformation == kNearIncompressible) addPenalty(t, t + N, b, b + N);
    fftForward(ctx, g, b, T, 2);
    specCombine(ctx, g, T, T + NS, S, S + NS, inv, model.deformation == kIncompressible, 1.0 / g.pointsPer(), T, T + NS);
    if (o2 == o1 + N) {
        fftInverse(ctx, g, T, o1, 2);
    } else {
        fftInverse(ctx, g, T, o1, 1);
        fftInverse(ctx, g, T + NS, o2, 1);
    }
}

// ------------------------------------------------------------------------------ gradient / objective
namespace {

// The trapezoid sum over a chunk of frames j0 .. j0+c-1 in one launch, accumulated in the
// order of the per-frame loop (same expression per frame as k_bf_accum, bit-identical).
__global__ void k_bf_accum_frames(std::size_t N, int j0, int c, int nt, double ht, const double* __restrict__ lam,
                                  const double* __restrict__ G, double* b1, double* b2, int first) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    double a1 = first ? 0.0 : b1[p], a2 = first ? 0.0 : b2[p];
    for (int k = 0; k < c; ++k) {
        const int j = j0 + k;
        const double w = ht * ((j == 0 || j == nt) ? 0.5 : 1.0);
        const double l = lam[static_cast<std::size_t>(j) * N + p];
        const double* g = G + static_cast<std::size_t>(k) * 2 * N;
        a1 += w * (l * g[p]);
        a2 += w * (l * g[N + p]);
    }
    b1[p] = a1;
    b2[p] = a2;
}

}  // namespace

// assembleBodyForce SL (src/inverse.cpp:58-64): b = sum_j w_j lam_j grad m_j, the gradients of
// the state frames by batched transforms (gradientBatch) and the sum in one launch per chunk.
void bodyForce(Ctx& ctx, const GridDims& g, int nt, const double* stateTraj, const double* adjTraj, double* b1,
               double* b2, double* gradTrajOut) {
    const std::size_t N = g.points();
    const double ht = 1.0 / nt;
    const int frames = nt + 1;
    // without an output trajectory the gradients go through a scratch of one chunk
    const int chunk = gradTrajOut ? frames
                                  : static_cast<int>(std::max<std::size_t>(
                                        1, std::min<std::size_t>(frames, (std::size_t(256) << 20) / (16 * N))));
    double* scratch = gradTrajOut ? nullptr : ctx.scratchBuf(20, sizeof(double) * 2 * N * chunk);
    for (int j0 = 0; j0 < frames; j0 += chunk) {
        const int c = std::min(chunk, frames - j0);
        double* gm = gradTrajOut ? gradTrajOut + static_cast<std::size_t>(j0) * 2 * N : scratch;
        gradientBatch(ctx, g, stateTraj + static_cast<std::size_t>(j0) * N, c, gm);
        {
            LaunchScope ls_(ctx, "k_bf_accum");
            k_bf_accum_frames<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, j0, c, nt, ht, adjTraj, gm, b1, b2,
                                                                      j0 == 0 ? 1 : 0);
        }
        VRG_LAUNCH_CHECK();
    }
}

// evaluateObjective / evaluateGradient (src/inverse.cpp:96-148) for the compressible and
// incompressible models.  stateOut / adjOut (nullable) receive the trajectories.
void evaluateObjective(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* mR,
                       const double* mT, const Model& model, int nt, double* scalars, double* stateOut,
                       double* stateStagesOut) {
    NvtxRange nv_("evaluateObjective");
    const std::size_t N = g.points();
    DBuf stateBuf;
    double* st = stateOut;
    if (!st) {
        stateBuf.alloc(sizeof(double) * (nt + 1) * N);
        st = stateBuf.d();
    }
    if (model.scheme != kSchemeSL) {
        HeunTransport heun(ctx, g, v1, v2, nt, model.scheme == kSchemeRK2A);
        DBuf stages;
        if (!stateStagesOut) stages.alloc(sizeof(double) * nt * N);
        heun.forward(mT, st, stateStagesOut ? stateStagesOut : stages.d(), true);
    } else {
        Solver solver(ctx, g, v1, v2, nt);
        solver.state(mT, st, true);
    }
    double* resid = ctx.scratchBuf(21, sizeof(double) * N);
    lincomb(ctx, N, 1.0, st + nt * N, -1.0, mR, resid);
    const double mismatch = 0.5 * dot(ctx, g, resid, nullptr, resid, nullptr);
    Weights w(g, model.norm);
    double* reg = ctx.scratchBuf(22, sizeof(double) * 2 * N);
    if (!(model.betaV > 0.0)) throw InvalidArgument("applyReg: beta must be positive");
    applyRealSymbol(ctx, g, v1, v2, reg, reg + N, w.regSymbol(model.betaV));
    const double regTerm = 0.5 * dot(ctx, g, reg, reg + N, v1, v2);
    const double penalty =
        model.deformation == kNearIncompressible ? divergencePenaltyValue(ctx, g, v1, v2, model.betaW) : 0.0;
    scalars[0] = mismatch + regTerm + penalty;
    scalars[1] = mismatch;
    scalars[2] = regTerm;
    scalars[3] = penalty;
}

void evaluateGradient(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* mR,
                      const double* mT, const Model& model, int nt, double* g1, double* g2, double* scalars,
                      double* stateOut, double* adjOut, const double* reuseState, double* gradTrajOut,
                      double* bodyOut, double* stateStagesOut, double* adjStagesOut) {
    NvtxRange nv_("evaluateGradient");
    const std::size_t N = g.points();
    DBuf stBuf, adBuf;
    double* st = stateOut;
    double* ad = adjOut;
    if (!st) {
        stBuf.alloc(sizeof(double) * (nt + 1) * N);
        st = stBuf.d();
    }
    if (!ad) {
        adBuf.alloc(sizeof(double) * (nt + 1) * N);
        ad = adBuf.d();
    }
    double* b = ctx.scratchBuf(23, sizeof(double) * 2 * N);
    double* resid = ctx.scratchBuf(21, sizeof(double) * N);
    double mismatch = 0.0;
    if (model.scheme != kSchemeSL) {  // RK2 / RK2A: Heun solves, stage-paired body force
        const bool anti = model.scheme == kSchemeRK2A;
        HeunTransport heun(ctx, g, v1, v2, nt, anti);
        DBuf stB, adB;
        if (!stateStagesOut) stB.alloc(sizeof(double) * nt * N);
        if (!adjStagesOut) adB.alloc(sizeof(double) * nt * N);
        double* stS = stateStagesOut ? stateStagesOut : stB.d();
        double* adS = adjStagesOut ? adjStagesOut : adB.d();
        if (reuseState) {
            if (reuseState != st) copy(ctx, (nt + 1) * N, reuseState, st);
            const long long f0 = ctx.ffts;
            heun.forwardStages(st, stS);
            ctx.ffts = f0;
        } else {
            heun.forward(mT, st, stS, true);
        }
        lincomb(ctx, N, 1.0, st + nt * N, -1.0, mR, resid);
        mismatch = 0.5 * dot(ctx, g, resid, nullptr, resid, nullptr);
        lincomb(ctx, N, -1.0, resid, 0.0, resid, resid);
        heun.backward(resid, ad, adS, true);
        bodyForceHeun(ctx, g, nt, anti, st, stS, ad, adS, b, b + N);
    } else {
        Solver solver(ctx, g, v1, v2, nt);
        if (reuseState) {
            if (reuseState != st) copy(ctx, (nt + 1) * N, reuseState, st);
        } else {
            solver.state(mT, st, true);
        }
        lincomb(ctx, N, 1.0, st + nt * N, -1.0, mR, resid);
        mismatch = 0.5 * dot(ctx, g, resid, nullptr, resid, nullptr);
        lincomb(ctx, N, -1.0, resid, 0.0, resid, resid);  // lambda1 = -1.0 * resid
        solver.adjoint(resid, ad, true);
        bodyForce(ctx, g, nt, st, ad, b, b + N, gradTrajOut);
    }
    Weights w(g, model.norm);
    if (!(model.betaV > 0.0)) throw InvalidArgument("applyReg: beta must be positive");
    applyRealSymbol(ctx, g, v1, v2, g1, g2, w.regSymbol(model.betaV));
    const double regTerm = 0.5 * dot(ctx, g, g1, g2, v1, v2);
    double penalty = 0.0;
    if (model.deformation == kNearIncompressible) {
        penalty = divergencePenaltyValue(ctx, g, v1, v2, model.betaW);
        double* pen = ctx.scratchBuf(42, sizeof(double) * 2 * N);
        divergencePenaltyGradient(ctx, g, v1, v2, model.betaW, pen, pen + N);
        axpby(ctx, N, 1.0, pen, 1.0, g1);
        axpby(ctx, N, 1.0, pen + N, 1.0, g2);
    }
    if (bodyOut) copy(ctx, 2 * N, b, bodyOut);
    if (model.deformation == kIncompressible) projectDivFree(ctx, g, b, b + N, b, b + N);
    axpby(ctx, N, 1.0, b, 1.0, g1);
    axpby(ctx, N, 1.0, b + N, 1.0, g2);
    scalars[0] = mismatch + regTerm + penalty;
    scalars[1] = mismatch;
    scalars[2] = regTerm;
    scalars[3] = penalty;
}

}  // namespace vrg
