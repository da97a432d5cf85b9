// Device GN Hessian matvec: fused SL incremental state (K6), fused SL incremental adjoint +
// trapezoid body force (K5 + K8), spectral regularisation / Leray / split wrapper (K7, K8).
#include <cstdlib>

#include "epilogues.cuh"
#include "evalband.cuh"
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

}  // namespace

Hessian::Hessian(Ctx& c, const GridDims& gd, const double* v1, const double* v2, const double* mR, const double* mT,
                 const Model& mdl, int steps, const double* stateTraj)
    : ctx(c), g(gd), model(mdl), nt(steps), solver(c, gd, v1, v2, steps), weights(gd, mdl.norm) {
    (void)mR;
    if (mdl.deformation == kNearIncompressible)
        throw NotSupported("HessianOperator: near-incompressible model is not implemented on the device");
    if (!(mdl.betaV > 0.0)) throw InvalidArgument("applyReg: beta must be positive");
    const std::size_t N = g.points();
    state_.alloc(sizeof(double) * (nt + 1) * N);
    if (stateTraj) {
        VRG_CUDA(cudaMemcpyAsync(state_.d(), stateTraj, sizeof(double) * (nt + 1) * N, cudaMemcpyDeviceToDevice,
                                 ctx.stream));
    } else {
        solver.state(mT, state_.d(), true);  // counts 2 + nt interps like solveState in the ctor
    }
    // Per-iterate invariants, not counted here: the reference recomputes them inside every
    // matvec and the per-matvec counters below include them.
    const long long f0 = ctx.ffts, i0 = ctx.interps;
    const bool hadFwd = !stateTraj;
    G_.alloc(sizeof(double) * (nt + 1) * 2 * N);
    GD_.alloc(sizeof(double) * nt * 2 * N);
    for (int j = 0; j <= nt; ++j) gradient(ctx, g, state_.d() + j * N, G_.d() + j * 2 * N, G_.d() + j * 2 * N + N);
    const double* Xf = solver.departure(kForward);
    work_.alloc(sizeof(double) * (11 * N + paddedPoints(g.n1, g.n2)));
    double* c2 = work_.d() + 11 * N;
    for (int j = 1; j <= nt; ++j) {
        const double* gp = G_.d() + (j - 1) * 2 * N;
        launchPrefilter(ctx, g, gp, solver.coef(), solver.tmp(), nullptr);
        launchPrefilter(ctx, g, gp + N, c2, solver.tmp(), nullptr);
        double* gd = GD_.d() + (j - 1) * 2 * N;
        launchEvaluate<2>(ctx, g, CoeffSet<2>{{solver.coef(), c2}}, Xf, Xf + N, EpiStore2{nullptr, gd, gd + N});
    }
    solver.departure(kBackward);
    solver.divVelocityAtDeparture(kBackward);
    ctx.ffts = f0;
    ctx.interps = i0;
    // lazily-built per-velocity work the reference does on the first apply
    // (charBwd 2 + dvDepBwd 1 interps, divv 3 FFTs; + charFwd 2 if the state was reused)
    lazyInterps_ = 3 + (hadFwd ? 0 : 2);
    // Band path (evalband.cuh) wherever the grid allows it: gather + epilogue + next row pass in
    // one kernel per step, bit-identical to the plain 3-kernel step and 6% faster per matvec at
    // 1024^2 on B200 (0.815 vs 0.867 ms).  VRG_FUSED_BANDS=0 selects the plain step.
    const char* env = std::getenv("VRG_FUSED_BANDS");
    const bool want = !(env && env[0] == '0');
    fused_ = useFusedBands && want && bandFusable(g) && colPassFusable(g) && bandBlocks(g) <= evalBlocks(g);
    if (const char* ge = std::getenv("VRG_GRAPHS")) useGraphs = ge[0] != '0';  // debugging switch
    lazyFfts_ = 3;
    spec_.alloc(sizeof(cplx) * 4 * g.specPoints());
    adjLog_.ensure(nt + 1, evalBlocks(g));
    weights.regSymbol(model.betaV);
    weights.invRegSymbol(model.betaV, -0.5);
    // every plan a matvec uses exists before any graph capture (plan creation allocates)
    for (int batch = 1; batch <= 2; ++batch) {
        ctx.plan(g, CUFFT_D2Z, batch);
        ctx.plan(g, CUFFT_Z2D, batch);
    }
    ctx.sync();
}

void Hessian::countDataTerm() {
    ctx.interps += 4LL * nt + 2 + lazyInterps_;
    ctx.ffts += (3 + 3LL * nt) + 3LL * (nt + 1) + lazyFfts_ + (model.deformation == kIncompressible ? 4 : 0);
    lazyInterps_ = 0;
    lazyFfts_ = 0;
}

void Hessian::dataTerm(const double* vt1, const double* vt2, double* b1, double* b2, const double* reg1,
                       const double* reg2, double* out1, double* out2) {
    const std::size_t N = g.points();
    const double ht = solver.ht;
    double* vtD = work_.d();
    double* mt[2] = {vtD + 2 * N, vtD + 3 * N};
    double* lam[2] = {vtD + 4 * N, vtD + 5 * N};
    double* c2 = vtD + 11 * N;  // padded coefficients of the second component
    const double* Xf = solver.departure(kForward);
    const double* Xb = solver.departure(kBackward);
    const double* dv = solver.divVelocity();
    const double* dvd = solver.divVelocityAtDeparture(kBackward);
    double* coef = solver.coef();
    double* tmp = solver.tmp();
    auto G = [&](int j) { return G_.d() + static_cast<std::size_t>(j) * 2 * N; };
    auto GD = [&](int j) { return GD_.d() + static_cast<std::size_t>(j - 1) * 2 * N; };  // j = 1..nt

    // incremental state (solveIncState SL, transport.cpp:322-342)
    launchPrefilter(ctx, g, vt1, coef, tmp, nullptr);
    launchPrefilter(ctx, g, vt2, c2, tmp, nullptr);
    launchEvaluate<2>(ctx, g, CoeffSet<2>{{coef, c2}}, Xf, Xf + N, EpiStore2{nullptr, vtD, vtD + N}, true);
    auto wOf = [&](int j) { return ht * ((j == 0 || j == nt) ? 0.5 : 1.0); };
    if (fused_) {
        // Band path: every step's gather kernel also row-filters its output (evalband.cuh), so
        // each step is [column pass] + [gather + epilogue + row pass].  R[.] ping-pong holds
        // the row-filtered m~_j, then the row-filtered lt_j.
        double* R[2] = {tmp, tmp + N};
        double* mtLast = mt[0];  // unfiltered m~(1) for the adjoint seed
        for (int j = 1; j <= nt; ++j) {
            EpiIncState epi{nullptr, vtD, vtD + N, GD(j), GD(j) + N, vt1, vt2, G(j), G(j) + N, 0.5 * ht,
                            j == nt ? mtLast : nullptr};
            if (j == 1) {
                launchEvalBand<EpiIncState, false>(ctx, g, CoeffSet<1>{{coef}}, Xf, Xf + N, epi, R[1], nullptr);
            } else {
                launchPrefilterCols(ctx, g, R[(j - 1) & 1], coef);
                launchEvalBand<EpiIncState, true>(ctx, g, CoeffSet<1>{{coef}}, Xf, Xf + N, epi, R[j & 1], nullptr);
            }
        }
        adjLog_.reset(ctx);
        EpiAdjointSeed seed{adjLog_.partial(nt), mtLast, nullptr, G(nt), G(nt) + N, wOf(nt), b1, b2, R[nt & 1],
                            adjLog_.flag(nt)};
        launchPointwise(ctx, g, seed);
        for (int j = nt; j >= 1; --j) {
            launchPrefilterCols(ctx, g, R[j & 1], coef);
            const bool last = j == 1;
            EpiAdjointBF epi{adjLog_.partial(j - 1), dvd, dv, ht, nullptr, G(j - 1), G(j - 1) + N, wOf(j - 1),
                             b1, b2, reg1, reg2, last ? out1 : nullptr, last ? out2 : nullptr};
            if (last)
                launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xb, Xb + N, epi, true);
            else
                launchEvalBand<EpiAdjointBF, true>(ctx, g, CoeffSet<1>{{coef}}, Xb, Xb + N, epi, R[(j - 1) & 1],
                                                   adjLog_.flag(j - 1));
        }
        adjLog_.finalize(ctx);
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
    adjLog_.reset(ctx);
    launchPointwise(ctx, g,
                    EpiAdjointSeed{adjLog_.partial(nt), mt[nt & 1], lam[nt & 1], G(nt), G(nt) + N, wOf(nt), b1, b2});
    for (int j = nt; j >= 1; --j) {
        launchPrefilter(ctx, g, lam[j & 1], coef, tmp, adjLog_.flag(j));
        const bool last = (j == 1) && out1;
        EpiAdjointBF epi{adjLog_.partial(j - 1), dvd, dv, ht, lam[(j - 1) & 1], G(j - 1), G(j - 1) + N, wOf(j - 1),
                         b1, b2, reg1, reg2, last ? out1 : nullptr, last ? out2 : nullptr};
        launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef}}, Xb, Xb + N, epi, true);
    }
    adjLog_.finalize(ctx);
}

void Hessian::checkLastGuard() { adjLog_.check(ctx, "adjoint", nt, false, true, nt); }

// Average device time of one launch of a matvec kernel class, `iters` back-to-back launches
// between two events on the context stream, with the operands of a mid-trajectory step
// (steady state after a matvec has run, so the operands are the ones the matvec produced).
double Hessian::benchKernel(int id, int iters) {
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
            case 1: {  // incremental-adjoint step + body force (K5+K8)
                EpiAdjointBF epi{adjLog_.partial(0), dvd, dv, ht, lam + N, G, G + N, ht, b, b + N,
                                 nullptr, nullptr, nullptr, nullptr};
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
                launchEvalBand<EpiIncState, true>(ctx, g, CoeffSet<1>{{coef}}, Xf, Xf + N, epi, tmp, nullptr);
                break;
            }
            case 8: {  // band incremental-adjoint + body-force step
                if (!fused_) throw NotSupported("bench kernel 8: band path not active on this grid");
                EpiAdjointBF epi{adjLog_.partial(0), dvd, dv, ht, nullptr, G, G + N, ht, b, b + N,
                                 nullptr, nullptr, nullptr, nullptr};
                launchEvalBand<EpiAdjointBF, true>(ctx, g, CoeffSet<1>{{coef}}, Xb, Xb + N, epi, tmp + N,
                                                   adjLog_.flag(0));
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
        GraphEntry e;
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
        it = graphs_.emplace(key, std::move(e)).first;
    }
    VRG_CUDA(cudaGraphLaunch(it->second.exec, ctx.stream));
    ctx.launches += it->second.launches;
    if (prof) {
        ctx.sync();
        ctx.profAccumulate(it->second.recs);
    }
}

Hessian::~Hessian() {
    for (auto& kv : graphs_) {
        cudaGraphExecDestroy(kv.second.exec);
        for (cudaEvent_t e : kv.second.events) cudaEventDestroy(e);
    }
}

void Hessian::apply(const double* vt1, const double* vt2, double* o1, double* o2) {
    replay(0, vt1, vt2, o1, o2, [&] { launchApply(vt1, vt2, o1, o2); });
    ctx.ffts += 4;
    countDataTerm();
    checkLastGuard();
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
        specCombine(ctx, g, S + 2 * NS, S + 3 * NS, S, S + NS, nullptr, true, 1.0 / N, S + 2 * NS, S + 3 * NS);
        if (o2 == o1 + N) {
            fftInverse(ctx, g, S + 2 * NS, o1, 2);
        } else {
            fftInverse(ctx, g, S + 2 * NS, o1, 1);
            fftInverse(ctx, g, S + 3 * NS, o2, 1);
        }
    } else {
        // reg = beta A vt, then the last adjoint step writes out = reg + b
        if (vt2 == vt1 + N) {
            fftForward(ctx, g, vt1, S, 2);
        } else {
            fftForward(ctx, g, vt1, S, 1);
            fftForward(ctx, g, vt2, S + NS, 1);
        }
        specScale(ctx, g, S, 2, regSym, 1.0 / N);
        fftInverse(ctx, g, S, reg, 2);
        dataTerm(vt1, vt2, b, b + N, reg, reg + N, o1, o2);
    }
}

void Hessian::applyDataTerm(const double* vt1, const double* vt2, double* o1, double* o2) {
    replay(1, vt1, vt2, o1, o2, [&] {
        const std::size_t N = g.points();
        double* b = work_.d() + 6 * N;
        dataTerm(vt1, vt2, b, b + N, nullptr, nullptr, nullptr, nullptr);
        if (model.deformation == kIncompressible) {
            cplx* T = spec_.as<cplx>() + 2 * g.specPoints();
            fftForward(ctx, g, b, T, 2);
            specCombine(ctx, g, T, T + g.specPoints(), nullptr, nullptr, nullptr, true, 1.0 / N, T, T + g.specPoints());
            if (o2 == o1 + N) {
                fftInverse(ctx, g, T, o1, 2);
            } else {
                fftInverse(ctx, g, T, o1, 1);
                fftInverse(ctx, g, T + g.specPoints(), o2, 1);
            }
        } else {
            copy(ctx, N, b, o1);
            copy(ctx, N, b + N, o2);
        }
    });
    countDataTerm();
    checkLastGuard();
}

void Hessian::applySplit(const double* s1, const double* s2, double* o1, double* o2) {
    replay(2, s1, s2, o1, o2, [&] { launchSplit(s1, s2, o1, o2); });
    ctx.ffts += 8;
    countDataTerm();
    checkLastGuard();
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
    specCombine(ctx, g, S, S + NS, nullptr, nullptr, inv, false, 1.0 / N, T, T + NS);
    fftInverse(ctx, g, T, t, 2);
    dataTerm(t, t + N, b, b + N, nullptr, nullptr, nullptr, nullptr);
    fftForward(ctx, g, b, T, 2);
    specCombine(ctx, g, T, T + NS, S, S + NS, inv, model.deformation == kIncompressible, 1.0 / N, T, T + NS);
    if (o2 == o1 + N) {
        fftInverse(ctx, g, T, o1, 2);
    } else {
        fftInverse(ctx, g, T, o1, 1);
        fftInverse(ctx, g, T + NS, o2, 1);
    }
}

// ------------------------------------------------------------------------------ gradient / objective
namespace {

__global__ void k_bf_accum(std::size_t N, double w, const double* __restrict__ lam, const double* __restrict__ g1,
                           const double* __restrict__ g2, double* b1, double* b2) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    b1[p] += w * (lam[p] * g1[p]);
    b2[p] += w * (lam[p] * g2[p]);
}

}  // namespace

// assembleBodyForce SL (src/inverse.cpp:58-64): b = sum_j w_j lam_j grad m_j.
void bodyForce(Ctx& ctx, const GridDims& g, int nt, const double* stateTraj, const double* adjTraj, double* b1,
               double* b2) {
    const std::size_t N = g.points();
    const double ht = 1.0 / nt;
    double* gm = ctx.scratchBuf(20, sizeof(double) * 2 * N);
    fill(ctx, N, 0.0, b1);
    fill(ctx, N, 0.0, b2);
    for (int j = 0; j <= nt; ++j) {
        const double w = ht * ((j == 0 || j == nt) ? 0.5 : 1.0);
        gradient(ctx, g, stateTraj + j * N, gm, gm + N);
        {
            LaunchScope ls_(ctx, "k_bf_accum");
            k_bf_accum<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, w, adjTraj + j * N, gm, gm + N, b1, b2);
        }
        VRG_LAUNCH_CHECK();
    }
}

// evaluateObjective / evaluateGradient (src/inverse.cpp:96-148) for the compressible and
// incompressible models.  stateOut / adjOut (nullable) receive the trajectories.
void evaluateObjective(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* mR,
                       const double* mT, const Model& model, int nt, double* scalars, double* stateOut) {
    if (model.deformation == kNearIncompressible) throw NotSupported("near-incompressible model not implemented");
    const std::size_t N = g.points();
    Solver solver(ctx, g, v1, v2, nt);
    DBuf stateBuf;
    double* st = stateOut;
    if (!st) {
        stateBuf.alloc(sizeof(double) * (nt + 1) * N);
        st = stateBuf.d();
    }
    solver.state(mT, st, true);
    double* resid = ctx.scratchBuf(21, sizeof(double) * N);
    lincomb(ctx, N, 1.0, st + nt * N, -1.0, mR, resid);
    const double mismatch = 0.5 * dot(ctx, g, resid, nullptr, resid, nullptr);
    Weights w(g, model.norm);
    double* reg = ctx.scratchBuf(22, sizeof(double) * 2 * N);
    if (!(model.betaV > 0.0)) throw InvalidArgument("applyReg: beta must be positive");
    applyRealSymbol(ctx, g, v1, v2, reg, reg + N, w.regSymbol(model.betaV));
    const double regTerm = 0.5 * dot(ctx, g, reg, reg + N, v1, v2);
    scalars[0] = mismatch + regTerm;
    scalars[1] = mismatch;
    scalars[2] = regTerm;
}

void evaluateGradient(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* mR,
                      const double* mT, const Model& model, int nt, double* g1, double* g2, double* scalars,
                      double* stateOut, double* adjOut, const double* reuseState) {
    if (model.deformation == kNearIncompressible) throw NotSupported("near-incompressible model not implemented");
    const std::size_t N = g.points();
    Solver solver(ctx, g, v1, v2, nt);
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
    if (reuseState) {
        if (reuseState != st) copy(ctx, (nt + 1) * N, reuseState, st);
    } else {
        solver.state(mT, st, true);
    }
    double* resid = ctx.scratchBuf(21, sizeof(double) * N);
    lincomb(ctx, N, 1.0, st + nt * N, -1.0, mR, resid);
    const double mismatch = 0.5 * dot(ctx, g, resid, nullptr, resid, nullptr);
    lincomb(ctx, N, -1.0, resid, 0.0, resid, resid);  // lambda1 = -1.0 * resid
    solver.adjoint(resid, ad, true);
    double* b = ctx.scratchBuf(23, sizeof(double) * 2 * N);
    bodyForce(ctx, g, nt, st, ad, b, b + N);
    Weights w(g, model.norm);
    if (!(model.betaV > 0.0)) throw InvalidArgument("applyReg: beta must be positive");
    applyRealSymbol(ctx, g, v1, v2, g1, g2, w.regSymbol(model.betaV));
    const double regTerm = 0.5 * dot(ctx, g, g1, g2, v1, v2);
    if (model.deformation == kIncompressible) projectDivFree(ctx, g, b, b + N, b, b + N);
    axpby(ctx, N, 1.0, b, 1.0, g1);
    axpby(ctx, N, 1.0, b + N, 1.0, g2);
    scalars[0] = mismatch + regTerm;
    scalars[1] = mismatch;
    scalars[2] = regTerm;
}

}  // namespace vrg
