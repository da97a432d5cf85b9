// Semi-Lagrangian transport kernels (K3 trace, K4 state step, K5 continuity step, K6
// incremental-state step) and the device transport::Solver.
#include <cmath>
#include <cstring>
#include <string>

#include <cstdlib>

#include "epilogues.cuh"
#include "evalband.cuh"
#include "transport.cuh"

namespace vrg {

// ------------------------------------------------------------------------------ epilogues
namespace {

// Star points x* = x - sgn*ht*v (src/transport.cpp:73-74), no FMA.
__global__ void k_star(const double* __restrict__ v1, const double* __restrict__ v2, int n1, int n2, int pairs,
                       double h1, double h2, double sgnHt, double* x1, double* x2) {
    const std::size_t N = static_cast<std::size_t>(n1) * n2 * pairs;
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const std::size_t row = p / n2;
    const int i1 = static_cast<int>(row % n1), i2 = static_cast<int>(p - row * n2);
    const double c1 = __dadd_rn(-kPi, __dmul_rn(h1, static_cast<double>(i1)));
    const double c2 = __dadd_rn(-kPi, __dmul_rn(h2, static_cast<double>(i2)));
    x1[p] = __dsub_rn(c1, __dmul_rn(sgnHt, v1[p]));
    x2[p] = __dsub_rn(c2, __dmul_rn(sgnHt, v2[p]));
}

// Maximum of |field| per pair into the step's guard slots (same block layout as k_evaluate).
__global__ void __launch_bounds__(kEvalBlock) k_fieldmax(const double* __restrict__ f, std::size_t N, double* partial,
                                                         unsigned blocksPer) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double g = 0.0;
    if (p < N) g = fmax(0.0, fabs(f[p]));
    __shared__ double red[kEvalBlock / 32];
    for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = g;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int w = 1; w < kEvalBlock / 32; ++w) m = fmax(m, red[w]);
        guardMax(partial + blockIdx.x / blocksPer, m);
    }
}

__global__ void k_ones(std::size_t N, double* y) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p < N) y[p] = 1.0;
}

}  // namespace

void launchFieldMax(Ctx& ctx, const GridDims& g, const double* f, double* partial) {
    {
        LaunchScope ls_(ctx, "k_fieldmax");
        k_fieldmax<<<evalBlocks(g), kEvalBlock, 0, ctx.stream>>>(f, g.points(), partial, evalBlocksPer(g));
    }
    VRG_LAUNCH_CHECK();
}

// ------------------------------------------------------------------------------ guard log
thread_local bool g_collectGuards = false;

void GuardLog::ensure(int nsteps, const GridDims& g) {
    if (nsteps <= steps && g.pairs == pairs) return;
    if (g.pairs > 1 && g.pointsPer() % kEvalBlock != 0)
        throw NotSupported("batched pairs: n1 * n2 must be a multiple of 256");
    steps = nsteps;
    pairs = g.pairs;
    buf.alloc(bytes());
}

void GuardLog::reset(Ctx& ctx) { VRG_CUDA(cudaMemsetAsync(buf.d(), 0, bytes(), ctx.stream)); }

void GuardLog::check(Ctx& ctx, const char* eq, int nt, bool forward, bool guard, int thresholdStep) {
    double* host = static_cast<double*>(ctx.hostStage(bytes()));
    VRG_CUDA(cudaMemcpyAsync(host, buf.d(), bytes(), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    const double* mx = host;
    const unsigned* fl = reinterpret_cast<const unsigned*>(host + static_cast<std::size_t>(steps) * pairs);
    if (pairs == 1 && !g_collectGuards) {
        checkHost(mx, fl, eq, nt, forward, guard, thresholdStep);
        return;
    }
    // a batch: every pair's verdict, nothing thrown (the non-finite flag is shared by the batch)
    pairStatus.assign(pairs, 0);
    pairError.assign(pairs, std::string());
    std::vector<double> m1(nt + 1);
    for (int k = 0; k < pairs; ++k) {
        for (int s = 0; s <= nt; ++s) m1[s] = mx[static_cast<std::size_t>(s) * pairs + k];
        try {
            checkHost(m1.data(), fl, eq, nt, forward, guard, thresholdStep);
        } catch (const BlowupError& e) {
            pairStatus[k] = kBlowup;
            pairError[k] = e.what();
        } catch (const InvalidArgument& e) {
            pairStatus[k] = kInvalidArgument;
            pairError[k] = e.what();
        }
    }
    if (!g_collectGuards)  // a batched operator used on its own: the first pair's error throws
        for (int k = 0; k < pairs; ++k) {
            if (pairStatus[k] == kBlowup) throw BlowupError(pairError[k]);
            if (pairStatus[k]) throw InvalidArgument(pairError[k]);
        }
}

void GuardLog::checkHost(const double* mx, const unsigned* fl, const char* eq, int nt, bool forward, bool guard,
                         int thresholdStep) {
    const double threshold = kBlowupFactor * mx[thresholdStep];
    for (int s = 1; s <= nt; ++s) {
        const int j = forward ? s : nt + 1 - s;    // step label (transport.cpp:221, 235)
        const int in = forward ? j - 1 : j;         // frame fed to the prefilter
        const int out = forward ? j : j - 1;        // frame produced
        if (fl[in]) throw InvalidArgument("prefilter: non-finite value");
        if (guard && mx[out] > threshold)
            throw BlowupError(std::string(eq) + " solve exceeded the blow-up guard at step " + std::to_string(j));
    }
}

// ------------------------------------------------------------------------------ helpers
int deriveSteps(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double cfl) {
    if (!(cfl > 0.0) || cfl > 20.0) throw InvalidArgument("cfl must lie in (0, 20]");
    const double m1 = normLinf(ctx, g.points(), v1);
    const double m2 = normLinf(ctx, g.points(), v2);
    double ratio = 0.0;
    ratio = std::max(ratio, m1 / (cfl * g.h1()));
    ratio = std::max(ratio, m2 / (cfl * g.h2()));
    const int nt = static_cast<int>(std::ceil(ratio));
    return std::max(2, nt);
}

void launchTrace(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* cv1,
                 const double* cv2, double ht, int dir, double* x1, double* x2) {
    const double sgn = dir == kForward ? 1.0 : -1.0;
    // star points staged in the output buffers, then overwritten by the departure points
    // (each thread reads its own star point before writing its departure point)
    double* s1 = ctx.scratchBuf(10, sizeof(double) * g.points());
    double* s2 = ctx.scratchBuf(11, sizeof(double) * g.points());
    {
        LaunchScope ls_(ctx, "k_star");
        k_star<<<grid1d(g.points(), 256), 256, 0, ctx.stream>>>(v1, v2, g.n1, g.n2, g.pairs, g.h1(), g.h2(), sgn * ht,
                                                                s1, s2);
    }
    VRG_LAUNCH_CHECK();
    EpiTrace epi{nullptr, v1, v2, x1, x2, g.n1, g.n2, g.h1(), g.h2(), sgn * 0.5 * ht};
    launchEvaluate<2>(ctx, g, CoeffSet<2>{{cv1, cv2}}, s1, s2, epi);
}

// ------------------------------------------------------------------------------ Solver
Solver::Solver(Ctx& c, const GridDims& gd, const double* vv1, const double* vv2, int steps)
    : ctx(c), g(gd), nt(steps), ht(1.0 / steps) {
    checkGrid(g.n1, g.n2);
    if (steps < 1) throw InvalidArgument("TimeGrid: nt must be >= 1");
    v.alloc(sizeof(double) * 2 * g.points());
    copy(ctx, g.points(), vv1, v.d());
    copy(ctx, g.points(), vv2, v.d() + g.points());
    if (anyNonFinite(ctx, 2 * g.points(), v.d())) throw InvalidArgument("transport velocity: non-finite value");
    coef_.alloc(sizeof(double) * paddedTotal(g));
    tmp_.alloc(sizeof(double) * 2 * g.points());
    log.ensure(nt + 1, g);
}

// Band path for the SL time loops (evalband.cuh) wherever the grid allows it: each step is the
// gather + epilogue + the next prefilter's row pass in one kernel, then the column pass; same
// arithmetic as prefilter + evaluate (the plain 3-kernel step, the generic-grid path).
bool Solver::bandPath() const { return bandFusable(g) && colPassFusable(g) && bandCellsFit(g); }

double* Solver::coef() { return coef_.d(); }
double* Solver::tmp() { return tmp_.d(); }

const double* Solver::departure(int dir) {
    if (!haveX_[dir]) {
        if (!haveCv_) {
            // both components in one batch (v is contiguous [v1 | v2])
            cv_.alloc(sizeof(double) * 2 * paddedTotal(g));
            launchPrefilterBatch(ctx, g, v1(), g.points(), 2, cv_.d(), paddedTotal(g), tmp_.d(), nullptr);
            haveCv_ = true;
        }
        X_[dir].alloc(sizeof(double) * 2 * g.points());
        launchTrace(ctx, g, v1(), v2(), cv_.d(), cv_.d() + paddedTotal(g), ht, dir, X_[dir].d(),
                    X_[dir].d() + g.points());
        ctx.interps += 2;  // traceCharacteristics evaluates both components (transport.cpp:77-78)
        haveX_[dir] = true;
    }
    return X_[dir].d();
}

const Cell* Solver::cells(int dir) {
    if (!haveCells_[dir]) {
        const double* X = departure(dir);
        cells_[dir].alloc(sizeof(Cell) * 2 * g.points());
        launchPackCells(ctx, g, X, cells_[dir].as<Cell>());
        haveCells_[dir] = true;
    }
    return cells_[dir].as<Cell>();
}

const double* Solver::divVelocity() {
    if (!haveDivv_) {
        divv_.alloc(sizeof(double) * g.points());
        divergence(ctx, g, v1(), v2(), divv_.d());  // counts 3 FFTs
        haveDivv_ = true;
    }
    return divv_.d();
}

const double* Solver::divVelocityAtDeparture(int dir) {
    if (!haveDvDep_[dir]) {
        const double* dv = divVelocity();
        const double* X = departure(dir);
        dvDep_[dir].alloc(sizeof(double) * g.points());
        launchPrefilter(ctx, g, dv, coef_.d(), tmp_.d(), nullptr);
        launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef_.d()}}, X, X + g.points(), EpiStore1{nullptr, dvDep_[dir].d()});
        ctx.interps += 1;
        haveDvDep_[dir] = true;
    }
    return dvDep_[dir].d();
}

void Solver::continuityStep(const double* u, double* out, int dir, double* guardPartial, unsigned* flag) {
    const double* X = departure(dir);
    const double* dv = divVelocity();
    const double* dvd = divVelocityAtDeparture(dir);
    launchPrefilter(ctx, g, u, coef_.d(), tmp_.d(), flag);
    EpiContinuity epi{guardPartial ? guardPartial : log.partial(0), dvd, dv, ht, out};
    launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef_.d()}}, X, X + g.points(), epi, true);
    ctx.interps += 1;
}

// Band form of a continuity loop (slAdjoint, transport.cpp:229-241, along kBackward; the SL
// Jacobian, transport.cpp:456-464, along kForward): step j writes its result to dst(j) (j = nt
// down to 1) and row-filters it for the next step; the prefilter input check of the next step
// (flag j-1) is done by step j's kernel, as in the plain path's prefilter.
template <class DstFn>
void Solver::continuityBand(const double* lam1, DstFn dst, int dir) {
    const double* X = departure(dir);
    const Cell* C = cells(dir);
    const double* dv = divVelocity();
    const double* dvd = divVelocityAtDeparture(dir);
    const std::size_t N = g.points();
    (void)X;
    launchPrefilter(ctx, g, lam1, coef_.d(), tmp_.d(), log.flag(nt));
    for (int j = nt; j >= 1; --j) {
        const EpiContinuity epi{log.partial(j - 1), dvd, dv, ht, dst(j)};
        if (j == 1) {  // the last step: no row pass
            launchEvalBand<EpiContinuity, true>(ctx, g, CoeffSet<1>{{coef_.d()}}, C, C + N, epi, nullptr, nullptr);
        } else {
            launchEvalBand<EpiContinuity, true>(ctx, g, CoeffSet<1>{{coef_.d()}}, C, C + N, epi, tmp_.d(),
                                                log.flag(j - 1));
            launchPrefilterCols(ctx, g, tmp_.d(), coef_.d());
        }
    }
    ctx.interps += nt;
}

void Solver::state(const double* m0, double* traj, bool guard) {
    NvtxRange nv_("Solver::solveState");
    const double* X = departure(kForward);
    const Cell* C = bandPath() ? cells(kForward) : nullptr;
    const std::size_t N = g.points();
    log.reset(ctx);
    copy(ctx, N, m0, traj);
    launchFieldMax(ctx, g, traj, log.partial(0));
    if (bandPath()) {
        launchPrefilter(ctx, g, traj, coef_.d(), tmp_.d(), log.flag(0));
        for (int j = 1; j <= nt; ++j) {
            const EpiStateStep epi{log.partial(j), traj + j * N};
            if (j == nt) {  // the last step: no row pass
                launchEvalBand<EpiStateStep, true>(ctx, g, CoeffSet<1>{{coef_.d()}}, C, C + N, epi, nullptr, nullptr);
            } else {
                launchEvalBand<EpiStateStep, true>(ctx, g, CoeffSet<1>{{coef_.d()}}, C, C + N, epi, tmp_.d(),
                                                   log.flag(j));
                launchPrefilterCols(ctx, g, tmp_.d(), coef_.d());
            }
        }
    } else {
        for (int j = 1; j <= nt; ++j) {
            launchPrefilter(ctx, g, traj + (j - 1) * N, coef_.d(), tmp_.d(), log.flag(j - 1));
            launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef_.d()}}, X, X + N, EpiStateStep{log.partial(j), traj + j * N},
                              true);
        }
    }
    ctx.interps += nt;
    log.check(ctx, "state", nt, true, guard, 0);
}

void Solver::stateFinal(const double* m0, double* out) {
    NvtxRange nv_("Solver::solveStateFinal");
    const double* X = departure(kForward);
    const Cell* C = bandPath() ? cells(kForward) : nullptr;
    const std::size_t N = g.points();
    double* buf = ctx.scratchBuf(12, sizeof(double) * 2 * N);
    log.reset(ctx);
    launchFieldMax(ctx, g, m0, log.partial(0));
    if (bandPath()) {
        launchPrefilter(ctx, g, m0, coef_.d(), tmp_.d(), log.flag(0));
        for (int j = 1; j <= nt; ++j) {
            double* dst = (j == nt) ? out : buf + (j % 2) * N;
            const EpiStateStep epi{log.partial(j), dst};
            if (j == nt) {  // the last step: no row pass
                launchEvalBand<EpiStateStep, true>(ctx, g, CoeffSet<1>{{coef_.d()}}, C, C + N, epi, nullptr, nullptr);
            } else {
                launchEvalBand<EpiStateStep, true>(ctx, g, CoeffSet<1>{{coef_.d()}}, C, C + N, epi, tmp_.d(),
                                                   log.flag(j));
                launchPrefilterCols(ctx, g, tmp_.d(), coef_.d());
            }
        }
    } else {
        const double* cur = m0;
        for (int j = 1; j <= nt; ++j) {
            double* dst = (j == nt) ? out : buf + (j % 2) * N;
            launchPrefilter(ctx, g, cur, coef_.d(), tmp_.d(), log.flag(j - 1));
            launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef_.d()}}, X, X + N, EpiStateStep{log.partial(j), dst}, true);
            cur = dst;
        }
    }
    ctx.interps += nt;
    log.check(ctx, "state", nt, true, true, 0);
}

void Solver::adjoint(const double* lam1, double* traj, bool guard) {
    NvtxRange nv_("Solver::solveAdjoint");
    const std::size_t N = g.points();
    log.reset(ctx);
    copy(ctx, N, lam1, traj + nt * N);
    launchFieldMax(ctx, g, traj + nt * N, log.partial(nt));
    if (bandPath()) {
        continuityBand(traj + nt * N, [&](int j) { return traj + (j - 1) * N; }, kBackward);
    } else {
        for (int j = nt; j >= 1; --j)
            continuityStep(traj + j * N, traj + (j - 1) * N, kBackward, log.partial(j - 1), log.flag(j));
    }
    log.check(ctx, "adjoint", nt, false, guard, nt);
}

void Solver::adjointFinal(const double* lam1, double* out) {
    NvtxRange nv_("Solver::solveAdjointFinal");
    const std::size_t N = g.points();
    double* buf = ctx.scratchBuf(12, sizeof(double) * 2 * N);
    log.reset(ctx);
    launchFieldMax(ctx, g, lam1, log.partial(nt));
    if (bandPath()) {
        continuityBand(lam1, [&](int j) { return (j == 1) ? out : buf + (j % 2) * N; }, kBackward);
    } else {
        const double* cur = lam1;
        for (int j = nt; j >= 1; --j) {
            double* dst = (j == 1) ? out : buf + (j % 2) * N;
            continuityStep(cur, dst, kBackward, log.partial(j - 1), log.flag(j));
            cur = dst;
        }
    }
    log.check(ctx, "adjoint", nt, false, true, nt);
}

void Solver::incState(const double* vt1, const double* vt2, const double* stateTraj, double* out) {
    const std::size_t N = g.points();
    const double* X = departure(kForward);
    // vt at departure (2 interps), then per step (grad m_{j-1})_D (2 interps), grad m_j, m~_D
    DBuf work(sizeof(double) * 8 * N);
    double* vtD = work.d();          // [vt1D | vt2D]
    double* gPrev = vtD + 2 * N;     // grad m_{j-1}
    double* gCur = gPrev + 2 * N;    // grad m_j
    double* gD = gCur + 2 * N;       // (grad m_{j-1})_D
    double* c2 = ctx.scratchBuf(13, sizeof(double) * paddedTotal(g));
    launchPrefilter(ctx, g, vt1, coef_.d(), tmp_.d(), nullptr);
    launchPrefilter(ctx, g, vt2, c2, tmp_.d(), nullptr);
    launchEvaluate<2>(ctx, g, CoeffSet<2>{{coef_.d(), c2}}, X, X + N, EpiStore2{nullptr, vtD, vtD + N}, true);
    ctx.interps += 2;
    gradient(ctx, g, stateTraj, gPrev, gPrev + N);
    fill(ctx, N, 0.0, out);
    for (int j = 1; j <= nt; ++j) {
        launchPrefilter(ctx, g, gPrev, coef_.d(), tmp_.d(), nullptr);
        launchPrefilter(ctx, g, gPrev + N, c2, tmp_.d(), nullptr);
        launchEvaluate<2>(ctx, g, CoeffSet<2>{{coef_.d(), c2}}, X, X + N, EpiStore2{nullptr, gD, gD + N}, true);
        gradient(ctx, g, stateTraj + j * N, gCur, gCur + N);
        EpiIncState epi{nullptr, vtD, vtD + N, gD, gD + N, vt1, vt2, gCur, gCur + N, 0.5 * ht, out + j * N};
        if (j == 1) {
            launchPointwise(ctx, g, epi);  // m~_0 = 0
        } else {
            launchPrefilter(ctx, g, out + (j - 1) * N, coef_.d(), tmp_.d(), nullptr);
            launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef_.d()}}, X, X + N, epi, true);
        }
        ctx.interps += 3;
        std::swap(gPrev, gCur);
    }
    ctx.sync();
}

namespace {
// m * v_i per component (hadamard(m, v[i]), divOfProduct of transport.cpp:31-36)
__global__ void k_mul2(std::size_t N, const double* __restrict__ m, const double* __restrict__ v1,
                       const double* __restrict__ v2, double* __restrict__ o1, double* __restrict__ o2) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    o1[p] = m[p] * v1[p];
    o2[p] = m[p] * v2[p];
}
}  // namespace

void Solver::incAdjointFullNewton(const double* vt1, const double* vt2, const double* lt1, const double* adj,
                                  double* traj, double* work, unsigned* flag) {
    const std::size_t N = g.points();
    const double* X = departure(kBackward);
    const double* dv = divVelocity();
    const double* dvd = divVelocityAtDeparture(kBackward);
    double* qCur = work;
    double* qPrev = work + N;
    double* qD = work + 2 * N;
    double* prod = work + 3 * N;  // 2N
    auto divProd = [&](const double* m, double* q) {
        {
            LaunchScope ls_(ctx, "k_mul2");
            k_mul2<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, m, vt1, vt2, prod, prod + N);
        }
        VRG_LAUNCH_CHECK();
        divergence(ctx, g, prod, prod + N, q);
    };
    if (traj + static_cast<std::size_t>(nt) * N != lt1) copy(ctx, N, lt1, traj + static_cast<std::size_t>(nt) * N);
    divProd(adj + static_cast<std::size_t>(nt) * N, qCur);
    for (int j = nt; j >= 1; --j) {
        launchPrefilter(ctx, g, qCur, coef_.d(), tmp_.d(), flag);
        launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef_.d()}}, X, X + N, EpiStore1{nullptr, qD}, true);
        divProd(adj + static_cast<std::size_t>(j - 1) * N, qPrev);
        launchPrefilter(ctx, g, traj + static_cast<std::size_t>(j) * N, coef_.d(), tmp_.d(), flag);
        launchEvaluate<1>(ctx, g, CoeffSet<1>{{coef_.d()}}, X, X + N,
                          EpiContinuityFN{nullptr, dvd, dv, qD, qPrev, ht, traj + static_cast<std::size_t>(j - 1) * N},
                          true);
        ctx.interps += 2;
        std::swap(qCur, qPrev);
    }
}

void Solver::jacobian(double* out) {
    const std::size_t N = g.points();
    double* buf = ctx.scratchBuf(12, sizeof(double) * 2 * N);
    {
        LaunchScope ls_(ctx, "k_ones");
        k_ones<<<grid1d(N, 256), 256, 0, ctx.stream>>>(N, buf);
    }
    VRG_LAUNCH_CHECK();
    log.reset(ctx);  // the steps' guard slots (unchecked: the Jacobian has no guard)
    if (bandPath()) {
        // nt forward continuity steps from 1; the band loop labels them nt .. 1, the last one
        // (label 1) writing out.  The steps read their input from the coefficients, so the
        // intermediate fields (unused) all go to buf, whose ones were prefiltered first.
        continuityBand(buf, [&](int j) { return (j == 1) ? out : buf; }, kForward);
    } else {
        const double* cur = buf;
        for (int j = 1; j <= nt; ++j) {
            double* dst = (j == nt) ? out : buf + (j % 2) * N;
            continuityStep(cur, dst, kForward, log.partial(0), nullptr);
            cur = dst;
        }
    }
    ctx.sync();
}

}  // namespace vrg
