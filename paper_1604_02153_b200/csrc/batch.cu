// Batched registration: P independent image pairs (configs 3 and 5b) solved in lockstep, with
// every transport, spectral and Krylov step of all pairs in the same kernel launches.
//
// The pairs are stacked (GridDims::pairs, common.cuh): a field of the batch is the P pairs'
// n1 x n2 fields one after the other, so the library's Solver / Hessian / spectral operators
// run on all pairs at once (band steps over P * n1 rows, cuFFT with P transforms per field,
// per-pair reductions).  The host driver below is inverse::newtonSolve (newton.cpp:24-159),
// solveKkt (precond.cpp:291-358), pcg (precond.cpp:38-85), applyTwoLevel (precond.cpp:264-289)
// and chebyshevSolve (precond.cpp:180-205) with one scalar state per pair: each pair takes
// exactly the decisions (and arithmetic, reductions included) of its own single-pair solve
// (csrc/precond.cu), and a pair that stops (converged Krylov solve, accepted line-search
// trial, converged Newton iteration) is masked out of the updates while the others go on.
// Coarse two-level operators are built per group of pairs with the same CFL-derived coarse
// step count.  Scope: Gauss-Newton SL with a fixed fine step count (NewtonConfig::ntOverride)
// and the Reg or two-level Chebyshev preconditioner; anything else is NotSupported (the
// per-pair solve covers it).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "batch.cuh"
#include "blas.cuh"
#include "evalband.cuh"
#include "heun.cuh"

namespace vrg {

namespace {

constexpr double kEmaxInflationB = 1.05;  // precond.cpp:18 (kEmaxInflation)

// Per-pair coefficients of a masked update (kernel parameter, no host -> device copy).
struct PairCoef {
    double a[kMaxBatchPairs];
    double b[kMaxBatchPairs];
    unsigned long long mask;
};

// Vectors of a batch: component blocks of P pairs (nPer values each); pair of element i.
__device__ __forceinline__ int pairOf(std::size_t i, std::size_t nPer, int P) {
    return static_cast<int>((i / nPer) % static_cast<std::size_t>(P));
}

// y += a_p x (axpby(a, x, 1, y): fma(x, a, y)), pairs in the mask
__global__ void k_axpy_pairs(std::size_t n, std::size_t nPer, int P, PairCoef c, const double* __restrict__ x,
                             double* y) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int p = pairOf(i, nPer, P);
        if ((c.mask >> p) & 1ull) y[i] = __fma_rn(x[i], c.a[p], y[i]);
    }
}

// out = a_p x + b_p y (lincomb: fma(x, a, y * b)), pairs in the mask
__global__ void k_lincomb_pairs(std::size_t n, std::size_t nPer, int P, PairCoef c, const double* __restrict__ x,
                                const double* __restrict__ y, double* out) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int p = pairOf(i, nPer, P);
        if ((c.mask >> p) & 1ull) out[i] = __fma_rn(x[i], c.a[p], __dmul_rn(y[i], c.b[p]));
    }
}

// chebyshevSolve's fused updates (precond.cu k_cheb_init / k_cheb_step) with per-pair bounds
__global__ void k_cheb_init_pairs(std::size_t n, std::size_t nPer, int P, PairCoef c, const double* __restrict__ rhs,
                                  double* __restrict__ r, double* __restrict__ d, double* __restrict__ x) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double ri = rhs[i];
        r[i] = ri;
        const double di = __fma_rn(ri, c.a[pairOf(i, nPer, P)], __dmul_rn(ri, 0.0));
        d[i] = di;
        x[i] = __fma_rn(di, 1.0, 0.0);
    }
}

__global__ void k_cheb_step_pairs(std::size_t n, std::size_t nPer, int P, PairCoef c, const double* __restrict__ ad,
                                  double* __restrict__ r, double* __restrict__ d, double* __restrict__ x) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int p = pairOf(i, nPer, P);
        const double ri = __fma_rn(ad[i], -1.0, r[i]);
        r[i] = ri;
        const double di = __fma_rn(d[i], c.a[p], __dmul_rn(ri, c.b[p]));
        d[i] = di;
        x[i] = __fma_rn(di, 1.0, x[i]);
    }
}

// non-finite flag per pair (anyNonFinite of each pair's vector)
__global__ void k_nonfinite_pairs(std::size_t n, std::size_t nPer, int P, const double* __restrict__ a,
                                  unsigned* flags) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        if (!isfinite(a[i])) atomicOr(flags + pairOf(i, nPer, P), 1u);
}

double secondsSinceB(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

PairCoef coefOf(const std::vector<double>& a, const std::vector<double>& b, const std::vector<char>& on) {
    PairCoef c{};
    c.mask = 0;
    for (std::size_t k = 0; k < on.size(); ++k) {
        c.a[k] = a.empty() ? 0.0 : a[k];
        c.b[k] = b.empty() ? 0.0 : b[k];
        if (on[k]) c.mask |= 1ull << k;
    }
    return c;
}

void axpyPairs(Ctx& ctx, const GridDims& g, int comps, const PairCoef& c, const double* x, double* y) {
    const std::size_t n = comps * g.points();
    LaunchScope ls_(ctx, "k_axpy_pairs");
    k_axpy_pairs<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, g.pointsPer(), g.pairs, c, x, y);
}

void lincombPairs(Ctx& ctx, const GridDims& g, int comps, const PairCoef& c, const double* x, const double* y,
                  double* out) {
    const std::size_t n = comps * g.points();
    LaunchScope ls_(ctx, "k_lincomb_pairs");
    k_lincomb_pairs<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, g.pointsPer(), g.pairs, c, x, y, out);
}

std::vector<char> nonFinitePairs(Ctx& ctx, const GridDims& g, int comps, const double* a) {
    const std::size_t n = comps * g.points();
    unsigned* flags = reinterpret_cast<unsigned*>(ctx.scratchBuf(215, sizeof(unsigned) * kMaxBatchPairs));
    VRG_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned) * g.pairs, ctx.stream));
    {
        LaunchScope ls_(ctx, "k_nonfinite");
        k_nonfinite_pairs<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, g.pointsPer(), g.pairs, a, flags);
    }
    VRG_LAUNCH_CHECK();
    std::vector<unsigned> h(g.pairs);
    VRG_CUDA(cudaMemcpyAsync(h.data(), flags, sizeof(unsigned) * g.pairs, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    std::vector<char> out(g.pairs);
    for (int k = 0; k < g.pairs; ++k) out[k] = h[k] != 0;
    return out;
}

std::vector<double> dotPairs(Ctx& ctx, const GridDims& g, const double* a, const double* b, bool vector) {
    const std::size_t N = g.points();
    std::vector<double> out(g.pairs);
    readPairs(ctx,
              launchDotPairs(ctx, g, a, b, vector ? a + N : nullptr, vector ? b + N : nullptr, g.h1() * g.h2(), 0),
              g.pairs, out.data());
    return out;
}

std::vector<double> linfPairs(Ctx& ctx, const GridDims& g, const double* a, bool vector) {
    std::vector<double> out(g.pairs);
    readPairs(ctx, launchMaxAbsPairs(ctx, g, a, vector ? a + g.points() : nullptr, 0), g.pairs, out.data());
    return out;
}

// Counter bookkeeping: the library's logical counters advance once per batched operation (one
// operation of each pair); the delta goes to the pairs that took part in it.
struct Counts {
    long long ffts = 0, interps = 0;
};
struct CountScope {
    Ctx& ctx;
    long long f0, i0;
    explicit CountScope(Ctx& c) : ctx(c), f0(c.ffts), i0(c.interps) {}
    void to(std::vector<Counts>& per, const std::vector<int>& ids, const std::vector<char>& on) {
        const long long df = ctx.ffts - f0, di = ctx.interps - i0;
        for (std::size_t k = 0; k < on.size(); ++k)
            if (on[k]) {
                per[ids[k]].ffts += df;
                per[ids[k]].interps += di;
            }
        skip();
    }
    // work whose counts were attributed elsewhere (nested scopes)
    void skip() {
        f0 = ctx.ffts;
        i0 = ctx.interps;
    }
};

}  // namespace

// Copies pair slots between two batches of `fields` fields (fields of srcP / dstP pairs, nPer
// values per pair): dst pair map[k].second <- src pair map[k].first.
void copyPairs(Ctx& ctx, const double* src, int srcP, double* dst, int dstP, std::size_t nPer, int fields,
               const std::vector<std::pair<int, int>>& map) {
    for (const auto& m : map)
        VRG_CUDA(cudaMemcpy2DAsync(dst + m.second * nPer, sizeof(double) * nPer * dstP, src + m.first * nPer,
                                   sizeof(double) * nPer * srcP, sizeof(double) * nPer, fields,
                                   cudaMemcpyDeviceToDevice, ctx.stream));
}

// evaluateObjective / evaluateGradient (inverse.cpp:96-148) for a batch, compressible or
// incompressible SL: per-pair scalars [objective, mismatch, regTerm, 0] and guard verdicts.
// A pair whose velocity is not finite gets the status of the Solver's check (transport.cpp:
// velocity validation) and is transported with v = 0 so that the other pairs go on.
std::vector<int> saneVelocities(Ctx& ctx, const GridDims& g, const double*& v, DBuf& fixed) {
    const auto bad = nonFinitePairs(ctx, g, 2, v);
    std::vector<int> status(g.pairs, 0);
    std::vector<std::pair<int, int>> keep;
    bool any = false;
    for (int k = 0; k < g.pairs; ++k) {
        if (bad[k]) {
            status[k] = kInvalidArgument;
            any = true;
        } else {
            keep.push_back({k, k});
        }
    }
    if (!any) return status;
    fixed.alloc(sizeof(double) * 2 * g.points());
    fill(ctx, 2 * g.points(), 0.0, fixed.d());
    copyPairs(ctx, v, g.pairs, fixed.d(), g.pairs, g.pointsPer(), 2, keep);
    v = fixed.d();
    return status;
}

void evaluateObjectiveBatch(Ctx& ctx, const GridDims& g, const double* v, const double* mR, const double* mT,
                            const Model& model, int nt, std::vector<double>& scalars, double* st,
                            std::vector<int>& status) {
    const std::size_t N = g.points();
    DBuf fixed;
    const auto vst = saneVelocities(ctx, g, v, fixed);
    {
        Solver solver(ctx, g, v, v + N, nt);
        solver.state(mT, st, true);
        status = solver.log.pairStatus;
    }
    for (int k = 0; k < g.pairs; ++k)
        if (vst[k]) status[k] = vst[k];
    double* resid = ctx.scratchBuf(21, sizeof(double) * N);
    lincomb(ctx, N, 1.0, st + nt * N, -1.0, mR, resid);
    const auto mis = dotPairs(ctx, g, resid, resid, false);
    Weights w(g, model.norm);
    double* reg = ctx.scratchBuf(22, sizeof(double) * 2 * N);
    applyRealSymbol(ctx, g, v, v + N, reg, reg + N, w.regSymbol(model.betaV));
    const auto rt = dotPairs(ctx, g, reg, v, true);
    scalars.assign(4 * g.pairs, 0.0);
    for (int k = 0; k < g.pairs; ++k) {
        const double mismatch = 0.5 * mis[k], regTerm = 0.5 * rt[k];
        scalars[4 * k] = mismatch + regTerm + 0.0;
        scalars[4 * k + 1] = mismatch;
        scalars[4 * k + 2] = regTerm;
    }
}

void evaluateGradientBatch(Ctx& ctx, const GridDims& g, const double* v, const double* mR, const double* mT,
                           const Model& model, int nt, double* grad, std::vector<double>& scalars, double* st,
                           double* ad, bool reuseState, double* gradTraj, std::vector<int>& status) {
    const std::size_t N = g.points();
    double* b = ctx.scratchBuf(23, sizeof(double) * 2 * N);
    double* resid = ctx.scratchBuf(21, sizeof(double) * N);
    DBuf fixed;
    status = saneVelocities(ctx, g, v, fixed);
    const std::vector<int> vst = status;
    std::vector<double> mis;
    {
        Solver solver(ctx, g, v, v + N, nt);
        if (!reuseState) {
            solver.state(mT, st, true);
            for (int k = 0; k < g.pairs; ++k)
                if (!status[k]) status[k] = solver.log.pairStatus[k];
        }
        lincomb(ctx, N, 1.0, st + nt * N, -1.0, mR, resid);
        mis = dotPairs(ctx, g, resid, resid, false);
        lincomb(ctx, N, -1.0, resid, 0.0, resid, resid);  // lambda1 = -1.0 * resid
        solver.adjoint(resid, ad, true);
        for (int k = 0; k < g.pairs; ++k)
            if (!status[k]) status[k] = solver.log.pairStatus[k];
        bodyForce(ctx, g, nt, st, ad, b, b + N, gradTraj);
    }
    Weights w(g, model.norm);
    applyRealSymbol(ctx, g, v, v + N, grad, grad + N, w.regSymbol(model.betaV));
    const auto rt = dotPairs(ctx, g, grad, v, true);
    if (model.deformation == kIncompressible) projectDivFree(ctx, g, b, b + N, b, b + N);
    axpby(ctx, N, 1.0, b, 1.0, grad);
    axpby(ctx, N, 1.0, b + N, 1.0, grad + N);
    scalars.assign(4 * g.pairs, 0.0);
    for (int k = 0; k < g.pairs; ++k) {
        const double mismatch = 0.5 * mis[k], regTerm = 0.5 * rt[k];
        scalars[4 * k] = mismatch + regTerm + 0.0;
        scalars[4 * k + 1] = mismatch;
        scalars[4 * k + 2] = regTerm;
    }
}

namespace {

// The coarse level of the two-level preconditioner for a batch (CoarseOperator per group of
// pairs with the same coarse step count, precond.cpp:207-240).
struct CoarseGroup {
    int nt = 0;
    std::vector<int> members;  // slots of the active batch
    GridDims g;
    DBuf mRc, mTc, vc, rc, sc;
    std::unique_ptr<Hessian> hess;
};

struct BatchKkt {
    Ctx& ctx;
    GridDims g, gc;
    const Model& model;
    const PrecondChoice& choice;
    Hessian& fine;
    std::vector<int>& ids;              // slot -> pair id
    std::vector<Counts>& counts;        // per pair id
    std::vector<double>& eMax;          // per pair id
    double eMin = 1.0;
    std::vector<int>& status;           // per pair id (0 ok)
    std::vector<std::string>& errors;   // per pair id
    const double* mR;
    const double* mT;
    const double* v;
    std::vector<CoarseGroup> groups;
    DBuf rcAll, scAll;

    BatchKkt(Ctx& c, const GridDims& gd, const Model& m, const PrecondChoice& ch, Hessian& h, std::vector<int>& id,
             std::vector<Counts>& cnt, std::vector<double>& em, std::vector<int>& st, std::vector<std::string>& er,
             const double* r, const double* t, const double* vv)
        : ctx(c), g(gd), gc(gd.n1 / 2, gd.n2 / 2, gd.pairs), model(m), choice(ch), fine(h), ids(id), counts(cnt),
          eMax(em), status(st), errors(er), mR(r), mT(t), v(vv) {}

    void fail(int slot, int code, const std::string& msg) {
        if (!status[ids[slot]]) {
            status[ids[slot]] = code;
            errors[ids[slot]] = msg;
        }
    }

    // restrictProblem + CoarseOperator per group (precond.cpp:163-171, 207-240)
    void buildCoarse(const std::vector<char>& on) {
        const int P = g.pairs;
        const std::size_t Nc = gc.points(), Ncp = gc.pointsPer();
        DBuf mRa(sizeof(double) * Nc), mTa(sizeof(double) * Nc), va(sizeof(double) * 2 * Nc);
        CountScope cs(ctx);
        resample(ctx, g, mR, gc, mRa.d());
        resample(ctx, g, mT, gc, mTa.d());
        resample(ctx, g, v, gc, va.d());
        resample(ctx, g, v + g.points(), gc, va.d() + Nc);
        cs.to(counts, ids, on);
        // coarse nt per pair (deriveSteps, transport.cpp:44-58, CFL 5)
        const auto m1 = linfPairs(ctx, gc, va.d(), false);
        const auto m2 = linfPairs(ctx, gc, va.d() + Nc, false);
        std::map<int, std::vector<int>> byNt;
        for (int k = 0; k < P; ++k) {
            if (!on[k]) continue;
            double ratio = 0.0;
            ratio = std::max(ratio, m1[k] / (kCoarseCfl * gc.h1()));
            ratio = std::max(ratio, m2[k] / (kCoarseCfl * gc.h2()));
            byNt[std::max(2, static_cast<int>(std::ceil(ratio)))].push_back(k);
        }
        rcAll.alloc(sizeof(double) * 2 * Nc);
        scAll.alloc(sizeof(double) * 2 * Nc);
        Model cm = model;
        cm.scheme = kSchemeSL;
        for (auto& kv : byNt) {
            CoarseGroup grp;
            grp.nt = kv.first;
            grp.members = kv.second;
            const int Pg = static_cast<int>(grp.members.size());
            grp.g = GridDims(gc.n1, gc.n2, Pg);
            std::vector<std::pair<int, int>> map;
            for (int j = 0; j < Pg; ++j) map.push_back({grp.members[j], j});
            grp.mRc.alloc(sizeof(double) * grp.g.points());
            grp.mTc.alloc(sizeof(double) * grp.g.points());
            grp.vc.alloc(sizeof(double) * 2 * grp.g.points());
            grp.rc.alloc(sizeof(double) * 2 * grp.g.points());
            grp.sc.alloc(sizeof(double) * 2 * grp.g.points());
            copyPairs(ctx, mRa.d(), P, grp.mRc.d(), Pg, Ncp, 1, map);
            copyPairs(ctx, mTa.d(), P, grp.mTc.d(), Pg, Ncp, 1, map);
            copyPairs(ctx, va.d(), P, grp.vc.d(), Pg, Ncp, 2, map);
            std::vector<char> gon(P, 0);
            for (int k : grp.members) gon[k] = 1;
            CountScope gs(ctx);
            grp.hess = std::make_unique<Hessian>(ctx, grp.g, grp.vc.d(), grp.vc.d() + grp.g.points(), grp.mRc.d(),
                                                 grp.mTc.d(), cm, grp.nt, nullptr);
            gs.to(counts, ids, gon);
            for (int j = 0; j < Pg; ++j)
                if (grp.hess->pairStatus[j]) fail(grp.members[j], grp.hess->pairStatus[j], grp.hess->pairError[j]);
            groups.push_back(std::move(grp));
        }
    }

    // applyTwoLevel (precond.cpp:264-289) for the pairs in `on`; z = r for the others' slots is
    // irrelevant (masked by the caller)
    void twoLevel(const double* r, double* z, const std::vector<char>& on) {
        const int P = g.pairs;
        const std::size_t N = g.points(), Nc = gc.points(), Ncp = gc.pointsPer();
        cplx* R = specScratch(ctx, g, 5, 2);
        cplx* C = specScratch(ctx, gc, 6, 2);
        CountScope cs(ctx);
        restrictLow(ctx, g, gc, r, R, C, rcAll.d(), static_cast<double>(Nc) / static_cast<double>(N));
        for (auto& grp : groups) {
            const int Pg = grp.g.pairs;
            std::vector<std::pair<int, int>> in, out;
            std::vector<char> gon(P, 0);
            bool any = false;
            for (int j = 0; j < Pg; ++j) {
                in.push_back({grp.members[j], j});
                out.push_back({j, grp.members[j]});
                gon[grp.members[j]] = on[grp.members[j]];
                any |= on[grp.members[j]] != 0;
            }
            if (!any) continue;
            copyPairs(ctx, rcAll.d(), P, grp.rc.d(), Pg, Ncp, 2, in);
            CountScope gs(ctx);
            grp.hess->beginDeferredGuards(choice.chebIters);
            chebyshev(grp, gon);
            grp.hess->endDeferredGuards();
            gs.to(counts, ids, gon);
            for (int j = 0; j < Pg; ++j)
                if (gon[grp.members[j]] && grp.hess->pairStatus[j])
                    fail(grp.members[j], grp.hess->pairStatus[j], grp.hess->pairError[j]);
            copyPairs(ctx, grp.sc.d(), Pg, scAll.d(), P, Ncp, 2, out);
        }
        cs.skip();       // the groups' counts went to their pairs
        ctx.ffts += 12;  // cutoff Low/High (8) + restrict (4), as applyTwoLevel counts
        const auto bad = nonFinitePairs(ctx, gc, 2, scAll.d());
        prolongAddHigh(ctx, g, gc, scAll.d(), C, R, z, static_cast<double>(N) / static_cast<double>(Nc));
        ctx.ffts += 4;
        cs.to(counts, ids, on);
        std::vector<std::pair<int, int>> fb;
        for (int k = 0; k < P; ++k)
            if (on[k] && bad[k]) {
                std::fprintf(stderr, "precond: coarse solve diverged, falling back to identity\n");
                fb.push_back({k, k});
            }
        if (!fb.empty()) copyPairs(ctx, r, P, z, P, g.pointsPer(), 2, fb);
    }

    // chebyshevSolve (precond.cpp:180-205) on a group, per-pair bounds [1, 1.05 eMax]
    void chebyshev(CoarseGroup& grp, const std::vector<char>& gon) {
        const GridDims& gg = grp.g;
        const int Pg = gg.pairs;
        const std::size_t n = 2 * gg.points();
        const int k = choice.chebIters;
        std::vector<double> theta(Pg), delta(Pg), sigma(Pg), rho(Pg), inv(Pg);
        for (int j = 0; j < Pg; ++j) {
            const double eMinJ = eMin, eMaxJ = kEmaxInflationB * eMax[ids[grp.members[j]]];
            if (!(eMaxJ > eMinJ) || !(eMinJ > 0.0)) throw InvalidArgument("chebyshevSolve: need eMax > eMin > 0");
            theta[j] = 0.5 * (eMaxJ + eMinJ);
            delta[j] = 0.5 * (eMaxJ - eMinJ);
            sigma[j] = theta[j] / delta[j];
            rho[j] = 1.0 / sigma[j];
            inv[j] = 1.0 / theta[j];
        }
        double* r = ctx.scratchBuf(220, sizeof(double) * n);
        double* d = ctx.scratchBuf(221, sizeof(double) * n);
        double* ad = ctx.scratchBuf(222, sizeof(double) * n);
        double* x = grp.sc.d();
        std::vector<char> all(Pg, 1);
        {
            LaunchScope ls_(ctx, "k_cheb_init");
            k_cheb_init_pairs<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, gg.pointsPer(), Pg, coefOf(inv, {}, all),
                                                                          grp.rc.d(), r, d, x);
        }
        VRG_LAUNCH_CHECK();
        std::vector<double> c1(Pg), c2(Pg);
        for (int it = 1; it <= k; ++it) {
            grp.hess->applySplit(d, d + gg.points(), ad, ad + gg.points());
            if (it == k) break;
            for (int j = 0; j < Pg; ++j) {
                const double rhoNew = 1.0 / (2.0 * sigma[j] - rho[j]);
                c1[j] = rhoNew * rho[j];
                c2[j] = 2.0 * rhoNew / delta[j];
                rho[j] = rhoNew;
            }
            LaunchScope ls_(ctx, "k_cheb_step");
            k_cheb_step_pairs<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, gg.pointsPer(), Pg, coefOf(c1, c2, all),
                                                                          ad, r, d, x);
        }
        VRG_LAUNCH_CHECK();
        (void)gon;
    }

    struct PcgState {
        int iterations = 0;
        bool converged = false, negativeCurvature = false, indefinite = false, done = false;
        double relResidual = 0.0;
    };

    // pcg (precond.cpp:38-85; csrc/precond.cu pcg, M branch) for the pairs in `on`
    std::vector<PcgState> pcgBatch(const double* b, const std::vector<double>& tol, int maxIter, bool useM,
                                   const std::vector<char>& on, double* x) {
        const int P = g.pairs;
        const std::size_t N = g.points(), n = 2 * N;
        double* r = ctx.scratchBuf(230, sizeof(double) * n);
        double* z = useM ? ctx.scratchBuf(231, sizeof(double) * n) : r;
        double* p = ctx.scratchBuf(232, sizeof(double) * n);
        double* ap = ctx.scratchBuf(233, sizeof(double) * n);
        std::vector<PcgState> st(P);
        std::vector<char> act = on;
        std::vector<double> ones(P, 1.0);
        fill(ctx, n, 0.0, x);  // every pair's slots; the pairs outside `on` are not used
        copy(ctx, n, b, r);
        if (useM) twoLevel(r, z, act);  // attributes its own counts
        CountScope cs(ctx);
        auto rz = dotPairs(ctx, g, r, z, true);
        std::vector<double> norm0(P, 0.0);
        for (int k = 0; k < P; ++k) {
            if (!act[k]) continue;
            if (rz[k] < 0.0 || !std::isfinite(rz[k])) {
                st[k].indefinite = true;
                act[k] = 0;
                continue;
            }
            norm0[k] = std::sqrt(std::max(rz[k], 0.0));
            if (!(norm0[k] > 0.0)) {
                st[k].converged = true;
                act[k] = 0;
            }
        }
        copy(ctx, n, z, p);
        for (int it = 0; it < maxIter; ++it) {
            bool any = false;
            for (int k = 0; k < P; ++k) any |= act[k] != 0;
            if (!any) break;
            fine.applySplit(p, p + N, ap, ap + N);
            cs.to(counts, ids, act);
            for (int k = 0; k < P; ++k)
                if (act[k] && fine.pairStatus[k]) {
                    fail(k, fine.pairStatus[k], fine.pairError[k]);
                    act[k] = 0;
                    st[k].done = true;
                }
            const auto pAp = dotPairs(ctx, g, p, ap, true);
            std::vector<double> alpha(P, 0.0), nalpha(P, 0.0);
            for (int k = 0; k < P; ++k) {
                if (!act[k]) continue;
                if (!(pAp[k] > 0.0)) {
                    st[k].negativeCurvature = true;
                    st[k].relResidual = std::sqrt(std::max(rz[k], 0.0)) / norm0[k];
                    act[k] = 0;
                    continue;
                }
                alpha[k] = rz[k] / pAp[k];
                nalpha[k] = -alpha[k];
            }
            axpyPairs(ctx, g, 2, coefOf(alpha, {}, act), p, x);
            axpyPairs(ctx, g, 2, coefOf(nalpha, {}, act), ap, r);
            cs.to(counts, ids, act);
            if (useM) twoLevel(r, z, act);
            cs.skip();
            const auto rzNew = dotPairs(ctx, g, r, z, true);
            std::vector<double> beta(P, 0.0);
            for (int k = 0; k < P; ++k) {
                if (!act[k]) continue;
                st[k].iterations = it + 1;
                if (rzNew[k] < 0.0 || !std::isfinite(rzNew[k])) {
                    st[k].indefinite = true;
                    act[k] = 0;
                    continue;
                }
                st[k].relResidual = std::sqrt(rzNew[k]) / norm0[k];
                if (st[k].relResidual <= tol[k]) {
                    st[k].converged = true;
                    act[k] = 0;
                    continue;
                }
                beta[k] = rzNew[k] / rz[k];
                rz[k] = rzNew[k];
            }
            lincombPairs(ctx, g, 2, coefOf(beta, ones, act), p, z, p);  // p = beta p + 1.0 z
        }
        return st;
    }
};

}  // namespace

// inverse::newtonSolve for a batch; see the file comment.
std::vector<SolverReport> newtonSolveBatch(Ctx& ctx, const GridDims& gAll, const double* mRAll, const double* mTAll,
                                           const Model& model, const NewtonConfig& cfg, const PrecondChoice& pc,
                                           double* vOut, std::vector<int>& status, std::vector<std::string>& errors) {
    NvtxRange nv_("newtonSolveBatch");
    CollectGuardsScope collect_;  // every transport guard reports per pair, nothing thrown
    const int P = gAll.pairs;
    if (P < 1 || P > kMaxBatchPairs) throw InvalidArgument("batched newtonSolve: 1 .. 64 pairs per batch");
    if (model.scheme != kSchemeSL || cfg.hessianMode != 0 || cfg.hasHessScheme || cfg.ntOverride <= 0 ||
        model.deformation == kNearIncompressible || ctx.fine.build || ctx.fine.gradient ||
        (pc.kind == kPcTwoLevel && (pc.coarseSolver != kCoarseCheb || pc.reestimateEachIteration)))
        throw NotSupported("batched newtonSolve: Gauss-Newton SL, fixed nt, Reg or two-level Chebyshev");
    if (gAll.pointsPer() % kEvalBlock != 0) throw NotSupported("batched pairs: n1 * n2 must be a multiple of 256");
    if (pc.kind == kPcTwoLevel && pc.chebIters < 1) throw InvalidArgument("solveKkt: chebIters must be >= 1");
    const auto tStart = std::chrono::steady_clock::now();
    const std::size_t Np = gAll.pointsPer();
    const int nt = cfg.ntOverride;
    status.assign(P, 0);
    errors.assign(P, std::string());
    std::vector<SolverReport> reports(P);
    std::vector<Counts> counts(P);
    std::vector<char> active(P, 1), carried(P, 0);
    std::vector<double> g0inf(P, 0.0), eMax(P, pc.eMax);

    DBuf vAll(sizeof(double) * 2 * gAll.points()), carriedAll(sizeof(double) * (nt + 1) * gAll.points()),
        finalAll(sizeof(double) * gAll.points());
    fill(ctx, 2 * gAll.points(), 0.0, vAll.d());
    copy(ctx, gAll.points(), mTAll, finalAll.d());

    // eigenvalue bounds at v = 0, once per solve (newton.cpp:36-40), per pair: the pairs' coarse
    // problems at v = 0 (all coarse nt = 2) as one batched coarse operator and their Lanczos
    // runs in lockstep (lanczosEmaxPairs), each pair's estimate that of its own estimateEigsAt
    if (pc.kind == kPcTwoLevel && !pc.hasEig) {
        std::vector<char> single(P, 1);  // pairs estimated on their own
        if (P > 1) {
            std::vector<int> idAll(P);
            for (int k = 0; k < P; ++k) idAll[k] = k;
            const std::vector<char> allOn(P, 1);
            CollectGuardsScope collect(true);
            CountScope cs(ctx);
            CoarseOperator coarse(ctx, gAll, nullptr, mRAll, mTAll, model, kCoarseCfl);
            cs.to(counts, idAll, allOn);
            std::vector<double> em;
            std::vector<char> fb;
            LinOpDev op = [&](const double* x, double* o) { coarse.applySplit(x, o); };
            coarse.hess->beginDeferredGuards(31);
            const bool done = lanczosEmaxPairs(ctx, coarse.gc, op, 30, 0x5eed, em, fb,
                                               [&](const std::vector<char>& on) { cs.to(counts, idAll, on); });
            coarse.hess->endDeferredGuards();
            if (done) {
                for (int k = 0; k < P; ++k) {
                    if (coarse.hess->pairStatus[k]) {  // estimateEigsAt would have thrown for this pair
                        status[k] = coarse.hess->pairStatus[k];
                        errors[k] = coarse.hess->pairError[k];
                        active[k] = 0;
                        single[k] = 0;
                    } else if (!fb[k]) {
                        eMax[k] = em[k];
                        single[k] = 0;
                    }
                }
            }
        }
        for (int k = 0; k < P; ++k) {
            if (!single[k]) continue;
            const long long f0 = ctx.ffts, i0 = ctx.interps;
            CollectGuardsScope one(false);  // a single-pair operation: its errors throw
            eMax[k] = estimateEigsAt(ctx, gAll.one(), nullptr, mRAll + k * Np, mTAll + k * Np, model, kCoarseCfl).second;
            counts[k].ffts += ctx.ffts - f0;
            counts[k].interps += ctx.interps - i0;
        }
    }

    for (int iter = 0; iter < cfg.maxOuterIter; ++iter) {
        std::vector<int> ids;
        for (int k = 0; k < P; ++k)
            if (active[k]) ids.push_back(k);
        if (ids.empty()) break;
        const auto tIter = std::chrono::steady_clock::now();
        const int PA = static_cast<int>(ids.size());
        const GridDims g(gAll.n1, gAll.n2, PA);
        const std::size_t N = g.points();
        std::vector<std::pair<int, int>> gather, scatter;
        for (int j = 0; j < PA; ++j) {
            gather.push_back({ids[j], j});
            scatter.push_back({j, ids[j]});
        }
        std::vector<int> st(P, 0);
        std::vector<std::string> er(P);
        DBuf vB(sizeof(double) * 2 * N), mRB(sizeof(double) * N), mTB(sizeof(double) * N);
        copyPairs(ctx, vAll.d(), P, vB.d(), PA, Np, 2, gather);
        copyPairs(ctx, mRAll, P, mRB.d(), PA, Np, 1, gather);
        copyPairs(ctx, mTAll, P, mTB.d(), PA, Np, 1, gather);
        double* v = vB.d();
        DBuf state(sizeof(double) * (nt + 1) * N), adjoint(sizeof(double) * (nt + 1) * N),
            grads(sizeof(double) * (nt + 1) * 2 * N), gBuf(sizeof(double) * 2 * N), dvBuf(sizeof(double) * 2 * N),
            tmpBuf(sizeof(double) * 2 * N), trialBuf(sizeof(double) * 2 * N),
            trialState(sizeof(double) * (nt + 1) * N);
        // reuse of the accepted trial's state (newton.cpp:54-56): every pair still iterating
        // after iteration 0 accepted a step at this nt
        const bool reuse = iter > 0;
        if (reuse) copyPairs(ctx, carriedAll.d(), P, state.d(), PA, Np, nt + 1, gather);
        std::vector<char> on(PA, 1);
        CountScope cs(ctx);
        std::vector<double> scal;
        std::vector<int> gst;
        evaluateGradientBatch(ctx, g, v, mRB.d(), mTB.d(), model, nt, gBuf.d(), scal, state.d(), adjoint.d(), reuse,
                              grads.d(), gst);
        // the reference's counts of evaluateGradient (inverse.cpp:119-148)
        cs.to(counts, ids, on);
        for (int j = 0; j < PA; ++j)
            if (gst[j]) {
                status[ids[j]] = gst[j];
                errors[ids[j]] = "evaluateGradient: transport failed";
                on[j] = 0;
            }
        const auto ginf = linfPairs(ctx, g, gBuf.d(), true);
        std::vector<IterationRecord> rec(PA);
        std::vector<double> eta(PA, 0.0), objective(PA), gdotd;
        for (int j = 0; j < PA; ++j) {
            const int k = ids[j];
            if (!on[j]) continue;
            if (iter == 0) g0inf[k] = std::max(ginf[j], 1e-300);
            const double grel = ginf[j] / g0inf[k];
            rec[j].iter = iter;
            rec[j].gradNormInf = ginf[j];
            rec[j].gradNormRel = grel;
            rec[j].objective = objective[j] = scal[4 * j];
            rec[j].mismatch = scal[4 * j + 1];
            rec[j].ffts = counts[k].ffts;
            rec[j].interps = counts[k].interps;
            reports[k].finalGradNormRel = grel;
            if (grel <= cfg.tolRelGrad || ginf[j] <= cfg.tolAbsGrad) {
                rec[j].wallTimeSec = secondsSinceB(tIter);
                reports[k].iterations.push_back(rec[j]);
                reports[k].status = kConverged;
                on[j] = 0;
                active[k] = 0;
                continue;
            }
            eta[j] = std::min(cfg.forcingCap, std::sqrt(grel));
        }
        for (int j = 0; j < PA; ++j)
            if (!on[j]) active[ids[j]] = 0;
        bool anyOn = false;
        for (int j = 0; j < PA; ++j) anyOn |= on[j] != 0;
        if (!anyOn) continue;

        // Hessian of the iterate (newton.cpp:83-96): state and grad m_j reused
        Hessian hess(ctx, g, v, v + N, mRB.d(), mTB.d(), model, nt, state.d(), 0, nullptr, grads.d());
        cs.to(counts, ids, on);
        lincomb(ctx, 2 * N, -1.0, gBuf.d(), 0.0, gBuf.d(), tmpBuf.d());  // rhs = -g
        // solveKkt (precond.cpp:291-358)
        {
            BatchKkt kkt(ctx, g, model, pc, hess, ids, counts, eMax, st, er, mRB.d(), mTB.d(), v);
            if (pc.hasEig) kkt.eMin = pc.eMin;
            const double* invHalf = hess.weights.invRegSymbol(model.betaV, -0.5);
            double* rhsSplit = ctx.scratchBuf(240, sizeof(double) * 2 * N);
            double* x = ctx.scratchBuf(241, sizeof(double) * 2 * N);
            applyRealSymbol(ctx, g, tmpBuf.d(), tmpBuf.d() + N, rhsSplit, rhsSplit + N, invHalf);
            cs.to(counts, ids, on);
            const bool twoLevel = pc.kind == kPcTwoLevel;
            if (twoLevel) kkt.buildCoarse(on);  // attributes its own counts
            cs.skip();
            for (int j = 0; j < PA; ++j)
                if (on[j] && st[ids[j]]) on[j] = 0;
            auto res = kkt.pcgBatch(rhsSplit, eta, cfg.maxInnerIter, twoLevel, on, x);
            // breakdown of the two-level preconditioner: re-estimate eMax and solve again
            // (precond.cpp:333-348), per pair on its own coarse operator
            std::vector<char> retry(PA, 0);
            bool anyRetry = false;
            for (int j = 0; j < PA; ++j)
                if (on[j] && !st[ids[j]] && res[j].indefinite && twoLevel) {
                    retry[j] = 1;
                    anyRetry = true;
                    const int k = ids[j];
                    const long long f0 = ctx.ffts, i0 = ctx.interps;
                    CollectGuardsScope single(false);
                    CoarseOperator co(ctx, g.one(), v + j * Np, mRB.d() + j * Np, mTB.d() + j * Np, model,
                                      kCoarseCfl);
                    co.hess->clearLazyCounts();  // the solve's coarse operator has done its lazy work
                    ctx.ffts = f0;
                    ctx.interps = i0;
                    eMax[k] = coarseLanczosEmax(ctx, co, 30, 0x5eed);
                    counts[k].ffts += ctx.ffts - f0;
                    counts[k].interps += ctx.interps - i0;
                    std::fprintf(stderr, "precond: re-estimated Chebyshev bound eMax=%.6g after breakdown\n", eMax[k]);
                }
            if (anyRetry) {
                // the other pairs' solutions stay in place: solve the retried pairs into x2
                double* x2 = ctx.scratchBuf(242, sizeof(double) * 2 * N);
                auto res2 = kkt.pcgBatch(rhsSplit, eta, cfg.maxInnerIter, true, retry, x2);
                std::vector<std::pair<int, int>> mv;
                for (int j = 0; j < PA; ++j)
                    if (retry[j]) {
                        res[j] = res2[j];
                        mv.push_back({j, j});
                    }
                copyPairs(ctx, x2, PA, x, PA, Np, 2, mv);
            }
            cs.skip();  // the Krylov solves and re-estimates attributed their counts
            applyRealSymbol(ctx, g, x, x + N, dvBuf.d(), dvBuf.d() + N, invHalf);
            cs.to(counts, ids, on);
            for (int j = 0; j < PA; ++j) {
                if (st[ids[j]]) {
                    status[ids[j]] = st[ids[j]];
                    errors[ids[j]] = er[ids[j]];
                    on[j] = 0;
                    active[ids[j]] = 0;
                }
                rec[j].innerIterations = res[j].iterations;
            }
        }
        double* dv = dvBuf.d();
        gdotd = dotPairs(ctx, g, gBuf.d(), dv, true);
        {
            // inner solve broke down: Sobolev-gradient fallback direction (newton.cpp:99-105)
            std::vector<char> fb(PA, 0);
            bool any = false;
            for (int j = 0; j < PA; ++j)
                if (on[j] && (!std::isfinite(gdotd[j]) || gdotd[j] >= 0.0)) fb[j] = any = 1;
            if (any) {
                Weights w(g, model.norm);
                CountScope fsc(ctx);
                applyRealSymbol(ctx, g, gBuf.d(), gBuf.d() + N, trialBuf.d(), trialBuf.d() + N,
                                w.invRegSymbol(model.betaV, -1.0));
                fsc.to(counts, ids, fb);
                std::vector<double> m1(PA, -1.0), z0(PA, 0.0);
                lincombPairs(ctx, g, 2, coefOf(z0, m1, fb), trialBuf.d(), trialBuf.d(), dv);
                const auto gd2 = dotPairs(ctx, g, gBuf.d(), dv, true);
                for (int j = 0; j < PA; ++j)
                    if (fb[j]) gdotd[j] = gd2[j];
            }
        }
        {
            CountScope dsc(ctx);
            divergence(ctx, g, dv, dv + N, tmpBuf.d());
            dsc.to(counts, ids, on);
            const auto dn = linfPairs(ctx, g, tmpBuf.d(), false);
            const auto vn = linfPairs(ctx, g, dv, true);
            for (int j = 0; j < PA; ++j) rec[j].searchDirDivRatio = dn[j] / std::max(vn[j], 1e-300);
        }
        // Armijo backtracking per pair (newton.cpp:109-131)
        std::vector<double> alpha(PA, 1.0);
        std::vector<char> searching = on, accepted(PA, 0);
        copy(ctx, 2 * N, v, trialBuf.d());  // the pairs not searching evaluate their own iterate
        std::vector<int> lsSteps(PA, 0);
        std::vector<double> ones(PA, 1.0);
        for (int step = 0; step < cfg.lsMaxSteps; ++step) {
            bool any = false;
            for (int j = 0; j < PA; ++j) any |= searching[j] != 0;
            if (!any) break;
            lincombPairs(ctx, g, 2, coefOf(ones, alpha, searching), v, dv, trialBuf.d());
            std::vector<double> ob;
            std::vector<int> ost;
            CountScope osc(ctx);
            evaluateObjectiveBatch(ctx, g, trialBuf.d(), mRB.d(), mTB.d(), model, nt, ob, trialState.d(), ost);
            osc.to(counts, ids, searching);
            std::vector<std::pair<int, int>> acc, accV;
            for (int j = 0; j < PA; ++j) {
                if (!searching[j]) continue;
                const bool blewUp = ost[j] == kBlowup;
                if (ost[j] && !blewUp) {  // a non-finite prefilter input: the reference throws
                    status[ids[j]] = ost[j];
                    errors[ids[j]] = "evaluateObjective: " + std::string("prefilter: non-finite value");
                    searching[j] = 0;
                    on[j] = 0;
                    active[ids[j]] = 0;
                    continue;
                }
                if (!blewUp && ob[4 * j] <= objective[j] + cfg.lsC1 * alpha[j] * gdotd[j]) {
                    accepted[j] = 1;
                    searching[j] = 0;
                    lsSteps[j] = step + 1;
                    acc.push_back({j, ids[j]});
                    accV.push_back({j, j});
                } else {
                    alpha[j] *= cfg.lsShrink;
                    lsSteps[j] = step + 1;
                }
            }
            if (!acc.empty()) {
                copyPairs(ctx, trialBuf.d(), PA, v, PA, Np, 2, accV);
                copyPairs(ctx, trialState.d(), PA, carriedAll.d(), P, Np, nt + 1, acc);
                std::vector<std::pair<int, int>> fin;
                for (const auto& a : acc) fin.push_back(a);
                copyPairs(ctx, trialState.d() + static_cast<std::size_t>(nt) * N, PA, finalAll.d(), P, Np, 1, fin);
            }
        }
        for (int j = 0; j < PA; ++j) {
            if (!on[j]) continue;
            const int k = ids[j];
            rec[j].lineSearchSteps = accepted[j] ? lsSteps[j] : cfg.lsMaxSteps;
            rec[j].stepLength = accepted[j] ? alpha[j] : 0.0;
            rec[j].wallTimeSec = secondsSinceB(tIter);
            rec[j].ffts = counts[k].ffts;
            rec[j].interps = counts[k].interps;
            reports[k].iterations.push_back(rec[j]);
            if (!accepted[j]) {
                reports[k].status = kLineSearchFailure;
                active[k] = 0;
                carried[k] = 0;
            } else {
                carried[k] = 1;
                if (iter + 1 == cfg.maxOuterIter) reports[k].status = kIterationLimit;
            }
        }
        copyPairs(ctx, v, PA, vAll.d(), P, Np, 2, scatter);
    }

    // final diagnostics per pair (newton.cpp:147-157): residuals, then the SL Jacobian of every
    // pair, the pairs grouped by their Jacobian step count (deriveSteps at CFL 0.2) and each
    // group solved as one batch (a pair's determinant is that of its own solve)
    const GridDims g1 = gAll.one();
    DBuf tmp(sizeof(double) * 2 * Np);
    for (int k = 0; k < P; ++k) {
        if (status[k]) continue;
        const double* mR = mRAll + k * Np;
        lincomb(ctx, Np, 1.0, mTAll + k * Np, -1.0, mR, tmp.d());
        const double residDenom = std::sqrt(dot(ctx, g1, tmp.d(), nullptr, tmp.d(), nullptr));
        lincomb(ctx, Np, 1.0, finalAll.d() + k * Np, -1.0, mR, tmp.d());
        const double residNum = std::sqrt(dot(ctx, g1, tmp.d(), nullptr, tmp.d(), nullptr));
        reports[k].finalResidualRel = residDenom > 0.0 ? residNum / residDenom : 0.0;
    }
    {
        const auto m1 = linfPairs(ctx, gAll, vAll.d(), false);
        const auto m2 = linfPairs(ctx, gAll, vAll.d() + gAll.points(), false);
        std::map<int, std::vector<int>> byNt;
        for (int k = 0; k < P; ++k) {
            if (status[k]) continue;
            double ratio = 0.0;
            ratio = std::max(ratio, m1[k] / (0.2 * gAll.h1()));
            ratio = std::max(ratio, m2[k] / (0.2 * gAll.h2()));
            byNt[std::max(2, static_cast<int>(std::ceil(ratio)))].push_back(k);
        }
        for (auto& kv : byNt) {
            const int Pg = static_cast<int>(kv.second.size());
            const GridDims gg(gAll.n1, gAll.n2, Pg);
            std::vector<std::pair<int, int>> map;
            for (int j = 0; j < Pg; ++j) map.push_back({kv.second[j], j});
            DBuf vg(sizeof(double) * 2 * gg.points()), jac(sizeof(double) * gg.points());
            copyPairs(ctx, vAll.d(), P, vg.d(), Pg, Np, 2, map);
            Solver js(ctx, gg, vg.d(), vg.d() + gg.points(), kv.first);
            js.jacobian(jac.d());
            std::vector<double> h(gg.points());
            VRG_CUDA(cudaMemcpyAsync(h.data(), jac.d(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, ctx.stream));
            ctx.sync();
            for (int j = 0; j < Pg; ++j) {
                const auto b = h.begin() + static_cast<std::ptrdiff_t>(j) * Np;
                reports[kv.second[j]].jacMin = *std::min_element(b, b + Np);
                reports[kv.second[j]].jacMax = *std::max_element(b, b + Np);
            }
        }
    }
    copy(ctx, 2 * gAll.points(), vAll.d(), vOut);
    ctx.sync();
    const double total = secondsSinceB(tStart);
    for (auto& r : reports) r.totalTimeSec = total;
    return reports;
}

}  // namespace vrg
