// K2: tensor-product cubic B-spline evaluation at one departure point per grid node, with a
// fused per-node epilogue.  Restates interp::evaluate (src/interp.cpp:87-127): wrap, cell,
// 4+4 weights, 16-tap periodic gather.  NF coefficient fields sharing one point set are
// evaluated together so the weights and indices are computed once (e.g. both components of
// a vector field, or the pair (grad m)_D).
//
// The epilogue functor receives (p, value[0..NF)) and returns the value the blow-up guard
// watches (|.|, NaN ignored like std::max in normLinf, src/field.cpp:59-65); block maxima
// go to guardPartials[blockIdx.x] when Epi::kGuard.
#pragma once

#include <algorithm>

#include "interp.cuh"

namespace vrg {

constexpr int kEvalBlock = 256;

// Epilogues declare `Pre` (operands loaded before the gather, see k_evaluate) and
// `prefetch(p)`; those without early operands use NoPre.
struct NoPre {};
#define VRG_NO_PREFETCH                 \
    using Pre = NoPre;                  \
    __device__ Pre prefetch(std::size_t) const { return {}; }

// Coefficient fields in the periodically padded layout ((n1+3) x (n2+3), see cellBase).
template <int NF>
struct CoeffSet {
    const double* c[NF];
};

// xStable: the departure points are not written by any kernel still in flight (the matvec
// time loops), so the cell computation runs before the programmatic-dependency wait.
// blockIdx.y: member of a batch of coefficient sets at the same points (coefficient offset
// csZ, epilogue index offset epiZ per member; guard-free epilogues only).
// Per-(step, pair) guard maximum: guard values are >= +0 (NaN skipped, inf kept), whose IEEE bit
// patterns order like unsigned integers, so an integer atomicMax on the bits is the maximum of
// the doubles (order-independent, hence run-to-run deterministic) and no reduction kernel
// follows the step.
__device__ __forceinline__ void guardMax(double* slot, double m) {
    atomicMax(reinterpret_cast<unsigned long long*>(slot), static_cast<unsigned long long>(__double_as_longlong(m)));
}


// Stacked pairs (GridDims::pairs): node p belongs to pair p / (n1 n2), whose coefficients are the
// pair's padded field (pair * paddedPoints(n1, n2) further on); n1 * n2 is then a multiple of
// the block size, so a block never straddles two pairs.
// First-tap row/column and weights of a departure point along one axis: from the coordinate
// or from its packed cell (interp.cuh: the per-iterate departure points of the SL loops).
__device__ __forceinline__ int depCell(double x, double invh, int n, double w[4]) { return cellBase(x, invh, n, w); }
__device__ __forceinline__ int depCell(Cell u, double, int, double w[4]) { return cellDecode(u, w); }

template <int NF, class Epi, class Dep = double>
__global__ void __launch_bounds__(kEvalBlock) k_evaluate(CoeffSet<NF> cs, const Dep* __restrict__ x1,
                                                         const Dep* __restrict__ x2, int n1, int n2, int xStable,
                                                         Epi epi, std::size_t csZ, std::size_t epiZ, int pairs) {
    const int Nper = n1 * n2;
    const int N = Nper * pairs;  // up to 2^31 points
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.y) {
#pragma unroll
        for (int f = 0; f < NF; ++f) cs.c[f] += blockIdx.y * csZ;
    }
    if (pairs > 1) {
        const std::size_t off = static_cast<std::size_t>(p / Nper) * paddedPoints(n1, n2);
#pragma unroll
        for (int f = 0; f < NF; ++f) cs.c[f] += off;
    }
    double guard = 0.0;
    if (!xStable) pdlWait();
    double w1[4], w2[4];
    int base = 0;
    if (p < N) {
        const int b1 = depCell(__ldg(x1 + p), n1 * (1.0 / kTwoPi), n1, w1);  // 1/h = n / 2pi
        const int b2 = depCell(__ldg(x2 + p), n2 * (1.0 / kTwoPi), n2, w2);
        base = b1 * (n2 + 3) + b2;
    }
    // epilogue operands that no in-flight kernel writes (per-iterate fields) are loaded now,
    // so their latency overlaps the departure-point loads and the gather
    typename Epi::Pre pre{};
    if (p < N) pre = epi.prefetch(p + blockIdx.y * epiZ);
    if (xStable) pdlWait();
    pdlTrigger();
    if (p < N) {
        const int PW = n2 + 3;
        // all 16 (x NF) taps are issued before any is consumed (one memory latency, not four)
        double tap[NF][16];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const double* c0 = cs.c[f] + base;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) tap[f][4 * a + b] = __ldg(c0 + a * PW + b);
        }
        // pin the taps in registers here: ptxas otherwise interleaves loads and FMAs in small
        // groups to save registers, serialising several memory latencies per thread
#pragma unroll
        for (int f = 0; f < NF; ++f)
#pragma unroll
            for (int i = 0; i < 16; ++i) asm volatile("" : "+d"(tap[f][i]));
        double val[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                double rowAcc = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) rowAcc += w2[b] * tap[f][4 * a + b];
                acc += w1[a] * rowAcc;
            }
            val[f] = acc;
        }
        const double gv = fabs(epi(p + blockIdx.y * epiZ, val, pre));
        if (gv == gv) guard = gv;  // NaN ignored, inf kept
    }
    if constexpr (Epi::kGuard) {
        __shared__ double red[kEvalBlock / 32];
        for (int o = 16; o > 0; o >>= 1) guard = fmax(guard, __shfl_xor_sync(0xffffffffu, guard, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = guard;
        __syncthreads();
        if (threadIdx.x == 0) {
            double m = red[0];
            for (int w = 1; w < kEvalBlock / 32; ++w) m = fmax(m, red[w]);
            guardMax(epi.guardPartials + blockIdx.x / ((Nper + kEvalBlock - 1) / kEvalBlock), m);
        }
    }
}

// Same block layout and guard reduction as k_evaluate, without the gather (values = 0):
// used where the interpolated field is identically zero (m~_0 = 0) or for pure pointwise work.
template <class Epi>
__global__ void __launch_bounds__(kEvalBlock) k_pointwise(std::size_t N, Epi epi, unsigned blocksPer) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double guard = 0.0;
    pdlWait();
    pdlTrigger();
    if (p < N) {
        const double z[2] = {0.0, 0.0};
        const double gv = fabs(epi(p, z, epi.prefetch(p)));
        if (gv == gv) guard = gv;
    }
    if constexpr (Epi::kGuard) {
        __shared__ double red[kEvalBlock / 32];
        for (int o = 16; o > 0; o >>= 1) guard = fmax(guard, __shfl_xor_sync(0xffffffffu, guard, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = guard;
        __syncthreads();
        if (threadIdx.x == 0) {
            double m = red[0];
            for (int w = 1; w < kEvalBlock / 32; ++w) m = fmax(m, red[w]);
            guardMax(epi.guardPartials + blockIdx.x / blocksPer, m);
        }
    }
}

inline unsigned evalBlocks(const GridDims& g) { return grid1d(g.points(), kEvalBlock).x; }
inline unsigned evalBlocksPer(const GridDims& g) { return grid1d(g.pointsPer(), kEvalBlock).x; }

template <class Epi>
void launchPointwise(Ctx& ctx, const GridDims& g, const Epi& epi) {
    {
        LaunchScope ls_(ctx, Epi::kName);
        launchPdl(1, k_pointwise<Epi>, grid1d(g.points(), kEvalBlock), dim3(kEvalBlock), 0, ctx.stream, g.points(), epi,
                  evalBlocksPer(g));
    }
}

template <int NF, class Epi, class Dep>
void launchEvaluate(Ctx& ctx, const GridDims& g, CoeffSet<NF> cs, const Dep* x1, const Dep* x2, const Epi& epi,
                    bool xStable = false) {
    const std::size_t N = g.points();
    {
        LaunchScope ls_(ctx, Epi::kName);
        launchPdl(1, k_evaluate<NF, Epi, Dep>, grid1d(N, kEvalBlock), dim3(kEvalBlock), 0, ctx.stream, cs, x1, x2, g.n1, g.n2,
                  xStable ? 1 : 0, epi, std::size_t(0), std::size_t(0), g.pairs);
    }
}

// `count` coefficient sets cs + k*csZ evaluated at the same points in one launch, the
// epilogue of member k at index p + k*epiZ (guard-free epilogues, e.g. EpiStore2).
template <int NF, class Epi, class Dep>
void launchEvaluateBatch(Ctx& ctx, const GridDims& g, CoeffSet<NF> cs, std::size_t csZ, int count, const Dep* x1,
                         const Dep* x2, const Epi& epi, std::size_t epiZ) {
    static_assert(!Epi::kGuard, "batched evaluate: guard-free epilogues only");
    const std::size_t N = g.points();
    {
        LaunchScope ls_(ctx, Epi::kName);
        launchPdl(1, k_evaluate<NF, Epi, Dep>, dim3(grid1d(N, kEvalBlock).x, count), dim3(kEvalBlock), 0, ctx.stream, cs,
                  x1, x2, g.n1, g.n2, 0, epi, csZ, epiZ, g.pairs);
    }
}



// Plain stores.
struct EpiStore1 {
    static constexpr const char* kName = "evaluate/store1";
    static constexpr bool kGuard = false;
    double* guardPartials = nullptr;
    double* out;
    VRG_NO_PREFETCH
    __device__ double operator()(std::size_t p, const double* v, const Pre&) const {
        out[p] = v[0];
        return 0.0;
    }
};

struct EpiStore2 {
    static constexpr const char* kName = "evaluate/store2";
    static constexpr bool kGuard = false;
    double* guardPartials = nullptr;
    double* out0;
    double* out1;
    VRG_NO_PREFETCH
    __device__ double operator()(std::size_t p, const double* v, const Pre&) const {
        out0[p] = v[0];
        out1[p] = v[1];
        return 0.0;
    }
};

}  // namespace vrg
