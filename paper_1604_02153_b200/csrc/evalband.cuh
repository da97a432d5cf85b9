// K2 + K1(rows) fused: B-spline evaluation with the step epilogue, one grid row per block,
// followed in the same kernel by the row pass of the next step's prefilter.
//
// In the matvec time loops every interpolated field (m~_j, lt_j) is produced by the previous
// step's gather, so the producer can row-filter it while the row is still in shared memory:
// a block owns one whole periodic row, so the row filter is exact inside the block
// (chunk-carry form of interp.cu) and only the column pass remains a separate kernel.  This
// removes one kernel and one field write+read per step.  The gather keeps the plain kernel's
// structure (256 threads, epilogue operands prefetched, programmatic dependent launch).
#pragma once

#include <atomic>
#include <type_traits>

#include "eval.cuh"

namespace vrg {

constexpr int kBandThreads = 256;

// Threads per row (one thread per 16-sample chunk in the row filter, n2 / TW nodes per thread
// in the gather): the largest of 256 / 128 / 64 / 32 dividing n2, so coarse and small grids
// (n2 = 32 .. 192) take the band path too.
inline int bandTW(int n2) {
    for (int tw : {256, 128, 64, 32})
        if (n2 % tw == 0) return tw;
    return 0;
}

// one block per row; n2 a multiple of 32 with its chunks (n2 / 16) within the row's threads
inline bool bandFusable(const GridDims& g) {
    const int tw = bandTW(g.n2);
    return tw && g.n2 >= 32 && g.n2 / kL <= tw;
}

// The SL time loops take the band path with packed departure cells (axes up to kCellMaxN).
inline bool bandCellsFit(const GridDims& g) { return g.n1 <= kCellMaxN && g.n2 <= kCellMaxN; }

// Doubles of shared memory one row needs (chunked row + chunk summaries + warp guard maxima).
__host__ __device__ inline int bandRowSmem(int n2, int tw) { return (n2 / kL) * (kCS + 3) + (tw + 31) / 32; }

inline std::size_t bandSmem(const GridDims& g) { return sizeof(double) * bandRowSmem(g.n2, bandTW(g.n2)); }

inline unsigned bandBlocks(const GridDims& g) { return static_cast<unsigned>(g.n1) * g.pairs; }

// Without a gather (kGather = false: m~_0 = 0, the first incremental-state step) the epilogue
// operands come from the immediate predecessor (vt_D), so the kernel waits before any load;
// with a gather only the coefficient field is produced by the predecessor and the departure
// points and epilogue operands are loaded before the programmatic-dependency wait.
// Coefficient load that stays behind griddepcontrol.wait.  The wait sits inside the node loop
// (first iteration) and ptxas hoists non-coherent (ld.global.nc / __ldg) gathers of the loop
// body above it, which reads the coefficients before the predecessor column pass has written
// them (seen in the SASS and as nondeterministic results under graph replay).  A coherent
// load is ordered by the wait.
// (A plain coherent load: the compiler keeps it behind the wait's memory clobber and shares
// the address arithmetic of the 16 taps, which an asm volatile load per tap did not.)
__device__ __forceinline__ double ldAfterWait(const double* p) { return *p; }

// Coefficient window of a slab-decomposed grid (slab.py): the coefficients hold `rows` padded
// rows, window row w = global grid row base + w (mod n1), instead of the whole periodically
// padded field.  A departure cell whose 4 tap rows fall outside the window sets *err.
struct BandWindow {
    int base = -1;
    int rows = 0;
    unsigned* err = nullptr;
};

// Resident blocks per SM the band kernel is compiled for (register cap 65536 / (256 x value)):
// 4 (64 registers) by default; an epilogue with more live state specialises it.
template <class Epi>
struct BandMinBlocks {
    static constexpr int value = 4;
};

// Barrier policies of one row's work: the whole block (k_eval_band) or one row worker of a
// strip block (k_eval_strip: named barrier `id` over the worker's TW threads).
struct BarBlock {
    __device__ void sync() const { __syncthreads(); }
    __device__ bool syncOr(bool p) const { return __syncthreads_or(p); }
};
template <int TW>
struct BarNamed {
    int id;
    __device__ void sync() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(TW) : "memory"); }
    __device__ bool syncOr(bool p) const {
        unsigned o;
        asm volatile(
            "{ .reg .pred pi, po;\n\t setp.ne.u32 pi, %1, 0;\n\t bar.red.or.pred po, %2, %3, pi;\n\t"
            " selp.u32 %0, 1, 0, po; }"
            : "=r"(o)
            : "r"(static_cast<unsigned>(p)), "r"(id), "n"(TW)
            : "memory");
        return o != 0;
    }
};

// One grid row r by TW threads (t = 0..TW-1): gather at the row's departure points, step
// epilogue, the row's guard maximum, then the exact periodic row filter in shared memory and
// the row-filtered output.  `sm` holds bandRowSmem(n2, TW) doubles.
// Stacked pairs (GridDims::pairs): r runs over all pairs' rows; row r belongs to pair r / n1,
// whose coefficients lie pair * paddedPoints(n1, n2) further on, and its guard maximum goes to
// the pair's slot (eval.cuh guardMax); slab windows keep one partial per local row.
template <class Epi, bool kGather, bool kWindow, int TW, class Bar, class Dep>
__device__ __forceinline__ void bandRow(CoeffSet<1> cs, const Dep* __restrict__ x1,
                                        const Dep* __restrict__ x2, int n1, int n2, const Epi& epi,
                                        double* __restrict__ rowOut, unsigned* nonfinite, const BandWindow& win,
                                        int r, int t, double* sm, Bar bar) {
    if (!kGather) pdlWait();
    const int pair = kWindow ? 0 : r / n1;
    if (!kWindow) cs.c[0] += static_cast<std::size_t>(pair) * paddedPoints(n1, n2);
    const int nc = n2 / kL;
    double* E = sm + nc * kCS;
    double* F0 = E + nc;
    double* P0 = F0 + nc;
    double* red = P0 + nc;
    const int per = n2 / TW;  // nodes per thread
    const int PW = n2 + 3;
    const double inv1 = n1 * (1.0 / kTwoPi), inv2 = n2 * (1.0 / kTwoPi);
    // padded-layout row of the first tap (cellBase) -> row of the coefficient array
    auto tapRow = [&](int b1) {
        if constexpr (kWindow) {
            int w = b1 - 1 - win.base;
            w += w < 0 ? n1 : 0;
            w -= w >= n1 ? n1 : 0;
            if (w < 0 || w + 3 >= win.rows) {
                atomicOr(win.err, 1u);
                w = 0;
            }
            return w;
        } else {
            return b1;
        }
    };

    double guard = 0.0;
    bool bad = false;
    // Software pipeline over the thread's nodes (incremental-state step, one-double epilogue
    // operand): the departure point and epilogue operand of node k+1 are loaded while node k's
    // taps are in flight, one memory round trip per node instead of two (the gather is latency
    // bound).  The adjoint step's four prefetched operands would cost a resident block per SM
    // (78 registers), which measured slower, so it keeps the plain order.
    constexpr bool kPipe = sizeof(typename Epi::Pre) <= sizeof(double);
    Dep xa{}, xb{};
    typename Epi::Pre pre{};
    // the unpipelined steps still run their departure cells one node ahead (two more registers:
    // the gather waits for one memory round trip per node instead of two; no spills at 64)
    constexpr bool kPipeDep = !kPipe && kGather;
    if constexpr (kPipe) {
        if (kGather) {
            xa = __ldg(x1 + r * n2 + t);
            xb = __ldg(x2 + r * n2 + t);
        }
        pre = epi.prefetch(r * n2 + t);
        if (kGather) pdlWait();
    } else if constexpr (kPipeDep) {
        xa = __ldg(x1 + r * n2 + t);
        xb = __ldg(x2 + r * n2 + t);
    }
    for (int k = 0; k < per; ++k) {
        const int col = t + TW * k;
        const int p = r * n2 + col;
        double w1[4], w2[4];
        int base = 0;
        typename Epi::Pre cur;
        if constexpr (kPipe) {
            if (kGather) {
                const int b1 = tapRow(depCell(xa, inv1, n1, w1));
                const int b2 = depCell(xb, inv2, n2, w2);
                base = b1 * PW + b2;
            }
            cur = pre;
            if (k + 1 < per) {
                if (kGather) {
                    xa = __ldg(x1 + p + TW);
                    xb = __ldg(x2 + p + TW);
                }
                pre = epi.prefetch(p + TW);
            }
        } else {
            if constexpr (kPipeDep) {
                const int b1 = tapRow(depCell(xa, inv1, n1, w1));
                const int b2 = depCell(xb, inv2, n2, w2);
                base = b1 * PW + b2;
                if (k + 1 < per) {
                    xa = __ldg(x1 + p + TW);
                    xb = __ldg(x2 + p + TW);
                }
            } else if (kGather) {
                const int b1 = tapRow(depCell(__ldg(x1 + p), inv1, n1, w1));
                const int b2 = depCell(__ldg(x2 + p), inv2, n2, w2);
                base = b1 * PW + b2;
            }
            cur = epi.prefetch(p);
            if (kGather && k == 0) pdlWait();
        }
        double val = 0.0;
        if (kGather) {
            double tap[16];
            const double* c0 = cs.c[0] + base;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) tap[4 * a + b] = ldAfterWait(c0 + a * PW + b);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                double rowAcc = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) rowAcc += w2[b] * tap[4 * a + b];
                val += w1[a] * rowAcc;
            }
        }
        const double o = epi(p, &val, cur);
        const double ao = fabs(o);
        if (ao == ao) guard = fmax(guard, ao);
        bad |= !isfinite(o);
        sm[slot(col)] = o;
    }
    if constexpr (Epi::kGuard) {
        for (int o = 16; o > 0; o >>= 1) guard = fmax(guard, __shfl_xor_sync(0xffffffffu, guard, o));
        if ((t & 31) == 0) red[t >> 5] = guard;
        bar.sync();
        if (t == 0) {
            double m = red[0];
            for (int w = 1; w < TW / 32; ++w) m = fmax(m, red[w]);
            if constexpr (kWindow)
                epi.guardPartials[r] = m;  // slab rows: per-row partials (slab.py reduces them)
            else
                guardMax(epi.guardPartials + pair, m);
        }
    }
    // the next prefilter's input check (checkFinite(u, "prefilter"), interp.cpp:76)
    if (bar.syncOr(bad) && t == 0 && nonfinite) atomicOr(nonfinite, 1u);
    if (!rowOut) return;  // the last step of a loop: nothing left to interpolate, no row pass

    // ---- row pass of the prefilter (exact: the whole periodic row is in shared memory)
    double f[kL];
    double2* s2 = reinterpret_cast<double2*>(sm + t * kCS);
    if (t < nc) {
#pragma unroll
        for (int k = 0; k < kL / 2; ++k) {
            const double2 v = s2[k];
            f[2 * k] = v.x;
            f[2 * k + 1] = v.y;
        }
        double b = 0.0;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) b = kZ * (f[k + 1] + b);
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < kL; ++k) a = f[k] + kZ * a;
        E[t] = a;
        F0[t] = f[0];
        P0[t] = b;
    }
    bar.sync();
    if (t < nc) {
        const ZPow zp;
        const int c = t;
        const int cm1 = c == 0 ? nc - 1 : c - 1, cm2 = cm1 == 0 ? nc - 1 : cm1 - 1;
        const int cp1 = c == nc - 1 ? 0 : c + 1, cp2 = cp1 == nc - 1 ? 0 : cp1 + 1;
        const double cp = E[cm1] + zp.p[kL] * E[cm2];
        const double cm = kZ * (F0[cp1] + P0[cp1]) + zp.p[kL + 1] * (F0[cp2] + P0[cp2]);
        double ym[kL];
        ym[kL - 1] = cm;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) ym[k] = kZ * (f[k + 1] + ym[k + 1]);
        double yp = cp;
#pragma unroll
        for (int k = 0; k < kL; k += 2) {
            yp = f[k] + kZ * yp;
            const double o0 = kSqrt3 * (yp + ym[k]);
            yp = f[k + 1] + kZ * yp;
            const double o1 = kSqrt3 * (yp + ym[k + 1]);
            s2[k / 2] = make_double2(o0, o1);
        }
    }
    bar.sync();
    double* dst = rowOut + static_cast<std::size_t>(r) * n2;
    for (int k = 0; k < per; ++k) {
        const int col = t + TW * k;
        dst[col] = sm[slot(col)];
    }
}

// Resident blocks per SM of the row-per-block kernel: the 256-thread count scaled to TW (same
// register cap).
template <class Epi, int TW>
constexpr int bandMinBlocks() {
    return BandMinBlocks<Epi>::value * (kBandThreads / TW);
}

// Departure points as packed cells (Dep = Cell, the SL time loops) or coordinates (Dep = double,
// slab windows).
template <class Epi, bool kGather, bool kWindow = false, int TW = kBandThreads, class Dep = Cell>
__global__ void __launch_bounds__(TW, (bandMinBlocks<Epi, TW>())) k_eval_band(CoeffSet<1> cs, const Dep* __restrict__ x1,
                                                            const Dep* __restrict__ x2, int n1, int n2, Epi epi,
                                                            double* __restrict__ rowOut, unsigned* nonfinite,
                                                            BandWindow win) {
    extern __shared__ __align__(16) double sm[];
    bandRow<Epi, kGather, kWindow, TW>(cs, x1, x2, n1, n2, epi, rowOut, nonfinite, win, blockIdx.x, threadIdx.x, sm,
                                       BarBlock{});
    pdlTrigger();  // at the end: the dependent column pass must not take this kernel's slots
}

// Strip form (large grids): one block (one per SM: its register file) owns W consecutive rows,
// one row worker of TW threads each (named barriers, no block-wide synchronisation), so the
// rows an SM gathers at the same time are neighbours and share their coefficient rows in L1 —
// with one block per row, consecutive rows land on different SMs and every SM fetches the 4
// tap rows of each of its rows from L2 (tap traffic 4.3x the coefficient field).
// Row workers per strip block: 7 x 128 threads (72 registers; ~7 rows per SM at 1024 rows on
// 148 SMs, one round) for every epilogue: with 6 workers the seed step needed 171 blocks, two
// rounds on 148 SMs (twice the time of a regular step), while 72 registers hold its state
// without spills (the 64-register row-per-block kernel is what needs BandMinBlocks = 3).
template <class Epi, int TW>
constexpr int stripWorkers() {
    return 7;
}

template <class Epi, bool kGather, int TW>
__global__ void __launch_bounds__(TW* stripWorkers<Epi, TW>(), 1)
    k_eval_strip(CoeffSet<1> cs, const Cell* __restrict__ x1, const Cell* __restrict__ x2, int n1, int n2, Epi epi,
                 double* __restrict__ rowOut, unsigned* nonfinite, int rows) {
    extern __shared__ __align__(16) double sm[];
    constexpr int W = stripWorkers<Epi, TW>();
    const int w = threadIdx.x / TW;
    const int t = threadIdx.x - w * TW;
    const int r = blockIdx.x * W + w;
    // r < rows is warp-uniform (TW is a multiple of 32); the vote tells the compiler so, which
    // keeps the row's loads on uniform memory descriptors (no R2UR per tap)
    if (__any_sync(0xffffffffu, r < rows))
        bandRow<Epi, kGather, false, TW>(cs, x1, x2, n1, n2, epi, rowOut, nonfinite, BandWindow{}, r, t,
                                         sm + w * bandRowSmem(n2, TW), BarNamed<TW>{1 + w});
    pdlTrigger();
}

// Row-to-SM mapping of the band step: 0 = by grid size (strip blocks when every SM gets >= 4
// rows), 1 = one block per row, 2 = strip blocks.  Only the kernel benchmark
// (vrg_hess_bench_kernel) sets it, to time both forms on the same operator.
inline std::atomic<int> g_bandMapping{0};

// Strip blocks where every SM gets >= 4 rows and a row's chunks fit 128 threads (n2 <= 2048).
// Measured on B200 (tools/sl_step_probe.py, ids +100/+200): at 1024^2 the state / incremental-
// state / adjoint band steps take 11.0 / 13.8 / 14.7 us as strips against 11.6 / 14.7 / 16.3 us
// with one block per row; at 2048^2 5% faster except the incremental-state step (1% slower); at
// 4096^2 (3 x 256-thread workers) 15-20% slower, so the row-per-block form stays there.
inline bool stripPath(const Ctx& ctx, const GridDims& g) {
    const bool fits = g.n2 % 128 == 0 && g.n2 / kL <= 128;
    if (g_bandMapping) return g_bandMapping == 2 && fits;
    return g.n1 >= 4 * ctx.numSMs && fits;
}

template <class Epi, bool kGather, int TW>
void launchEvalStrip(Ctx& ctx, const GridDims& g, CoeffSet<1> cs, const Cell* x1, const Cell* x2, const Epi& epi,
                     double* rowOut, unsigned* nonfinite) {
    constexpr int W = stripWorkers<Epi, TW>();
    constexpr int kThreads = W * TW;
    const std::size_t smem = sizeof(double) * W * bandRowSmem(g.n2, TW);
    static std::mutex mu;
    static bool attr[64] = {};
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!attr[ctx.device]) {
            VRG_CUDA(cudaFuncSetAttribute(k_eval_strip<Epi, kGather, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          200 * 1024));
            attr[ctx.device] = true;
        }
    }
    const int rows = g.n1 * g.pairs;
    launchPdl(1, k_eval_strip<Epi, kGather, TW>, dim3((rows + W - 1) / W), dim3(kThreads), smem, ctx.stream, cs, x1,
              x2, g.n1, g.n2, epi, rowOut, nonfinite, rows);
}

template <class Epi, bool kGather>
void launchEvalBand(Ctx& ctx, const GridDims& g, CoeffSet<1> cs, const Cell* x1, const Cell* x2, const Epi& epi,
                    double* rowOut, unsigned* nonfinite) {
    LaunchScope ls_(ctx, Epi::kName);
    if (stripPath(ctx, g)) {
        launchEvalStrip<Epi, kGather, 128>(ctx, g, cs, x1, x2, epi, rowOut, nonfinite);
        return;
    }
    const std::size_t smem = bandSmem(g);
    const dim3 grid(bandBlocks(g));
    switch (bandTW(g.n2)) {
        case 256:
            launchPdl(1, k_eval_band<Epi, kGather, false, 256>, grid, dim3(256), smem, ctx.stream, cs, x1, x2, g.n1,
                      g.n2, epi, rowOut, nonfinite, BandWindow{});
            break;
        case 128:
            launchPdl(1, k_eval_band<Epi, kGather, false, 128>, grid, dim3(128), smem, ctx.stream, cs, x1, x2, g.n1,
                      g.n2, epi, rowOut, nonfinite, BandWindow{});
            break;
        case 64:
            launchPdl(1, k_eval_band<Epi, kGather, false, 64>, grid, dim3(64), smem, ctx.stream, cs, x1, x2, g.n1, g.n2,
                      epi, rowOut, nonfinite, BandWindow{});
            break;
        default:
            launchPdl(1, k_eval_band<Epi, kGather, false, 32>, grid, dim3(32), smem, ctx.stream, cs, x1, x2, g.n1, g.n2,
                      epi, rowOut, nonfinite, BandWindow{});
            break;
    }
}

// Slab launch: L local rows (blocks) of a grid with n1 global rows, coefficients in a window.
template <class Epi, bool kGather>
void launchEvalBandWindow(Ctx& ctx, int n1, int L, int n2, CoeffSet<1> cs, const double* x1, const double* x2,
                          const Epi& epi, double* rowOut, unsigned* nonfinite, BandWindow win) {
    LaunchScope ls_(ctx, Epi::kName);
    const GridDims gl(L, n2);
    if (bandTW(n2) != kBandThreads) throw NotSupported("slab step: the row length must be a multiple of 256");
    launchPdl(1, k_eval_band<Epi, kGather, true, kBandThreads, double>, dim3(L), dim3(kBandThreads), bandSmem(gl), ctx.stream, cs, x1, x2,
              n1, n2, epi, rowOut, nonfinite, win);
}

}  // namespace vrg
