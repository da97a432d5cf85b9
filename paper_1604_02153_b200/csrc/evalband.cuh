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

#include "eval.cuh"

namespace vrg {

constexpr int kBandThreads = 256;

// one block per row; n2 a multiple of 256 up to 4096 (chunks per row <= threads)
inline bool bandFusable(const GridDims& g) { return g.n2 >= 256 && g.n2 <= 4096 && g.n2 % 256 == 0; }

inline std::size_t bandSmem(const GridDims& g) {
    const int nc = g.n2 / kL;
    return sizeof(double) * (static_cast<std::size_t>(nc) * kCS + 3 * nc);
}

inline unsigned bandBlocks(const GridDims& g) { return static_cast<unsigned>(g.n1); }

// Without a gather (kGather = false: m~_0 = 0, the first incremental-state step) the epilogue
// operands come from the immediate predecessor (vt_D), so the kernel waits before any load;
// with a gather only the coefficient field is produced by the predecessor and the departure
// points and epilogue operands are loaded before the programmatic-dependency wait.
// Coefficient load that stays behind griddepcontrol.wait.  The wait sits inside the node loop
// (first iteration) and ptxas hoists non-coherent (ld.global.nc / __ldg) gathers of the loop
// body above it, which reads the coefficients before the predecessor column pass has written
// them (seen in the SASS and as nondeterministic results under graph replay).  A coherent
// load is ordered by the wait.
__device__ __forceinline__ double ldAfterWait(const double* p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

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

template <class Epi, bool kGather, bool kWindow = false>
__global__ void __launch_bounds__(kBandThreads, BandMinBlocks<Epi>::value) k_eval_band(CoeffSet<1> cs, const double* __restrict__ x1,
                                                            const double* __restrict__ x2, int n1, int n2, Epi epi,
                                                            double* __restrict__ rowOut, unsigned* nonfinite,
                                                            BandWindow win = BandWindow{}) {
    if (!kGather) pdlWait();
    extern __shared__ __align__(16) double sm[];
    const int nc = n2 / kL;
    double* E = sm + nc * kCS;
    double* F0 = E + nc;
    double* P0 = F0 + nc;
    const int t = threadIdx.x;
    const int r = blockIdx.x;
    const int per = n2 / kBandThreads;  // nodes per thread (<= 16)
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
    double xa = 0.0, xb = 0.0;
    typename Epi::Pre pre{};
    if constexpr (kPipe) {
        if (kGather) {
            xa = __ldg(x1 + r * n2 + t);
            xb = __ldg(x2 + r * n2 + t);
        }
        pre = epi.prefetch(r * n2 + t);
        if (kGather) pdlWait();
    }
    for (int k = 0; k < per; ++k) {
        const int col = t + kBandThreads * k;
        const int p = r * n2 + col;
        double w1[4], w2[4];
        int base = 0;
        typename Epi::Pre cur;
        if constexpr (kPipe) {
            if (kGather) {
                const int b1 = tapRow(cellBase(xa, inv1, n1, w1));
                const int b2 = cellBase(xb, inv2, n2, w2);
                base = b1 * PW + b2;

            }
            cur = pre;
            if (k + 1 < per) {
                if (kGather) {
                    xa = __ldg(x1 + p + kBandThreads);
                    xb = __ldg(x2 + p + kBandThreads);
                }
                pre = epi.prefetch(p + kBandThreads);
            }
        } else {
            if (kGather) {
                const int b1 = tapRow(cellBase(__ldg(x1 + p), inv1, n1, w1));
                const int b2 = cellBase(__ldg(x2 + p), inv2, n2, w2);
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
        __shared__ double red[kBandThreads / 32];
        for (int o = 16; o > 0; o >>= 1) guard = fmax(guard, __shfl_xor_sync(0xffffffffu, guard, o));
        if ((t & 31) == 0) red[t >> 5] = guard;
        __syncthreads();
        if (t == 0) {
            double m = red[0];
            for (int w = 1; w < kBandThreads / 32; ++w) m = fmax(m, red[w]);
            epi.guardPartials[blockIdx.x] = m;
        }
    }
    // the next prefilter's input check (checkFinite(u, "prefilter"), interp.cpp:76)
    if (__syncthreads_or(bad) && t == 0 && nonfinite) atomicOr(nonfinite, 1u);

    // ---- row pass of the prefilter (exact: the whole periodic row is in the block)
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
    __syncthreads();
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
    __syncthreads();
    double* dst = rowOut + static_cast<std::size_t>(r) * n2;
    for (int k = 0; k < per; ++k) {
        const int col = t + kBandThreads * k;
        dst[col] = sm[slot(col)];
    }
    pdlTrigger();  // at the end: the dependent column pass must not take this kernel's slots
}

template <class Epi, bool kGather>
void launchEvalBand(Ctx& ctx, const GridDims& g, CoeffSet<1> cs, const double* x1, const double* x2, const Epi& epi,
                    double* rowOut, unsigned* nonfinite) {
    LaunchScope ls_(ctx, Epi::kName);
    launchPdl(1, k_eval_band<Epi, kGather>, dim3(bandBlocks(g)), dim3(kBandThreads), bandSmem(g), ctx.stream, cs, x1,
              x2, g.n1, g.n2, epi, rowOut, nonfinite, BandWindow{});
}

// Slab launch: L local rows (blocks) of a grid with n1 global rows, coefficients in a window.
template <class Epi, bool kGather>
void launchEvalBandWindow(Ctx& ctx, int n1, int L, int n2, CoeffSet<1> cs, const double* x1, const double* x2,
                          const Epi& epi, double* rowOut, unsigned* nonfinite, BandWindow win) {
    LaunchScope ls_(ctx, Epi::kName);
    const GridDims gl(L, n2);
    launchPdl(1, k_eval_band<Epi, kGather, true>, dim3(L), dim3(kBandThreads), bandSmem(gl), ctx.stream, cs, x1, x2,
              n1, n2, epi, rowOut, nonfinite, win);
}

}  // namespace vrg
