// K2 + K1(rows) fused: B-spline evaluation with the step epilogue over full-width row bands,
// followed in the same kernel by the row pass of the next step's prefilter.
//
// In the matvec time loops every interpolated field (m~_j, lt_j) is produced by the previous
// step's gather, so the producer can row-filter it while the band is still in shared memory:
// a block owns B = 4096/n2 whole rows (256 chunks of 16 samples), so the periodic row filter
// is exact inside the block (chunk-carry form of interp.cu) and only the column pass remains
// as a separate kernel.  This removes one kernel and one field write+read per step.
#pragma once

#include "eval.cuh"

namespace vrg {

constexpr int kBandThreads = 256;

// Band kernels need n2 a power of two in [32, 4096] and n1 divisible by 4096/n2.
inline bool bandFusable(const GridDims& g) {
    const int n2 = g.n2;
    if (n2 < 32 || n2 > 4096 || (n2 & (n2 - 1)) != 0) return false;
    const int B = 4096 / n2;
    return g.n1 % B == 0;
}

inline int bandLineStride(int n2) { return (n2 / kL) * kCS; }  // even

inline std::size_t bandSmem(const GridDims& g) {
    const int B = 4096 / g.n2;
    return sizeof(double) * (static_cast<std::size_t>(B) * bandLineStride(g.n2) + 3 * kBandThreads);
}

inline unsigned bandBlocks(const GridDims& g) { return static_cast<unsigned>(g.n1 / (4096 / g.n2)); }

template <class Epi, bool kGather>
__global__ void __launch_bounds__(kBandThreads) k_eval_band(CoeffSet<1> cs, const double* __restrict__ x1,
                                                            const double* __restrict__ x2, int n1, int n2,
                                                            int log2n2, Epi epi, double* __restrict__ rowOut,
                                                            unsigned* nonfinite) {
    extern __shared__ __align__(16) double sm[];
    const int nc = n2 / kL;         // chunks per row
    const int B = kBandThreads / nc;  // rows per band
    const int LS = nc * kCS;
    const int r0 = blockIdx.x * B;
    double* E = sm + B * LS;
    double* F0 = E + kBandThreads;
    double* P0 = F0 + kBandThreads;
    const int t = threadIdx.x;
    const int PW = n2 + 3;
    const double inv1 = n1 * (1.0 / kTwoPi), inv2 = n2 * (1.0 / kTwoPi);

    // ---- gather + epilogue, 16 nodes per thread, coalesced along the rows
    double guard = 0.0;
    bool bad = false;
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
        const int idx = t + kBandThreads * k;
        const int lr = idx >> log2n2, col = idx - (lr << log2n2);
        const int p = (r0 + lr) * n2 + col;
        double val = 0.0;
        if (kGather) {
            double w1[4], w2[4];
            const int b1 = cellBase(__ldg(x1 + p), inv1, n1, w1);
            const int b2 = cellBase(__ldg(x2 + p), inv2, n2, w2);
            const double* c0 = cs.c[0] + b1 * PW + b2;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const double* row = c0 + a * PW;
                double rowAcc = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) rowAcc += w2[b] * __ldg(row + b);
                val += w1[a] * rowAcc;
            }
        }
        const double o = epi(p, &val, epi.prefetch(p));
        const double ao = fabs(o);
        if (ao == ao) guard = fmax(guard, ao);
        bad |= !isfinite(o);
        sm[lr * LS + slot(col)] = o;
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

    // ---- row pass of the prefilter on the band (exact: whole periodic rows in the block)
    const int l = t / nc, c = t - l * nc;
    double2* s2 = reinterpret_cast<double2*>(sm + l * LS + c * kCS);
    double f[kL];
#pragma unroll
    for (int k = 0; k < kL / 2; ++k) {
        const double2 v = s2[k];
        f[2 * k] = v.x;
        f[2 * k + 1] = v.y;
    }
    {
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
    {
        const ZPow zp;
        const int base = l * nc;
        const int cm1 = c == 0 ? nc - 1 : c - 1, cm2 = cm1 == 0 ? nc - 1 : cm1 - 1;
        const int cp1 = c == nc - 1 ? 0 : c + 1, cp2 = cp1 == nc - 1 ? 0 : cp1 + 1;
        const double cp = E[base + cm1] + zp.p[kL] * E[base + cm2];
        const double cm = kZ * (F0[base + cp1] + P0[base + cp1]) + zp.p[kL + 1] * (F0[base + cp2] + P0[base + cp2]);
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
    double* dst = rowOut + static_cast<std::size_t>(r0) * n2;
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
        const int idx = t + kBandThreads * k;
        const int lr = idx >> log2n2, col = idx - (lr << log2n2);
        dst[idx] = sm[lr * LS + slot(col)];
    }
}

template <class Epi, bool kGather>
void launchEvalBand(Ctx& ctx, const GridDims& g, CoeffSet<1> cs, const double* x1, const double* x2, const Epi& epi,
                    double* rowOut, unsigned* nonfinite) {
    int log2n2 = 0;
    while ((1 << log2n2) < g.n2) ++log2n2;
    {
        LaunchScope ls_(ctx, Epi::kName);
        k_eval_band<Epi, kGather><<<bandBlocks(g), kBandThreads, bandSmem(g), ctx.stream>>>(cs, x1, x2, g.n1, g.n2,
                                                                                            log2n2, epi, rowOut,
                                                                                            nonfinite);
    }
    VRG_LAUNCH_CHECK();
}

}  // namespace vrg
