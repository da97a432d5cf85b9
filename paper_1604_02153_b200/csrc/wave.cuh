// Building blocks of the persistent dataflow ("wavefront") matvec kernel (inverse.cu, k_wave).
//
// The band path runs every SL step of the GN matvec as two grid-wide kernels (gather +
// epilogue + row pass, then the column pass), and each kernel boundary drains and refills the
// memory pipeline (~3-4 us of a 16 us step on B200).  The dependencies between the two halves
// are local, though: the column pass of a 256-row segment needs the row-filtered rows of that
// segment plus a 32-row halo (the chunk-carry reach), and the gather of a row needs the
// coefficient rows within the departure displacement (+ the 4-tap stencil).  k_wave therefore
// runs the whole time loop in one launch: resident blocks take tasks from a global queue in a
// topological order (row tasks and column-segment tasks, step after step) and each task waits
// only for the row groups / segments it reads, through release/acquire counters in global
// memory.  Dispatch is in queue order, so the earliest unfinished task always has its
// dependencies satisfied (no deadlock, also when not every block is resident).
//
// Data produced inside the kernel is read with coherent loads (plain ld.global), never with
// __ldg / ld.global.nc, whose cache is not kept coherent within a kernel.
#pragma once

#include "evalband.cuh"
#include "interp.cuh"

namespace vrg {

constexpr int kWaveThreads = 256;
constexpr int kWaveRG = 16;     // rows per completion group of the row tasks
constexpr int kWaveHalo = 32;   // chunk-carry reach of the column pass (2 chunks of 16)

__device__ __forceinline__ unsigned ldAcquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void waitAtLeast(const unsigned* p, unsigned target) {
    if (ldAcquire(p) >= target) return;
    while (ldAcquire(p) < target) __nanosleep(64);
}
// Called by all threads of the block after the task's stores: publishes them with release
// semantics at gpu scope (bar.sync orders the block's stores before thread 0's fence).
__device__ __forceinline__ void signalDone(unsigned* c0, unsigned* c1 = nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(c0, 1u);
        if (c1) atomicAdd(c1, 1u);
    }
}

// Coherent load kept in program order relative to the other volatile loads (lets ptxas
// consume taps as they arrive instead of holding all 16 in registers at once).
__device__ __forceinline__ double ldCoherent(const double* p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// One grid row of an SL step: gather at the departure points of row r from the padded
// coefficients (coherent loads), the step epilogue, and, if kFilter, the row pass of the next
// prefilter into rowOut.  Same arithmetic as k_eval_band (evalband.cuh), 256 threads.
// Guard maxima of the epilogue go to epi.guardPartials[r].
template <class Epi, bool kGather, bool kFilter>
__device__ __forceinline__ void waveRowTask(const double* coef, const double* __restrict__ x1,
                                            const double* __restrict__ x2, int n1, int n2, int r, const Epi& epi,
                                            double* rowOut, unsigned* nonfinite, double* sm, double* red, double* Y) {
    const int nc = n2 / kL;
    double* E = sm + nc * kCS;
    double* F0 = E + nc;
    double* P0 = F0 + nc;
    const int t = threadIdx.x;
    const int per = n2 / kWaveThreads;
    const int PW = n2 + 3;
    const double inv1 = n1 * (1.0 / kTwoPi), inv2 = n2 * (1.0 / kTwoPi);
    double guard = 0.0;
    bool bad = false;
    for (int k = 0; k < per; ++k) {
        const int col = t + kWaveThreads * k;
        const int p = r * n2 + col;
        double w1[4], w2[4];
        int base = 0;
        if (kGather) {
            const int b1 = cellBase(__ldg(x1 + p), inv1, n1, w1);
            const int b2 = cellBase(__ldg(x2 + p), inv2, n2, w2);
            base = b1 * PW + b2;
        }
        const typename Epi::Pre pre = epi.prefetch(p);
        double val = 0.0;
        if (kGather) {
            const double* c0 = coef + base;
            double tap[16];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) tap[4 * a + b] = ldCoherent(c0 + a * PW + b);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                double rowAcc = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) rowAcc += w2[b] * tap[4 * a + b];
                val += w1[a] * rowAcc;
            }
        }
        const double o = epi(p, &val, pre);
        const double ao = fabs(o);
        if (ao == ao) guard = fmax(guard, ao);
        bad |= !isfinite(o);
        if (kFilter) sm[slot(col)] = o;
    }
    if constexpr (Epi::kGuard) {
        for (int o = 16; o > 0; o >>= 1) guard = fmax(guard, __shfl_xor_sync(0xffffffffu, guard, o));
        if ((t & 31) == 0) red[t >> 5] = guard;
        __syncthreads();
        if (t == 0) {
            double m = red[0];
            for (int w = 1; w < kWaveThreads / 32; ++w) m = fmax(m, red[w]);
            epi.guardPartials[r] = m;
        }
    }
    if (__syncthreads_or(bad) && t == 0 && nonfinite) atomicOr(nonfinite, 1u);
    if (!kFilter) return;

    // row pass of the prefilter (pfSeg / k_eval_band arithmetic, whole periodic row); the
    // chunk samples are re-read from shared memory in each sweep instead of being held in
    // registers (the persistent kernel has less register room than k_eval_band)
    double2* s2 = reinterpret_cast<double2*>(sm + t * kCS);
    const double* f = sm + t * kCS;
    if (t < nc) {
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
        // anticausal sweep kept in the shared scratch Y ([k][thread], conflict-free)
        double ym = cm;
        Y[(kL - 1) * kWaveThreads + t] = ym;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) {
            ym = kZ * (f[k + 1] + ym);
            Y[k * kWaveThreads + t] = ym;
        }
        double yp = cp;
#pragma unroll
        for (int k = 0; k < kL; k += 2) {
            const double2 v = s2[k / 2];
            yp = v.x + kZ * yp;
            const double o0 = kSqrt3 * (yp + Y[k * kWaveThreads + t]);
            yp = v.y + kZ * yp;
            const double o1 = kSqrt3 * (yp + Y[(k + 1) * kWaveThreads + t]);
            s2[k / 2] = make_double2(o0, o1);
        }
    }
    __syncthreads();
    double* dst = rowOut + static_cast<std::size_t>(r) * n2;
    for (int k = 0; k < per; ++k) {
        const int col = t + kWaveThreads * k;
        dst[col] = sm[slot(col)];
    }
}

// Column pass of one segment (rows s*SR .. s*SR+SR-1) for the CW = 256 / (SR/16) columns of
// group cg, output in the padded coefficient layout: the pfColsReg arithmetic (interp.cu),
// one thread per interior 16-row chunk, with the 2-chunk halo summaries computed by threads
// 0 .. 4 CW - 1.
__device__ __forceinline__ void waveColsTask(const double* in, double* out, int n1, int n2, int SR, int CW, int s,
                                             int cg, double* sm, double* Y) {
    const int icr = SR / kL;   // interior chunk rows
    const int CR = icr + 4;    // with the halo
    double* E = sm;            // [CR][CW]
    double* F0 = E + CR * CW;
    double* P0 = F0 + CR * CW;
    const int t = threadIdx.x;
    const int col = t % CW;
    const int gc = cg * CW + col;
    const int nChunkRows = n1 / kL;
    auto chunkSrc = [&](int ci) {
        int q = (s * icr - 2 + ci) % nChunkRows;
        q = q < 0 ? q + nChunkRows : q;
        return in + static_cast<std::size_t>(q) * kL * n2 + gc;
    };
    auto summarize = [&](int ci) {
        const double* src = chunkSrc(ci);
        double f[kL];
#pragma unroll
        for (int k = 0; k < kL; ++k) f[k] = src[static_cast<std::size_t>(k) * n2];
        double b = 0.0;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) b = kZ * (f[k + 1] + b);
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < kL; ++k) a = f[k] + kZ * a;
        E[ci * CW + col] = a;
        F0[ci * CW + col] = f[0];
        P0[ci * CW + col] = b;
    };
    if (t < 4 * CW) {  // halo chunk rows 0, 1, icr+2, icr+3
        const int h = t / CW;
        summarize(h < 2 ? h : icr + h);
    }
    const bool interior = t < icr * CW;
    const int ci = 2 + t / CW;
    if (interior) summarize(ci);
    __syncthreads();
    if (interior) {
        // both sweeps re-read the chunk (L1 hits) rather than keeping it in registers
        const double* src = chunkSrc(ci);
        const ZPow zp;
        const double cp = E[(ci - 1) * CW + col] + zp.p[kL] * E[(ci - 2) * CW + col];
        const double cm = kZ * (F0[(ci + 1) * CW + col] + P0[(ci + 1) * CW + col]) +
                          zp.p[kL + 1] * (F0[(ci + 2) * CW + col] + P0[(ci + 2) * CW + col]);
        double ym = cm;
        Y[(kL - 1) * kWaveThreads + t] = ym;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) {
            ym = kZ * (src[static_cast<std::size_t>(k + 1) * n2] + ym);
            Y[k * kWaveThreads + t] = ym;
        }
        const int PW = n2 + 3;
        const int colX = gc == n2 - 1 ? 0 : (gc == 0 ? n2 + 1 : (gc == 1 ? n2 + 2 : -1));
        const int r0 = s * SR + (ci - 2) * kL;  // first output row
        const bool edgeRows = r0 == 0 || r0 + kL == n1;
        double yp = cp;
#pragma unroll
        for (int k = 0; k < kL; ++k) {
            yp = src[static_cast<std::size_t>(k) * n2] + kZ * yp;
            const double v = kSqrt3 * (yp + Y[k * kWaveThreads + t]);
            const int q = r0 + k;
            double* r1 = out + static_cast<std::size_t>(q + 1) * PW;
            r1[gc + 1] = v;
            if (colX >= 0) r1[colX] = v;
            if (edgeRows) {
                const int rowX = q == n1 - 1 ? 0 : (q == 0 ? n1 + 1 : (q == 1 ? n1 + 2 : -1));
                if (rowX >= 0) {
                    double* r2 = out + static_cast<std::size_t>(rowX) * PW;
                    r2[gc + 1] = v;
                    if (colX >= 0) r2[colX] = v;
                }
            }
        }
    }
}

// column-task width for a segment height: one thread per interior chunk
inline int waveColsWidth(int SR) { return kWaveThreads / (SR / kL); }
inline std::size_t waveColsSmem(int SR) { return sizeof(double) * 3 * (SR / kL + 4) * waveColsWidth(SR); }
// dynamic shared memory of k_wave: the larger task layout, then the sweep scratch Y
inline std::size_t waveSmemBase(const GridDims& g, int SR) {
    return (std::max(bandSmem(g), waveColsSmem(SR)) + 15) / 16 * 16;
}
inline std::size_t waveSmemFor(const GridDims& g, int SR) {
    return waveSmemBase(g, SR) + sizeof(double) * kL * kWaveThreads;
}

}  // namespace vrg
