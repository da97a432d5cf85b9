// Alternating-direction SL step: one kernel per time step with the whole prefilter fused.
//
// The periodic cubic B-spline prefilter is separable, C = P_row P_col m = P_col P_row m, and
// each 1-D filter needs whole lines.  The band path (evalband.cuh) fuses the row pass into the
// step's gather kernel and leaves the column pass as a second kernel per step.  Here the steps
// alternate between two kernel shapes so that no separate pass remains:
//
//   kind A (a block owns R whole ROWS):  input q = P_col m_{j-1} (column-filtered field).  The
//     block stages the rows of q within the departure reach of its own rows (its R rows plus H
//     on each side, a "strip"), row-filters them in shared memory (the rows are complete) into
//     the coefficients, gathers its nodes from shared memory, applies the step epilogue, and
//     row-filters its own new rows: p = P_row m_j, the input of the next (kind B) step.
//   kind B (a block owns R whole COLUMNS): the same with rows and columns exchanged: stages the
//     columns of p within the reach, column-filters them into the coefficients, gathers,
//     and writes q = P_col m_j for the next kind A step.
//
// Per step this moves the strip of the input (R+2H)/R times (L2-resident at the grid sizes
// where lines fit in shared memory), the departure points, the epilogue operands and two
// output fields, with the 16 taps of every node served from shared memory; there is no
// coefficient field in HBM and no second kernel.  Lines of up to ~1100 samples fit (the
// strip of 2H+R lines lives in shared memory), i.e. grids up to 1024 x 1024; larger grids use
// the band path.  The arithmetic of the taps, weights and accumulation is the band kernel's;
// the coefficients differ from the band path's by the order of the two (commuting) 1-D
// filters, i.e. at rounding level.
//
// H = ceil(reach) + 2 lines, reach = the largest departure displacement across lines (cells)
// over the step's characteristics, computed once per velocity (adiReach).  A node whose taps
// fall outside the strip sets *err (the caller then falls back; never silent).
#pragma once

#include "eval.cuh"

namespace vrg {

constexpr int kAdiThreads = 512;
constexpr int kAdiMaxPer = 14;  // nodes per thread: R * line <= kAdiMaxPer * kAdiThreads
constexpr int kAdiMaxSmem = 227 * 1024 - 2048;  // dynamic shared memory per block (+ static, <= 227 KB)

struct AdiPlan {
    bool ok = false;
    int R[2] = {0, 0};       // lines owned per block: [0] kind A (rows), [1] kind B (columns)
    int blocks[2] = {0, 0};
    int H[2] = {0, 0};       // strip halo (lines on each side) per kind
    std::size_t smem[2] = {0, 0};
};

// stride of one staged line: element k at slot(k) (chunk-padded, conflict-free chunk walks),
// + 2 so that consecutive lines start in different 16-byte bank groups
__host__ __device__ constexpr int adiLineStride(int n) { return n + 2 * (n / kL) + 2; }

inline std::size_t adiSmem(int n, int S) {
    return sizeof(double) * (static_cast<std::size_t>(S) * adiLineStride(n) + 3 * static_cast<std::size_t>(S) * (n / kL));
}

// Exact periodic prefilter of `nl` staged lines of length n, in place (chunk-carry form of
// interp.cu / evalband.cuh; every chunk is exact up to z^32 ~ 5e-19 relative).
__device__ __forceinline__ void adiFilterLines(double* sm, int LS, int nl, int n, double* E, double* F0, double* P0) {
    const int nc = n / kL;
    const int tasks = nl * nc;
    for (int task = threadIdx.x; task < tasks; task += blockDim.x) {
        const int l = task / nc, c = task - l * nc;
        const double2* s2 = reinterpret_cast<const double2*>(sm + l * LS + c * kCS);
        double f[kL];
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
        E[task] = a;
        F0[task] = f[0];
        P0[task] = b;
    }
    __syncthreads();
    for (int task = threadIdx.x; task < tasks; task += blockDim.x) {
        const int l = task / nc, c = task - l * nc;
        double2* s2 = reinterpret_cast<double2*>(sm + l * LS + c * kCS);
        double f[kL];
#pragma unroll
        for (int k = 0; k < kL / 2; ++k) {
            const double2 v = s2[k];
            f[2 * k] = v.x;
            f[2 * k + 1] = v.y;
        }
        const ZPow zp;
        const int o = l * nc;
        const int cm1 = c == 0 ? nc - 1 : c - 1, cm2 = cm1 == 0 ? nc - 1 : cm1 - 1;
        const int cp1 = c == nc - 1 ? 0 : c + 1, cp2 = cp1 == nc - 1 ? 0 : cp1 + 1;
        const double cp = E[o + cm1] + zp.p[kL] * E[o + cm2];
        const double cm = kZ * (F0[o + cp1] + P0[o + cp1]) + zp.p[kL + 1] * (F0[o + cp2] + P0[o + cp2]);
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
}

__device__ __forceinline__ void adiCp8(double* dst, const double* src) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(src));
}
__device__ __forceinline__ void adiCp16(double* dst, const double* src) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(src));
}
__device__ __forceinline__ void adiCpWait() { asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory"); }

// kDir 0: kind A (rows), 1: kind B (columns).  `in` = the input filtered along the other axis
// (unpadded n1 x n2), `filtOut` = this step's output filtered along the owned axis (may be
// null for the last step of a solve).  kGather = false: the interpolated field is zero (m~_0).
// The departure points and epilogue operands (per-velocity fields, never written by the
// predecessor) are loaded into registers before the programmatic-dependency wait, so their
// latency overlaps the predecessor's tail and the strip staging; the strip goes global ->
// shared with cp.async (all of it in flight at once).
template <class Epi, int kDir, bool kGather>
__global__ void __launch_bounds__(kAdiThreads, 1)
    k_adi_step(const double* __restrict__ in, const double* __restrict__ x1, const double* __restrict__ x2, int n1,
               int n2, int R, int H, Epi epi, double* __restrict__ filtOut, unsigned* nonfinite, unsigned* err) {
    extern __shared__ __align__(16) double sm[];
    const int n = kDir == 0 ? n2 : n1;       // line length
    const int nLines = kDir == 0 ? n1 : n2;  // lines of the grid along the owned axis
    const int LS = adiLineStride(n);
    const int base = blockIdx.x * R;
    const int Rb = min(R, nLines - base);
    const int S = Rb + 2 * H;
    const int nc = n / kL;
    double* E = sm + static_cast<std::size_t>(R + 2 * H) * LS;
    double* F0 = E + (R + 2 * H) * nc;
    double* P0 = F0 + (R + 2 * H) * nc;
    const int t = threadIdx.x;
    const int nodes = Rb * n;
    auto nodeOf = [&](int idx) -> std::size_t {
        if (kDir == 0) return static_cast<std::size_t>(base) * n2 + idx;  // rows base.. are contiguous
        const int row = idx / Rb;
        return static_cast<std::size_t>(row) * n2 + base + (idx - row * Rb);
    };
    // ---- prologue (independent of the predecessor): departure points, epilogue operands
    double xa[kAdiMaxPer], xb[kAdiMaxPer];
    typename Epi::Pre pre[kAdiMaxPer];
#pragma unroll
    for (int k = 0; k < kAdiMaxPer; ++k) {
        const int idx = t + k * kAdiThreads;
        if (idx < nodes) {
            const std::size_t p = nodeOf(idx);
            if (kGather) {
                xa[k] = __ldg(x1 + p);
                xb[k] = __ldg(x2 + p);
            }
            pre[k] = epi.prefetch(p);
        }
    }
    pdlWait();
    pdlTrigger();
    // ---- stage the strip: lines base-H .. base+Rb+H-1 (periodic) of `in`
    if (kGather) {
        const int warp = t >> 5, lane = t & 31;
        if (kDir == 0) {  // rows: 16-byte granules of contiguous rows
            for (int l = warp; l < S; l += kAdiThreads / 32) {
                int gl = base - H + l;
                gl += gl < 0 ? nLines : 0;
                gl -= gl >= nLines ? nLines : 0;
                const double* src = in + static_cast<std::size_t>(gl) * n2;
                double* dst = sm + l * LS;
                for (int k = 2 * lane; k < n; k += 64) adiCp16(dst + slot(k), src + k);
            }
        } else {  // columns: one grid row per warp iteration, lane l -> strip line l (S <= 32 per pass)
            for (int k = warp; k < n; k += kAdiThreads / 32) {
                const double* src = in + static_cast<std::size_t>(k) * n2;
                for (int l = lane; l < S; l += 32) {
                    int gl = base - H + l;
                    gl += gl < 0 ? nLines : 0;
                    gl -= gl >= nLines ? nLines : 0;
                    adiCp8(sm + l * LS + slot(k), src + gl);
                }
            }
        }
        adiCpWait();
        __syncthreads();
        adiFilterLines(sm, LS, S, n, E, F0, P0);
    }
    // ---- gather + epilogue for the block's nodes (kept in registers)
    const double inv1 = n1 * (1.0 / kTwoPi), inv2 = n2 * (1.0 / kTwoPi);
    double vals[kAdiMaxPer];
    double guard = 0.0;
    bool bad = false, outside = false;
#pragma unroll
    for (int k = 0; k < kAdiMaxPer; ++k) {
        const int idx = t + k * kAdiThreads;
        if (idx >= nodes) break;
        const std::size_t p = nodeOf(idx);
        double val = 0.0;
        if (kGather) {
            double w1[4], w2[4];
            const int b1 = cellBase(xa[k], inv1, n1, w1);  // padded index: tap rows b1-1 .. b1+2
            const int b2 = cellBase(xb[k], inv2, n2, w2);
            // strip line of the first tap along the owned axis, positions along the line
            int l0 = (kDir == 0 ? b1 : b2) - 1 - (base - H);
            l0 += l0 < 0 ? nLines : 0;
            l0 -= l0 >= nLines ? nLines : 0;
            if (l0 < 0 || l0 + 3 >= S) {
                outside = true;
                l0 = 0;
            }
            int pos[4];
            {
                int q = (kDir == 0 ? b2 : b1) - 1;
                q += q < 0 ? n : 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    pos[u] = slot(q);
                    q = q + 1 == n ? 0 : q + 1;
                }
            }
            double tap[16];
            const double* L0 = sm + l0 * LS;
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    tap[4 * a + b] = kDir == 0 ? L0[a * LS + pos[b]] : L0[b * LS + pos[a]];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                double rowAcc = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) rowAcc += w2[b] * tap[4 * a + b];
                val += w1[a] * rowAcc;
            }
        }
        const double o = epi(p, &val, pre[k]);
        const double ao = fabs(o);
        if (ao == ao) guard = fmax(guard, ao);
        bad |= !isfinite(o);
        vals[k] = o;
    }
    if (outside) atomicOr(err, 1u);
    if constexpr (Epi::kGuard) {
        __shared__ double red[kAdiThreads / 32];
        for (int o = 16; o > 0; o >>= 1) guard = fmax(guard, __shfl_xor_sync(0xffffffffu, guard, o));
        if ((t & 31) == 0) red[t >> 5] = guard;
        __syncthreads();
        if (t == 0) {
            double m = red[0];
            for (int w = 1; w < kAdiThreads / 32; ++w) m = fmax(m, red[w]);
            epi.guardPartials[blockIdx.x] = m;
        }
    }
    // the next prefilter's input check (checkFinite(u, "prefilter"), interp.cpp:76)
    if (__syncthreads_or(bad) && t == 0 && nonfinite) atomicOr(nonfinite, 1u);
    if (!filtOut) return;
    // ---- own lines of the new field -> filtered along the owned axis -> filtOut
#pragma unroll
    for (int k = 0; k < kAdiMaxPer; ++k) {
        const int idx = t + k * kAdiThreads;
        if (idx >= nodes) break;
        int l, pos;
        if (kDir == 0) {
            l = idx / n2;
            pos = idx - l * n2;
        } else {
            pos = idx / Rb;
            l = idx - pos * Rb;
        }
        sm[l * LS + slot(pos)] = vals[k];
    }
    __syncthreads();
    adiFilterLines(sm, LS, Rb, n, E, F0, P0);
    if (kDir == 0) {
        for (int i = t; i < nodes; i += kAdiThreads) {
            const int l = i / n2, k = i - l * n2;
            filtOut[static_cast<std::size_t>(base + l) * n2 + k] = sm[l * LS + slot(k)];
        }
    } else {
        for (int i = t; i < nodes; i += kAdiThreads) {
            const int k = i / Rb, l = i - k * Rb;
            filtOut[static_cast<std::size_t>(k) * n2 + base + l] = sm[l * LS + slot(k)];
        }
    }
}

// Plan for a grid and a reach (cells): lines per block for both kinds, strip halo, smem.
AdiPlan adiPlan(const Ctx& ctx, const GridDims& g, double reachRows, double reachCols);

template <class Epi, bool kGather>
void launchAdiStep(Ctx& ctx, const GridDims& g, const AdiPlan& pl, int dir, const double* in, const double* x1,
                   const double* x2, const Epi& epi, double* filtOut, unsigned* nonfinite, unsigned* err) {
    static bool attr[2] = {false, false};  // per template instance: opt in to > 48 KB of shared memory
    if (!attr[dir]) {
        if (dir == 0)
            VRG_CUDA(cudaFuncSetAttribute(k_adi_step<Epi, 0, kGather>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kAdiMaxSmem));
        else
            VRG_CUDA(cudaFuncSetAttribute(k_adi_step<Epi, 1, kGather>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kAdiMaxSmem));
        attr[dir] = true;
    }
    LaunchScope ls_(ctx, Epi::kName);
    if (dir == 0)
        launchPdl(1, k_adi_step<Epi, 0, kGather>, dim3(pl.blocks[0]), dim3(kAdiThreads), pl.smem[0], ctx.stream, in, x1,
                  x2, g.n1, g.n2, pl.R[0], pl.H[0], epi, filtOut, nonfinite, err);
    else
        launchPdl(1, k_adi_step<Epi, 1, kGather>, dim3(pl.blocks[1]), dim3(kAdiThreads), pl.smem[1], ctx.stream, in, x1,
                  x2, g.n1, g.n2, pl.R[1], pl.H[1], epi, filtOut, nonfinite, err);
}

// Largest departure displacement along each axis (cells, minimum image), both characteristics
// given; +inf if any point is non-finite.
void adiReach(Ctx& ctx, const GridDims& g, const double* X, double& rows, double& cols);

}  // namespace vrg
