// K1: periodic cubic B-spline prefilter (interp::prefilter, src/interp.cpp:75-85) as two
// shared-memory-tiled recursive-filter passes.  See interp.cuh for the algorithm.
#include "interp.cuh"

namespace vrg {

namespace {

constexpr int kRowThreads = 256;
constexpr int kColBX = 32;  // columns per column-pass block (one warp across)
constexpr int kColBY = 8;   // chunk-threads per column
constexpr int kColRows = kChunk * kColBY;

__device__ __forceinline__ int wrapStep(int j, int n) { return j == n ? 0 : j; }

__device__ __forceinline__ int wrapAny(int j, int n) {
    j %= n;
    return j < 0 ? j + n : j;
}

// Filters one chunk [a, a+lc) of a periodic line of length n whose samples are at(k) for
// k in [0,n).  Results are written to y[0..lc).
template <class At>
__device__ __forceinline__ void filterChunk(const At& at, int n, int a, int lc, double y[kChunk]) {
    // anticausal: y-_k = z (f_{k+1} + y-_{k+1}), started at k = a+lc-1+kWarm with 0
    double ym = 0.0;
    int j = wrapAny(a + lc + kWarm, n);  // index of f_{k+1} for k = a+lc-1+kWarm-1 ... walk down
    // walk k from a+lc-2+kWarm down to a+lc-1 (warm-up), consuming f_{k+1}
    for (int t = 0; t < kWarm; ++t) {
        j = (j == 0 ? n : j) - 1;  // f index a+lc+kWarm-1-t
        ym = kZ * (at(j) + ym);
    }
    // now ym = y-_{a+lc-1}; j = index of a+lc
#pragma unroll
    for (int i = kChunk - 1; i >= 0; --i) {
        if (i < lc) {
            y[i] = ym;
            j = (j == 0 ? n : j) - 1;  // index a+i
            ym = kZ * (at(j) + ym);     // y-_{a+i-1}
        }
    }
    // causal: y+_k = f_k + z y+_{k-1}, started at k = a-kWarm with 0
    double yp = 0.0;
    j = wrapAny(a - kWarm, n);
    for (int t = 0; t < kWarm; ++t) {
        yp = at(j) + kZ * yp;
        j = wrapStep(j + 1, n);
    }
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
        if (i < lc) {
            yp = at(j) + kZ * yp;
            j = wrapStep(j + 1, n);
            y[i] = kSqrt3 * (yp + y[i]);
        }
    }
}

// Row pass: each block stages `rows` whole rows (length n2, padded stride n2+1 to avoid
// bank conflicts), filters chunks in place, stores coalesced.
__global__ void __launch_bounds__(kRowThreads) k_prefilter_rows(const double* __restrict__ u, double* __restrict__ out,
                                                                 int n1, int n2, int rows, unsigned* nonfinite) {
    extern __shared__ double s[];
    const int stride = n2 + 1;
    const int row0 = blockIdx.x * rows;
    const int nrows = min(rows, n1 - row0);
    const int total = nrows * n2;
    bool bad = false;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int r = idx / n2, c = idx - r * n2;
        const double x = u[static_cast<std::size_t>(row0 + r) * n2 + c];
        bad |= !isfinite(x);
        s[r * stride + c] = x;
    }
    if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1u);
    if (!nonfinite) __syncthreads();

    const int chunks = (n2 + kChunk - 1) / kChunk;
    const int task = threadIdx.x;
    const int r = task / chunks;
    const int a = (task - r * chunks) * kChunk;
    const bool active = r < nrows;
    double y[kChunk];
    int lc = 0;
    if (active) {
        lc = min(kChunk, n2 - a);
        const double* line = s + r * stride;
        filterChunk([line](int k) { return line[k]; }, n2, a, lc, y);
    }
    __syncthreads();
    if (active) {
        double* line = s + r * stride;
#pragma unroll
        for (int i = 0; i < kChunk; ++i)
            if (i < lc) line[a + i] = y[i];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int rr = idx / n2, c = idx - rr * n2;
        out[static_cast<std::size_t>(row0 + rr) * n2 + c] = s[rr * stride + c];
    }
}

// Column pass: block = 32 columns x kColRows rows (+kWarm halo rows each side, periodic),
// thread (tx, ty) filters rows [ty*kChunk, +kChunk) of column tx reading the staged tile.
__global__ void __launch_bounds__(kColBX* kColBY) k_prefilter_cols(const double* __restrict__ in,
                                                                   double* __restrict__ out, int n1, int n2) {
    extern __shared__ double s[];
    const int c0 = blockIdx.x * kColBX;
    const int r0 = blockIdx.y * kColRows;
    const int tileRows = kColRows + 2 * kWarm;
    const int tid = threadIdx.y * kColBX + threadIdx.x;
    const int ncols = min(kColBX, n2 - c0);
    for (int idx = tid; idx < tileRows * kColBX; idx += kColBX * kColBY) {
        const int rr = idx / kColBX, cc = idx - rr * kColBX;
        if (cc < ncols) {
            const int gr = wrapAny(r0 - kWarm + rr, n1);
            s[idx] = in[static_cast<std::size_t>(gr) * n2 + c0 + cc];
        }
    }
    __syncthreads();
    const int tx = threadIdx.x;
    const int rs = r0 + threadIdx.y * kChunk;  // first output row of this chunk
    if (tx >= ncols || rs >= n1) return;
    const int lc = min(kChunk, n1 - rs);
    // Local line: tile row index t <-> global row r0 - kWarm + t.  The chunk's recurrences only
    // touch rows [rs-kWarm, rs+lc+kWarm), all inside the tile, so no wrap is needed here.
    const double* col = s + tx;
    const int base = threadIdx.y * kChunk;  // tile row of (rs - kWarm)
    double y[kChunk];
    // anticausal
    double ym = 0.0;
    int t = base + kWarm + lc + kWarm;  // tile row of f_{rs+lc+kWarm}
    for (int k = 0; k < kWarm; ++k) {
        --t;
        ym = kZ * (col[t * kColBX] + ym);
    }
#pragma unroll
    for (int i = kChunk - 1; i >= 0; --i) {
        if (i < lc) {
            y[i] = ym;
            --t;
            ym = kZ * (col[t * kColBX] + ym);
        }
    }
    double yp = 0.0;
    t = base;
    for (int k = 0; k < kWarm; ++k, ++t) yp = col[t * kColBX] + kZ * yp;
#pragma unroll
    for (int i = 0; i < kChunk; ++i) {
        if (i < lc) {
            yp = col[t * kColBX] + kZ * yp;
            ++t;
            out[static_cast<std::size_t>(rs + i) * n2 + c0 + tx] = kSqrt3 * (yp + y[i]);
        }
    }
}

// ------------------------------------------------------------------------------ fast path
// Exact chunk-carry form for axes with n % 16 == 0 and n >= 32.  Each thread owns a chunk of
// 16 samples and runs both recurrences from a zero state:
//   A_k = f_k + z A_{k-1}  (A_{-1} = 0),   B_k = z (f_{k+1} + B_{k+1})  (B_15 = 0).
// The true values are A_k + z^(k+1) c+ and B_k + z^(15-k) c-, with carries from the
// neighbouring chunks of the same periodic line
//   c+ = E[c-1] + z^16 E[c-2],                               E = A_15 of a chunk,
//   c- = z (F0[c+1] + P0[c+1]) + z^17 (F0[c+2] + P0[c+2]),   F0 = f_0, P0 = B_0,
// exact up to z^32 ~ 5e-19 relative.  A block filters a segment of R samples of `lines`
// lines plus a 2-chunk halo on each side (periodic), so any segment is exact on its own.
// Loads go global -> shared with cp.async (no register staging, full memory-level
// parallelism); shared layout pads one slot per 16-chunk so the per-thread chunk walks are
// bank-conflict free.
constexpr int kHalo = 2 * kL;
constexpr int kLines = 8;  // lines per segment block (power of two)
constexpr int kLinesLog2 = kLines == 16 ? 4 : kLines == 8 ? 3 : kLines == 4 ? 2 : 1;


__device__ __forceinline__ void cpAsync8(double* dst, const double* src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}

__device__ __forceinline__ void cpAsyncWaitAll() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}


__device__ __forceinline__ void cpAsync16(double* dst, const double* src) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}


// kRows: lines are rows (positions along axis 1, contiguous); else lines are columns.
// kPadOut (columns pass only): write the coefficients in the periodically padded layout
// (n1+3) x (n2+3), padded(i+1, j+1) = c(i, j) with one wrap row/column before and two after,
// which the evaluation kernels index without any wrap logic.
// kR: interior samples per segment (compile time, so every staging loop fully unrolls);
// the block has kLines * (kR/16 + 4) threads, one per chunk.
template <bool kRows, bool kPadOut, int kR>
__device__ __forceinline__ void pfSeg(const double* __restrict__ in, double* __restrict__ out, int n1, int n2, int LS,
                                      unsigned* nonfinite, int bx, int by, int t, double* sm, bool active) {
    constexpr int S = kR + 2 * kHalo;   // samples staged per line
    constexpr int nch = S / kL;         // chunks per line segment
    constexpr int NT = kLines * nch;    // threads
    const int n = kRows ? n2 : n1;      // line length
    const int nLines = kRows ? n1 : n2;
    const int p0 = bx * kR;             // first interior position
    const int l0 = by * kLines;
    const int lines = active ? min(kLines, nLines - l0) : 0;  // inactive: barriers only
    double* E = sm + kLines * LS;
    double* F0 = E + kLines * nch;
    double* P0 = F0 + kLines * nch;
    // ---- stage global -> shared (periodic halo)
    if (kRows) {
        // S/2 pairs per line, 8 pairs per thread (kLines * S/2 = 8 * NT)
        constexpr int PPL = S / 2;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int i = t + k * NT;
            const int l = i / PPL, pp = i - l * PPL;
            if (l < lines) {
                int q = p0 - kHalo + 2 * pp;
                q = q < 0 ? q + n : (q >= n ? q - n : q);
                cpAsync16(sm + l * LS + slot(2 * pp), in + static_cast<std::size_t>(l0 + l) * n2 + q);
            }
        }
    } else {
        const int l = t & (kLines - 1);
        const int pb = t >> kLinesLog2;  // 0 .. nch-1, stride nch
        if (l < lines) {
            const double* src = in + l0 + l;
            double* dst = sm + l * LS;
#pragma unroll
            for (int i = 0; i < kL; ++i) {  // S = kL * nch positions, nch per sweep
                const int p = pb + i * nch;
                int q = p0 - kHalo + p;
                q = q < 0 ? q + n : (q >= n ? q - n : q);
                cpAsync8(dst + slot(p), src + static_cast<std::size_t>(q) * n2);
            }
        }
    }
    cpAsyncWaitAll();
    __syncthreads();

    // ---- phase 1: zero-state chunk summaries
    const int l = t / nch, c = t - l * nch;
    const bool mine = l < lines;
    double2* s2 = reinterpret_cast<double2*>(sm + l * LS + c * kCS);
    double f[kL];
    bool bad = false;
    if (mine) {
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
        for (int k = 0; k < kL; ++k) {
            a = f[k] + kZ * a;
            bad |= !isfinite(f[k]);
        }
        E[t] = a;
        F0[t] = f[0];
        P0[t] = b;
    }
    if (nonfinite) {
        if (__syncthreads_or(bad) && t == 0) atomicOr(nonfinite, 1u);
    } else {
        __syncthreads();
    }
    // ---- phase 2: both recurrences again from the true chunk-boundary states
    if (mine && c >= 2 && c < nch - 2) {
        const ZPow zp;
        const double cp = E[t - 1] + zp.p[kL] * E[t - 2];  // true y+ before the chunk
        const double cm = kZ * (F0[t + 1] + P0[t + 1]) + zp.p[kL + 1] * (F0[t + 2] + P0[t + 2]);
        double ym[kL];
        ym[kL - 1] = cm;  // true y- at the chunk's last sample
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

    // ---- store the interior
    if (kRows) {
        constexpr int PPL = kR / 2;  // interior pairs per line
        for (int i = t; i < kLines * PPL; i += NT) {
            const int ll = i / PPL, pp = i - ll * PPL;
            if (ll < lines)
                reinterpret_cast<double2*>(out + static_cast<std::size_t>(l0 + ll) * n2 + p0)[pp] =
                    *reinterpret_cast<const double2*>(sm + ll * LS + slot(2 * pp + kHalo));
        }
    } else {
        const int ll = t & (kLines - 1);
        const int pb = t >> kLinesLog2;
        if (ll < lines) {
            const double* src = sm + ll * LS;
            const int col = l0 + ll;
            if (kPadOut) {
                const int PW = n2 + 3;
                const int colX = col == n2 - 1 ? 0 : (col == 0 ? n2 + 1 : (col == 1 ? n2 + 2 : -1));
                const bool edgeRows = p0 == 0 || p0 + kR == n1;  // segment holds row 0, 1 or n1-1
#pragma unroll
                for (int i = 0; i < (kR + nch - 1) / nch; ++i) {
                    const int p = pb + i * nch;
                    if (p < kR) {
                        const double v = src[slot(p + kHalo)];
                        const int q = p0 + p;
                        double* r1 = out + static_cast<std::size_t>(q + 1) * PW;
                        r1[col + 1] = v;
                        if (colX >= 0) r1[colX] = v;
                        if (edgeRows) {
                            const int rowX = q == n1 - 1 ? 0 : (q == 0 ? n1 + 1 : (q == 1 ? n1 + 2 : -1));
                            if (rowX >= 0) {
                                double* r2 = out + static_cast<std::size_t>(rowX) * PW;
                                r2[col + 1] = v;
                                if (colX >= 0) r2[colX] = v;
                            }
                        }
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < (kR + nch - 1) / nch; ++i) {
                    const int p = pb + i * nch;
                    if (p < kR) out[static_cast<std::size_t>(p0 + p) * n2 + col] = src[slot(p + kHalo)];
                }
            }
        }
    }
}

// blockIdx.z: field of a batch (input / output strides inZ / outZ doubles).
template <bool kRows, bool kPadOut, int kR>
__global__ void __launch_bounds__(kLines*(kR / kL + 4)) k_pf_seg(const double* __restrict__ in,
                                                                 double* __restrict__ out, int n1, int n2, int LS,
                                                                 unsigned* nonfinite, std::size_t inZ, std::size_t outZ) {
    extern __shared__ __align__(16) double sm[];
    pdlWait();  // the input is the predecessor's output
    pdlTrigger();
    pfSeg<kRows, kPadOut, kR>(in + blockIdx.z * inZ, out + blockIdx.z * outZ, n1, n2, LS, nonfinite, blockIdx.x,
                              blockIdx.y, threadIdx.x, sm, true);
}

// Periodic padding of an unpadded field (for coefficient sets that arrive unpadded).
__global__ void k_pad(const double* __restrict__ c, double* __restrict__ out, int n1, int n2) {
    const int PW = n2 + 3, PH = n1 + 3;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= PW || i >= PH) return;
    int si = i - 1, sj = j - 1;
    si = si < 0 ? si + n1 : (si >= n1 ? si - n1 : si);
    sj = sj < 0 ? sj + n2 : (sj >= n2 ? sj - n2 : sj);
    out[static_cast<std::size_t>(i) * PW + j] = c[static_cast<std::size_t>(si) * n2 + sj];
}

__global__ void k_unpad(const double* __restrict__ pc, double* __restrict__ out, int n1, int n2) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= n2) return;
    out[static_cast<std::size_t>(i) * n2 + j] = pc[static_cast<std::size_t>(i + 1) * (n2 + 3) + j + 1];
}

struct SegPlan {
    int R = 0, LS = 0, threads = 0;
    std::size_t smem = 0;
    bool ok = false;
};

SegPlan segPlan(int n) {
    SegPlan p;
    for (int r : {256, 128, 64, 32})
        if (n >= 32 && n % r == 0) {
            p.R = r;
            break;
        }
    if (!p.R) return p;
    const int nch = (p.R + 2 * kHalo) / kL;
    const int base = nch * kCS;
    p.LS = base + ((2 - base % 16) + 16) % 16;  // even, = 2 mod 16 (conflict-free column loads)
    p.threads = kLines * nch;
    p.smem = sizeof(double) * (static_cast<std::size_t>(kLines) * p.LS + 3 * kLines * nch);
    p.ok = true;
    return p;
}

template <bool kRows, bool kPad, int kR>
void launchSeg(Ctx& ctx, const GridDims& g, const SegPlan& p, const double* in, double* out, unsigned* nonfinite,
               int count, std::size_t inZ, std::size_t outZ) {
    const int n = kRows ? g.n2 : g.n1, lines = kRows ? g.n1 : g.n2;
    launchPdl(2, k_pf_seg<kRows, kPad, kR>, dim3(n / kR, (lines + kLines - 1) / kLines, count), dim3(p.threads),
              p.smem, ctx.stream, in, out, g.n1, g.n2, p.LS, nonfinite, inZ, outZ);
}

template <bool kRows, bool kPad>
void launchSegR(Ctx& ctx, const GridDims& g, const SegPlan& p, const double* in, double* out, unsigned* nonfinite,
                int count = 1, std::size_t inZ = 0, std::size_t outZ = 0) {
    switch (p.R) {
        case 256: launchSeg<kRows, kPad, 256>(ctx, g, p, in, out, nonfinite, count, inZ, outZ); break;
        case 128: launchSeg<kRows, kPad, 128>(ctx, g, p, in, out, nonfinite, count, inZ, outZ); break;
        case 64: launchSeg<kRows, kPad, 64>(ctx, g, p, in, out, nonfinite, count, inZ, outZ); break;
        default: launchSeg<kRows, kPad, 32>(ctx, g, p, in, out, nonfinite, count, inZ, outZ); break;
    }
}

// Column pass with the samples in registers: thread (column c0+col, chunk row cr) loads the
// 16 rows of its chunk straight from global memory (each load coalesced over the 16 columns of
// the block), so no shared staging of samples is needed; only the chunk summaries go through
// shared memory.  kCR = kR/16 + 4 chunk rows (2-chunk periodic halo above and below); output
// in the padded coefficient layout.
constexpr int kColW = 16;

template <int kR>
struct ColsShared {
    static constexpr int kCR = kR / kL + 4;
    double E[kCR][kColW], F0[kCR][kColW], P0[kCR][kColW];
};

// One column segment (block coordinates bx = row segment, by = column group); all threads of
// the block take part in the barrier whether or not their column exists (loop-safe).
template <int kR>
__device__ __forceinline__ void pfColsReg(const double* __restrict__ in, double* __restrict__ out, int n1, int n2,
                                          int bx, int by, int t, ColsShared<kR>& sh) {
    constexpr int kCR = kR / kL + 4;
    const int col = t & (kColW - 1);
    const int cr = t / kColW;
    const int gc = by * kColW + col;
    const int p0 = bx * kR;
    const bool active = gc < n2;
    double f[kL];
    if (active) {
        int q = p0 - kHalo + cr * kL;  // first row of this chunk (may wrap)
        q = q < 0 ? q + n1 : (q >= n1 ? q - n1 : q);
        const double* src = in + gc;
#pragma unroll
        for (int k = 0; k < kL; ++k) {
            f[k] = __ldg(src + static_cast<std::size_t>(q) * n2);
            q = q + 1 == n1 ? 0 : q + 1;
        }
        double b = 0.0;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) b = kZ * (f[k + 1] + b);
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < kL; ++k) a = f[k] + kZ * a;
        sh.E[cr][col] = a;
        sh.F0[cr][col] = f[0];
        sh.P0[cr][col] = b;
    }
    __syncthreads();
    if (active && cr >= 2 && cr < kCR - 2) {
        const ZPow zp;
        const double cp = sh.E[cr - 1][col] + zp.p[kL] * sh.E[cr - 2][col];
        const double cm = kZ * (sh.F0[cr + 1][col] + sh.P0[cr + 1][col]) +
                          zp.p[kL + 1] * (sh.F0[cr + 2][col] + sh.P0[cr + 2][col]);
        double ym[kL];
        ym[kL - 1] = cm;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) ym[k] = kZ * (f[k + 1] + ym[k + 1]);
        const int PW = n2 + 3;
        const int colX = gc == n2 - 1 ? 0 : (gc == 0 ? n2 + 1 : (gc == 1 ? n2 + 2 : -1));
        const int r0 = p0 + (cr - 2) * kL;  // first output row
        const bool edgeRows = r0 == 0 || r0 + kL == n1;
        double yp = cp;
#pragma unroll
        for (int k = 0; k < kL; ++k) {
            yp = f[k] + kZ * yp;
            const double v = kSqrt3 * (yp + ym[k]);
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

template <int kR>
__global__ void __launch_bounds__(kColW*(kR / kL + 4)) k_pf_cols_reg(const double* __restrict__ in,
                                                                     double* __restrict__ out, int n1, int n2,
                                                                     std::size_t inZ, std::size_t outZ) {
    __shared__ ColsShared<kR> sh;
    pdlWait();  // the input is the predecessor's output
    pfColsReg<kR>(in + blockIdx.z * inZ, out + blockIdx.z * outZ, n1, n2, blockIdx.x, blockIdx.y, threadIdx.x, sh);
    pdlTrigger();  // at the end (common.cuh kPdlMask)
}

template <int kR>
void launchColsReg(Ctx& ctx, const GridDims& g, const double* in, double* out, int count, std::size_t inZ,
                   std::size_t outZ) {
    launchPdl(2, k_pf_cols_reg<kR>, dim3(g.n1 / kR, (g.n2 + kColW - 1) / kColW, count), dim3(kColW * (kR / kL + 4)),
              0, ctx.stream, in, out, g.n1, g.n2, inZ, outZ);
}

// Column pass into the padded layout; false if n1 is not a multiple of 32.  `count` fields at
// strides inZ / outZ doubles (one launch).
bool launchColumnPass(Ctx& ctx, const GridDims& g, const double* in, double* out, int count = 1, std::size_t inZ = 0,
                      std::size_t outZ = 0) {
    SegPlan pc = segPlan(g.n1);
    if (!pc.ok) return false;
    {
        LaunchScope ls_(ctx, "k_prefilter_cols");
        switch (pc.R) {
            case 256: launchColsReg<256>(ctx, g, in, out, count, inZ, outZ); break;
            case 128: launchColsReg<128>(ctx, g, in, out, count, inZ, outZ); break;
            case 64: launchColsReg<64>(ctx, g, in, out, count, inZ, outZ); break;
            default: launchColsReg<32>(ctx, g, in, out, count, inZ, outZ); break;
        }
    }
    VRG_LAUNCH_CHECK();
    return true;
}

// Column pass of a slab's coefficient window (slab.py): `in` holds winRows + 64 row-filtered
// rows (window rows -32 .. winRows+31, i.e. the halo the chunk carry needs is already there,
// exchanged from the neighbouring slabs), `out` the winRows x (n2+3) window with the columns
// periodically padded like the full layout.  Same per-chunk arithmetic as pfColsReg, no wrap
// along axis 1.  Block: 16 columns x (16 output chunks + 4 halo chunks).
__global__ void __launch_bounds__(kColW * 20) k_slab_cols(const double* __restrict__ in, double* __restrict__ out,
                                                          int winRows, int n2) {
    __shared__ double E[20][kColW], F0[20][kColW], P0[20][kColW];
    pdlWait();
    pdlTrigger();
    const int t = threadIdx.x;
    const int col = t % kColW;
    const int cr = t / kColW;
    const int gc = blockIdx.y * kColW + col;
    const int inChunks = winRows / kL + 4;
    const int ic = blockIdx.x * 16 + cr;  // input chunk (output chunk + 2)
    const bool active = gc < n2 && ic < inChunks;
    double f[kL];
    if (active) {
        const double* src = in + static_cast<std::size_t>(ic) * kL * n2 + gc;
#pragma unroll
        for (int k = 0; k < kL; ++k) f[k] = __ldg(src + static_cast<std::size_t>(k) * n2);
        double b = 0.0;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) b = kZ * (f[k + 1] + b);
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < kL; ++k) a = f[k] + kZ * a;
        E[cr][col] = a;
        F0[cr][col] = f[0];
        P0[cr][col] = b;
    }
    __syncthreads();
    if (active && cr >= 2 && cr < 18 && ic < inChunks - 2) {
        const ZPow zp;
        const double cp = E[cr - 1][col] + zp.p[kL] * E[cr - 2][col];
        const double cm = kZ * (F0[cr + 1][col] + P0[cr + 1][col]) + zp.p[kL + 1] * (F0[cr + 2][col] + P0[cr + 2][col]);
        double ym[kL];
        ym[kL - 1] = cm;
#pragma unroll
        for (int k = kL - 2; k >= 0; --k) ym[k] = kZ * (f[k + 1] + ym[k + 1]);
        const int PW = n2 + 3;
        const int colX = gc == n2 - 1 ? 0 : (gc == 0 ? n2 + 1 : (gc == 1 ? n2 + 2 : -1));
        const int r0 = (ic - 2) * kL;  // first window row
        double yp = cp;
#pragma unroll
        for (int k = 0; k < kL; ++k) {
            yp = f[k] + kZ * yp;
            const double v = kSqrt3 * (yp + ym[k]);
            double* r1 = out + static_cast<std::size_t>(r0 + k) * PW;
            r1[gc + 1] = v;
            if (colX >= 0) r1[colX] = v;
        }
    }
}

}  // namespace

bool colPassFusable(const GridDims& g) { return segPlan(g.n1).ok; }

void launchSlabCols(Ctx& ctx, int winRows, int n2, const double* inHalo, double* window) {
    if (winRows % kL != 0 || winRows <= 0) throw InvalidArgument("slab column pass: window rows must be a multiple of 16");
    LaunchScope ls_(ctx, "k_slab_cols");
    launchPdl(2, k_slab_cols, dim3((winRows / kL + 15) / 16, (n2 + kColW - 1) / kColW), dim3(kColW * 20), 0,
              ctx.stream, inHalo, window, winRows, n2);
}

void launchPrefilterBatch(Ctx& ctx, const GridDims& g, const double* u, std::size_t uStride, int count, double* c,
                          std::size_t cStride, double* tmp, unsigned* nonfinite) {
    if (count <= 0) return;
    const SegPlan pr = segPlan(g.n2), pc = segPlan(g.n1);
    const bool packed = g.pairs == 1 || (uStride == g.points() && cStride == paddedTotal(g));
    if (!(pr.ok && pc.ok) || !packed || uStride < g.points() || cStride < paddedTotal(g)) {
        for (int k = 0; k < count; ++k) launchPrefilter(ctx, g, u + k * uStride, c + k * cStride, tmp, nonfinite);
        return;
    }
    {
        // rows are independent: the pairs' rows form one (pairs * n1) x n2 row set
        LaunchScope ls_(ctx, "k_prefilter_rows");
        launchSegR<true, false>(ctx, GridDims(g.n1 * g.pairs, g.n2), pr, u, tmp, nonfinite, count, uStride,
                                g.points());
    }
    VRG_LAUNCH_CHECK();
    // columns are periodic per pair: count * pairs column sets, one pair's field apart
    launchColumnPass(ctx, g.one(), tmp, c, count * g.pairs, g.pointsPer(), paddedPoints(g.n1, g.n2));
}

void launchPrefilterRows(Ctx& ctx, const GridDims& g, const double* u, double* rowFiltered, unsigned* nonfinite) {
    const SegPlan pr = segPlan(g.n2);
    if (!pr.ok) throw NotSupported("prefilter row pass: n2 must be a multiple of 32");
    launchSegR<true, false>(ctx, GridDims(g.n1 * g.pairs, g.n2), pr, u, rowFiltered, nonfinite);
    VRG_LAUNCH_CHECK();
}

void launchPrefilterCols(Ctx& ctx, const GridDims& g, const double* rowFiltered, double* c) {
    if (!launchColumnPass(ctx, g.one(), rowFiltered, c, g.pairs, g.pointsPer(), paddedPoints(g.n1, g.n2)))
        throw NotSupported("prefilter column pass: n1 must be a multiple of 32");
}

void launchPrefilter(Ctx& ctx, const GridDims& g, const double* u, double* c, double* tmp, unsigned* nonfinite) {
    const SegPlan pr = segPlan(g.n2), pc = segPlan(g.n1);
    if (pr.ok && pc.ok) {
        {
            LaunchScope ls_(ctx, "k_prefilter_rows");
            launchSegR<true, false>(ctx, GridDims(g.n1 * g.pairs, g.n2), pr, u, tmp, nonfinite);
        }
        VRG_LAUNCH_CHECK();
        launchColumnPass(ctx, g.one(), tmp, c, g.pairs, g.pointsPer(), paddedPoints(g.n1, g.n2));
        return;
    }
    if (g.pairs > 1) {  // generic path: pair by pair
        for (int k = 0; k < g.pairs; ++k)
            launchPrefilter(ctx, g.one(), u + k * g.pointsPer(), c + k * paddedPoints(g.n1, g.n2), tmp, nonfinite);
        return;
    }
    double* tmp2 = tmp + g.points();  // unpadded column-pass output of the generic path
    // generic path (small or non-multiple-of-16 axes): warm-up recurrences
    const int chunks = (g.n2 + kChunk - 1) / kChunk;
    if (chunks > kRowThreads) throw NotSupported("prefilter: n2 > 8192 not supported");
    const int rows = std::max(1, kRowThreads / chunks);
    const std::size_t smemRows = static_cast<std::size_t>(rows) * (g.n2 + 1) * sizeof(double);
    static std::mutex mu;
    static std::vector<bool> attrDone(64, false);
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!attrDone[ctx.device]) {
            VRG_CUDA(cudaFuncSetAttribute(k_prefilter_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
            VRG_CUDA(cudaFuncSetAttribute(k_prefilter_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
            attrDone[ctx.device] = true;
        }
    }
    {
        LaunchScope ls_(ctx, "k_prefilter_rows");
        k_prefilter_rows<<<(g.n1 + rows - 1) / rows, kRowThreads, smemRows, ctx.stream>>>(u, tmp, g.n1, g.n2, rows,
                                                                                          nonfinite);
    }
    VRG_LAUNCH_CHECK();
    const std::size_t smemCols = static_cast<std::size_t>(kColRows + 2 * kWarm) * kColBX * sizeof(double);
    dim3 grid((g.n2 + kColBX - 1) / kColBX, (g.n1 + kColRows - 1) / kColRows);
    {
        LaunchScope ls_(ctx, "k_prefilter_cols");
        k_prefilter_cols<<<grid, dim3(kColBX, kColBY), smemCols, ctx.stream>>>(tmp, tmp2, g.n1, g.n2);
    }
    VRG_LAUNCH_CHECK();
    launchPad(ctx, g, tmp2, c);
}

void launchPad(Ctx& ctx, const GridDims& g, const double* c, double* padded) {
    {
        LaunchScope ls_(ctx, "k_pad");
        k_pad<<<dim3((g.n2 + 3 + 127) / 128, g.n1 + 3), 128, 0, ctx.stream>>>(c, padded, g.n1, g.n2);
    }
    VRG_LAUNCH_CHECK();
}

void launchUnpad(Ctx& ctx, const GridDims& g, const double* padded, double* c) {
    {
        LaunchScope ls_(ctx, "k_unpad");
        k_unpad<<<dim3((g.n2 + 127) / 128, g.n1), 128, 0, ctx.stream>>>(padded, c, g.n1, g.n2);
    }
    VRG_LAUNCH_CHECK();
}

namespace {
// Departure cells of N nodes (x1 = X[0..N), x2 = X[N..2N)): cells[p] / cells[N + p].
__global__ void k_pack_cells(const double* __restrict__ X, std::size_t N, int n1, int n2, Cell* __restrict__ cells) {
    const std::size_t p = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= N) return;
    cells[p] = cellPack(X[p], n1 * (1.0 / kTwoPi), n1);
    cells[N + p] = cellPack(X[N + p], n2 * (1.0 / kTwoPi), n2);
}
}  // namespace

void launchPackCells(Ctx& ctx, const GridDims& g, const double* X, Cell* cells) {
    if (g.n1 > kCellMaxN || g.n2 > kCellMaxN) throw NotSupported("departure cells: axis longer than 8192");
    const std::size_t N = g.points();
    {
        LaunchScope ls_(ctx, "k_pack_cells");
        k_pack_cells<<<static_cast<unsigned>((N + 255) / 256), 256, 0, ctx.stream>>>(X, N, g.n1, g.n2, cells);
    }
    VRG_LAUNCH_CHECK();
}

}  // namespace vrg
