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
// Exact chunk-carry form (lines of length n, n % 16 == 0, n >= 32): each thread owns a chunk
// of 16 samples held in registers and runs both recurrences with zero initial state:
//   A_k = f_k + z A_{k-1}  (A_{-1} = 0),   B_k = z (f_{k+1} + B_{k+1})  (B_15 = 0).
// The true values are A_k + z^(k+1) c+ and B_k + z^(15-k) c-, with carries from the
// neighbouring chunks of the same (periodic) line
//   c+ = E[c-1] + z^16 E[c-2],                      E = A_15 of a chunk,
//   c- = z (F0[c+1] + P0[c+1]) + z^17 (F0[c+2] + P0[c+2]),   F0 = f_0, P0 = B_0,
// exact up to z^32 ~ 5e-19 relative.  No warm-up work, every sample read once.
constexpr int kL = 16;

// z^i, i = 0..17, folded to compile-time constants.
struct ZPow {
    static constexpr double pw(int i) { return i == 0 ? 1.0 : kZ * pw(i - 1); }
    double p[18];
    __device__ constexpr ZPow() : p{pw(0), pw(1), pw(2), pw(3), pw(4), pw(5), pw(6), pw(7), pw(8),
                                     pw(9), pw(10), pw(11), pw(12), pw(13), pw(14), pw(15), pw(16), pw(17)} {}
};

// Filters the 16 samples at s[0..15] (smem, contiguous) in place given the line's chunk tables.
__device__ __forceinline__ void chunkPhase1(const double* s, double A[kL], double B[kL], double& e, double& f0,
                                            double& p0) {
    double f[kL];
#pragma unroll
    for (int k = 0; k < kL; ++k) f[k] = s[k];
    B[kL - 1] = 0.0;
#pragma unroll
    for (int k = kL - 2; k >= 0; --k) B[k] = kZ * (f[k + 1] + B[k + 1]);
    double p = 0.0;
#pragma unroll
    for (int k = 0; k < kL; ++k) {
        p = f[k] + kZ * p;
        A[k] = p;
    }
    e = A[kL - 1];
    f0 = f[0];
    p0 = B[0];
}

__device__ __forceinline__ void chunkPhase2(double* s, const double A[kL], const double B[kL], double cp, double cm,
                                            const ZPow& zp) {
#pragma unroll
    for (int k = 0; k < kL; ++k) s[k] = kSqrt3 * ((A[k] + zp.p[k + 1] * cp) + (B[k] + zp.p[kL - 1 - k] * cm));
}

// Row pass: `rows` whole rows per block, row-major smem with one pad slot per 16-chunk.
__global__ void __launch_bounds__(256) k_pf_rows(const double* __restrict__ u, double* __restrict__ out, int n1,
                                                 int n2, int rows, unsigned* nonfinite) {
    extern __shared__ double sm[];
    const int nc = n2 / kL;
    const int stride = n2 + nc;
    double* E = sm + rows * stride;
    double* F0 = E + rows * nc;
    double* P0 = F0 + rows * nc;
    const int row0 = blockIdx.x * rows;
    const int nrows = min(rows, n1 - row0);
    const int halfTotal = nrows * n2 / 2;
    const double2* u2 = reinterpret_cast<const double2*>(u + static_cast<std::size_t>(row0) * n2);
    bool bad = false;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < halfTotal; idx += blockDim.x) {
        const double2 v = u2[idx];
        const int i = 2 * idx;
        const int r = i / n2, col = i - r * n2;
        double* d = sm + r * stride + col + col / kL;
        d[0] = v.x;
        d[1] = v.y;
        bad |= !isfinite(v.x) || !isfinite(v.y);
    }
    if (nonfinite) {
        if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1u);
    } else {
        __syncthreads();
    }
    const int t = threadIdx.x;
    const int r = t / nc, c = t - r * nc;
    const bool active = r < nrows;
    double A[kL], B[kL];
    double* s = sm + r * stride + c * (kL + 1);
    if (active) chunkPhase1(s, A, B, E[t], F0[t], P0[t]);
    __syncthreads();
    if (active) {
        const ZPow zp;
        const int base = r * nc;
        const int cm1 = c == 0 ? nc - 1 : c - 1, cm2 = cm1 == 0 ? nc - 1 : cm1 - 1;
        const int cp1 = c == nc - 1 ? 0 : c + 1, cp2 = cp1 == nc - 1 ? 0 : cp1 + 1;
        const double carryP = E[base + cm1] + zp.p[kL] * E[base + cm2];
        const double carryM = kZ * (F0[base + cp1] + P0[base + cp1]) + zp.p[kL + 1] * (F0[base + cp2] + P0[base + cp2]);
        chunkPhase2(s, A, B, carryP, carryM, zp);
    }
    __syncthreads();
    double2* o2 = reinterpret_cast<double2*>(out + static_cast<std::size_t>(row0) * n2);
#pragma unroll 4
    for (int idx = threadIdx.x; idx < halfTotal; idx += blockDim.x) {
        const int i = 2 * idx;
        const int rr = i / n2, col = i - rr * n2;
        const double* d = sm + rr * stride + col + col / kL;
        o2[idx] = make_double2(d[0], d[1]);
    }
}

// Column pass: `W` whole columns per block, column-major smem (one pad per 16-chunk, column
// stride = 4 mod 16 double-banks so the tile loads are conflict-free).
__global__ void __launch_bounds__(512, 1) k_pf_cols(const double* __restrict__ in, double* __restrict__ out, int n1,
                                                  int n2, int W, int colStride) {
    extern __shared__ double sm[];
    const int nc = n1 / kL;
    double* E = sm + W * colStride;
    double* F0 = E + W * nc;
    double* P0 = F0 + W * nc;
    const int c0 = blockIdx.x * W;
    const int ncols = min(W, n2 - c0);
    const int total = n1 * W;
#pragma unroll 8
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int row = idx / W, w = idx - row * W;
        if (w < ncols) sm[w * colStride + row + row / kL] = in[static_cast<std::size_t>(row) * n2 + c0 + w];
    }
    __syncthreads();
    const int t = threadIdx.x;
    const int w = t / nc, c = t - w * nc;
    const bool active = w < ncols;
    double A[kL], B[kL];
    double* s = sm + w * colStride + c * (kL + 1);
    if (active) chunkPhase1(s, A, B, E[t], F0[t], P0[t]);
    __syncthreads();
    if (active) {
        const ZPow zp;
        const int base = w * nc;
        const int cm1 = c == 0 ? nc - 1 : c - 1, cm2 = cm1 == 0 ? nc - 1 : cm1 - 1;
        const int cp1 = c == nc - 1 ? 0 : c + 1, cp2 = cp1 == nc - 1 ? 0 : cp1 + 1;
        const double carryP = E[base + cm1] + zp.p[kL] * E[base + cm2];
        const double carryM = kZ * (F0[base + cp1] + P0[base + cp1]) + zp.p[kL + 1] * (F0[base + cp2] + P0[base + cp2]);
        chunkPhase2(s, A, B, carryP, carryM, zp);
    }
    __syncthreads();
#pragma unroll 8
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int row = idx / W, ww = idx - row * W;
        if (ww < ncols) out[static_cast<std::size_t>(row) * n2 + c0 + ww] = sm[ww * colStride + row + row / kL];
    }
}

struct FastPlan {
    int rows = 0, rowThreads = 0;
    std::size_t rowSmem = 0;
    int W = 0, colThreads = 0, colStride = 0;
    std::size_t colSmem = 0;
};

bool fastAxis(int n) { return n >= 32 && n % kL == 0 && n <= 16384; }

FastPlan fastPlan(const GridDims& g) {
    FastPlan p;
    const int nc2 = g.n2 / kL;
    p.rows = std::max(1, 256 / nc2);
    p.rowThreads = p.rows * nc2;
    p.rowSmem = sizeof(double) * (static_cast<std::size_t>(p.rows) * (g.n2 + nc2) + 3 * p.rows * nc2);
    const int nc1 = g.n1 / kL;
    p.W = std::max(2, 4096 / g.n1);
    p.colThreads = p.W * nc1;
    const int base = g.n1 + nc1;
    p.colStride = base + ((4 - base % 16) + 16) % 16;
    p.colSmem = sizeof(double) * (static_cast<std::size_t>(p.W) * p.colStride + 3 * p.W * nc1);
    return p;
}

}  // namespace

void launchPrefilter(Ctx& ctx, const GridDims& g, const double* u, double* c, double* tmp, unsigned* nonfinite) {
    static std::mutex mu0;
    static std::vector<bool> attr0(64, false);
    {
        std::lock_guard<std::mutex> lock(mu0);
        if (!attr0[ctx.device]) {
            VRG_CUDA(cudaFuncSetAttribute(k_pf_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            VRG_CUDA(cudaFuncSetAttribute(k_pf_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            attr0[ctx.device] = true;
        }
    }
    if (fastAxis(g.n1) && fastAxis(g.n2)) {
        const FastPlan p = fastPlan(g);
        if (p.rowThreads <= 256 && p.colThreads <= 512 && p.rowSmem <= 200 * 1024 && p.colSmem <= 200 * 1024) {
            {
                LaunchScope ls_(ctx, "k_prefilter_rows");
                k_pf_rows<<<(g.n1 + p.rows - 1) / p.rows, p.rowThreads, p.rowSmem, ctx.stream>>>(u, tmp, g.n1, g.n2,
                                                                                                 p.rows, nonfinite);
            }
            VRG_LAUNCH_CHECK();
            {
                LaunchScope ls_(ctx, "k_prefilter_cols");
                k_pf_cols<<<(g.n2 + p.W - 1) / p.W, p.colThreads, p.colSmem, ctx.stream>>>(tmp, c, g.n1, g.n2, p.W,
                                                                                           p.colStride);
            }
            VRG_LAUNCH_CHECK();
            return;
        }
    }
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
        k_prefilter_cols<<<grid, dim3(kColBX, kColBY), smemCols, ctx.stream>>>(tmp, c, g.n1, g.n2);
    }
    VRG_LAUNCH_CHECK();
}

}  // namespace vrg
