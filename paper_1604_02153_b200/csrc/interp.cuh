// Periodic cubic B-spline interpolation on sm_100a: prefilter (K1) and evaluation at departure
// points with fused epilogues (K2).  Restates interp::prefilter / interp::evaluate
// (src/interp.cpp:16-127) with a GPU-shaped algorithm; see DESIGN.md "K1/K2".
#pragma once

#include "common.cuh"

namespace vrg {

// Recursive-filter form of the periodic prefilter.  The exact inverse of circulant
// [1/6, 2/3, 1/6] is c_k = sqrt(3) * sum_m z^|m| f_{k+m}, z = sqrt(3)-2; it splits into a
// causal recurrence y+_k = f_k + z y+_{k-1} and an anticausal one y-_k = z (f_{k+1} + y-_{k+1}),
// c = sqrt(3) (y+ + y-).  Each thread filters a chunk of kChunk outputs, starting both
// recurrences kWarm samples outside the chunk (periodic wrap); the neglected tail is
// 2.4 |z|^(kWarm+1) max|f| < 1e-16 max|f|.  The reference solves the same system exactly with
// Thomas + Sherman-Morrison (src/interp.cpp:16-57); both agree to rounding.
constexpr double kZ = -0.26794919243112270647;   // sqrt(3) - 2
constexpr double kSqrt3 = 1.7320508075688772935;
constexpr int kWarm = 28;
constexpr int kChunk = 32;
constexpr int kL = 16;  // chunk of the exact chunk-carry filter (interp.cu)

// z^i, i = 0..17, folded to compile-time constants.
struct ZPow {
    static constexpr double pw(int i) { return i == 0 ? 1.0 : kZ * pw(i - 1); }
    double p[18];
    __device__ constexpr ZPow() : p{pw(0), pw(1), pw(2), pw(3), pw(4), pw(5), pw(6), pw(7), pw(8),
                                     pw(9), pw(10), pw(11), pw(12), pw(13), pw(14), pw(15), pw(16), pw(17)} {}
};

// Shared layout of one staged line: chunk c (16 samples) at offset kCS*c, kCS = 18 doubles, so
// chunk starts are 16-byte aligned (16-byte cp.async and LDS.128/STS.128) and consecutive
// chunks fall in distinct 16-byte bank groups.
constexpr int kCS = 18;
__device__ __forceinline__ int slot(int p) { return p + 2 * (p >> 4); }

// Launches the two prefilter passes (rows of length n2, then columns of length n1) on
// ctx.stream: c = P u, written in the periodically padded layout of paddedPoints(n1, n2)
// doubles (see cellBase).  `tmp` holds 2*n1*n2 doubles.  If `nonfinite` is non-null, a
// non-finite input value sets *nonfinite = 1 (checkFinite(u, "prefilter"), interp.cpp:76).
void launchPrefilter(Ctx& ctx, const GridDims& g, const double* u, double* c, double* tmp, unsigned* nonfinite);
// `count` fields u + k*uStride -> padded coefficients c + k*cStride in two launches (rows, then
// columns, blockIdx.z = field); tmp holds count*n1*n2 doubles.  Grids off the segment path
// loop over launchPrefilter (tmp then needs 2*n1*n2).
void launchPrefilterBatch(Ctx& ctx, const GridDims& g, const double* u, std::size_t uStride, int count, double* c,
                          std::size_t cStride, double* tmp, unsigned* nonfinite);
// Column pass only (input already row-filtered, e.g. by a fused band kernel, evalband.cuh).
bool colPassFusable(const GridDims& g);
void launchPrefilterCols(Ctx& ctx, const GridDims& g, const double* rowFiltered, double* c);
// Row pass only (rowFiltered unpadded n1 x n2); used per slab, whose rows are complete.
void launchPrefilterRows(Ctx& ctx, const GridDims& g, const double* u, double* rowFiltered, unsigned* nonfinite);
// Column pass of a slab's coefficient window from winRows + 64 row-filtered rows (slab.py).
void launchSlabCols(Ctx& ctx, int winRows, int n2, const double* inHalo, double* window);

// B-spline weights, src/interp.cpp:59-65 (the /6 as a multiply by 1/6: <= 1 ulp apart).
__device__ __forceinline__ void bsplineWeights(double f, double w[4]) {
    constexpr double k6 = 1.0 / 6.0;
    const double f2 = f * f, f3 = f2 * f;
    w[0] = (1.0 - 3.0 * f + 3.0 * f2 - f3) * k6;
    w[1] = (3.0 * f3 - 6.0 * f2 + 4.0) * k6;
    w[2] = (-3.0 * f3 + 3.0 * f2 + 3.0 * f + 1.0) * k6;
    w[3] = f3 * k6;
}

// Cell index and fractional offset of a coordinate along one axis, src/interp.cpp:100-109.
// The reference divides by 2pi and by h; here both are multiplies by the reciprocals
// (`invh` = 1/h), which moves s by at most an ulp — the spline is C2 across cell and wrap
// boundaries, so a flipped floor() changes the value only at rounding level.
__device__ __forceinline__ void cellOf(double x, double invh, int n, int idx[4], double w[4]) {
    constexpr double kInv2Pi = 1.0 / kTwoPi;
    const double xw = __dsub_rn(x, __dmul_rn(kTwoPi, floor(__dadd_rn(x, kPi) * kInv2Pi)));
    const double s = __dadd_rn(xw, kPi) * invh;
    const double bf = floor(s);
    bsplineWeights(s - bf, w);
    int b = static_cast<int>(bf) - 1;
    // b in [-1, n] for finite wrapped points; wrapIndex of src/interp.cpp:67-71
    b = b < 0 ? b + n : (b >= n ? b - n : b);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        idx[t] = b;
        b = (b + 1 == n) ? 0 : b + 1;
    }
}

// Same cell computation for the periodically padded coefficient layout ((n1+3) x (n2+3),
// padded(i+1, j+1) = c(i, j)): returns the padded index of the first tap, taps are
// first + 0..3 along the axis with no wrap.
__device__ __forceinline__ int cellBase(double x, double invh, int n, double w[4]) {
    constexpr double kInv2Pi = 1.0 / kTwoPi;
    const double xw = __dsub_rn(x, __dmul_rn(kTwoPi, floor(__dadd_rn(x, kPi) * kInv2Pi)));
    const double s = __dadd_rn(xw, kPi) * invh;
    const double bf = floor(s);
    bsplineWeights(s - bf, w);
    // in [0, n] for finite wrapped points; clamped so that no input (NaN, or a coordinate too
    // large for the wrap to be exact) can address outside the padded field
    const int b = static_cast<int>(fmin(fmax(bf, 0.0), static_cast<double>(n)));
    return b >= n ? b - n : b;
}

// Departure cells: the per-iterate departure points of the SL time loops, reduced once to what
// the gather needs.  One 64-bit word per node and axis: the padded-layout first-tap index b
// (cellBase; 13 bits, axes up to kCellMaxN = 8192, the prefilter's own limit) above the
// fractional offset s - floor(s) as a 51-bit fixed-point fraction.  s = (x_wrapped + pi)/h >= 2
// has an ulp >= 2^-51, so there the fraction is stored exactly; below s = 2 (the first two
// cells) it is rounded to 2^-51 (<= 2.2e-16 absolute on the weights).  Decoding costs four integer ops and one add instead of the wrap,
// two floors, a float->int conversion and the clamps per axis (the band kernels are
// issue-bound: profiles/r2s3_ncu_sl_step.md).
using Cell = unsigned long long;
constexpr int kCellMaxN = 8192;

__device__ __forceinline__ Cell cellPack(double x, double invh, int n) {
    constexpr double kInv2Pi = 1.0 / kTwoPi;
    const double xw = __dsub_rn(x, __dmul_rn(kTwoPi, floor(__dadd_rn(x, kPi) * kInv2Pi)));
    const double s = __dadd_rn(xw, kPi) * invh;
    const double bf = floor(s);
    const double f = s - bf;
    int b = static_cast<int>(fmin(fmax(bf, 0.0), static_cast<double>(n)));
    b = b >= n ? b - n : b;
    constexpr Cell kMax = (Cell(1) << 51) - 1;
    Cell q = (f == f) ? __double2ull_rn(f * 2251799813685248.0) : 0ull;  // f * 2^51
    q = q > kMax ? kMax : q;
    return (static_cast<Cell>(b) << 51) | q;
}

// Padded first-tap index and weights of a packed cell: the fraction's 51 bits become the top of
// a [1, 2) mantissa.  The weights keep the reference's polynomials (an 11-operation regrouping
// was 2-3% faster per band step but moved a FFT-sensitive default-path Newton record of config 2
// past 10x the reference's own rounding floor).
__device__ __forceinline__ int cellDecode(Cell u, double w[4]) {
    const unsigned hi = static_cast<unsigned>(u >> 32), lo = static_cast<unsigned>(u);
    const unsigned mhi = (__funnelshift_l(lo, hi, 1) & 0xFFFFFu) | 0x3FF00000u;
    bsplineWeights(__hiloint2double(static_cast<int>(mhi), static_cast<int>(lo << 1)) - 1.0, w);
    return static_cast<int>(hi >> 19);
}

constexpr std::size_t paddedPoints(int n1, int n2) {
    return static_cast<std::size_t>(n1 + 3) * static_cast<std::size_t>(n2 + 3);
}
// padded coefficients of one field of a grid or batch (the pairs' padded fields one after another)
inline std::size_t paddedTotal(const GridDims& g) { return paddedPoints(g.n1, g.n2) * g.pairs; }

// Departure cells of the departure points X = [x1 | x2] of a grid (or batch), cells = [c1 | c2].
void launchPackCells(Ctx& ctx, const GridDims& g, const double* X, Cell* cells);

// Pads / unpads a coefficient field (used at the C ABI, whose coefficients are unpadded).
void launchPad(Ctx& ctx, const GridDims& g, const double* c, double* padded);
void launchUnpad(Ctx& ctx, const GridDims& g, const double* padded, double* c);

}  // namespace vrg
