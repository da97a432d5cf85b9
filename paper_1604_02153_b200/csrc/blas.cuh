// K9: BLAS-1 and reductions on device fields (src/field.cpp:19-119).
#pragma once

#include "common.cuh"

namespace vrg {

constexpr int kReduceThreads = 256;
constexpr int kReduceBlocks = 592;  // 4 x 148 SMs
constexpr int kReduceTicketSlots = 64;  // per-pair tickets of the fused reductions (pairs per batch)

// Launch-only reductions: the result lands in a device scalar (slot 0..31 of the context's
// reduction area) and stays stream-ordered.
double* launchDot(Ctx& ctx, std::size_t n, const double* a0, const double* b0, const double* a1, const double* b1,
                  double scale, int slot);
// the same reduction with the result written to `out` (any device double)
void launchDotInto(Ctx& ctx, std::size_t n, const double* a0, const double* b0, const double* a1, const double* b1,
                   double scale, double* out);
double* launchMaxAbs(Ctx& ctx, std::size_t n, const double* a0, const double* a1, double scale, int slot);

// grid size of the element-wise kernels (grid-stride loops, at most 8 blocks of 256 per SM)
unsigned elemBlocks(const Ctx& ctx, std::size_t n);

// Per-pair reductions of a batch (GridDims::pairs): results for every pair in a device array
// (slot 0..7), each bit-identical to the single-field reduction of that pair; a0/b0 (a1/b1) are
// fields of the batch.  readPairs copies P results to the host (synchronises).
double* launchDotPairs(Ctx& ctx, const GridDims& g, const double* a0, const double* b0, const double* a1,
                       const double* b1, double scale, int slot);
double* launchMaxAbsPairs(Ctx& ctx, const GridDims& g, const double* a0, const double* a1, int slot);
void readPairs(Ctx& ctx, const double* dev, int P, double* host);

// Synchronous host-visible reductions.
double readScalar(Ctx& ctx, const double* dev);
// dot (field.cpp:47-54): h1*h2*sum(a0*b0) + h1*h2*sum(a1*b1) (a1/b1 may be null).
double dot(Ctx& ctx, const GridDims& g, const double* a0, const double* a1, const double* b0, const double* b1);
// normLinf (field.cpp:59-65) over one or two fields.
double normLinf(Ctx& ctx, std::size_t n, const double* a0, const double* a1 = nullptr);
bool anyNonFinite(Ctx& ctx, std::size_t n, const double* a0, const double* a1 = nullptr);

// y = a*x + b*y ; out = a*x + b*y ; fill ; copy
void axpby(Ctx& ctx, std::size_t n, double a, const double* x, double b, double* y);
// y = y + (-c[0]) * x with c a device scalar: the same arithmetic as axpby(ctx, n, -c, x, 1, y)
// without reading c on the host (stream-ordered Gram-Schmidt)
void axpyNegDevCoef(Ctx& ctx, std::size_t n, const double* c, const double* x, double* y);
void lincomb(Ctx& ctx, std::size_t n, double a, const double* x, double b, const double* y, double* out);
void fill(Ctx& ctx, std::size_t n, double v, double* y);
void copy(Ctx& ctx, std::size_t n, const double* src, double* dst);

}  // namespace vrg
