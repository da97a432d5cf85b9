// K7: pseudospectral operators = cuFFT D2Z/Z2D + fused per-mode symbol kernels.
// Restates spectral:: (src/spectral.cpp:16-223) and fft:: (src/fft.cpp:57-82).  The 1/N of
// the inverse transform (src/fft.cpp:74-75) is folded into the symbol kernels.
#pragma once

#include <map>
#include <memory>

#include "common.cuh"

namespace vrg {

enum RegNorm : int { kH1 = 1, kH2 = 2, kH3 = 3 };

// SpectralWeights (src/spectral.cpp:46-66) on the half spectrum, computed on the host with
// the reference's formula (exact integer arithmetic in fp64) and uploaded; (beta*gammaReg)^p
// tables use std::pow on the host like applyInvReg (src/spectral.cpp:127), so every symbol is
// bit-identical to the reference's.
struct Weights {
    GridDims g;
    int norm = kH2;
    std::map<double, DBuf> regSymbols;                  // beta -> beta*gamma
    std::map<std::pair<double, double>, DBuf> symbols;  // (beta, power) -> (beta*gammaReg)^power
    Weights(const GridDims& g, int norm);
    // beta*gamma (applyReg)
    const double* regSymbol(double beta);
    // (beta*gammaReg)^power (applyInvReg)
    const double* invRegSymbol(double beta, double power);

private:
    const double* makeSymbol(int kind, double beta, double power, DBuf& b);
};

using cplx = double2;

// Spectra scratch: the context keeps per-grid complex buffers.
cplx* specScratch(Ctx& ctx, const GridDims& g, int slot, int count);

void fftForward(Ctx& ctx, const GridDims& g, const double* u, cplx* s, int batch);   // D2Z, batch fields contiguous
void fftInverse(Ctx& ctx, const GridDims& g, cplx* s, double* u, int batch);         // Z2D (destroys s)

// Field-level operators (device pointers, stream-ordered on ctx.stream).
void gradient(Ctx& ctx, const GridDims& g, const double* u, double* g1, double* g2);
// Gradients of `count` contiguous fields u_f -> G + 2f*N = [d1 u_f | d2 u_f] with batched
// transforms (one D2Z, one symbol launch, one Z2D per chunk of gradientChunk fields); same
// arithmetic per field as gradient().
void gradientBatch(Ctx& ctx, const GridDims& g, const double* u, int count, double* G);
int gradientChunk(const GridDims& g, int count);
// applyHelmholtz (spectral.cpp:214-223): (1 - Lap) u with Nyquist-zeroed waves; 2 FFTs
void applyHelmholtz(Ctx& ctx, const GridDims& g, const double* u, double* out);
// near-incompressible penalty (inverse.cpp:17-28): -betaW grad((1 - Lap) div v) (8 FFTs) and
// 1/2 betaW (<w, w> + <grad w, grad w>), w = div v (6 FFTs)
void divergencePenaltyGradient(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double betaW,
                               double* o1, double* o2);
double divergencePenaltyValue(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double betaW);
void divergence(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double* out);
// out_i = IFFT(sym * FFT(v_i)); v and out are 2 contiguous fields when `pair`.
void applyRealSymbol(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double* o1, double* o2,
                     const double* sym);
void projectDivFree(Ctx& ctx, const GridDims& g, const double* b1, const double* b2, double* o1, double* o2);
void resample(Ctx& ctx, const GridDims& src, const double* u, const GridDims& dst, double* out);
// Low/high band of the n/4 cut-off filter from one forward transform; outputs may be null.
void cutoff(Ctx& ctx, const GridDims& g, const double* u, double* low, double* high);
void gaussianSmooth(Ctx& ctx, const GridDims& g, const double* u, double sigma, double* out);

// Spectral building blocks used by the fused operators.
// s[f] *= sym * scale for nf spectra of one grid (sym may be null = 1).
void specScale(Ctx& ctx, const GridDims& g, cplx* s, int nf, const double* sym, double scale);
// Leray projection in place on two spectra (src/spectral.cpp:133-155).
void specLeray(Ctx& ctx, const GridDims& g, cplx* s1, cplx* s2);
// out = (sym*(optional Leray)(b) + add) * scale, elementwise on two spectra.
void specCombine(Ctx& ctx, const GridDims& g, const cplx* b1, const cplx* b2, const cplx* a1, const cplx* a2,
                 const double* sym, bool leray, double scale, cplx* o1, cplx* o2);

}  // namespace vrg
