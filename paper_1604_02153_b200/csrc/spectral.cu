// K7 implementation: cuFFT plans from the context cache + symbol kernels.
#include <algorithm>
#include <cmath>

#include "blas.cuh"
#include "spectral.cuh"

namespace vrg {

namespace {

constexpr int kSpecBlock = 256;

__device__ __forceinline__ int waveOf(int idx, int n) { return idx <= n / 2 ? idx : idx - n; }  // fft.cpp:80
__device__ __forceinline__ double waveNyq0(int idx, int n) {                                     // spectral.cpp:31-33
    return idx == n / 2 ? 0.0 : static_cast<double>(waveOf(idx, n));
}

__device__ __forceinline__ cplx cmulI(double k, cplx v) { return make_double2(-k * v.y, k * v.x); }  // (i k) * v
__device__ __forceinline__ cplx cscale(cplx v, double a) { return make_double2(v.x * a, v.y * a); }

__global__ void k_grad(const cplx* __restrict__ s, cplx* __restrict__ o1, cplx* __restrict__ o2, int n1, int n2,
                       int pairs, double scale) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;  // mode of the pair's spectrum (stacked pairs)
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    const cplx v = s[i];
    o1[i] = cscale(cmulI(waveNyq0(r, n1), v), scale);
    o2[i] = cscale(cmulI(waveNyq0(c, n2), v), scale);
}

// k_grad over a batch of spectra (blockIdx.y = field): field f's gradient spectra at
// o + 2f*NS (axis 0) and o + (2f+1)*NS (axis 1), the [g1 | g2] layout of a gradient trajectory.
__global__ void k_grad_batch(const cplx* __restrict__ s, cplx* __restrict__ o, int n1, int n2, int pairs,
                             double scale) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;  // one field of the batch (all pairs)
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t f = blockIdx.y;
    const std::size_t li = i % nPer;
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    const cplx v = s[f * n + i];
    o[2 * f * n + i] = cscale(cmulI(waveNyq0(r, n1), v), scale);
    o[(2 * f + 1) * n + i] = cscale(cmulI(waveNyq0(c, n2), v), scale);
}

__global__ void k_div(const cplx* __restrict__ s1, const cplx* __restrict__ s2, cplx* __restrict__ o, int n1, int n2,
                      int pairs, double scale) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;  // mode of the pair's spectrum (stacked pairs)
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    const cplx a = cmulI(waveNyq0(r, n1), s1[i]);
    const cplx b = cmulI(waveNyq0(c, n2), s2[i]);
    o[i] = cscale(make_double2(a.x + b.x, a.y + b.y), scale);
}

// applyHelmholtz symbol 1 + k1^2 + k2^2 with Nyquist-zeroed waves (spectral.cpp:214-223)
__global__ void k_helm(cplx* s, int n1, int n2, int pairs, double scale) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;  // mode of the pair's spectrum (stacked pairs)
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    const double k1 = waveNyq0(r, n1), k2 = waveNyq0(c, n2);
    s[i] = cscale(s[i], (1.0 + k1 * k1 + k2 * k2) * scale);
}

__global__ void k_scale(cplx* s, std::size_t n, std::size_t nPer, int nf, const double* __restrict__ sym,
                        double scale) {
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double m = sym ? sym[i % nPer] * scale : scale;
    for (int f = 0; f < nf; ++f) s[f * n + i] = cscale(s[f * n + i], m);
}

__device__ __forceinline__ void leray(int r, int c, int n1, int n2, cplx& s1, cplx& s2) {
    const double k1 = waveNyq0(r, n1), k2 = waveNyq0(c, n2);
    const double ksq = k1 * k1 + k2 * k2;
    if (ksq == 0.0) return;  // mean and pure-Nyquist modes pass through
    const cplx kdotb = make_double2(k1 * s1.x + k2 * s2.x, k1 * s1.y + k2 * s2.y);
    s1 = make_double2(s1.x - k1 * kdotb.x / ksq, s1.y - k1 * kdotb.y / ksq);
    s2 = make_double2(s2.x - k2 * kdotb.x / ksq, s2.y - k2 * kdotb.y / ksq);
}

__global__ void k_leray(cplx* s1, cplx* s2, int n1, int n2, int pairs) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;  // mode of the pair's spectrum (stacked pairs)
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    cplx a = s1[i], b = s2[i];
    leray(r, c, n1, n2, a, b);
    s1[i] = a;
    s2[i] = b;
}

__global__ void k_combine(const cplx* __restrict__ b1, const cplx* __restrict__ b2, const cplx* __restrict__ a1,
                          const cplx* __restrict__ a2, const double* __restrict__ sym, bool doLeray, double scale,
                          cplx* o1, cplx* o2, int n1, int n2, int pairs) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;
    cplx x = b1[i], y = b2[i];
    if (doLeray) {
        const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
        leray(r, c, n1, n2, x, y);
    }
    if (sym) {
        const double m = sym[li];
        x = cscale(x, m);
        y = cscale(y, m);
    }
    if (a1) {
        x = make_double2(x.x + a1[i].x, x.y + a1[i].y);
        y = make_double2(y.x + a2[i].x, y.y + a2[i].y);
    }
    o1[i] = cscale(x, scale);
    o2[i] = cscale(y, scale);
}

// spectral::resample (src/spectral.cpp:157-179) from source spectrum to target spectrum.
__global__ void k_resample(const cplx* __restrict__ s, int sn1, int sn2, cplx* __restrict__ t, int tn1, int tn2,
                           int pairs, double amp, double scale) {
    const int tc = tn2 / 2 + 1, sc = sn2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(tn1) * tc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t pair = i / nPer, li = i - pair * nPer;
    s += pair * static_cast<std::size_t>(sn1) * sc;
    const int rt = static_cast<int>(li / tc), c = static_cast<int>(li - static_cast<std::size_t>(rt) * tc);
    const int band1 = min(sn1, tn1) / 2, band2 = min(sn2, tn2) / 2;
    const int k1 = waveOf(rt, tn1), k2 = waveOf(c, tn2);
    cplx v = make_double2(0.0, 0.0);
    if (abs(k1) < band1 && abs(k2) < band2) {
        const int rs = k1 >= 0 ? k1 : k1 + sn1;
        v = cscale(s[static_cast<std::size_t>(rs) * sc + c], amp);
    }
    t[i] = cscale(v, scale);
}

// spectral::cutoffFilter (src/spectral.cpp:188-203): both bands from one spectrum.
__global__ void k_cutoff(const cplx* __restrict__ s, cplx* lo, cplx* hi, int n1, int n2, int pairs, double scale) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;  // mode of the pair's spectrum (stacked pairs)
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    const bool low = abs(waveOf(r, n1)) < n1 / 4 && abs(waveOf(c, n2)) < n2 / 4;
    const cplx v = cscale(s[i], scale);
    const cplx z = make_double2(0.0, 0.0);
    if (lo) lo[i] = low ? v : z;
    if (hi) hi[i] = low ? z : v;
}

__global__ void k_gauss(cplx* s, int n1, int n2, int pairs, double s1, double s2, double scale) {
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;  // mode of the pair's spectrum (stacked pairs)
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    const double k1 = waveOf(r, n1), k2 = waveOf(c, n2);
    s[i] = cscale(s[i], exp(-0.5 * (k1 * k1 * s1 * s1 + k2 * k2 * s2 * s2)) * scale);
}

inline dim3 specGrid(const GridDims& g) { return grid1d(g.specPoints(), kSpecBlock); }

}  // namespace

// ------------------------------------------------------------------------------ weights
namespace {
// SpectralWeights::make (spectral.cpp:46-66) and the symbols of applyReg / applyInvReg
// (spectral.cpp:109-131) on the half spectrum, computed on the device: gamma = ksq^order by the
// same sequence of multiplies as the reference; kind 0 -> beta*gamma; kind 1 ->
// (beta*gammaReg)^power with gammaReg(0) = 1.  The powers the solver uses are done with
// correctly rounded operations (-1: 1/x, -1/2: 1/sqrt(x), within an ulp of std::pow); others
// use the device pow (<= 2 ulp).  At 4096^2 the host loop with std::pow took ~0.2 s per symbol.
__global__ void k_weight_symbol(double* __restrict__ out, int n1, int n2, int order, int kind, double beta,
                                double power) {
    constexpr int pairs = 1;  // one pair's symbol table
    const int nc = n2 / 2 + 1;
    const std::size_t nPer = static_cast<std::size_t>(n1) * nc;
    const std::size_t n = nPer * pairs;
    const std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const std::size_t li = i % nPer;  // mode of the pair's spectrum (stacked pairs)
    const int r = static_cast<int>(li / nc), c = static_cast<int>(li - static_cast<std::size_t>(r) * nc);
    const double k1 = r <= n1 / 2 ? r : r - n1;
    const double k2 = c <= n2 / 2 ? c : c - n2;
    const double ksq = __dadd_rn(__dmul_rn(k1, k1), __dmul_rn(k2, k2));
    double val = 1.0;
    for (int p = 0; p < order; ++p) val = __dmul_rn(val, ksq);
    if (kind == 0) {
        out[i] = __dmul_rn(beta, val);
        return;
    }
    const double x = __dmul_rn(beta, val == 0.0 ? 1.0 : val);
    double y;
    if (power == -1.0)
        y = __ddiv_rn(1.0, x);
    else if (power == -0.5)
        y = __ddiv_rn(1.0, __dsqrt_rn(x));
    else if (power == 1.0)
        y = x;
    else
        y = pow(x, power);
    out[i] = y;
}
}  // namespace

Weights::Weights(const GridDims& gd, int nrm) : g(gd.one()), norm(nrm) {}  // one pair's symbols

const double* Weights::makeSymbol(int kind, double beta, double power, DBuf& b) {
    const int order = norm == kH1 ? 1 : norm == kH3 ? 3 : 2;
    b.alloc(sizeof(double) * g.specPoints());
    // the stream of the library call in progress (symbols are consumed on it); else a blocking
    // launch so that any stream may read the result
    cudaStream_t s = g_allocStream;
    k_weight_symbol<<<grid1d(g.specPoints(), 256), 256, 0, s>>>(b.d(), g.n1, g.n2, order, kind, beta, power);
    VRG_LAUNCH_CHECK();
    if (s == nullptr) VRG_CUDA(cudaStreamSynchronize(nullptr));
    return b.d();
}

const double* Weights::regSymbol(double beta) {
    auto it = regSymbols.find(beta);
    if (it != regSymbols.end()) return it->second.d();
    return makeSymbol(0, beta, 1.0, regSymbols[beta]);
}

const double* Weights::invRegSymbol(double beta, double power) {
    auto key = std::make_pair(beta, power);
    auto it = symbols.find(key);
    if (it != symbols.end()) return it->second.d();
    return makeSymbol(1, beta, power, symbols[key]);
}

// ------------------------------------------------------------------------------ FFT
cplx* specScratch(Ctx& ctx, const GridDims& g, int slot, int count) {
    return reinterpret_cast<cplx*>(ctx.scratchBuf(1000 + slot, sizeof(cplx) * g.specPoints() * count));
}

void fftForward(Ctx& ctx, const GridDims& g, const double* u, cplx* s, int batch) {
    cufftHandle p = ctx.plan(g, CUFFT_D2Z, batch);
    LaunchScope ls_(ctx, "cufft_d2z", false);
    VRG_CUFFT(cufftExecD2Z(p, const_cast<double*>(u), reinterpret_cast<cufftDoubleComplex*>(s)));
}

void fftInverse(Ctx& ctx, const GridDims& g, cplx* s, double* u, int batch) {
    cufftHandle p = ctx.plan(g, CUFFT_Z2D, batch);
    LaunchScope ls_(ctx, "cufft_z2d", false);
    VRG_CUFFT(cufftExecZ2D(p, reinterpret_cast<cufftDoubleComplex*>(s), u));
}

// Forward transform of a vector field (batched when the components are contiguous).
static void fftForward2(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, cplx* s) {
    if (v2 == v1 + g.points()) {
        fftForward(ctx, g, v1, s, 2);
    } else {
        fftForward(ctx, g, v1, s, 1);
        fftForward(ctx, g, v2, s + g.specPoints(), 1);
    }
}

static void fftInverse2(Ctx& ctx, const GridDims& g, cplx* s, double* o1, double* o2) {
    if (o2 == o1 + g.points()) {
        fftInverse(ctx, g, s, o1, 2);
    } else {
        fftInverse(ctx, g, s, o1, 1);
        fftInverse(ctx, g, s + g.specPoints(), o2, 1);
    }
}

// ------------------------------------------------------------------------------ operators
void gradient(Ctx& ctx, const GridDims& g, const double* u, double* g1, double* g2) {
    cplx* s = specScratch(ctx, g, 0, 1);
    cplx* o = specScratch(ctx, g, 1, 2);
    fftForward(ctx, g, u, s, 1);
    {
        LaunchScope ls_(ctx, "k_grad");
        k_grad<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s, o, o + g.specPoints(), g.n1, g.n2, g.pairs,
                                                            1.0 / g.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    fftInverse2(ctx, g, o, g1, g2);
    ctx.ffts += 3;
}

int gradientChunk(const GridDims& g, int count) {
    // spectra of the chunk (3 per field) within 256 MiB of scratch
    const std::size_t perField = 3 * sizeof(cplx) * g.specPoints();
    const std::size_t cap = std::size_t(256) << 20;
    return static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(count, cap / perField)));
}

void gradientBatch(Ctx& ctx, const GridDims& g, const double* u, int count, double* G) {
    const std::size_t N = g.points(), NS = g.specPoints();
    const int chunk = gradientChunk(g, count);
    cplx* s = specScratch(ctx, g, 7, chunk);
    cplx* o = specScratch(ctx, g, 8, 2 * chunk);
    for (int f0 = 0; f0 < count; f0 += chunk) {
        const int c = std::min(chunk, count - f0);
        fftForward(ctx, g, u + f0 * N, s, c);
        {
            LaunchScope ls_(ctx, "k_grad");
            const dim3 grid(specGrid(g).x, c);
            k_grad_batch<<<grid, kSpecBlock, 0, ctx.stream>>>(s, o, g.n1, g.n2, g.pairs, 1.0 / g.pointsPer());
        }
        VRG_LAUNCH_CHECK();
        fftInverse(ctx, g, o, G + 2 * f0 * N, 2 * c);
    }
    ctx.ffts += 3LL * count;
    (void)NS;
}

void divergence(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double* out) {
    cplx* s = specScratch(ctx, g, 1, 2);
    cplx* o = specScratch(ctx, g, 0, 1);
    fftForward2(ctx, g, v1, v2, s);
    {
        LaunchScope ls_(ctx, "k_div");
        k_div<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s, s + g.specPoints(), o, g.n1, g.n2, g.pairs,
                                                           1.0 / g.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    fftInverse(ctx, g, o, out, 1);
    ctx.ffts += 3;
}

void applyRealSymbol(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double* o1, double* o2,
                     const double* sym) {
    cplx* s = specScratch(ctx, g, 1, 2);
    fftForward2(ctx, g, v1, v2, s);
    specScale(ctx, g, s, 2, sym, 1.0 / g.pointsPer());
    fftInverse2(ctx, g, s, o1, o2);
    ctx.ffts += 4;
}

void applyHelmholtz(Ctx& ctx, const GridDims& g, const double* u, double* out) {
    cplx* s = specScratch(ctx, g, 0, 1);
    fftForward(ctx, g, u, s, 1);
    {
        LaunchScope ls_(ctx, "k_helm");
        k_helm<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s, g.n1, g.n2, g.pairs, 1.0 / g.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    fftInverse(ctx, g, s, out, 1);
    ctx.ffts += 2;
}

void divergencePenaltyGradient(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double betaW,
                               double* o1, double* o2) {
    double* w = ctx.scratchBuf(40, sizeof(double) * g.points());
    divergence(ctx, g, v1, v2, w);
    applyHelmholtz(ctx, g, w, w);
    gradient(ctx, g, w, o1, o2);
    lincomb(ctx, g.points(), -betaW, o1, 0.0, o1, o1);
    lincomb(ctx, g.points(), -betaW, o2, 0.0, o2, o2);
}

double divergencePenaltyValue(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double betaW) {
    const std::size_t N = g.points();
    double* w = ctx.scratchBuf(40, sizeof(double) * N);
    double* gw = ctx.scratchBuf(41, sizeof(double) * 2 * N);
    divergence(ctx, g, v1, v2, w);
    gradient(ctx, g, w, gw, gw + N);
    return 0.5 * betaW * (dot(ctx, g, w, nullptr, w, nullptr) + dot(ctx, g, gw, gw + N, gw, gw + N));
}

void projectDivFree(Ctx& ctx, const GridDims& g, const double* b1, const double* b2, double* o1, double* o2) {
    cplx* s = specScratch(ctx, g, 1, 2);
    fftForward2(ctx, g, b1, b2, s);
    {
        LaunchScope ls_(ctx, "k_leray");
        k_leray<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s, s + g.specPoints(), g.n1, g.n2, g.pairs);
    }
    VRG_LAUNCH_CHECK();
    specScale(ctx, g, s, 2, nullptr, 1.0 / g.pointsPer());
    fftInverse2(ctx, g, s, o1, o2);
    ctx.ffts += 4;
}

void resample(Ctx& ctx, const GridDims& src, const double* u, const GridDims& dst, double* out) {
    if (src.pairs != dst.pairs) throw InvalidArgument("resample: source and target batches differ");
    if (src == dst) {
        if (out != u) VRG_CUDA(cudaMemcpyAsync(out, u, sizeof(double) * src.points(), cudaMemcpyDeviceToDevice, ctx.stream));
        return;
    }
    cplx* s = specScratch(ctx, src, 2, 1);
    cplx* t = specScratch(ctx, dst, 3, 1);
    fftForward(ctx, src, u, s, 1);
    const double amp = static_cast<double>(dst.points()) / static_cast<double>(src.points());
    {
        LaunchScope ls_(ctx, "k_resample");
        k_resample<<<specGrid(dst), kSpecBlock, 0, ctx.stream>>>(s, src.n1, src.n2, t, dst.n1, dst.n2, dst.pairs, amp,
                                                                 1.0 / dst.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    fftInverse(ctx, dst, t, out, 1);
    ctx.ffts += 2;
}

void cutoff(Ctx& ctx, const GridDims& g, const double* u, double* low, double* high) {
    cplx* s = specScratch(ctx, g, 0, 1);
    cplx* o = specScratch(ctx, g, 1, 2);
    fftForward(ctx, g, u, s, 1);
    {
        LaunchScope ls_(ctx, "k_cutoff");
        k_cutoff<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s, low ? o : nullptr, high ? o + g.specPoints() : nullptr,
                                                             g.n1, g.n2, g.pairs, 1.0 / g.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    if (low) fftInverse(ctx, g, o, low, 1);
    if (high) fftInverse(ctx, g, o + g.specPoints(), high, 1);
    ctx.ffts += (low ? 2 : 0) + (high ? 2 : 0);
}

void gaussianSmooth(Ctx& ctx, const GridDims& g, const double* u, double sigma, double* out) {
    cplx* s = specScratch(ctx, g, 0, 1);
    fftForward(ctx, g, u, s, 1);
    {
        LaunchScope ls_(ctx, "k_gauss");
        k_gauss<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s, g.n1, g.n2, g.pairs, sigma * g.h1(), sigma * g.h2(),
                                                            1.0 / g.pointsPer());
    }
    VRG_LAUNCH_CHECK();
    fftInverse(ctx, g, s, out, 1);
    ctx.ffts += 2;
}

void specScale(Ctx& ctx, const GridDims& g, cplx* s, int nf, const double* sym, double scale) {
    {
        LaunchScope ls_(ctx, "k_scale");
        k_scale<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s, g.specPoints(), g.specPer(), nf, sym, scale);
    }
    VRG_LAUNCH_CHECK();
}

void specLeray(Ctx& ctx, const GridDims& g, cplx* s1, cplx* s2) {
    {
        LaunchScope ls_(ctx, "k_leray");
        k_leray<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(s1, s2, g.n1, g.n2, g.pairs);
    }
    VRG_LAUNCH_CHECK();
}

void specCombine(Ctx& ctx, const GridDims& g, const cplx* b1, const cplx* b2, const cplx* a1, const cplx* a2,
                 const double* sym, bool doLeray, double scale, cplx* o1, cplx* o2) {
    {
        LaunchScope ls_(ctx, "k_combine");
        k_combine<<<specGrid(g), kSpecBlock, 0, ctx.stream>>>(b1, b2, a1, a2, sym, doLeray, scale, o1, o2, g.n1, g.n2,
                                                               g.pairs);
    }
    VRG_LAUNCH_CHECK();
}

}  // namespace vrg
