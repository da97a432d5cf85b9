// CPU FFT backing the FFTW3-API shim (see fftw3.h).  Test infrastructure for the oracle build.
//
// * complex FFT of any length: iterative radix-2 for powers of two, recursive mixed radix
//   (smallest prime factor first, direct DFT for the prime leaf) otherwise;
// * real transforms of even length via the half-length complex packing trick;
// * 2-D transforms row pass then column pass (columns processed in cache blocks).
// Plans are immutable after creation, so execution is thread-safe (FFTW new-array API
// guarantee the reference relies on, proj/core/src/fft.cpp:15-16).
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <memory>
#include <vector>

namespace {

using cplx = std::complex<double>;
constexpr double kTwoPi = 6.283185307179586476925286766559;

struct Fft1D {
    int n = 0;
    bool pow2 = false;
    std::vector<cplx> twFwd;  // exp(-2 pi i j / n), j < n
    std::vector<int> rev;     // bit reversal (pow2 only)

    explicit Fft1D(int len) : n(len) {
#ifdef VRG_SHIM_MIXED_RADIX_ONLY
        pow2 = false;  // alternative rounding: the recursive mixed-radix path for every length
#else
        pow2 = n > 0 && (n & (n - 1)) == 0;
#endif
        twFwd.resize(n);
        for (int j = 0; j < n; ++j) {
            const double a = -kTwoPi * static_cast<double>(j) / static_cast<double>(n);
            twFwd[j] = cplx(std::cos(a), std::sin(a));
        }
        if (pow2) {
            rev.resize(n);
            int bits = 0;
            while ((1 << bits) < n) ++bits;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int b = 0; b < bits; ++b)
                    if (i & (1 << b)) r |= 1 << (bits - 1 - b);
                rev[i] = r;
            }
        }
    }

    cplx tw(long long j, int sign) const {  // exp(sign * 2 pi i j / n)
        const cplx w = twFwd[static_cast<std::size_t>(j % n)];
        return sign < 0 ? w : std::conj(w);
    }

    // In-place transform of x[0..n).  sign = -1 forward, +1 backward (unnormalised).
    void run(cplx* x, int sign) const {
        if (n <= 1) return;
        if (pow2) {
            for (int i = 0; i < n; ++i)
                if (i < rev[i]) std::swap(x[i], x[rev[i]]);
            const double sg = sign < 0 ? 1.0 : -1.0;  // conjugate twiddles for the backward transform
            double* xd = reinterpret_cast<double*>(x);
            const double* tw0 = reinterpret_cast<const double*>(twFwd.data());
            for (int len = 2; len <= n; len <<= 1) {
                const int half = len >> 1;
                const int step = n / len;
                for (int i = 0; i < n; i += len) {
                    for (int k = 0; k < half; ++k) {
                        const double wr = tw0[2 * k * step], wi = sg * tw0[2 * k * step + 1];
                        double* a = xd + 2 * (i + k);
                        double* b = xd + 2 * (i + k + half);
                        const double tr = wr * b[0] - wi * b[1], ti = wr * b[1] + wi * b[0];
                        b[0] = a[0] - tr;
                        b[1] = a[1] - ti;
                        a[0] += tr;
                        a[1] += ti;
                    }
                }
            }
            return;
        }
        std::vector<cplx> out(n), scratch(n);
        mixed(x, 1, out.data(), n, sign, scratch.data());
        std::memcpy(x, out.data(), sizeof(cplx) * n);
    }

    // out[0..len) = DFT_len of in[0], in[s], in[2s], ...; twiddles from the length-n table
    // (len divides n, so exp(2 pi i j/len) = tw(j * n/len)).
    void mixed(const cplx* in, int s, cplx* out, int len, int sign, cplx* scratch) const {
        if (len == 1) {
            out[0] = in[0];
            return;
        }
        int p = 2;
        while (p * p <= len && len % p != 0) ++p;
        if (len % p != 0) p = len;  // prime
        const int m = len / p;
        const long long unit = n / len;
        if (m == 1) {  // direct DFT of prime length
            for (int k = 0; k < p; ++k) {
                cplx acc = 0.0;
                for (int r = 0; r < p; ++r)
                    acc += in[static_cast<std::size_t>(r) * s] * tw(unit * ((static_cast<long long>(r) * k) % p), sign);
                out[k] = acc;
            }
            return;
        }
        // sub-transforms Y_r = DFT_m(in[r s + j p s])
        for (int r = 0; r < p; ++r) mixed(in + static_cast<std::size_t>(r) * s, s * p, scratch + static_cast<std::size_t>(r) * m, m, sign, out);
        // X[k + m q] = sum_r (w_len^{r k} Y_r[k]) w_p^{r q}
        std::vector<cplx> t(p);
        for (int k = 0; k < m; ++k) {
            for (int r = 0; r < p; ++r) t[r] = scratch[static_cast<std::size_t>(r) * m + k] * tw(unit * static_cast<long long>(r) * k, sign);
            for (int q = 0; q < p; ++q) {
                cplx acc = 0.0;
                for (int r = 0; r < p; ++r) acc += t[r] * tw(unit * m * ((static_cast<long long>(r) * q) % p), sign);
                out[k + static_cast<std::size_t>(m) * q] = acc;
            }
        }
    }
};

// Real <-> half-complex of even length n via a length n/2 complex transform.
struct RealFft {
    int n;
    Fft1D half;
    std::vector<cplx> w;  // exp(-2 pi i k / n), k <= n/2
    explicit RealFft(int len) : n(len), half(len / 2) {
        w.resize(n / 2 + 1);
        for (int k = 0; k <= n / 2; ++k) {
            const double a = -kTwoPi * k / static_cast<double>(n);
            w[k] = cplx(std::cos(a), std::sin(a));
        }
    }
    // x real [n] -> X[0..n/2]
    void forward(const double* x, cplx* X, cplx* z) const {
        const int m = n / 2;
        for (int j = 0; j < m; ++j) z[j] = cplx(x[2 * j], x[2 * j + 1]);
        half.run(z, -1);
        for (int k = 0; k <= m; ++k) {
            const cplx zk = z[k % m];
            const cplx zc = std::conj(z[(m - k) % m]);
            const cplx e = 0.5 * (zk + zc);
            const cplx o = cplx(0.0, -0.5) * (zk - zc);
            X[k] = e + w[k] * o;
        }
    }
    // X[0..n/2] (imag of DC/Nyquist ignored) -> x real [n], unnormalised
    void backward(const cplx* Xin, double* x, cplx* z) const {
        const int m = n / 2;
        cplx X0(Xin[0].real(), 0.0), Xm(Xin[m].real(), 0.0);
        for (int k = 0; k < m; ++k) {
            const cplx a = k == 0 ? X0 : Xin[k];
            const cplx bsrc = (m - k) == m ? Xm : Xin[m - k];
            const cplx b = std::conj(k == 0 ? Xm : bsrc);
            const cplx e2 = a + b;                 // 2 E_k
            const cplx o2 = (a - b) / w[k];        // 2 O_k
            z[k] = e2 + cplx(0.0, 1.0) * o2;
        }
        half.run(z, +1);
        for (int j = 0; j < m; ++j) {
            x[2 * j] = z[j].real();
            x[2 * j + 1] = z[j].imag();
        }
    }
};

}  // namespace

struct fftw_plan_s {
    int n0, n1;
    bool r2c;
    std::unique_ptr<RealFft> row;
    std::unique_ptr<Fft1D> col;
};

namespace {

fftw_plan makePlan(int n0, int n1, bool r2c) {
    auto* p = new fftw_plan_s;
    p->n0 = n0;
    p->n1 = n1;
    p->r2c = r2c;
    p->row = std::make_unique<RealFft>(n1);
    p->col = std::make_unique<Fft1D>(n0);
    return p;
}

constexpr int kColBlock = 16;

void columnPass(const fftw_plan_s* p, cplx* data, int sign) {
    const int n0 = p->n0, nc = p->n1 / 2 + 1;
    std::vector<cplx> buf(static_cast<std::size_t>(kColBlock) * n0);
    for (int c0 = 0; c0 < nc; c0 += kColBlock) {
        const int cb = std::min(kColBlock, nc - c0);
        for (int r = 0; r < n0; ++r)
            for (int b = 0; b < cb; ++b) buf[static_cast<std::size_t>(b) * n0 + r] = data[static_cast<std::size_t>(r) * nc + c0 + b];
        for (int b = 0; b < cb; ++b) p->col->run(buf.data() + static_cast<std::size_t>(b) * n0, sign);
        for (int r = 0; r < n0; ++r)
            for (int b = 0; b < cb; ++b) data[static_cast<std::size_t>(r) * nc + c0 + b] = buf[static_cast<std::size_t>(b) * n0 + r];
    }
}

}  // namespace

extern "C" {

fftw_plan fftw_plan_dft_r2c_2d(int n0, int n1, double*, fftw_complex*, unsigned) {
    if (n0 < 1 || n1 < 2 || (n1 % 2) != 0) return nullptr;
    return makePlan(n0, n1, true);
}

fftw_plan fftw_plan_dft_c2r_2d(int n0, int n1, fftw_complex*, double*, unsigned) {
    if (n0 < 1 || n1 < 2 || (n1 % 2) != 0) return nullptr;
    return makePlan(n0, n1, false);
}

void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* outRaw) {
    cplx* out = reinterpret_cast<cplx*>(outRaw);
    const int n0 = p->n0, n1 = p->n1, nc = n1 / 2 + 1;
    std::vector<cplx> z(n1 / 2 + 1);
    for (int r = 0; r < n0; ++r) p->row->forward(in + static_cast<std::size_t>(r) * n1, out + static_cast<std::size_t>(r) * nc, z.data());
    columnPass(p, out, -1);
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* inRaw, double* out) {
    cplx* in = reinterpret_cast<cplx*>(inRaw);
    const int n0 = p->n0, n1 = p->n1, nc = n1 / 2 + 1;
    columnPass(p, in, +1);
    std::vector<cplx> z(n1 / 2 + 1);
    for (int r = 0; r < n0; ++r) p->row->backward(in + static_cast<std::size_t>(r) * nc, out + static_cast<std::size_t>(r) * n1, z.data());
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
