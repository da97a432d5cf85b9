// veloreg::spectral over libvrg: the drop-in for proj/core/src/spectral.cpp (API
// include/veloreg/spectral.hpp:12-56, unmodified).  Every operator is cuFFT + a fused symbol
// kernel on the device (vrg_gradient, vrg_apply_reg, ...); FFT counts follow the reference's
// per-transform counting (kept by libvrg and forwarded per call).
#include <stdexcept>

#include "veloreg/spectral.hpp"
#include "vrg_device.hpp"

namespace veloreg::spectral {

using vrgdev::DevBuf;
using vrgdev::Session;

namespace {

int normCode(RegNorm n) { return n == RegNorm::H1Semi ? VRG_H1SEMI : n == RegNorm::H3Semi ? VRG_H3SEMI : VRG_H2SEMI; }

int order(RegNorm n) { return n == RegNorm::H1Semi ? 1 : n == RegNorm::H3Semi ? 3 : 2; }

int wave(int idx, int n) { return idx <= n / 2 ? idx : idx - n; }  // fft.cpp:80

Session session() { return Session(vrgdev::threadDevice()); }

}  // namespace

// The host tables the accessors expose (HessianOperator::weights(), precond::applyRegPrecond):
// gamma = |k|^(2p) over the full n1 x n2 mode layout, gammaRegularized with the k=0 entry 1
// (spectral.cpp:46-66).  The device operators build the same symbols on the device.
SpectralWeights SpectralWeights::make(const Grid& g, RegNorm norm) {
    SpectralWeights w;
    w.norm = norm;
    w.grid = g;
    const std::size_t N = static_cast<std::size_t>(g.points());
    w.gamma.assign(N, 0.0);
    w.gammaRegularized.assign(N, 0.0);
    const int p = order(norm);
    for (int r = 0; r < g.n[0]; ++r) {
        const double a = wave(r, g.n[0]);
        for (int c = 0; c < g.n[1]; ++c) {
            const double b = wave(c, g.n[1]);
            const double k2 = a * a + b * b;
            double y = 1.0;
            for (int i = 0; i < p; ++i) y *= k2;
            const std::size_t at = static_cast<std::size_t>(g.index(r, c));
            w.gamma[at] = y;
            w.gammaRegularized[at] = y == 0.0 ? 1.0 : y;
        }
    }
    return w;
}

VectorField gradient(const ScalarField& u) {
    const Grid& g = u.grid;
    auto s = session();
    DevBuf du = vrgdev::deviceField(s, u), o(s, 2 * static_cast<std::size_t>(g.points()));
    s.check(vrg_gradient(s.ctx(), g.n[0], g.n[1], du.get(), o.get(), o.at(g.points())));
    return vrgdev::hostVector(s, g, o.get());
}

ScalarField divergence(const VectorField& v) {
    checkSameGrid(v[0], v[1]);
    const Grid& g = v.grid();
    auto s = session();
    DevBuf dv = vrgdev::deviceVector(s, v), o(s, g.points());
    s.check(vrg_divergence(s.ctx(), g.n[0], g.n[1], dv.get(), dv.at(g.points()), o.get()));
    return vrgdev::hostField(s, g, o.get());
}

VectorField applyReg(const VectorField& v, const SpectralWeights& w, double beta) {
    if (beta <= 0.0) throw std::invalid_argument("applyReg: beta must be positive");
    const Grid& g = v.grid();
    const std::size_t N = g.points();
    auto s = session();
    DevBuf dv = vrgdev::deviceVector(s, v), o(s, 2 * N);
    s.check(vrg_apply_reg(s.ctx(), g.n[0], g.n[1], normCode(w.norm), beta, dv.get(), dv.at(N), o.get(), o.at(N)));
    return vrgdev::hostVector(s, g, o.get());
}

VectorField applyInvReg(const VectorField& v, const SpectralWeights& w, double beta, double power) {
    if (beta <= 0.0) throw std::invalid_argument("applyInvReg: beta must be positive");
    const Grid& g = v.grid();
    const std::size_t N = g.points();
    auto s = session();
    DevBuf dv = vrgdev::deviceVector(s, v), o(s, 2 * N);
    s.check(vrg_apply_inv_reg(s.ctx(), g.n[0], g.n[1], normCode(w.norm), beta, power, dv.get(), dv.at(N), o.get(),
                              o.at(N)));
    return vrgdev::hostVector(s, g, o.get());
}

VectorField projectDivFree(const VectorField& b) {
    checkSameGrid(b[0], b[1]);
    const Grid& g = b.grid();
    const std::size_t N = g.points();
    auto s = session();
    DevBuf db = vrgdev::deviceVector(s, b), o(s, 2 * N);
    s.check(vrg_project_div_free(s.ctx(), g.n[0], g.n[1], db.get(), db.at(N), o.get(), o.at(N)));
    return vrgdev::hostVector(s, g, o.get());
}

ScalarField resample(const ScalarField& u, const Grid& target) {
    if (u.grid == target) return u;  // spectral.cpp:159: no transform, no count
    auto s = session();
    DevBuf du = vrgdev::deviceField(s, u), o(s, target.points());
    s.check(vrg_resample(s.ctx(), u.grid.n[0], u.grid.n[1], du.get(), target.n[0], target.n[1], o.get()));
    return vrgdev::hostField(s, target, o.get());
}

VectorField resample(const VectorField& u, const Grid& target) {
    VectorField out;
    out[0] = resample(u[0], target);
    out[1] = resample(u[1], target);
    return out;
}

ScalarField cutoffFilter(const ScalarField& u, Band band) {
    const Grid& g = u.grid;
    auto s = session();
    DevBuf du = vrgdev::deviceField(s, u), o(s, g.points());
    s.check(vrg_cutoff(s.ctx(), g.n[0], g.n[1], du.get(), band == Band::Low ? VRG_BAND_LOW : VRG_BAND_HIGH, o.get()));
    return vrgdev::hostField(s, g, o.get());
}

VectorField cutoffFilter(const VectorField& u, Band band) {
    VectorField out;
    out[0] = cutoffFilter(u[0], band);
    out[1] = cutoffFilter(u[1], band);
    return out;
}

ScalarField gaussianSmooth(const ScalarField& u, double sigmaGridPoints) {
    const Grid& g = u.grid;
    auto s = session();
    DevBuf du = vrgdev::deviceField(s, u), o(s, g.points());
    s.check(vrg_gaussian_smooth(s.ctx(), g.n[0], g.n[1], du.get(), sigmaGridPoints, o.get()));
    return vrgdev::hostField(s, g, o.get());
}

ScalarField applyHelmholtz(const ScalarField& u) {
    const Grid& g = u.grid;
    auto s = session();
    DevBuf du = vrgdev::deviceField(s, u), o(s, g.points());
    s.check(vrg_apply_helmholtz(s.ctx(), g.n[0], g.n[1], du.get(), o.get()));
    return vrgdev::hostField(s, g, o.get());
}

}  // namespace veloreg::spectral
