// veloreg::interp over libvrg: the drop-in for proj/core/src/interp.cpp (API
// include/veloreg/interp.hpp:11-34, unmodified).  The periodic cubic B-spline prefilter (the
// chunk-carry recursive filter) and the 16-tap evaluation run on the device.
#include <stdexcept>

#include "veloreg/interp.hpp"
#include "vrg_device.hpp"

namespace veloreg::interp {

using vrgdev::DevBuf;
using vrgdev::Session;

// interp.cpp:75-85: coefficients of the cyclic tridiagonal system per axis
SplineCoefficients prefilter(const ScalarField& u) {
    checkFinite(u, "prefilter");
    const Grid& g = u.grid;
    Session s(vrgdev::threadDevice());
    DevBuf du = vrgdev::deviceField(s, u), c(s, g.points());
    s.check(vrg_prefilter(s.ctx(), g.n[0], g.n[1], du.get(), c.get()));
    SplineCoefficients out;
    out.grid = g;
    out.c.assign(static_cast<std::size_t>(g.points()), 0.0);
    vrgdev::download(s, out.c, c.get());
    return out;
}

// interp.cpp:87-127: wrap, cell, weights, 4 x 4 taps; one interpolation counted
ScalarField evaluate(const SplineCoefficients& c, const PointSet& pts) {
    if (pts.grid != c.grid) throw std::invalid_argument("evaluate: point set does not match coefficient grid");
    const Grid& g = c.grid;
    const std::size_t N = g.points();
    Session s(vrgdev::threadDevice());
    DevBuf dc(s, N), x(s, 2 * N), o(s, N);
    vrgdev::upload(s, dc.get(), c.c);
    vrgdev::upload(s, x.get(), pts.x1);
    vrgdev::upload(s, x.at(N), pts.x2);
    s.check(vrg_evaluate(s.ctx(), g.n[0], g.n[1], dc.get(), x.get(), x.at(N), o.get()));
    return vrgdev::hostField(s, g, o.get());
}

}  // namespace veloreg::interp
