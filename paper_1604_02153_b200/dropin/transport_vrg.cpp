// veloreg::transport over libvrg: the drop-in for proj/core/src/transport.cpp.  Same public API
// (include/veloreg/transport.hpp:18-113, unmodified), same argument checks and messages, same
// lazy per-velocity caches and operation counts (kept by libvrg's Solver), same BlowupError
// messages; the solves run on the device (vrg_solver_*).
#include <cstdio>
#include <stdexcept>
#include <string>

#include "veloreg/transport.hpp"
#include "vrg_device.hpp"

namespace veloreg::transport {

using vrgdev::DevBuf;
using vrgdev::Session;

namespace {

int schemeCode(Scheme s) {
    return s == Scheme::SL ? VRG_SCHEME_SL : s == Scheme::RK2 ? VRG_SCHEME_RK2 : VRG_SCHEME_RK2A;
}

}  // namespace

// transport.cpp:40-42
TimeGrid::TimeGrid(int steps) : nt(steps), ht(1.0 / steps) {
    if (steps < 1) throw std::invalid_argument("TimeGrid: nt must be >= 1");
}

// transport.cpp:44-50: max(2, ceil(max_i ||v_i||_inf / (cfl h_i))), the maxima on the device
int deriveSteps(const VectorField& v, double cfl) {
    if (!(cfl > 0.0) || cfl > 20.0) throw std::invalid_argument("cfl must lie in (0, 20]");
    const Grid& g = v.grid();
    Session s(vrgdev::threadDevice());
    DevBuf dv = vrgdev::deviceVector(s, v);
    int nt = 0;
    s.check(vrg_derive_steps(s.ctx(), g.n[0], g.n[1], dv.get(), dv.at(g.points()), cfl, &nt));
    return nt;
}

// transport.cpp:52-58
TimeGrid makeTimeGrid(const VectorField& v, const SchemeConfig& cfg) {
    if (cfg.ntOverride) return TimeGrid(*cfg.ntOverride);
    if (cfg.scheme != Scheme::SL && cfg.cfl > 0.5)
        std::fprintf(stderr, "transport: warning: CFL %.3g > 0.5 with an explicit RK2 scheme\n", cfg.cfl);
    return TimeGrid(deriveSteps(v, cfg.cfl));
}

// transport.cpp:60-89: Heun departure points, traced on the device (vrg_trace)
Characteristics traceCharacteristics(const VectorField& v, double ht, TraceDirection dir) {
    if (!(ht > 0.0)) throw std::invalid_argument("traceCharacteristics: ht must be positive");
    checkFinite(v, "traceCharacteristics velocity");
    const Grid& g = v.grid();
    const std::size_t N = g.points();
    Session s(vrgdev::threadDevice());
    DevBuf dv = vrgdev::deviceVector(s, v);
    DevBuf x(s, 2 * N);
    s.check(vrg_trace(s.ctx(), g.n[0], g.n[1], dv.get(), dv.at(N), ht,
                      dir == TraceDirection::Forward ? VRG_FORWARD : VRG_BACKWARD, x.get(), x.at(N)));
    Characteristics out{interp::PointSet(g), dir, ht};
    vrgdev::download(s, out.departure.x1, x.get());
    vrgdev::download(s, out.departure.x2, x.at(N));
    return out;
}

// The pImpl: host copies of the constructor arguments (the accessors return them) and the
// device solver, which owns the lazily built characteristics and div v caches.
struct Solver::Impl {
    VectorField v;
    TimeGrid tg;
    SchemeConfig cfg;
    vrgdev::Device* dev;
    DevBuf dv;
    vrg_solver_t h = nullptr;

    Impl(const VectorField& vel, const TimeGrid& grid, const SchemeConfig& config)
        : v(vel), tg(grid), cfg(config), dev(&vrgdev::threadDevice()) {}

    ~Impl() {
        if (h) {
            std::lock_guard<std::mutex> lock(dev->mu);
            vrg_solver_destroy(h);
        }
    }

    std::size_t N() const { return static_cast<std::size_t>(v.grid().points()); }
    bool isSL() const { return cfg.scheme == Scheme::SL; }

    // first use creates the device solver (after the ctor's finiteness check)
    vrg_solver_t handle(const Session& s) {
        if (!h) {
            const Grid& g = v.grid();
            dv = vrgdev::deviceVector(s, v);
            s.check(vrg_solver_create_ex(s.ctx(), g.n[0], g.n[1], dv.get(), dv.at(N()), tg.nt, schemeCode(cfg.scheme),
                                         &h));
        }
        return h;
    }

    TransportSolution solution(const Session& s, const double* traj) {
        TransportSolution out;
        out.nodes.frames = vrgdev::hostFrames(s, v.grid(), traj, tg.nt + 1);
        if (!isSL()) {
            DevBuf st(s, static_cast<std::size_t>(tg.nt) * N());
            s.check(vrg_solver_stages(h, st.get()));
            out.stages = vrgdev::hostFrames(s, v.grid(), st.get(), tg.nt);
        }
        return out;
    }
};

// transport.cpp:244-247
Solver::Solver(const VectorField& v, const TimeGrid& tg, const SchemeConfig& cfg)
    : impl_(std::make_unique<Impl>(v, tg, cfg)) {
    checkFinite(v, "transport velocity");
}

Solver::~Solver() = default;
Solver::Solver(Solver&&) noexcept = default;
Solver& Solver::operator=(Solver&&) noexcept = default;

const VectorField& Solver::velocity() const { return impl_->v; }
const TimeGrid& Solver::timeGrid() const { return impl_->tg; }
const SchemeConfig& Solver::config() const { return impl_->cfg; }

// transport.cpp:257-260 (slState / heunForward, guarded)
TransportSolution Solver::solveState(const ScalarField& m0) const {
    checkSameGrid(m0, impl_->v[0]);
    Impl& I = *impl_;
    Session s(*I.dev);
    vrg_solver_t h = I.handle(s);
    DevBuf m = vrgdev::deviceField(s, m0);
    DevBuf traj(s, (I.tg.nt + 1) * I.N());
    s.check(vrg_solver_state(h, m.get(), traj.get()));
    return I.solution(s, traj.get());
}

// transport.cpp:262-265 (slAdjoint / heunBackward, guarded)
TransportSolution Solver::solveAdjoint(const ScalarField& lambda1) const {
    checkSameGrid(lambda1, impl_->v[0]);
    Impl& I = *impl_;
    Session s(*I.dev);
    vrg_solver_t h = I.handle(s);
    DevBuf l = vrgdev::deviceField(s, lambda1);
    DevBuf traj(s, (I.tg.nt + 1) * I.N());
    s.check(vrg_solver_adjoint(h, l.get(), traj.get()));
    return I.solution(s, traj.get());
}

// transport.cpp:267-289
ScalarField Solver::solveStateFinal(const ScalarField& m0) const {
    checkSameGrid(m0, impl_->v[0]);
    Impl& I = *impl_;
    Session s(*I.dev);
    vrg_solver_t h = I.handle(s);
    DevBuf m = vrgdev::deviceField(s, m0);
    DevBuf out(s, I.N());
    s.check(vrg_solver_state_final(h, m.get(), out.get()));
    return vrgdev::hostField(s, I.v.grid(), out.get());
}

// transport.cpp:291-309
ScalarField Solver::solveAdjointFinal(const ScalarField& lambda1) const {
    checkSameGrid(lambda1, impl_->v[0]);
    Impl& I = *impl_;
    Session s(*I.dev);
    vrg_solver_t h = I.handle(s);
    DevBuf l = vrgdev::deviceField(s, lambda1);
    DevBuf out(s, I.N());
    s.check(vrg_solver_adjoint_final(h, l.get(), out.get()));
    return vrgdev::hostField(s, I.v.grid(), out.get());
}

// transport.cpp:311-377: argument checks on the host, the solve on the device (the RK2 / RK2A
// predictor fields of `state` are recomputed there from its nodes, the same arithmetic)
Trajectory Solver::solveIncState(const VectorField& vtilde, const TransportSolution& state) const {
    Impl& I = *impl_;
    if (state.nodes.steps() != I.tg.nt) throw std::invalid_argument("solveIncState: trajectory length mismatch");
    checkSameGrid(vtilde[0], I.v[0]);
    if (!I.isSL() && !state.hasStages())
        throw std::invalid_argument("solveIncState: state solution lacks the RK2 stage fields");
    Session s(*I.dev);
    vrg_solver_t h = I.handle(s);
    DevBuf vt = vrgdev::deviceVector(s, vtilde);
    DevBuf st = vrgdev::deviceFrames(s, state.nodes.frames);
    DevBuf traj(s, (I.tg.nt + 1) * I.N());
    s.check(vrg_solver_incstate(h, vt.get(), vt.at(I.N()), st.get(), traj.get()));
    Trajectory out;
    out.frames = vrgdev::hostFrames(s, I.v.grid(), traj.get(), I.tg.nt + 1);
    return out;
}

// transport.cpp:380-454
Trajectory Solver::solveIncAdjoint(const VectorField& vtilde, const ScalarField& lambdaTilde1,
                                   const TransportSolution* adjoint, HessianMode mode) const {
    Impl& I = *impl_;
    checkSameGrid(lambdaTilde1, I.v[0]);
    const bool fullNewton = mode == HessianMode::FullNewton;
    if (fullNewton) {
        if (adjoint == nullptr)
            throw std::invalid_argument("solveIncAdjoint: full Newton mode requires the adjoint trajectory");
        if (adjoint->nodes.steps() != I.tg.nt) throw std::invalid_argument("solveIncAdjoint: trajectory length mismatch");
        if (!I.isSL() && !adjoint->hasStages())
            throw std::invalid_argument("solveIncAdjoint: adjoint solution lacks the RK2 stage fields");
    }
    Session s(*I.dev);
    vrg_solver_t h = I.handle(s);
    DevBuf vt = vrgdev::deviceVector(s, vtilde);
    DevBuf lt = vrgdev::deviceField(s, lambdaTilde1);
    DevBuf adj;
    if (fullNewton) adj = vrgdev::deviceFrames(s, adjoint->nodes.frames);
    DevBuf traj(s, (I.tg.nt + 1) * I.N());
    s.check(vrg_solver_incadjoint(h, vt.get(), vt.at(I.N()), lt.get(), fullNewton ? adj.get() : nullptr,
                                  fullNewton ? VRG_FULL_NEWTON : VRG_GAUSS_NEWTON, traj.get()));
    Trajectory out;
    out.frames = vrgdev::hostFrames(s, I.v.grid(), traj.get(), I.tg.nt + 1);
    return out;
}

// transport.cpp:456-464 (SL) and the Heun variant
ScalarField Solver::jacobianDeterminant() const {
    Impl& I = *impl_;
    Session s(*I.dev);
    vrg_solver_t h = I.handle(s);
    DevBuf out(s, I.N());
    s.check(vrg_solver_jacobian(h, out.get()));
    return vrgdev::hostField(s, I.v.grid(), out.get());
}

// Free-function forms (transport.hpp:103-111): each builds a fresh Solver.
Trajectory solveState(const VectorField& v, const ScalarField& m0, const TimeGrid& tg, const SchemeConfig& cfg) {
    return Solver(v, tg, cfg).solveState(m0).nodes;
}

Trajectory solveAdjoint(const VectorField& v, const ScalarField& lambda1, const TimeGrid& tg,
                        const SchemeConfig& cfg) {
    return Solver(v, tg, cfg).solveAdjoint(lambda1).nodes;
}

Trajectory solveIncState(const VectorField& v, const VectorField& vtilde, const TransportSolution& state,
                         const TimeGrid& tg, const SchemeConfig& cfg) {
    return Solver(v, tg, cfg).solveIncState(vtilde, state);
}

Trajectory solveIncAdjoint(const VectorField& v, const VectorField& vtilde, const ScalarField& lambdaTilde1,
                           const TransportSolution* adjoint, HessianMode mode, const TimeGrid& tg,
                           const SchemeConfig& cfg) {
    return Solver(v, tg, cfg).solveIncAdjoint(vtilde, lambdaTilde1, adjoint, mode);
}

ScalarField jacobianDet(const VectorField& v, const TimeGrid& tg, const SchemeConfig& cfg) {
    return Solver(v, tg, cfg).jacobianDeterminant();
}

}  // namespace veloreg::transport
