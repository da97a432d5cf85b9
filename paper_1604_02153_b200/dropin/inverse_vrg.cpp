// veloreg::inverse over libvrg: the drop-in for proj/core/src/inverse.cpp (API
// include/veloreg/inverse.hpp:60-105, unmodified).  evaluateObjective / evaluateGradient and the
// HessianOperator pImpl run on the device (vrg_evaluate_*_ex, vrg_hess_*); the operator keeps
// its per-iterate invariants (state, grad m_j, departure points, ...) resident in HBM between
// applies.  The reference's Newton driver (newton.cpp) and preconditioner (precond.cpp) call
// these unchanged.
#include <stdexcept>

#include "veloreg/inverse.hpp"
#include "vrg_device.hpp"

namespace veloreg::inverse {

using transport::Scheme;
using transport::TransportSolution;
using vrgdev::DevBuf;
using vrgdev::Session;

namespace {

int schemeCode(Scheme s) {
    return s == Scheme::SL ? VRG_SCHEME_SL : s == Scheme::RK2 ? VRG_SCHEME_RK2 : VRG_SCHEME_RK2A;
}

vrg_model modelOf(const Model& m) {
    vrg_model r;
    r.norm = m.norm == spectral::RegNorm::H1Semi ? VRG_H1SEMI : m.norm == spectral::RegNorm::H3Semi ? VRG_H3SEMI : VRG_H2SEMI;
    r.beta_v = m.betaV;
    r.deformation = m.deformation == Deformation::Compressible     ? VRG_COMPRESSIBLE
                    : m.deformation == Deformation::Incompressible ? VRG_INCOMPRESSIBLE
                                                                   : VRG_NEAR_INCOMPRESSIBLE;
    r.beta_w = m.betaW;
    return r;
}

TransportSolution solutionOf(const Session& s, const Grid& g, const DevBuf& nodes, const DevBuf& stages, int nt) {
    TransportSolution out;
    out.nodes.frames = vrgdev::hostFrames(s, g, nodes.get(), nt + 1);
    if (stages) out.stages = vrgdev::hostFrames(s, g, stages.get(), nt);
    return out;
}

// Checks the reference makes before its transport solves (transport.cpp:244-247, 257-258).
void checkVelocityAndTemplate(const VectorField& v, const ScalarField& templateImage, bool needTemplate) {
    checkFinite(v, "transport velocity");
    if (needTemplate) checkSameGrid(templateImage, v[0]);
}

}  // namespace

// inverse.cpp:96-117
ObjectiveResult evaluateObjective(const VectorField& v, const problems::RegistrationProblem& problem,
                                  const Model& model, const transport::TimeGrid& tg,
                                  const transport::SchemeConfig& cfg) {
    if (problem.reference.grid != v.grid())
        throw std::invalid_argument("evaluateObjective: problem and velocity grids differ");
    checkVelocityAndTemplate(v, problem.templateImage, true);
    const Grid& g = v.grid();
    const std::size_t N = g.points();
    const bool rk = cfg.scheme != Scheme::SL;
    Session s(vrgdev::threadDevice());
    DevBuf dv = vrgdev::deviceVector(s, v), mR = vrgdev::deviceField(s, problem.reference),
           mT = vrgdev::deviceField(s, problem.templateImage);
    DevBuf st(s, (tg.nt + 1) * N), stS;
    if (rk) stS = DevBuf(s, tg.nt * N);
    const vrg_model m = modelOf(model);
    double sc[4] = {0, 0, 0, 0};
    s.check(vrg_evaluate_objective_ex(s.ctx(), g.n[0], g.n[1], dv.get(), dv.at(N), mR.get(), mT.get(), &m,
                                      schemeCode(cfg.scheme), tg.nt, st.get(), rk ? stS.get() : nullptr, sc));
    ObjectiveResult res;
    res.objective = sc[0];
    res.mismatch = sc[1];
    res.regTerm = sc[2];
    res.penaltyTerm = sc[3];
    res.state = solutionOf(s, g, st, stS, tg.nt);
    return res;
}

// inverse.cpp:119-148
GradientResult evaluateGradient(const VectorField& v, const problems::RegistrationProblem& problem,
                                const Model& model, const transport::TimeGrid& tg,
                                const transport::SchemeConfig& cfg, const TransportSolution* reuseState) {
    if (problem.reference.grid != v.grid())
        throw std::invalid_argument("evaluateGradient: problem and velocity grids differ");
    checkVelocityAndTemplate(v, problem.templateImage, reuseState == nullptr);
    if (reuseState && reuseState->nodes.steps() != tg.nt)
        throw std::invalid_argument("evaluateGradient: reused state has wrong step count");
    const bool rk = cfg.scheme != Scheme::SL;
    if (rk && reuseState && !reuseState->hasStages())  // assembleBodyForce, inverse.cpp:71-72
        throw std::invalid_argument("assembleBodyForce: RK2 assembly requires stage fields");
    const Grid& g = v.grid();
    const std::size_t N = g.points();
    Session s(vrgdev::threadDevice());
    DevBuf dv = vrgdev::deviceVector(s, v), mR = vrgdev::deviceField(s, problem.reference),
           mT = vrgdev::deviceField(s, problem.templateImage);
    DevBuf reuse;
    if (reuseState) reuse = vrgdev::deviceFrames(s, reuseState->nodes.frames);
    DevBuf gr(s, 2 * N), body(s, 2 * N), st(s, (tg.nt + 1) * N), ad(s, (tg.nt + 1) * N), stS, adS;
    if (rk) {
        stS = DevBuf(s, tg.nt * N);
        adS = DevBuf(s, tg.nt * N);
    }
    const vrg_model m = modelOf(model);
    double sc[4] = {0, 0, 0, 0};
    s.check(vrg_evaluate_gradient_ex(s.ctx(), g.n[0], g.n[1], dv.get(), dv.at(N), mR.get(), mT.get(), &m,
                                     schemeCode(cfg.scheme), tg.nt, reuseState ? reuse.get() : nullptr, gr.get(),
                                     gr.at(N), body.get(), st.get(), rk ? stS.get() : nullptr, ad.get(),
                                     rk ? adS.get() : nullptr, sc));
    GradientResult res;
    res.timeGrid = tg;
    res.g = vrgdev::hostVector(s, g, gr.get());
    res.bodyForce = vrgdev::hostVector(s, g, body.get());
    res.objective = sc[0];
    res.mismatch = sc[1];
    res.regTerm = sc[2];
    res.penaltyTerm = sc[3];
    res.state = solutionOf(s, g, st, stS, tg.nt);
    res.adjoint = solutionOf(s, g, ad, adS, tg.nt);
    return res;
}

// The pImpl: the device operator (vrg_hess_t) with its resident per-iterate invariants, plus
// the host members the accessors return.
struct HessianOperator::Impl {
    Model model;
    spectral::SpectralWeights weights;
    Grid grid;
    vrgdev::Device* dev;
    vrg_hess_t h = nullptr;
    const char* deferredError = nullptr;  // what the reference would throw at apply time

    Impl(const VectorField& v, const problems::RegistrationProblem& problem, const Model& mdl,
         const transport::TimeGrid& tg, const transport::SchemeConfig& cfg, transport::HessianMode mode,
         const TransportSolution* reuseState, const TransportSolution* reuseAdjoint)
        : model(mdl),
          weights(spectral::SpectralWeights::make(v.grid(), mdl.norm)),
          grid(v.grid()),
          dev(&vrgdev::threadDevice()) {
        // inverse.cpp:158-175: the state is reused (copied) or solved here; full Newton also
        // reuses or solves the adjoint
        const bool fullNewton = mode == transport::HessianMode::FullNewton;
        checkVelocityAndTemplate(v, problem.templateImage, reuseState == nullptr);
        const bool rk = cfg.scheme != Scheme::SL;
        if (reuseState && reuseState->nodes.steps() != tg.nt)
            deferredError = "solveIncState: trajectory length mismatch";
        else if (rk && reuseState && !reuseState->hasStages())
            deferredError = "solveIncState: state solution lacks the RK2 stage fields";
        if (fullNewton && reuseAdjoint && reuseAdjoint->nodes.steps() != tg.nt) deferredError = "solveIncAdjoint: trajectory length mismatch";
        const std::size_t N = grid.points();
        Session s(*dev);
        DevBuf dv = vrgdev::deviceVector(s, v), mR = vrgdev::deviceField(s, problem.reference),
               mT = vrgdev::deviceField(s, problem.templateImage);
        DevBuf st, ad;
        const bool useState = reuseState && !deferredError;
        if (useState) st = vrgdev::deviceFrames(s, reuseState->nodes.frames);
        if (fullNewton && reuseAdjoint && !deferredError) ad = vrgdev::deviceFrames(s, reuseAdjoint->nodes.frames);
        const vrg_model m = modelOf(model);
        s.check(vrg_hess_create_ex(s.ctx(), grid.n[0], grid.n[1], dv.get(), dv.at(N), mR.get(), mT.get(), &m,
                                   schemeCode(cfg.scheme), tg.nt, fullNewton ? VRG_FULL_NEWTON : VRG_GAUSS_NEWTON,
                                   useState ? st.get() : nullptr, ad ? ad.get() : nullptr, &h));
    }

    ~Impl() {
        if (h) {
            std::lock_guard<std::mutex> lock(dev->mu);
            vrg_hess_destroy(h);
        }
    }

    VectorField call(int (*fn)(vrg_hess_t, const double*, const double*, double*, double*), const VectorField& vt) {
        // dataTerm -> solveIncState: trajectory checks, then checkSameGrid (transport.cpp:313-315)
        if (deferredError) throw std::invalid_argument(deferredError);
        if (vt[0].grid != grid || vt[1].grid != grid) throw std::invalid_argument("field grids do not match");
        const std::size_t N = grid.points();
        Session s(*dev);
        DevBuf dvt = vrgdev::deviceVector(s, vt), o(s, 2 * N);
        s.check(fn(h, dvt.get(), dvt.at(N), o.get(), o.at(N)));
        return vrgdev::hostVector(s, grid, o.get());
    }
};

HessianOperator::HessianOperator(const VectorField& v, const problems::RegistrationProblem& problem,
                                 const Model& model, const transport::TimeGrid& tg,
                                 const transport::SchemeConfig& cfg, transport::HessianMode mode,
                                 const TransportSolution* state, const TransportSolution* adjoint)
    : impl_(std::make_unique<Impl>(v, problem, model, tg, cfg, mode, state, adjoint)) {}

HessianOperator::~HessianOperator() = default;

// inverse.cpp:229-233: beta A[vt] + K[data term], one device matvec (CUDA-graph replay)
VectorField HessianOperator::apply(const VectorField& vtilde) const { return impl_->call(vrg_hess_apply, vtilde); }

// inverse.cpp:235-237
VectorField HessianOperator::applyDataTerm(const VectorField& vtilde) const {
    return impl_->call(vrg_hess_apply_data, vtilde);
}

const Model& HessianOperator::model() const { return impl_->model; }
const spectral::SpectralWeights& HessianOperator::weights() const { return impl_->weights; }
const Grid& HessianOperator::grid() const { return impl_->grid; }

// inverse.cpp:243-249
VectorField hessianMatvec(const VectorField& vtilde, const VectorField& v, const problems::RegistrationProblem& problem,
                          const Model& model, const transport::TimeGrid& tg, const transport::SchemeConfig& cfg,
                          transport::HessianMode mode) {
    HessianOperator op(v, problem, model, tg, cfg, mode);
    return op.apply(vtilde);
}

}  // namespace veloreg::inverse
