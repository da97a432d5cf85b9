// C-ABI over the UNMODIFIED reference library (/root/reference/proj/core), compiled into
// oracle/_ref/libveloreg_ref.so by oracle/Makefile.  TEST INFRASTRUCTURE ONLY: it is the
// checker the parity tests and the bench's CPU-baseline leg call through ctypes; no product
// path links or loads it.
//
// Every entry point forwards to the reference's public API (citations relative to
// /root/reference) with plain pointers and sizes; exceptions are mapped to status codes:
//   0 ok, 1 std::invalid_argument, 2 transport::BlowupError, 3 other std::exception.
#include <cstring>
#include <memory>
#include <string>

#include "veloreg/counters.hpp"
#include "veloreg/io.hpp"
#include "veloreg/field.hpp"
#include "veloreg/interp.hpp"
#include "veloreg/inverse.hpp"
#include "veloreg/newton.hpp"
#include "veloreg/precond.hpp"
#include "veloreg/problems.hpp"
#include "veloreg/spectral.hpp"
#include "veloreg/transport.hpp"

using namespace veloreg;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const transport::BlowupError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

ScalarField sf(int n1, int n2, const double* p) {
    ScalarField u{Grid(n1, n2)};
    std::memcpy(u.v.data(), p, sizeof(double) * u.v.size());
    return u;
}

VectorField vf(int n1, int n2, const double* a, const double* b) {
    VectorField v;
    v[0] = sf(n1, n2, a);
    v[1] = sf(n1, n2, b);
    return v;
}

void put(const ScalarField& u, double* out) { std::memcpy(out, u.v.data(), sizeof(double) * u.v.size()); }

void putTraj(const transport::Trajectory& t, double* out) {
    std::size_t off = 0;
    for (const ScalarField& f : t.frames) {
        put(f, out + off);
        off += f.v.size();
    }
}

spectral::RegNorm normOf(int k) {
    return k == 1 ? spectral::RegNorm::H1Semi : k == 3 ? spectral::RegNorm::H3Semi : spectral::RegNorm::H2Semi;
}

inverse::Deformation defOf(int k) {
    return k == 1 ? inverse::Deformation::Incompressible
                  : k == 2 ? inverse::Deformation::NearIncompressible : inverse::Deformation::Compressible;
}

int g_scheme = 0;  // 0 SL, 1 RK2, 2 RK2A for the operators built through this wrapper

transport::SchemeConfig slCfg(int nt, double cfl) {
    transport::SchemeConfig c{g_scheme == 1 ? transport::Scheme::RK2 : g_scheme == 2 ? transport::Scheme::RK2A
                                                                                    : transport::Scheme::SL,
                              cfl, std::nullopt};
    if (nt > 0) c.ntOverride = nt;
    return c;
}

problems::RegistrationProblem problemOf(int n1, int n2, const double* mR, const double* mT) {
    problems::RegistrationProblem p;
    p.reference = sf(n1, n2, mR);
    p.templateImage = sf(n1, n2, mT);
    p.provenance = "synthetic";
    return p;
}

double g_betaW = 1e-1;  // Model::betaW default (inverse.hpp:21)

inverse::Model modelOf(int norm, double beta, int deform) {
    inverse::Model m;
    m.norm = normOf(norm);
    m.betaV = beta;
    m.deformation = defOf(deform);
    m.betaW = g_betaW;
    return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_counters_reset() { counters::reset(); }
void ref_set_penalty_weight(double betaW) { g_betaW = betaW; }
void ref_set_scheme(int scheme) { g_scheme = scheme; }
void ref_counters(long long* ffts, long long* interps) {
    const auto s = counters::snapshot();
    *ffts = s.ffts;
    *interps = s.interps;
}

// interp.hpp:30-34
int ref_prefilter(int n1, int n2, const double* u, double* c) {
    return guarded([&] {
        auto sc = interp::prefilter(sf(n1, n2, u));
        std::memcpy(c, sc.c.data(), sizeof(double) * sc.c.size());
    });
}

int ref_evaluate(int n1, int n2, const double* c, const double* x1, const double* x2, double* out) {
    return guarded([&] {
        const Grid g(n1, n2);
        interp::SplineCoefficients sc{g, std::vector<double>(c, c + g.points())};
        interp::PointSet pts(g);
        std::memcpy(pts.x1.data(), x1, sizeof(double) * g.points());
        std::memcpy(pts.x2.data(), x2, sizeof(double) * g.points());
        put(interp::evaluate(sc, pts), out);
    });
}

// transport.hpp:44-58
int ref_derive_steps(int n1, int n2, const double* v1, const double* v2, double cfl, int* nt) {
    return guarded([&] { *nt = transport::deriveSteps(vf(n1, n2, v1, v2), cfl); });
}

// transport.cpp:60-89
int ref_trace(int n1, int n2, const double* v1, const double* v2, double ht, int backward, double* x1, double* x2) {
    return guarded([&] {
        auto ch = transport::traceCharacteristics(vf(n1, n2, v1, v2), ht,
                                                  backward ? transport::TraceDirection::Backward
                                                           : transport::TraceDirection::Forward);
        std::memcpy(x1, ch.departure.x1.data(), sizeof(double) * n1 * n2);
        std::memcpy(x2, ch.departure.x2.data(), sizeof(double) * n1 * n2);
    });
}

// Solver::solveState / solveAdjoint / solveIncState / solveIncAdjoint (SL), transport.cpp:257-454
int ref_solve_state(int n1, int n2, const double* v1, const double* v2, int nt, const double* m0, double* traj) {
    return guarded([&] {
        transport::Solver s(vf(n1, n2, v1, v2), transport::TimeGrid(nt), slCfg(nt, 1.0));
        putTraj(s.solveState(sf(n1, n2, m0)).nodes, traj);
    });
}

int ref_solve_adjoint(int n1, int n2, const double* v1, const double* v2, int nt, const double* lam1, double* traj) {
    return guarded([&] {
        transport::Solver s(vf(n1, n2, v1, v2), transport::TimeGrid(nt), slCfg(nt, 1.0));
        putTraj(s.solveAdjoint(sf(n1, n2, lam1)).nodes, traj);
    });
}

int ref_solve_state_final(int n1, int n2, const double* v1, const double* v2, int nt, const double* m0, double* out) {
    return guarded([&] {
        transport::Solver s(vf(n1, n2, v1, v2), transport::TimeGrid(nt), slCfg(nt, 1.0));
        put(s.solveStateFinal(sf(n1, n2, m0)), out);
    });
}

int ref_solve_adjoint_final(int n1, int n2, const double* v1, const double* v2, int nt, const double* lam1, double* out) {
    return guarded([&] {
        transport::Solver s(vf(n1, n2, v1, v2), transport::TimeGrid(nt), slCfg(nt, 1.0));
        put(s.solveAdjointFinal(sf(n1, n2, lam1)), out);
    });
}

int ref_solve_incstate(int n1, int n2, const double* v1, const double* v2, int nt, const double* m0,
                       const double* vt1, const double* vt2, double* traj) {
    return guarded([&] {
        transport::Solver s(vf(n1, n2, v1, v2), transport::TimeGrid(nt), slCfg(nt, 1.0));
        auto st = s.solveState(sf(n1, n2, m0));
        putTraj(s.solveIncState(vf(n1, n2, vt1, vt2), st), traj);
    });
}

int ref_solve_incadjoint_gn(int n1, int n2, const double* v1, const double* v2, int nt, const double* lt1,
                            double* traj) {
    return guarded([&] {
        transport::Solver s(vf(n1, n2, v1, v2), transport::TimeGrid(nt), slCfg(nt, 1.0));
        VectorField z(Grid(n1, n2));
        putTraj(s.solveIncAdjoint(z, sf(n1, n2, lt1), nullptr, transport::HessianMode::GaussNewton), traj);
    });
}

// full-Newton incremental adjoint (transport.cpp:403-453) with the adjoint solved from adjSeed
// here (so the RK2 schemes have its stage fields)
int ref_solve_incadjoint_fn(int n1, int n2, const double* v1, const double* v2, int nt, const double* vt1,
                            const double* vt2, const double* lt1, const double* adjSeed, double* traj) {
    return guarded([&] {
        transport::Solver s(vf(n1, n2, v1, v2), transport::TimeGrid(nt), slCfg(nt, 1.0));
        transport::TransportSolution adj = s.solveAdjoint(sf(n1, n2, adjSeed));
        putTraj(s.solveIncAdjoint(vf(n1, n2, vt1, vt2), sf(n1, n2, lt1), &adj, transport::HessianMode::FullNewton),
                traj);
    });
}

int ref_jacobian_det(int n1, int n2, const double* v1, const double* v2, int nt, double cfl, double* out) {
    return guarded([&] {
        VectorField v = vf(n1, n2, v1, v2);
        auto cfg = slCfg(nt, cfl);
        put(transport::jacobianDet(v, transport::makeTimeGrid(v, cfg), cfg), out);
    });
}

// spectral.hpp:27-56
int ref_gradient(int n1, int n2, const double* u, double* g1, double* g2) {
    return guarded([&] {
        VectorField g = spectral::gradient(sf(n1, n2, u));
        put(g[0], g1);
        put(g[1], g2);
    });
}

int ref_divergence(int n1, int n2, const double* v1, const double* v2, double* out) {
    return guarded([&] { put(spectral::divergence(vf(n1, n2, v1, v2)), out); });
}

int ref_apply_reg(int n1, int n2, int norm, double beta, const double* v1, const double* v2, double* o1, double* o2) {
    return guarded([&] {
        auto w = spectral::SpectralWeights::make(Grid(n1, n2), normOf(norm));
        VectorField o = spectral::applyReg(vf(n1, n2, v1, v2), w, beta);
        put(o[0], o1);
        put(o[1], o2);
    });
}

int ref_apply_inv_reg(int n1, int n2, int norm, double beta, double power, const double* v1, const double* v2,
                      double* o1, double* o2) {
    return guarded([&] {
        auto w = spectral::SpectralWeights::make(Grid(n1, n2), normOf(norm));
        VectorField o = spectral::applyInvReg(vf(n1, n2, v1, v2), w, beta, power);
        put(o[0], o1);
        put(o[1], o2);
    });
}

int ref_project_div_free(int n1, int n2, const double* v1, const double* v2, double* o1, double* o2) {
    return guarded([&] {
        VectorField o = spectral::projectDivFree(vf(n1, n2, v1, v2));
        put(o[0], o1);
        put(o[1], o2);
    });
}

int ref_resample(int n1, int n2, const double* u, int t1, int t2, double* out) {
    return guarded([&] { put(spectral::resample(sf(n1, n2, u), Grid(t1, t2)), out); });
}

int ref_cutoff(int n1, int n2, const double* u, int high, double* out) {
    return guarded([&] {
        put(spectral::cutoffFilter(sf(n1, n2, u), high ? spectral::Band::High : spectral::Band::Low), out);
    });
}

int ref_apply_helmholtz(int n1, int n2, const double* u, double* out) {
    return guarded([&] { put(spectral::applyHelmholtz(sf(n1, n2, u)), out); });
}

int ref_gaussian_smooth(int n1, int n2, const double* u, double sigma, double* out) {
    return guarded([&] { put(spectral::gaussianSmooth(sf(n1, n2, u), sigma), out); });
}

// problems.cpp:87-118 (mt19937_64 + normal_distribution)
int ref_random_bandlimited_field(int n1, int n2, unsigned long long seed, double* out) {
    return guarded([&] { put(problems::randomBandLimitedField(Grid(n1, n2), seed), out); });
}

// ---- HessianOperator handle (inverse.hpp:74-97) -------------------------------------------
struct RefHess {
    problems::RegistrationProblem problem;
    std::unique_ptr<inverse::HessianOperator> op;
};

void* ref_hess_create_mode(int n1, int n2, const double* v1, const double* v2, const double* mR, const double* mT,
                           int norm, double beta, int deform, int nt, int mode, int* status) {
    RefHess* h = nullptr;
    *status = guarded([&] {
        auto* hh = new RefHess;
        hh->problem = problemOf(n1, n2, mR, mT);
        hh->op = std::make_unique<inverse::HessianOperator>(
            vf(n1, n2, v1, v2), hh->problem, modelOf(norm, beta, deform), transport::TimeGrid(nt), slCfg(nt, 1.0),
            mode == 1 ? transport::HessianMode::FullNewton : transport::HessianMode::GaussNewton);
        h = hh;
    });
    return h;
}

void* ref_hess_create(int n1, int n2, const double* v1, const double* v2, const double* mR, const double* mT,
                      int norm, double beta, int deform, int nt, int* status) {
    return ref_hess_create_mode(n1, n2, v1, v2, mR, mT, norm, beta, deform, nt, 0, status);
}

int ref_hess_apply(void* handle, const double* vt1, const double* vt2, int dataOnly, double* o1, double* o2) {
    return guarded([&] {
        auto* h = static_cast<RefHess*>(handle);
        const Grid& g = h->op->grid();
        VectorField vt = vf(g.n[0], g.n[1], vt1, vt2);
        VectorField o = dataOnly ? h->op->applyDataTerm(vt) : h->op->apply(vt);
        put(o[0], o1);
        put(o[1], o2);
    });
}

void ref_hess_destroy(void* handle) { delete static_cast<RefHess*>(handle); }

// ---- gradient / objective (inverse.cpp:96-148) ---------------------------------------------
int ref_evaluate_gradient(int n1, int n2, const double* v1, const double* v2, const double* mR, const double* mT,
                          int norm, double beta, int deform, int nt, double* g1, double* g2, double* scalars) {
    return guarded([&] {
        auto p = problemOf(n1, n2, mR, mT);
        auto r = inverse::evaluateGradient(vf(n1, n2, v1, v2), p, modelOf(norm, beta, deform), transport::TimeGrid(nt),
                                           slCfg(nt, 1.0));
        put(r.g[0], g1);
        put(r.g[1], g2);
        scalars[0] = r.objective;
        scalars[1] = r.mismatch;
        scalars[2] = r.regTerm;
    });
}

int ref_evaluate_objective(int n1, int n2, const double* v1, const double* v2, const double* mR, const double* mT,
                           int norm, double beta, int deform, int nt, double* scalars) {
    return guarded([&] {
        auto p = problemOf(n1, n2, mR, mT);
        auto r = inverse::evaluateObjective(vf(n1, n2, v1, v2), p, modelOf(norm, beta, deform), transport::TimeGrid(nt),
                                            slCfg(nt, 1.0));
        scalars[0] = r.objective;
        scalars[1] = r.mismatch;
        scalars[2] = r.regTerm;
    });
}

// ---- preconditioner pieces (precond.hpp) ----------------------------------------------------
// Coarse split Hessian at fine velocity v (coarse scheme SL CFL 5, newton.cpp:16).
struct RefCoarse {
    problems::RegistrationProblem problem;
    std::unique_ptr<precond::CoarseOperator> op;
};

void* ref_coarse_create(int n1, int n2, const double* v1, const double* v2, const double* mR, const double* mT,
                        int norm, double beta, int deform, double coarseCfl, int* status) {
    RefCoarse* h = nullptr;
    *status = guarded([&] {
        auto* hh = new RefCoarse;
        hh->problem = problemOf(n1, n2, mR, mT);
        hh->op = std::make_unique<precond::CoarseOperator>(vf(n1, n2, v1, v2), hh->problem, modelOf(norm, beta, deform),
                                                           slCfg(0, coarseCfl));
        h = hh;
    });
    return h;
}

int ref_coarse_split_apply(void* handle, const double* s1, const double* s2, double* o1, double* o2) {
    return guarded([&] {
        auto* h = static_cast<RefCoarse*>(handle);
        const Grid& g = h->op->grid();
        VectorField o = h->op->applySplitHessian(vf(g.n[0], g.n[1], s1, s2));
        put(o[0], o1);
        put(o[1], o2);
    });
}

int ref_two_level_apply(void* handle, int n1, int n2, const double* r1, const double* r2, int cheb, int chebIters,
                        double epsScale, double outerTol, double eMin, double eMax, double* o1, double* o2) {
    return guarded([&] {
        auto* h = static_cast<RefCoarse*>(handle);
        precond::PrecondChoice pc;
        pc.kind = precond::PrecondKind::TwoLevel;
        pc.coarseSolver = cheb ? precond::CoarseSolverKind::Cheb : precond::CoarseSolverKind::Pcg;
        pc.chebIters = chebIters;
        pc.epsScale = epsScale;
        VectorField o = precond::applyTwoLevel(vf(n1, n2, r1, r2), *h->op, pc, outerTol, eMin, eMax);
        put(o[0], o1);
        put(o[1], o2);
    });
}

void ref_coarse_destroy(void* handle) { delete static_cast<RefCoarse*>(handle); }

int ref_estimate_eigs(int n1, int n2, const double* mR, const double* mT, int norm, double beta, int deform,
                      double* eMin, double* eMax) {
    return guarded([&] {
        auto p = problemOf(n1, n2, mR, mT);
        auto e = precond::estimateEigs(p, modelOf(norm, beta, deform), slCfg(0, 5.0));
        *eMin = e.first;
        *eMax = e.second;
    });
}

// ---- full registration (newton.cpp:24-159) --------------------------------------------------
// cfgI: [maxOuterIter, maxInnerIter, ntOverride(0=CFL), pcKind(0 reg,1 2L), coarse(0 pcg,1 cheb), chebIters]
// cfgD: [tolRelGrad, tolAbsGrad, gradCfl, epsScale]
// rep:  per iteration 10 doubles [iter, gradNormInf, gradNormRel, objective, mismatch, inner, lsSteps,
//       stepLength, ffts, interps]; summary [status, nIter, finalGradNormRel, finalResidualRel, jacMin, jacMax]
int ref_newton_solve(int n1, int n2, const double* mR, const double* mT, int norm, double beta, int deform,
                     const int* cfgI, const double* cfgD, double* v1, double* v2, double* rep, int repCap,
                     double* summary) {
    return guarded([&] {
        auto p = problemOf(n1, n2, mR, mT);
        inverse::NewtonConfig cfg;
        cfg.maxOuterIter = cfgI[0];
        cfg.maxInnerIter = cfgI[1];
        cfg.gradScheme = slCfg(cfgI[2], cfgD[2]);
        cfg.tolRelGrad = cfgD[0];
        cfg.tolAbsGrad = cfgD[1];
        precond::PrecondChoice pc;
        pc.kind = cfgI[3] ? precond::PrecondKind::TwoLevel : precond::PrecondKind::Reg;
        pc.coarseSolver = cfgI[4] ? precond::CoarseSolverKind::Cheb : precond::CoarseSolverKind::Pcg;
        pc.chebIters = cfgI[5];
        pc.epsScale = cfgD[3];
        cfg.hessianMode = cfgI[6] == 1 ? transport::HessianMode::FullNewton : transport::HessianMode::GaussNewton;
        auto [v, r] = inverse::newtonSolve(p, modelOf(norm, beta, deform), cfg, pc);
        put(v[0], v1);
        put(v[1], v2);
        int k = 0;
        for (const auto& it : r.iterations) {
            if (k >= repCap) break;
            double* row = rep + 10 * k++;
            row[0] = it.iter;
            row[1] = it.gradNormInf;
            row[2] = it.gradNormRel;
            row[3] = it.objective;
            row[4] = it.mismatch;
            row[5] = it.innerIterations;
            row[6] = it.lineSearchSteps;
            row[7] = it.stepLength;
            row[8] = static_cast<double>(it.ffts);
            row[9] = static_cast<double>(it.interps);
        }
        summary[0] = static_cast<double>(static_cast<int>(r.status));
        summary[1] = static_cast<double>(r.iterations.size());
        summary[2] = r.finalGradNormRel;
        summary[3] = r.finalResidualRel;
        summary[4] = r.jacMin;
        summary[5] = r.jacMax;
    });
}

}  // extern "C"


// ---- io (io.cpp) ----------------------------------------------------------------------------
extern "C" {
int ref_write_field(const char* path, int n1, int n2, int comps, const double* data) {
    return guarded([&] {
        const std::size_t N = static_cast<std::size_t>(n1) * n2;
        if (comps == 1) {
            io::writeField(path, sf(n1, n2, data));
        } else {
            io::writeField(path, vf(n1, n2, data, data + N));
        }
    });
}

int ref_read_field(const char* path, int* n1, int* n2, int* comps, double* data, long long cap) {
    return guarded([&] {
        const int nc = io::fieldComponents(path);
        *comps = nc;
        if (nc == 1) {
            ScalarField u = io::readScalarField(path);
            *n1 = u.grid.n[0];
            *n2 = u.grid.n[1];
            if (data && static_cast<long long>(u.v.size()) <= cap) put(u, data);
        } else {
            VectorField u = io::readVectorField(path);
            *n1 = u.grid().n[0];
            *n2 = u.grid().n[1];
            const std::size_t N = u[0].v.size();
            if (data && static_cast<long long>(2 * N) <= cap) {
                put(u[0], data);
                put(u[1], data + N);
            }
        }
    });
}

}
