// Device-resident preconditioning and Krylov layer (include/veloreg/precond.hpp): two-level
// preconditioner with the coarse split Hessian, Chebyshev and PCG, Lanczos eMax, solveKkt.
// Control flow is host C++ (as in the reference); every vector lives in HBM and every
// operator application is a libvrg kernel sequence.  Vectors are vector fields stored as two
// contiguous fp64 fields [c0 | c1].
#pragma once

#include <functional>
#include <memory>

#include "inverse.cuh"

namespace vrg {

using LinOpDev = std::function<void(const double* in, double* out)>;

enum PrecondKind : int { kPcReg = 0, kPcTwoLevel = 1 };
enum CoarseSolverKind : int { kCoarsePcg = 0, kCoarseCheb = 1 };

// precond::PrecondChoice (precond.hpp:16-23)
struct PrecondChoice {
    int kind = kPcReg;
    int coarseSolver = kCoarseCheb;
    double epsScale = 0.1;
    int chebIters = 10;
    bool hasEig = false;
    double eMin = 1.0, eMax = 10.0;
    bool reestimateEachIteration = false;
};

// Vector-field BLAS on contiguous [c0 | c1] device vectors (field.cpp:19-119 semantics).
double vdot(Ctx& ctx, const GridDims& g, const double* a, const double* b);
double vnormL2(Ctx& ctx, const GridDims& g, const double* a);
double vnormLinf(Ctx& ctx, const GridDims& g, const double* a);

// problems::randomBandLimitedField / Velocity (problems.cpp:87-118): libstdc++ mt19937_64 +
// normal_distribution on the host (bit-identical draws), band limit and scaling on the device.
void randomBandLimitedField(Ctx& ctx, const GridDims& g, std::uint64_t seed, double* out);
void randomBandLimitedVelocity(Ctx& ctx, const GridDims& g, std::uint64_t seed, double* out);

// precond::CoarseOperator (precond.cpp:207-240): restricted problem and velocity on the
// half grid, coarse nt from the CFL rule, coarse GN Hessian (runs a coarse state solve).
class CoarseOperator {
public:
    CoarseOperator(Ctx& ctx, const GridDims& fine, const double* v, const double* mR, const double* mT,
                   const Model& model, double coarseCfl);
    Ctx& ctx;
    GridDims fine, gc;
    int nt = 0;
    DBuf mRc, mTc, vc;
    std::unique_ptr<Hessian> hess;
    void applySplit(const double* s, double* out) { hess->applySplit(s, s + gc.points(), out, out + gc.points()); }
};

// chebyshevSolve (precond.cpp:180-205), x_0 = 0, exactly k operator applications.
void chebyshevSolve(Ctx& ctx, const GridDims& g, const LinOpDev& op, const double* rhs, int k, double eMin,
                    double eMax, double* x);

struct PcgOut {
    int iterations = 0;
    bool converged = false, negativeCurvature = false, indefinitePreconditioner = false;
    double relResidual = 0.0;
};
// pcg (precond.cpp:38-85): residual measured in the preconditioned norm sqrt(r'Mr).
PcgOut pcg(Ctx& ctx, const GridDims& g, const LinOpDev& A, const double* b, const LinOpDev* M, double tol,
           int maxIter, double* x);

double tridiagMaxEig(const std::vector<double>& alpha, const std::vector<double>& beta);
// lanczosEmax (precond.cpp:134-161) with the power-iteration fallback (precond.cpp:119-132).
double lanczosEmax(Ctx& ctx, const GridDims& g, const LinOpDev& op, int steps, std::uint64_t seed);

// Two-level restriction / prolongation of a (batched) vector field between g and its half grid
// gc (cutoffFilter Low + resample, resample + cutoffFilter High; precond.cpp:266-268, 286-287);
// R and C hold the two components' spectra of every pair.
void restrictLow(Ctx& ctx, const GridDims& g, const GridDims& gc, const double* r, cplx* R, cplx* C, double* rc,
                 double ampDown);
void prolongAddHigh(Ctx& ctx, const GridDims& g, const GridDims& gc, const double* sc, cplx* C, cplx* R, double* out,
                    double ampUp);

// applyTwoLevel (precond.cpp:264-289); returns false when the coarse solve diverged and the
// identity fallback was taken.
bool applyTwoLevel(Ctx& ctx, const GridDims& g, const double* r, CoarseOperator& coarse, const PrecondChoice& choice,
                   double outerTol, double eMin, double eMax, double* out);

// lanczosEmax of a coarse operator's split Hessian with its guard checks deferred (precond.cpp:134-161)
double coarseLanczosEmax(Ctx& ctx, CoarseOperator& coarse, int steps, std::uint64_t seed);

// lanczosEmax on the stacked pairs of a batch in lockstep: one operator application and one
// orthogonalisation launch (a thread-block cluster per pair) per step for all pairs, each pair's
// arithmetic that of lanczosEmax on it alone.  emax[k]: pair k's estimate; fallback[k]: pair k
// needs lanczosEmax's power-iteration fallback (non-finite beta / no step) from the caller.
// counted(on) after each operator application, with the pairs that took part in it.  False
// (nothing decided) when the batch does not fit the cluster kernel (coarse grids above 128^2).
bool lanczosEmaxPairs(Ctx& ctx, const GridDims& g, const LinOpDev& op, int steps, std::uint64_t seed,
                      std::vector<double>& emax, std::vector<char>& fallback,
                      const std::function<void(const std::vector<char>&)>& counted);

// estimateEigsAt / estimateEigs (precond.cpp:242-258): (1, Lanczos eMax of the coarse split
// Hessian at v; v = nullptr means v = 0).
std::pair<double, double> estimateEigsAt(Ctx& ctx, const GridDims& g, const double* v, const double* mR,
                                         const double* mT, const Model& model, double coarseCfl,
                                         std::uint64_t seed = 0x5eed);

struct KktResult {
    int iterations = 0;
    bool negativeCurvature = false, converged = false;
    double relResidual = 0.0, totalTimeSec = 0.0, precondTimeSec = 0.0;
};
// solveKkt (precond.cpp:291-358).  `solution` receives delta-v (2 contiguous fields).
KktResult solveKkt(Ctx& ctx, Hessian& hess, const double* rhs, double tol, int maxIter, const PrecondChoice& choice,
                   const double* mR, const double* mT, const double* v, double coarseCfl, double* solution);
// The same with the fine split operator A(s) = M^{-1/2} Q M^{-1/2} s + s given as a LinOp
// (precond::LinOp, precond.hpp:25), M = beta A from `weights`.
KktResult solveKktOp(Ctx& ctx, const GridDims& g, const Model& model, Weights& weights, const LinOpDev& A,
                     const double* rhs, double tol, int maxIter, const PrecondChoice& choice, const double* mR,
                     const double* mT, const double* v, double coarseCfl, double* solution);

// Fine GN operator whose data term Q comes from Ctx::fine (an external, e.g. slab-decomposed,
// implementation): applySplit mirrors Hessian::launchSplit's spectral steps around the hook and
// bumps the reference's counters per matvec (Hessian::countDataTerm).
class ExternalFineOperator {
public:
    ExternalFineOperator(Ctx& ctx, const GridDims& g, const double* v, const Model& model, int nt, Weights& weights);
    void applySplit(const double* s, double* o);

private:
    Ctx& ctx_;
    GridDims g_;
    Model model_;
    int nt_;
    Weights& weights_;
    long long lazyInterps_ = 5, lazyFfts_ = 3;  // charFwd + charBwd + dvDep, div v (state reused)
};

// inverse::newtonSolve (newton.cpp:24-159) ---------------------------------------------------
struct NewtonConfig {
    int maxOuterIter = 50;
    double tolRelGrad = 1e-2;
    double tolAbsGrad = 1e-5;
    int maxInnerIter = 500;
    double forcingCap = 0.5;
    double lsC1 = 1e-4;
    double lsShrink = 0.5;
    int lsMaxSteps = 20;
    double gradCfl = 1.0;
    int ntOverride = 0;  // 0 = CFL-derived
    int hessianMode = 0;  // 0 Gauss-Newton, 1 full Newton (NewtonConfig::hessianMode)
    // NewtonConfig::hessScheme (inverse.hpp:35-40): the Hessian's own transport scheme and step
    // count (CFL-derived from its own cfl unless hessNtOverride > 0); absent = gradient's
    bool hasHessScheme = false;
    int hessScheme = 0;
    double hessCfl = 0.2;
    int hessNtOverride = 0;
};

struct IterationRecord {
    int iter = 0;
    double gradNormInf = 0, gradNormRel = 0, objective = 0, mismatch = 0;
    int innerIterations = 0, lineSearchSteps = 0;
    double stepLength = 0, searchDirDivRatio = 0, wallTimeSec = 0;
    long long ffts = 0, interps = 0;
};

enum SolveStatus : int { kConverged = 0, kIterationLimit = 1, kLineSearchFailure = 2 };

struct SolverReport {
    std::vector<IterationRecord> iterations;
    int status = kIterationLimit;
    double finalGradNormRel = 0, finalResidualRel = 0, jacMin = 1, jacMax = 1, totalTimeSec = 0;
};

constexpr double kCoarseCfl = 5.0;  // kCoarseScheme (newton.cpp:16)

SolverReport newtonSolve(Ctx& ctx, const GridDims& g, const double* mR, const double* mT, const Model& model,
                         const NewtonConfig& cfg, const PrecondChoice& pc, double* vOut);

}  // namespace vrg
