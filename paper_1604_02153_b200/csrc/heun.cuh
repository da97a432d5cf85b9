// RK2 / RK2A (antisymmetric) spectral transport: Heun steps with pseudospectral advection
// (transport.cpp:129-195, 267-309, 345-377, 426-464; inverse.cpp:30-88), SURVEY §8f f4.
//
// All derivatives are spectral (cuFFT); every right-hand side is a few FFTs plus pointwise work,
// so the scheme is FFT bound.  The combinations are evaluated with the reference's rounding
// steps (no contraction into FMAs): y + a x as __dadd_rn(y, __dmul_rn(a, x)).  Trajectories
// are (nt+1) node fields plus nt stage (Heun predictor) fields, as TransportSolution holds them.
#pragma once

#include "transport.cuh"

namespace vrg {

enum TransportScheme : int { kSchemeSL = 0, kSchemeRK2 = 1, kSchemeRK2A = 2 };

class HeunTransport {
public:
    HeunTransport(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, int nt, bool antisymmetric);
    Ctx& ctx;
    GridDims g;
    int nt;
    double ht;
    bool anti;
    DBuf v;  // [v1 | v2]
    GuardLog log;

    const double* divVelocity();  // lazy, 3 FFTs on first use (transport.cpp:114-118)
    // d_t m = F(m) (forward) and d_tau lambda = B(lambda) (reversed time)
    void forwardRhs(const double* m, double* out);
    void backwardRhs(const double* lam, double* out);
    // heunForward / heunBackward with the guard (state / adjoint) when `guard`
    void forward(const double* m0, double* nodes, double* stages, bool guard);
    void backward(const double* lam1, double* nodes, double* stages, bool guard);
    void stateFinal(const double* m0, double* out);
    void adjointFinal(const double* lam1, double* out);
    // Heun predictors of a trajectory's steps recomputed from its nodes (the C ABI passes
    // nodes only); forward: pred_j = m_{j-1} + ht F(m_{j-1}), backward: pred_{j-1} = lam_j + ht B(lam_j)
    void forwardStages(const double* nodes, double* stages);
    void backwardStages(const double* nodes, double* stages);
    // solveIncState RK2 (transport.cpp:345-377): source -S(m)[vt] at nodes and stages
    void incState(const double* vt1, const double* vt2, const double* stNodes, const double* stStages, double* out);
    // solveIncAdjoint full Newton RK2 (transport.cpp:426-453)
    void incAdjointFullNewton(const double* vt1, const double* vt2, const double* lt1, const double* adjNodes,
                              const double* adjStages, double* out);
    // jacobianDeterminant RK2 (transport.cpp:470-485)
    void jacobian(double* out);

private:
    DBuf divv_;
    bool haveDivv_ = false;
    DBuf work_;  // 8N
    double* w(int i) { return work_.d() + static_cast<std::size_t>(i) * g.points(); }
    void heunStep(const double* y, double* yNext, double* pred, bool fwd, const double* src1, const double* src2);
};

// v . grad(m) (advectBy, transport.cpp:22-28) and div(m v) (divOfProduct, transport.cpp:31-36)
void advectBy(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* m, double* out);
void divOfProduct(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* m, double* out);
// S(m)^T mu = (mu grad m - m grad mu + grad(mu m)) / 2 (inverse.cpp:32-44)
void antisymmetricForceTerm(Ctx& ctx, const GridDims& g, const double* m, const double* mu, double* o1, double* o2);
// assembleBodyForce for RK2/RK2A (inverse.cpp:67-87): b = sum over steps of the stage pairs
void bodyForceHeun(Ctx& ctx, const GridDims& g, int nt, bool anti, const double* stNodes, const double* stStages,
                   const double* adNodes, const double* adStages, double* b1, double* b2);

}  // namespace vrg
