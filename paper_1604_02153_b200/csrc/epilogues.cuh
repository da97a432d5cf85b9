// Epilogues of the SL transport steps (shared by transport.cu and inverse.cu).
#pragma once

#include "eval.cuh"

namespace vrg {

// K3 epilogue: X_D = x - sgn*0.5*ht*(v + v(x*)), evaluated with the reference's operation
// order and no FMA contraction (src/transport.cpp:84-85), so X_D is bit-identical.
struct EpiTrace {
    static constexpr const char* kName = "evaluate/trace";
    static constexpr bool kGuard = false;
    double* guardPartials = nullptr;
    const double* v1;
    const double* v2;
    double* x1;
    double* x2;
    int n1, n2;  // one pair's grid (stacked pairs: node p is node p mod n1 n2 of its pair)
    double h1, h2, sgnHalfHt;
    VRG_NO_PREFETCH
    __device__ double operator()(std::size_t p, const double* vs, const Pre&) const {
        const std::size_t row = p / n2;
        const int i1 = static_cast<int>(row % n1), i2 = static_cast<int>(p - row * n2);
        const double c1 = __dadd_rn(-kPi, __dmul_rn(h1, static_cast<double>(i1)));
        const double c2 = __dadd_rn(-kPi, __dmul_rn(h2, static_cast<double>(i2)));
        x1[p] = __dsub_rn(c1, __dmul_rn(sgnHalfHt, __dadd_rn(v1[p], vs[0])));
        x2[p] = __dsub_rn(c2, __dmul_rn(sgnHalfHt, __dadd_rn(v2[p], vs[1])));
        return 0.0;
    }
};

// K4 epilogue: m_j = I[m_{j-1}](X_D) with the guard watching |m_j|.
struct EpiStateStep {
    static constexpr const char* kName = "evaluate/state_step";
    static constexpr bool kGuard = true;
    double* guardPartials;
    double* out;
    VRG_NO_PREFETCH
    __device__ double operator()(std::size_t p, const double* v, const Pre&) const {
        out[p] = v[0];
        return v[0];
    }
};

// K5 epilogue (slContinuityStep, src/transport.cpp:206-210).
struct EpiContinuity {
    static constexpr const char* kName = "evaluate/continuity";
    static constexpr bool kGuard = true;
    double* guardPartials;
    const double* dvDep;
    const double* dv;
    double ht;
    double* out;
    struct Pre {
        double dvDep, dv;
    };
    __device__ Pre prefetch(std::size_t p) const { return {dvDep[p], dv[p]}; }
    __device__ double operator()(std::size_t p, const double* v, const Pre& q) const {
        const double uD = v[0];
        const double f0 = uD * q.dvDep;
        const double pred = uD + ht * f0;
        const double o = uD + 0.5 * ht * (f0 + pred * q.dv);
        out[p] = o;
        return o;
    }
};

// Full-Newton SL incremental adjoint step (solveIncAdjoint, src/transport.cpp:409-418): the
// continuity step with the source q = div(lambda vt) at the departure points (qD) and at the
// arrival points of the next time node (qPrev).
struct EpiContinuityFN {
    static constexpr const char* kName = "evaluate/continuity_fn";
    static constexpr bool kGuard = false;
    double* guardPartials = nullptr;
    const double* dvDep;
    const double* dv;
    const double* qD;
    const double* qPrev;
    double ht;
    double* out;
    struct Pre {
        double dvDep, dv, qD, qPrev;
    };
    __device__ Pre prefetch(std::size_t p) const { return {dvDep[p], dv[p], qD[p], qPrev[p]}; }
    __device__ double operator()(std::size_t p, const double* v, const Pre& q) const {
        const double lamTD = v[0];
        const double f0 = lamTD * q.dvDep + q.qD;
        const double pred = lamTD + ht * f0;
        const double o = lamTD + 0.5 * ht * (f0 + pred * q.dv + q.qPrev);
        out[p] = o;
        return o;
    }
};

// K6 epilogue (solveIncState SL, src/transport.cpp:333-338).
struct EpiIncState {
    static constexpr const char* kName = "evaluate/incstate";
    static constexpr bool kGuard = false;
    double* guardPartials = nullptr;
    const double* vt1D;
    const double* vt2D;
    const double* gd1;
    const double* gd2;
    const double* vt1;
    const double* vt2;
    const double* g1;
    const double* g2;
    double halfHt;
    double* out;
    // the whole source term is independent of the gathered value
    struct Pre {
        double s;
    };
    __device__ Pre prefetch(std::size_t p) const {
        // GD_j / G_j are read once per matvec: streamed with evict-first so the per-matvec
        // fields (vt, vt_D, X_D) stay L2-resident across the nt steps
        const double sPrevD = -(vt1D[p] * __ldcs(gd1 + p) + vt2D[p] * __ldcs(gd2 + p));
        const double sCur = -(vt1[p] * __ldcs(g1 + p) + vt2[p] * __ldcs(g2 + p));
        return {halfHt * (sPrevD + sCur)};
    }
    __device__ double operator()(std::size_t p, const double* v, const Pre& q) const {
        const double o = v[0] + q.s;
        if (out) out[p] = o;  // null in the fused band path (only the row-filtered field is kept)
        return o;
    }
};

}  // namespace vrg
