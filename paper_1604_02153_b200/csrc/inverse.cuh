// Reduced-space operators on the device: inverse::HessianOperator (GN, SL) and the
// gradient/objective evaluations (include/veloreg/inverse.hpp:60-97, src/inverse.cpp:96-233).
#pragma once

#include <memory>

#include "transport.cuh"

namespace vrg {

enum Deformation : int { kCompressible = 0, kIncompressible = 1, kNearIncompressible = 2 };

struct Model {
    int norm = kH2;
    double betaV = 1e-2;
    int deformation = kCompressible;
    double betaW = 1e-1;
    int scheme = 0;  // transport scheme (heun.cuh TransportScheme); SchemeConfig in the reference
};

// GN Hessian at one velocity iterate, everything device-resident.
//
// Per-iterate invariants are built once in the constructor and reused by every matvec
// (they are pure functions of (v, m_T), so results are bit-identical to recomputing them as
// the reference does per call, src/inverse.cpp:177-187):
//   state m_j (j=0..nt), G_j = grad m_j, GD_j = (grad m_{j-1})_D at the forward departure
//   points (j=1..nt), X_D in both directions, div v and (div v)_D backward.
class Hessian {
public:
    // `stateTraj` (nullable): reuse a state trajectory (HessianOperator ctor, inverse.cpp:162-172).
    // hmode: 0 Gauss-Newton, 1 full Newton (HessianMode, transport.hpp; the full-Newton
    // operator solves the adjoint in the ctor, inverse.cpp:164-172)
    Hessian(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* mR, const double* mT,
            const Model& model, int nt, const double* stateTraj, int hmode = 0, const double* adjTraj = nullptr,
            const double* gradTraj = nullptr);  // gradTraj: grad m_j of stateTraj ((nt+1) x 2N), reused

    Ctx& ctx;
    GridDims g;
    Model model;
    int nt;
    Solver solver;
    Weights weights;

    // out = beta A vt + K[b(vt)]  (HessianOperator::apply, inverse.cpp:229-233)
    void apply(const double* vt1, const double* vt2, double* o1, double* o2);
    // out = K[b(vt)]  (applyDataTerm, inverse.cpp:235-237)
    void applyDataTerm(const double* vt1, const double* vt2, double* o1, double* o2);
    // out = M^{-1/2} Q M^{-1/2} s + s  (applySplitHessianOf, precond.cpp:20-26)
    void applySplit(const double* s1, const double* s2, double* o1, double* o2);

    ~Hessian();
    Hessian(const Hessian&) = delete;
    Hessian& operator=(const Hessian&) = delete;

    const double* state() const { return state_.d(); }
    bool useGraphs = true;  // false for the RK2/RK2A operator (host-checked Heun guards)
    // ms per launch of a matvec kernel class (0 incstate step, 1 adjoint+body-force step,
    // 2 prefilter (both passes), 3 two-field evaluate), timed back to back.
    double benchKernel(int id, int iters);
    // device-visible guard check result of the last data term (throws like solveAdjoint).
    void checkLastGuard();
    // Deferred guard checks for a device-resident loop of matvecs (the coarse Chebyshev
    // solve): between begin and end, each matvec appends its per-step guard maxima and flags
    // to a device log instead of synchronising; endDeferredGuards() reads the log once and
    // throws the first error in call order (the one the reference would have thrown).  GN SL
    // operators only; otherwise the checks stay immediate.
    void beginDeferredGuards(int maxCalls);
    void endDeferredGuards();
    // Queued matvecs (apply batches, C ABI vrg_hess_apply_batch / _host_batch): apply() without
    // the per-matvec host round trip.  The matvec's guard maxima and prefilter flags go to
    // pinned host slot `slot` (0 or 1) in stream order; checkQueued(slot) waits for that copy
    // only and throws what apply() would have thrown, so the host checks matvec i while matvec
    // i+1 runs.  queuedGuards(): GN SL/RK operators of one pair (elsewhere apply() is used).
    bool queuedGuards() const;
    void applyQueued(const double* vt1, const double* vt2, double* o1, double* o2, int slot);
    void checkQueued(int slot);
    // counter increments of one data term in the reference (steady state)
    void countDataTerm();
    // forget the lazily-built per-velocity work still to be counted (an operator rebuilt for a
    // problem whose operator already ran, batch.cu)
    void clearLazyCounts() {
        lazyInterps_ = 0;
        lazyFfts_ = 0;
    }
    // a batch of stacked pairs (GridDims::pairs > 1): the guard verdicts of the matvecs so far
    // (0 ok, else the C ABI status of the error the reference would throw; first error kept)
    // instead of exceptions
    std::vector<int> pairStatus;
    std::vector<std::string> pairError;

private:
    // b = sum_j w_j lt_j grad m_j of the GN incremental adjoint seeded with -m~(1).
    // If regOut1/2 non-null, the last step also writes out = reg + b (compressible fusion).
    void dataTerm(const double* vt1, const double* vt2, double* b1, double* b2, const double* reg1,
                  const double* reg2, double* out1, double* out2);

    void launchApply(const double* vt1, const double* vt2, double* o1, double* o2);
    void launchSplit(const double* s1, const double* s2, double* o1, double* o2);
    template <class F>
    void replay(int kind, const double* a, const double* b, const double* c, const double* d, F&& launchSeq);
    struct GraphKey {
        int kind;
        const double *a, *b, *c, *d;
        bool operator<(const GraphKey& o) const { return std::tie(kind, a, b, c, d) < std::tie(o.kind, o.a, o.b, o.c, o.d); }
    };
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        long long launches = 0;
        std::vector<Ctx::ProfRec> recs;   // profiled variant: event pairs inside the graph
        std::vector<cudaEvent_t> events;  // owned by the graph
    };
    std::map<GraphKey, GraphEntry> graphs_;

    DBuf state_;  // (nt+1) N
    DBuf G_;      // (nt+1) x [g1 | g2]
    DBuf GD_;     // nt x [gd1 | gd2], GD_[j-1] = (grad m_{j-1})_D
    DBuf work_;   // vtD (2N), mt ping-pong (2N), lam ping-pong (2N), b (2N), coef2 (N), reg (2N)
    DBuf spec_;   // 4 half spectra
    // Guard log of the data term's adjoint; queued matvecs alternate between the two (the graph
    // of slot s writes guardLogs_[s]: its readback overlaps the next matvec)
    GuardLog guardLogs_[2];
    GuardLog* adjLog_ = &guardLogs_[0];
    bool deferring_ = false;
    int deferCap_ = 0, deferCount_ = 0;
    DBuf deferMax_, deferFlags_;
    void guardAfterMatvec();
    cudaStream_t guardStream_ = nullptr;  // queued matvecs: guard readback of slot s into hostGuard_
    double* hostGuard_ = nullptr;         // pinned, 2 slots of guardSlotBytes()
    std::size_t guardSlotBytes() const { return (guardLogs_[0].bytes() + 15) / 16 * 16; }
    double* hostGuardSlot(int slot) const {
        return reinterpret_cast<double*>(reinterpret_cast<char*>(hostGuard_) + slot * guardSlotBytes());
    }
    cudaEvent_t evGuard_[2] = {nullptr, nullptr}, evDone_[2] = {nullptr, nullptr};
    long long lazyInterps_ = 0, lazyFfts_ = 0;
    bool fused_ = false;  // band kernels (gather + row pass) in the time loops, evalband.cuh
    int mode_ = 0;        // 1: full Newton
    DBuf adj_;            // full Newton: adjoint trajectory lambda_j, (nt+1) N
    DBuf fn_;             // full Newton: m~ and lt trajectories (2 (nt+1) N), work (7N)
    DBuf fnFlag_;         // full Newton: non-finite prefilter input
    void dataTermFN(const double* vt1, const double* vt2, double* b1, double* b2, const double* reg1,
                    const double* reg2, double* out1, double* out2);
    void addPenalty(const double* vt1, const double* vt2, double* b1, double* b2);
    // beta A vt on a second stream, joined before the data term's last step consumes it
    cudaStream_t aux_ = nullptr;
    cudaEvent_t evFork_ = nullptr, evJoin_ = nullptr;
    bool regPending_ = false;
    void waitReg();
    // RK2 / RK2A scheme (heun.cuh)
    std::unique_ptr<class HeunTransport> heun_;
    DBuf stStages_, adjStages_;
    void initHeun(const double* mR, const double* mT, const double* stateTraj, const double* adjTraj);
    void dataTermHeun(const double* vt1, const double* vt2, double* b1, double* b2, const double* reg1,
                      const double* reg2, double* out1, double* out2);

public:
    bool bandPath() const { return fused_; }
    // nodes, edges and programmatic (PDL) edges of the last captured matvec graph
    int graphInfo_[3] = {0, 0, 0};
    // device buffers of the per-iterate invariants: state (nt+1)N, G (nt+1)2N, GD nt 2N
    const double* gradTraj() const { return G_.d(); }
    const double* gradDepTraj() const { return GD_.d(); }
};

// One SL step of a slab-decomposed grid (C ABI vrg_slab_step).
void slabStep(Ctx& ctx, int kind, int n1, int n2, int L, int winBase, int winRows, const double* coef,
              const double* x1, const double* x2, const double* const* ops, int nops, double ht, double w,
              double* rowOut, double* guardPartials, unsigned* flag, unsigned* winErr);

void bodyForce(Ctx& ctx, const GridDims& g, int nt, const double* stateTraj, const double* adjTraj, double* b1,
               double* b2, double* gradTrajOut = nullptr);  // gradTrajOut: keeps grad m_j ((nt+1) x 2N)
// scalars[4] = [objective, mismatch, regTerm, penaltyTerm] (ObjectiveResult / GradientResult,
// inverse.hpp:47-58).  Nullable outputs: the state (and adjoint) trajectories, their RK2 / RK2A
// Heun predictor fields (nt fields each; ignored for SL), the body force before the Leray
// projection (GradientResult::bodyForce, 2 fields), grad m_j of the SL state ((nt+1) x 2N).
void evaluateObjective(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* mR,
                       const double* mT, const Model& model, int nt, double* scalars, double* stateOut,
                       double* stateStagesOut = nullptr);
void evaluateGradient(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* mR,
                      const double* mT, const Model& model, int nt, double* g1, double* g2, double* scalars,
                      double* stateOut, double* adjOut, const double* reuseState, double* gradTrajOut = nullptr,
                      double* bodyOut = nullptr, double* stateStagesOut = nullptr, double* adjStagesOut = nullptr);

}  // namespace vrg
