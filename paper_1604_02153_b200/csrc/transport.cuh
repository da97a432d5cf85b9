// Semi-Lagrangian transport on the device: transport::Solver (include/veloreg/transport.hpp:
// 71-100, src/transport.cpp:91-454), SL branches only.  The RK2/RK2A spectral schemes are out
// of scope and raise NotSupported at the C ABI.
#pragma once

#include <string>
#include <vector>

#include "blas.cuh"
#include "eval.cuh"
#include "spectral.cuh"

namespace vrg {

enum Direction : int { kForward = 0, kBackward = 1 };

// transport::deriveSteps (src/transport.cpp:44-50) on device fields.
int deriveSteps(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, double cfl);

// traceCharacteristics (src/transport.cpp:60-89), from the prefiltered velocity
// coefficients (cv1, cv2) so both directions share one prefilter.
void launchTrace(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, const double* cv1,
                 const double* cv2, double ht, int dir, double* x1, double* x2);

// Block maxima of |f| into guard partials (evaluate block layout).
void launchFieldMax(Ctx& ctx, const GridDims& g, const double* f, double* partial);

// Per-step guard bookkeeping for one solve: block maxima per step, reduced per step, plus the
// prefilter non-finite flags, read back once when the solve ends.
// Batched solves (batch.cu) collect every pair's guard verdict instead of throwing, whatever
// the number of pairs of an operator (a coarse group can hold a single pair); set for the
// duration of a batched solve on the calling thread.
extern thread_local bool g_collectGuards;
struct CollectGuardsScope {
    bool prev;
    explicit CollectGuardsScope(bool on = true) : prev(g_collectGuards) { g_collectGuards = on; }
    ~CollectGuardsScope() { g_collectGuards = prev; }
};

struct GuardLog {
    int steps = 0;        // number of step slots (nt+1)
    int pairs = 1;
    // one device buffer: steps x pairs doubles of per-step guard maxima (atomic max, eval.cuh
    // guardMax), then steps unsigned prefilter flags; read back in one copy into the context's
    // pinned staging (Ctx::hostStage)
    DBuf buf;
    std::size_t bytes() const { return sizeof(double) * steps * pairs + sizeof(unsigned) * steps; }
    double* stepMax() const { return buf.d(); }
    unsigned* flags() const { return reinterpret_cast<unsigned*>(buf.d() + static_cast<std::size_t>(steps) * pairs); }
    // batch (pairs > 1): check() records each pair's verdict instead of throwing (0 ok, else the
    // C ABI status of the error the reference would throw) and its message
    std::vector<int> pairStatus;
    std::vector<std::string> pairError;
    void ensure(int nsteps, const GridDims& g);
    // the kernels' guard slot of a step (one per pair)
    double* partial(int step) const { return stepMax() + static_cast<std::size_t>(step) * pairs; }
    unsigned* flag(int step) const { return flags() + step; }
    void reset(Ctx& ctx);
    // Host readback; throws the reference's first error in solve order.
    //   order: steps visited, each (prefilter-input step index, output step index).
    void check(Ctx& ctx, const char* eq, int nt, bool forward, bool guard, int thresholdStep);
    // The same decisions on host copies of stepMax / flags (deferred checks).
    static void checkHost(const double* mx, const unsigned* fl, const char* eq, int nt, bool forward, bool guard,
                          int thresholdStep);
};

class Solver {
public:
    Solver(Ctx& ctx, const GridDims& g, const double* v1, const double* v2, int nt);
    Ctx& ctx;
    GridDims g;
    int nt;
    double ht;
    DBuf v;  // [v1 | v2]

    const double* v1() const { return v.d(); }
    const double* v2() const { return v.d() + g.points(); }

    // Lazy per-velocity caches (src/transport.cpp:107-127), with the reference's counter
    // increments when first built.
    const double* departure(int dir);  // [x1 | x2]
    // The departure points packed for the gathers of the band path (interp.cuh: Cell), [c1 | c2];
    // built once per direction from departure(dir), no counter increments.
    const Cell* cells(int dir);
    const double* divVelocity();
    const double* divVelocityAtDeparture(int dir);

    // Scratch owned by the solver.
    double* coef();
    bool bandPath() const;
    double* tmp();

    // slState (src/transport.cpp:214-227): traj = (nt+1) fields, traj[0] = m0.
    void state(const double* m0, double* traj, bool guard);
    // solveStateFinal (src/transport.cpp:267-278): out = m(1), two ping-pong buffers.
    void stateFinal(const double* m0, double* out);
    // slAdjoint (src/transport.cpp:229-241): traj[nt] = lam1, marching back.
    void adjoint(const double* lam1, double* traj, bool guard);
    void adjointFinal(const double* lam1, double* out);
    // solveIncState SL (src/transport.cpp:322-342): out trajectory (nt+1) fields.
    void incState(const double* vt1, const double* vt2, const double* stateTraj, double* out);
    // solveIncAdjoint, full-Newton SL (src/transport.cpp:403-420): traj (nt+1 frames, traj[nt] =
    // lt1) from the adjoint trajectory `adj`; work holds 5N; a non-finite prefilter input sets
    // *flag.  No guard (as in the reference).
    void incAdjointFullNewton(const double* vt1, const double* vt2, const double* lt1, const double* adj,
                              double* traj, double* work, unsigned* flag);

    // jacobianDeterminant SL (src/transport.cpp:456-464).
    void jacobian(double* out);

    // One SL continuity step (slContinuityStep, src/transport.cpp:200-212) of u along dir.
    void continuityStep(const double* u, double* out, int dir, double* guardPartial, unsigned* flag);

    GuardLog log;


private:
    template <class DstFn>
    void continuityBand(const double* lam1, DstFn dst, int dir);
    DBuf cv_;  // prefiltered velocity [c1 | c2]
    DBuf X_[2], cells_[2];
    DBuf divv_, dvDep_[2];
    DBuf coef_, tmp_;
    bool haveCv_ = false, haveX_[2] = {false, false}, haveCells_[2] = {false, false}, haveDivv_ = false, haveDvDep_[2] = {false, false};
};

}  // namespace vrg
