/* vrg.h — C ABI of libvrg, the B200-native (sm_100a) drop-in for the reduced-space
 * Gauss–Newton Hessian-matvec path of the reference solver `veloreg`
 * (arXiv 1604.02153; reference C++ API in /root/reference/proj/core/include/veloreg).
 *
 * Every entry point replaces one reference interface, cited as path:line relative to
 * /root/reference/proj/core.  Conventions:
 *   - plain C: int status, opaque handles, plain pointers and sizes, no exceptions;
 *   - fields are fp64 arrays of n1*n2 values, row-major, axis 1 fastest, node (i1,i2) at
 *     (-pi + i1*2pi/n1, -pi + i2*2pi/n2) (include/veloreg/field.hpp:13-54); a trajectory is
 *     (nt+1) consecutive fields; a vector field is two pointers (components 0 and 1);
 *   - unless a name ends in _host, array arguments are DEVICE pointers on the context's
 *     device; calls are ordered on the context's stream; calls that return host-visible
 *     results (scalars, errors) synchronise that stream;
 *   - status codes mirror the reference's exception types: VRG_INVALID_ARGUMENT for
 *     std::invalid_argument, VRG_BLOWUP for transport::BlowupError (transport.hpp:35-38);
 *     the message (identical to the reference's what()) is returned by vrg_last_error(ctx);
 *   - operation counters follow counters.hpp:1-23 semantics; read them per context with
 *     vrg_counters and add them to the process counters the host keeps.
 */
#ifndef VRG_H
#define VRG_H

#ifdef __cplusplus
extern "C" {
#endif

#define VRG_OK 0
#define VRG_INVALID_ARGUMENT 1
#define VRG_BLOWUP 2
#define VRG_RUNTIME_ERROR 3
#define VRG_NOT_SUPPORTED 4

/* enum values shared with the reference */
#define VRG_H1SEMI 1 /* spectral::RegNorm (spectral.hpp:12) */
#define VRG_H2SEMI 2
#define VRG_H3SEMI 3
#define VRG_COMPRESSIBLE 0 /* inverse::Deformation (inverse.hpp:15) */
#define VRG_INCOMPRESSIBLE 1
#define VRG_NEAR_INCOMPRESSIBLE 2
#define VRG_FORWARD 0 /* transport::TraceDirection (transport.hpp:15) */
#define VRG_BACKWARD 1
#define VRG_GAUSS_NEWTON 0 /* transport::HessianMode (transport.hpp:16) */
#define VRG_FULL_NEWTON 1

/* transport schemes (transport::Scheme, transport.hpp) */
#define VRG_SCHEME_SL 0
#define VRG_SCHEME_RK2 1
#define VRG_SCHEME_RK2A 2
#define VRG_BAND_LOW 0 /* spectral::Band (spectral.hpp:44) */
#define VRG_BAND_HIGH 1

/* inverse::Model (inverse.hpp:18-23), passed per call to the _ex entry points: the legacy entry
 * points take norm / beta / deformation as arguments and betaW / the scheme from the context
 * (vrg_set_penalty_weight, vrg_set_scheme); the _ex ones take everything per call, so operators
 * with different models can share one context. */
typedef struct vrg_model_s {
    int norm;          /* VRG_H1SEMI .. VRG_H3SEMI (spectral::RegNorm) */
    double beta_v;     /* Model::betaV */
    int deformation;   /* VRG_COMPRESSIBLE, VRG_INCOMPRESSIBLE, VRG_NEAR_INCOMPRESSIBLE */
    double beta_w;     /* Model::betaW (near-incompressible penalty weight), default 0.1 */
} vrg_model;
/* transport::SchemeConfig (transport.hpp:23-27) */
typedef struct vrg_scheme_cfg_s {
    int scheme;        /* VRG_SCHEME_SL / _RK2 / _RK2A */
    double cfl;
    int nt_override;   /* 0 = none (CFL-derived step count) */
} vrg_scheme_cfg;
/* inverse::NewtonConfig (inverse.hpp:25-41) */
typedef struct vrg_newton_cfg_s {
    int max_outer_iter;        /* 50 */
    double tol_rel_grad;       /* 1e-2 */
    double tol_abs_grad;       /* 1e-5 */
    int max_inner_iter;        /* 500 */
    double forcing_cap;        /* 0.5 */
    double ls_c1;              /* 1e-4 */
    double ls_shrink;          /* 0.5 */
    int ls_max_steps;          /* 20 */
    int hessian_mode;          /* VRG_GAUSS_NEWTON / VRG_FULL_NEWTON */
    vrg_scheme_cfg grad_scheme;  /* {SL, 1.0, none} */
    int has_hess_scheme;       /* NewtonConfig::hessScheme engaged (0: the gradient's) */
    vrg_scheme_cfg hess_scheme;
} vrg_newton_cfg;
/* precond::PrecondChoice (precond.hpp:19-27) */
typedef struct vrg_precond_choice_s {
    int kind;                  /* 0 Reg (default), 1 TwoLevel */
    int coarse_solver;         /* 0 Pcg, 1 Cheb (default) */
    double eps_scale;          /* 0.1 */
    int cheb_iters;            /* 10 */
    int has_eig;               /* eigEstimate engaged */
    double emin, emax;
    int reestimate_each_iteration;
} vrg_precond_choice;

typedef struct vrg_ctx_s* vrg_ctx_t;
typedef struct vrg_solver_s* vrg_solver_t;
typedef struct vrg_hess_s* vrg_hess_t;
typedef struct vrg_coarse_s* vrg_coarse_t;

/* ---- context / memory (no reference counterpart: the device runtime under the pImpls) ---- */
const char* vrg_version(void);
int vrg_ctx_create(int device, void* cuda_stream /* nullable: own stream */, vrg_ctx_t* out);
/* the CUDA stream the context launches on (its own non-blocking stream when created with a
 * NULL stream), for callers that order their own work with the library's */
void* vrg_ctx_stream(vrg_ctx_t ctx);
/* Model::betaW (inverse.hpp:21), the H1 penalty weight on div v of the near-incompressible
 * model (deformation 2), used by the calls on this context; default 0.1 as in the reference */
int vrg_set_penalty_weight(vrg_ctx_t ctx, double beta_w);
/* SchemeConfig::scheme (VRG_SCHEME_SL default, VRG_SCHEME_RK2, VRG_SCHEME_RK2A: Heun steps with
 * spectral advection, transport.cpp:129-195) of the solvers, operators, gradients and Newton
 * solves created on this context; the two-level preconditioner's coarse problem stays SL(5)
 * as in the reference (precond.cpp kCoarseScheme) */
int vrg_set_scheme(vrg_ctx_t ctx, int scheme);
void vrg_ctx_destroy(vrg_ctx_t ctx);
const char* vrg_last_error(vrg_ctx_t ctx); /* ctx may be NULL: last error of this thread */
int vrg_sync(vrg_ctx_t ctx);
/* device memory for use in the context's stream order (stream-ordered block cache: no device
 * synchronisation on free); vrg_free takes only vrg_malloc blocks of the same context */
int vrg_malloc(vrg_ctx_t ctx, unsigned long long bytes, void** out);
int vrg_free(vrg_ctx_t ctx, void* p);
int vrg_host_alloc(vrg_ctx_t ctx, unsigned long long bytes, void** out); /* pinned */
int vrg_host_free(vrg_ctx_t ctx, void* p);
int vrg_copy_h2d(vrg_ctx_t ctx, void* dst, const void* src, unsigned long long bytes);
int vrg_copy_d2h(vrg_ctx_t ctx, void* dst, const void* src, unsigned long long bytes);
/* counters::snapshot / counters::reset (counters.hpp:16-20, counters.cpp:10-22), per context */
int vrg_counters(vrg_ctx_t ctx, long long* ffts, long long* interps);
int vrg_counters_reset(vrg_ctx_t ctx);
/* instrumentation (no reference counterpart): kernels this library launched on the context,
 * and an optional CUDA-event profile per launch site.  vrg_profile_dump writes lines
 * "tag<TAB>launches<TAB>total_ms" and resets the profile. */
int vrg_launch_count(vrg_ctx_t ctx, long long* launches);
int vrg_profile(vrg_ctx_t ctx, int enable);
int vrg_profile_dump(vrg_ctx_t ctx, char* buf, int cap);

/* ---- field BLAS-1 (field.hpp:62-80, field.cpp:19-119) ---- */
int vrg_dot(vrg_ctx_t ctx, int n1, int n2, const double* a1, const double* a2, const double* b1, const double* b2,
            double* out); /* a2/b2 may be NULL for scalar fields */
int vrg_norm_linf(vrg_ctx_t ctx, int n1, int n2, const double* a1, const double* a2, double* out);
int vrg_axpy(vrg_ctx_t ctx, unsigned long long n, double a, const double* x, double* y);

/* ---- interp (interp.hpp:27-34) ---- */
int vrg_prefilter(vrg_ctx_t ctx, int n1, int n2, const double* u, double* c);
int vrg_evaluate(vrg_ctx_t ctx, int n1, int n2, const double* c, const double* x1, const double* x2, double* out);

/* ---- transport (transport.hpp:18-113) ---- */
int vrg_derive_steps(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, double cfl, int* nt);
int vrg_trace(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, double ht, int direction,
              double* x1, double* x2); /* traceCharacteristics, transport.hpp:49 */
/* transport::Solver (transport.hpp:71-100), scheme SL. */
int vrg_solver_create(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, int nt, vrg_solver_t* out);
/* transport::Solver(v, TimeGrid(nt), SchemeConfig{scheme}) with the scheme given per call */
int vrg_solver_create_ex(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, int nt, int scheme,
                         vrg_solver_t* out);
/* TransportSolution::stages (transport.hpp:61-66): the nt Heun predictor fields of the solver's
 * last state / adjoint solve (RK2 / RK2A; VRG_NOT_SUPPORTED for SL, whose stages are empty) */
int vrg_solver_stages(vrg_solver_t s, double* out);
void vrg_solver_destroy(vrg_solver_t s);
int vrg_solver_state(vrg_solver_t s, const double* m0, double* traj);        /* solveState */
int vrg_solver_adjoint(vrg_solver_t s, const double* lam1, double* traj);    /* solveAdjoint */
int vrg_solver_state_final(vrg_solver_t s, const double* m0, double* out);   /* solveStateFinal */
int vrg_solver_adjoint_final(vrg_solver_t s, const double* lam1, double* out); /* solveAdjointFinal */
int vrg_solver_incstate(vrg_solver_t s, const double* vt1, const double* vt2, const double* state_traj,
                        double* traj); /* solveIncState */
int vrg_solver_incadjoint(vrg_solver_t s, const double* vt1, const double* vt2, const double* lt1,
                          const double* adjoint_traj /* nullable */, int mode, double* traj); /* solveIncAdjoint */
int vrg_solver_jacobian(vrg_solver_t s, double* out);                        /* jacobianDeterminant */
int vrg_solver_departure(vrg_solver_t s, int direction, double* x1, double* x2); /* cached Characteristics */

/* ---- spectral (spectral.hpp:27-56) ---- */
int vrg_gradient(vrg_ctx_t ctx, int n1, int n2, const double* u, double* g1, double* g2);
int vrg_divergence(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, double* out);
int vrg_apply_reg(vrg_ctx_t ctx, int n1, int n2, int norm, double beta, const double* v1, const double* v2,
                  double* o1, double* o2);
int vrg_apply_inv_reg(vrg_ctx_t ctx, int n1, int n2, int norm, double beta, double power, const double* v1,
                      const double* v2, double* o1, double* o2);
int vrg_project_div_free(vrg_ctx_t ctx, int n1, int n2, const double* b1, const double* b2, double* o1, double* o2);
int vrg_resample(vrg_ctx_t ctx, int n1, int n2, const double* u, int t1, int t2, double* out);
int vrg_cutoff(vrg_ctx_t ctx, int n1, int n2, const double* u, int band, double* out);
int vrg_gaussian_smooth(vrg_ctx_t ctx, int n1, int n2, const double* u, double sigma, double* out);
/* applyHelmholtz (spectral.hpp:56, spectral.cpp:214-223): (1 - Lap) u, Nyquist-zeroed waves */
int vrg_apply_helmholtz(vrg_ctx_t ctx, int n1, int n2, const double* u, double* out);
/* assembleBodyForce, SL scheme (inverse.cpp:50-65): b = sum_j w_j lambda_j grad m_j, trapezoid
 * weights ht/2 at the ends, ht inside; state_traj / adj_traj = (nt+1) contiguous fields each */
int vrg_body_force(vrg_ctx_t ctx, int n1, int n2, int nt, const double* state_traj, const double* adj_traj,
                   double* b1, double* b2);

/* ---- inverse (inverse.hpp:60-105) ---- */
/* inverse::HessianOperator(v, problem, model, tg, cfg{SL}, mode, state) (inverse.hpp:74-80).
 * state_traj: nullable device trajectory to reuse (inverse.cpp:162-172). */
int vrg_hess_create(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                    const double* mT, int norm, double beta, int deformation, int nt, int mode,
                    const double* state_traj, vrg_hess_t* out);
/* inverse::HessianOperator(v, problem, model, TimeGrid(nt), SchemeConfig{scheme}, mode, state,
 * adjoint) (inverse.hpp:74-80): model and scheme per call; state_traj / adjoint_traj (nullable)
 * are the reused trajectories (inverse.cpp:162-172), copied; the adjoint is used in full-Newton
 * mode only.  RK2 / RK2A predictor fields are recomputed from the nodes (same arithmetic). */
int vrg_hess_create_ex(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                       const double* mT, const vrg_model* model, int scheme, int nt, int mode,
                       const double* state_traj, const double* adjoint_traj, vrg_hess_t* out);
/* A Gauss-Newton SL HessianOperator of `pairs` stacked image pairs (batch fields: pair after pair,
 * v1 / v2 / mR / mT each pairs x n1 x n2 device doubles); apply / apply_data / apply_split then
 * take and return batch fields, each pair's result equal to its own operator's. */
int vrg_hess_create_batch(vrg_ctx_t ctx, int n1, int n2, int pairs, const double* v1, const double* v2,
                          const double* mR, const double* mT, int norm, double beta, int deformation, int nt,
                          vrg_hess_t* out);
void vrg_hess_destroy(vrg_hess_t h);
int vrg_hess_apply(vrg_hess_t h, const double* vt1, const double* vt2, double* o1, double* o2);      /* apply */
int vrg_hess_apply_data(vrg_hess_t h, const double* vt1, const double* vt2, double* o1, double* o2); /* applyDataTerm */
/* applySplitHessianOf (precond.cpp:20-26): M^{-1/2} Q M^{-1/2} s + s */
int vrg_hess_apply_split(vrg_hess_t h, const double* s1, const double* s2, double* o1, double* o2);
/* apply() from HOST buffers: H2D of vtilde, matvec, D2H of the result (the drop-in call a
 * host-side caller of HessianOperator::apply makes; value semantics of inverse.hpp:83). */
int vrg_hess_apply_host(vrg_hess_t h, const double* vt1, const double* vt2, double* o1, double* o2);
/* k independent apply_host calls (inputs vt1[i], vt2[i] -> outputs o1[i], o2[i], host buffers,
 * pinned for overlap) with the host<->device copies of neighbouring matvecs overlapped with the
 * compute of the current one (two copy streams, two device slots), and each matvec's guard
 * checked on the host while the next one runs.  Same results and error behaviour as k
 * apply_host calls in order: the first failing matvec's error is returned, the outputs before
 * it are delivered, the failing one's and later ones are not written. */
int vrg_hess_apply_host_batch(vrg_hess_t h, int k, const double* const* vt1, const double* const* vt2,
                              double* const* o1, double* const* o2);
/* k apply calls on DEVICE buffers queued back to back (HessianOperator::apply, inverse.cpp:
 * 229-233, repeated): each matvec's guard is checked on the host while the next one runs, so
 * the device never waits for the host between matvecs.  Same results as k apply calls; on an
 * error (the first failing matvec's, as apply would throw it) the outputs of the matvecs before
 * it are final and the failing one's and the next one's may have been written. */
int vrg_hess_apply_batch(vrg_hess_t h, int k, const double* const* vt1, const double* const* vt2, double* const* o1,
                         double* const* o2);
int vrg_hess_state(vrg_hess_t h, double* traj); /* copy of the held state trajectory */
/* instrumentation: average ms of one launch of a matvec kernel class (0 incremental-state
 * step, 1 incremental-adjoint + body-force step, 2 prefilter (both passes), 3 two-field
 * evaluate, 4 column pass, 5 D2D copy, 6 axpy, 7 band incremental-state step, 8 band
 * incremental-adjoint step, 9 SL state step band form (gather + next row pass, then column
 * pass), 10 SL state step plain form (prefilter + gather)), `iters` back-to-back launches on the context stream (bench.py roofline) */
int vrg_hess_bench_kernel(vrg_hess_t h, int kernel, int iters, double* ms_per_launch);
/* instrumentation: row-to-SM mapping of the band steps for operators created afterwards (0 = by
 * grid size, 1 = one block per grid row, 2 = strip blocks of consecutive rows where the row
 * length allows it); process-wide, returns the previous mode.  Both forms compute identical
 * bits; tests and the kernel benchmark use it to compare them. */
int vrg_band_mapping(int mode);
/* 1 when the time loops run the band kernels (gather + epilogue + next row pass fused; ids 7
 * and 8 of vrg_hess_bench_kernel), 0 for the plain 3-kernel step */
/* instrumentation: nodes, edges and programmatic-dependent-launch edges of the operator's last
 * captured matvec graph (info[3]) */
int vrg_hess_graph_info(vrg_hess_t h, int* info);
int vrg_hess_band_path(vrg_hess_t h, int* band);
/* device pointers of the operator's per-iterate invariants (read only, owned by h):
 * [0] state m_j, (nt+1) fields; [1] grad m_j, (nt+1) x [d1 | d2]; [2] (grad m_{j-1})_D, nt x
 * [d1 | d2]; [3] forward departure points [x1 | x2]; [4] backward departure points; [5] div v;
 * [6] (div v) at the backward departure points.  Used to set up slab-decomposed operators. */
int vrg_hess_buffers(vrg_hess_t h, const double** ptrs);

/* ---- slab decomposition (host orchestration in slab.py) ----------
 * A slab owns rows r0 .. r0+L-1 of an n1 x n2 grid.  Its coefficient window holds winRows
 * padded rows (n2+3 columns, periodic column padding), window row w = grid row winBase + w
 * (mod n1).  The prefilter of a slab field is: vrg_prefilter_rows on the L local rows, halo
 * exchange of the row-filtered rows (winRows + 64 rows: window - 32 .. window + winRows + 31),
 * then vrg_slab_cols.  Row pass only: rowFiltered = n1 x n2 (unpadded). */
int vrg_prefilter_rows(vrg_ctx_t ctx, int n1, int n2, const double* u, double* rowFiltered, unsigned* nonfinite);
int vrg_slab_cols(vrg_ctx_t ctx, int winRows, int n2, const double* inHalo, double* window);
/* One SL step over the slab's L rows (band kernel: gather from the window at the departure
 * points x1/x2 of the local rows (global coordinates), epilogue, and the row pass of the result
 * into rowOut).  kind / operand fields `ops` (each L x n2):
 *   0 store            out = I[c](X)                                   ops: out
 *   1 incstate         m~ = I[c](X) + ht/2 (-vtD.GD - vt.G)            ops: vtD1 vtD2 gd1 gd2 vt1 vt2 g1 g2
 *   2 incstate, m~_0=0 (no gather)                                     ops: as 1
 *   3/4 last incstate + adjoint seed (gather / no gather): returns lt(1) = -m~(1), b = w lt(1) G
 *                                                                      ops: as 1, b1 b2
 *   5 adjoint + body force  b += w lt G                                ops: dvD dv g1 g2 b1 b2
 *   6 last adjoint step     out = reg + b + w lt G                     ops: as 5, reg1 reg2 out1 out2
 *   7 state step        out = I[c](X)  (guarded)                       ops: out
 * guardPartials: L per-row maxima |result| (kinds 3-7); nonfinite: set if a result is not
 * finite; winErr: set if a departure cell's taps fall outside the window. */
int vrg_slab_step(vrg_ctx_t ctx, int kind, int n1, int n2, int L, int winBase, int winRows, const double* coef,
                  const double* x1, const double* x2, const double* const* ops, int nops, double ht, double w,
                  double* rowOut, double* guardPartials, unsigned* nonfinite, unsigned* winErr);

/* evaluateGradient / evaluateObjective (inverse.hpp:60-71); scalars = [objective, mismatch, regTerm] */
int vrg_evaluate_gradient(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                          const double* mT, int norm, double beta, int deformation, int nt, double* g1, double* g2,
                          double* scalars);
int vrg_evaluate_objective(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                           const double* mT, int norm, double beta, int deformation, int nt, double* scalars);

/* evaluateGradient(v, problem, model, TimeGrid(nt), {scheme}, reuseState) (inverse.hpp:65-68,
 * inverse.cpp:119-148) with every GradientResult member: g, bodyForce (before the Leray
 * projection), state and adjoint trajectories ((nt+1) fields each) and their Heun predictor
 * fields (nt fields each, RK2 / RK2A only); scalars = [objective, mismatch, regTerm, penaltyTerm].
 * reuse_state and every output except g1/g2/scalars are nullable. */
int vrg_evaluate_gradient_ex(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                             const double* mT, const vrg_model* model, int scheme, int nt, const double* reuse_state,
                             double* g1, double* g2, double* body /* [b1 | b2] */, double* state_traj,
                             double* state_stages, double* adjoint_traj, double* adjoint_stages, double* scalars);
/* evaluateObjective (inverse.hpp:60-63, inverse.cpp:96-117): ObjectiveResult with the state */
int vrg_evaluate_objective_ex(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                              const double* mT, const vrg_model* model, int scheme, int nt, double* state_traj,
                              double* state_stages, double* scalars);

/* ---- precond (precond.hpp:25-95) ---- */
/* problems::randomBandLimitedField (problems.hpp:45): libstdc++ mt19937_64 + normal draws */
int vrg_random_bandlimited_field(vrg_ctx_t ctx, int n1, int n2, unsigned long long seed, double* out);
/* precond::CoarseOperator(vFine, problem, model, coarseScheme{SL, cfl}) (precond.hpp:56-70);
 * v1/v2 may be NULL for v = 0. */
int vrg_coarse_create(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                      const double* mT, int norm, double beta, int deformation, double coarse_cfl, vrg_coarse_t* out);
void vrg_coarse_destroy(vrg_coarse_t c);
int vrg_coarse_info(vrg_coarse_t c, int* n1c, int* n2c, int* nt); /* grid() and the CFL-derived coarse nt */
/* CoarseOperator::applySplitHessian; s/out are coarse-grid fields */
int vrg_coarse_apply_split(vrg_coarse_t c, const double* s1, const double* s2, double* o1, double* o2);
/* applyTwoLevel(r, coarse, choice, outerTol, eMin, eMax) (precond.hpp:74-78); coarse_solver 0 = PCG, 1 = CHEB.
 * Returns VRG_OK; *fallback = 1 when the coarse solve diverged and the identity was applied. */
int vrg_two_level_apply(vrg_coarse_t c, const double* r1, const double* r2, int coarse_solver, int cheb_iters,
                        double eps_scale, double outer_tol, double emin, double emax, double* o1, double* o2,
                        int* fallback);
/* estimateEigs / estimateEigsAt (precond.hpp:40-53): Lanczos(30) eMax of the coarse split Hessian */
int vrg_estimate_eigs(vrg_ctx_t ctx, int n1, int n2, const double* v1, const double* v2, const double* mR,
                      const double* mT, int norm, double beta, int deformation, double coarse_cfl,
                      unsigned long long seed, double* emin, double* emax);
/* solveKkt(hess, rhs, tol, maxIter, choice, problem, v, coarseScheme) (precond.hpp:93-95).
 * pc_int = [kind(0 reg, 1 two-level), coarse_solver, cheb_iters, has_eig]; pc_dbl = [eps_scale, emin, emax];
 * result = [iterations, converged, negative_curvature, rel_residual, total_s, precond_s]. */
int vrg_solve_kkt(vrg_hess_t h, const double* rhs1, const double* rhs2, double tol, int max_iter, const int* pc_int,
                  const double* pc_dbl, const double* mR, const double* mT, const double* v1, const double* v2,
                  double coarse_cfl, double* sol1, double* sol2, double* result);

/* ---- newton (newton.hpp:10-12): inverse::newtonSolve on HOST images mR/mT, v returned on the host.
 * cfg_int = [maxOuterIter, maxInnerIter, ntOverride(0 = CFL), lsMaxSteps, hessianMode (VRG_GAUSS_NEWTON |
 *            VRG_FULL_NEWTON)]
 * cfg_dbl = [tolRelGrad, tolAbsGrad, forcingCap, lsC1, lsShrink, gradCfl]
 * pc_int / pc_dbl as for vrg_solve_kkt (has_eig = 0: estimated at v = 0 like newton.cpp:36-40)
 * records: per outer iteration 12 doubles [iter, gradNormInf, gradNormRel, objective, mismatch,
 *          innerIterations, lineSearchSteps, stepLength, searchDirDivRatio, wallTimeSec, ffts, interps]
 * summary = [status(0 converged, 1 iteration limit, 2 line-search failure), n_iterations,
 *            finalGradNormRel, finalResidualRel, jacMin, jacMax, totalTimeSec] */
int vrg_newton_solve(vrg_ctx_t ctx, int n1, int n2, const double* mR_host, const double* mT_host, int norm,
                     double beta, int deformation, const int* cfg_int, const double* cfg_dbl, const int* pc_int,
                     const double* pc_dbl, double* v1_host, double* v2_host, double* records, int records_cap,
                     double* summary);

/* inverse::newtonSolve for `pairs` independent image pairs at once (configs 3 and 5b: batches of
 * pairs on one GPU): the pairs' transport, spectral and Krylov steps run in the same kernel
 * launches (stacked fields, one scalar state per pair), each pair taking the decisions of its own
 * newtonSolve.  mR/mT/v1/v2: pairs x n1 x n2 doubles (pair after pair); cfg/pc as for
 * vrg_newton_solve (Gauss-Newton SL with cfg_int[2] = ntOverride > 0; Reg or two-level Chebyshev);
 * records: pairs x records_cap x 12, summary: pairs x 7, pair_status: per pair 0 or the status
 * of the error that pair's solve raised (message on stderr).  n1 * n2 a multiple of 256,
 * 1 <= pairs <= 64. */
int vrg_newton_solve_batch(vrg_ctx_t ctx, int n1, int n2, int pairs, const double* mR_host, const double* mT_host,
                           int norm, double beta, int deformation, const int* cfg_int, const double* cfg_dbl,
                           const int* pc_int, const double* pc_dbl, double* v1_host, double* v2_host, double* records,
                           int records_cap, double* summary, int* pair_status);

/* newtonSolve with the whole NewtonConfig (hessScheme included) and PrecondChoice per call;
 * records / summary as for vrg_newton_solve */
int vrg_newton_solve_ex(vrg_ctx_t ctx, int n1, int n2, const double* mR_host, const double* mT_host,
                        const vrg_model* model, const vrg_newton_cfg* cfg, const vrg_precond_choice* pc,
                        double* v1_host, double* v2_host, double* records, int records_cap, double* summary);

/* ---- external fine operator (the precond::LinOp plug-in point, precond.hpp:25, as used by
 * solveKkt's split Hessian, precond.cpp:20-26,313).  While set, vrg_newton_solve does not build
 * its own fine HessianOperator (newton.cpp:90-96): it calls build(user, v, nt) once per outer
 * iteration (v = 2 contiguous device fields) and data_term(user, vt, b) per fine matvec
 * (b = K[b(vt)], inverse.cpp:235-237, 2 contiguous device fields), on the context's stream;
 * the spectral parts of the split operator, the preconditioner, gradient, objective and line
 * search stay in the library.  A nonzero callback return fails the solve (VRG_RUNTIME_ERROR).
 * Gauss-Newton, compressible, SL only.  Pass NULL callbacks to clear. */
typedef int (*vrg_fine_build_fn)(void* user, const double* v, int nt);
typedef int (*vrg_fine_data_term_fn)(void* user, const double* vt, double* b);
int vrg_set_fine_operator(vrg_ctx_t ctx, vrg_fine_build_fn build, vrg_fine_data_term_fn data_term, void* user);
/* External (e.g. slab-decomposed) implementations of everything transport-heavy in newtonSolve,
 * so the driver (newton.cpp:24-159, precond.cpp:291-358: host control, whole-grid vectors) does
 * no whole-grid transport itself.  build / data_term: as vrg_set_fine_operator.  Optional pairs:
 *   gradient(user, v, nt, reuse, g, m1, scalars): evaluateGradient (inverse.cpp:119-148) once per
 *     outer iteration; reuse = 1: the state of the last objective call (the accepted line-search
 *     trial) is this iterate's (newton.cpp:54-56); m1 = m(1);
 *   objective(user, v, nt, m1, scalars): evaluateObjective (inverse.cpp:96-117) per line-search
 *     trial; return 2 for transport::BlowupError (newton.cpp:118-122);
 *   coarse_build(user, v, &ntc) per solveKkt (precond::CoarseOperator, precond.cpp:207-240: the
 *     restricted problem, coarse nt from CFL 5); two_level(user, r, z, k, emin, emax_inflated)
 *     per application of the two-level CHEB(k) preconditioner (applyTwoLevel, precond.cpp:
 *     264-289; return 3 when the coarse solve diverged and z = r); coarse_emax(user, &emax,
 *     &applications) for the Chebyshev bound re-estimate after a breakdown (lanczosEmax from the
 *     0x5eed probe, precond.cpp:338-347).
 * v, g, r, z: 2 contiguous device fields; m1: one field; scalars = [objective, mismatch,
 * regTerm, penaltyTerm].  The driver adds the reference's logical operation counts for the
 * work the hooks do.  NULL ops clears. */
typedef int (*vrg_gradient_fn)(void* user, const double* v, int nt, int reuse, double* g, double* m1, double* scalars);
typedef int (*vrg_objective_fn)(void* user, const double* v, int nt, double* m1, double* scalars);
typedef int (*vrg_coarse_build_fn)(void* user, const double* v, int* coarse_nt);
typedef int (*vrg_two_level_fn)(void* user, const double* r, double* z, int cheb_iters, double emin, double emax);
typedef int (*vrg_coarse_emax_fn)(void* user, double* emax, int* applications);
typedef int (*vrg_split_fn)(void* user, const double* s, double* o);
typedef struct vrg_external_ops_s {
    vrg_fine_build_fn build;
    vrg_fine_data_term_fn data_term;
    vrg_gradient_fn gradient;       /* nullable (with objective) */
    vrg_objective_fn objective;
    vrg_coarse_build_fn coarse_build;  /* nullable (with two_level and coarse_emax) */
    vrg_two_level_fn two_level;
    vrg_coarse_emax_fn coarse_emax;
    vrg_split_fn split;             /* nullable: the whole split matvec M^{-1/2} Q M^{-1/2} s + s
                                       (precond.cpp:20-26) instead of data_term + the driver's FFTs */
    void* user;
} vrg_external_ops;
int vrg_set_external_ops(vrg_ctx_t ctx, const vrg_external_ops* ops);

#ifdef __cplusplus
}
#endif

#endif /* VRG_H */
