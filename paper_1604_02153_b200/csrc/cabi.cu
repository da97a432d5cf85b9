// extern "C" boundary of libvrg (include/vrg.h).  Exceptions never cross it: each entry point
// maps them to the status codes the reference's exception types correspond to.
#include <cstdio>
#include <mutex>
#include <unordered_map>
#include <cstring>
#include <map>

#include <memory>

#include "../../include/vrg.h"
#include "batch.cuh"
#include "evalband.cuh"
#include "heun.cuh"
#include "precond.cuh"

struct vrg_ctx_s {
    vrg::Ctx ctx;
    double betaW = 1e-1;  // Model::betaW of the near-incompressible model (inverse.hpp:21)
    int scheme = 0;       // SchemeConfig::scheme for the calls on this context (SL, RK2, RK2A)
    // vrg_malloc blocks (the stream-ordered block cache of the context's stream): pointer -> size
    std::mutex allocMu;
    std::unordered_map<void*, std::size_t> allocs;
    vrg_ctx_s(int dev, cudaStream_t s) : ctx(dev, s) {}
    ~vrg_ctx_s() {
        for (auto& kv : allocs) vrg::cachedFree(kv.first, kv.second, ctx.stream);
    }
};
struct vrg_solver_s {
    vrg_ctx_s* owner;
    vrg::Solver solver;
    std::unique_ptr<vrg::HeunTransport> heun;  // RK2 / RK2A solver (scheme != SL)
    vrg::DBuf stages;                           // nt predictor fields of the last trajectory
};
// Copy streams and events of the pipelined host-buffer batch (vrg_hess_apply_host_batch).
struct HostPipe {
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t start = nullptr, evIn[2] = {}, evComp[2] = {}, evOut[2] = {};
    void init() {
        if (in) return;
        VRG_CUDA(cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking));
        VRG_CUDA(cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&start, &evIn[0], &evIn[1], &evComp[0], &evComp[1], &evOut[0], &evOut[1]})
            VRG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    ~HostPipe() {
        if (!in) return;
        cudaStreamSynchronize(in);
        cudaStreamSynchronize(out);
        for (cudaEvent_t e : {start, evIn[0], evIn[1], evComp[0], evComp[1], evOut[0], evOut[1]}) cudaEventDestroy(e);
        cudaStreamDestroy(in);
        cudaStreamDestroy(out);
    }
};

struct vrg_hess_s {
    vrg_ctx_s* owner;
    vrg::Hessian hess;
    vrg::DBuf io;     // device staging for the host-buffer entry points
    HostPipe pipe;    // copy streams of the batch entry point
};

namespace {

thread_local std::string g_threadErr;
thread_local double g_betaW = 1e-1;  // betaW of the context of the call in progress (modelOf)
thread_local int g_scheme = 0;       // transport scheme of the context of the call in progress

template <class F>
int guarded(vrg_ctx_s* c, F&& f) {
    std::string msg;
    int code = VRG_OK;
    try {
        if (c) VRG_CUDA(cudaSetDevice(c->ctx.device));
        if (c) {
            vrg::AllocStreamScope as_(c->ctx.stream);
            g_betaW = c->betaW;
            g_scheme = c->scheme;
            f();
        } else {
            f();
        }
        return VRG_OK;
    } catch (const vrg::BlowupError& e) {
        code = VRG_BLOWUP;
        msg = e.what();
    } catch (const std::invalid_argument& e) {
        code = VRG_INVALID_ARGUMENT;
        msg = e.what();
    } catch (const vrg::NotSupported& e) {
        code = VRG_NOT_SUPPORTED;
        msg = e.what();
    } catch (const std::exception& e) {
        code = VRG_RUNTIME_ERROR;
        msg = e.what();
    }
    g_threadErr = msg;
    if (c) c->ctx.err = msg;
    return code;
}

vrg::GridDims dims(int n1, int n2) {
    vrg::checkGrid(n1, n2);
    return vrg::GridDims(n1, n2);
}

vrg::Model modelOf(int norm, double beta, int deformation) {
    if (norm < 1 || norm > 3) throw vrg::InvalidArgument("unknown regularization norm");
    if (deformation < 0 || deformation > 2) throw vrg::InvalidArgument("unknown deformation model");
    vrg::Model m;
    m.norm = norm;
    m.betaV = beta;
    m.deformation = deformation;
    m.betaW = g_betaW;
    m.scheme = g_scheme;
    return m;
}

// Model and scheme given per call (the _ex entry points): no context state involved.
vrg::Model modelEx(const vrg_model* m, int scheme) {
    if (!m) throw vrg::InvalidArgument("null model");
    if (scheme < VRG_SCHEME_SL || scheme > VRG_SCHEME_RK2A) throw vrg::InvalidArgument("unknown transport scheme");
    if (!(m->beta_w >= 0.0)) throw vrg::InvalidArgument("near-incompressible penalty weight must be >= 0");
    vrg::Model r = modelOf(m->norm, m->beta_v, m->deformation);
    r.betaW = m->beta_w;
    r.scheme = scheme;
    return r;
}

}  // namespace

extern "C" {

const char* vrg_version(void) { return "vrg 0.1 (sm_100a)"; }

int vrg_ctx_create(int device, void* stream, vrg_ctx_t* out) {
    *out = nullptr;
    return guarded(nullptr, [&] { *out = new vrg_ctx_s(device, static_cast<cudaStream_t>(stream)); });
}

void vrg_ctx_destroy(vrg_ctx_t c) { delete c; }

void* vrg_ctx_stream(vrg_ctx_t c) { return c ? static_cast<void*>(c->ctx.stream) : nullptr; }

int vrg_set_scheme(vrg_ctx_t c, int scheme) {
    return guarded(c, [&] {
        if (scheme < VRG_SCHEME_SL || scheme > VRG_SCHEME_RK2A) throw vrg::InvalidArgument("unknown transport scheme");
        c->scheme = scheme;
    });
}

int vrg_set_penalty_weight(vrg_ctx_t c, double betaW) {
    return guarded(c, [&] {
        if (!(betaW >= 0.0)) throw vrg::InvalidArgument("near-incompressible penalty weight must be >= 0");
        c->betaW = betaW;
    });
}

const char* vrg_last_error(vrg_ctx_t c) { return c ? c->ctx.err.c_str() : g_threadErr.c_str(); }

int vrg_sync(vrg_ctx_t c) {
    return guarded(c, [&] { c->ctx.sync(); });
}

// Device memory in the context's stream order, from the stream-ordered block cache: a drop-in
// allocates the fields of every call (DevBuf), and cudaMalloc / cudaFree per call (the latter
// synchronising the device) dominated the reference driver's time over the device pImpls.
int vrg_malloc(vrg_ctx_t c, unsigned long long bytes, void** out) {
    return guarded(c, [&] {
        std::size_t got = 0;
        *out = vrg::cachedAlloc(bytes ? bytes : 1, c->ctx.stream, &got);
        std::lock_guard<std::mutex> lock(c->allocMu);
        c->allocs[*out] = got;
    });
}

int vrg_free(vrg_ctx_t c, void* p) {
    return guarded(c, [&] {
        if (!p) return;
        std::size_t got = 0;
        {
            std::lock_guard<std::mutex> lock(c->allocMu);
            auto it = c->allocs.find(p);
            if (it == c->allocs.end()) throw vrg::InvalidArgument("vrg_free: not a vrg_malloc block of this context");
            got = it->second;
            c->allocs.erase(it);
        }
        vrg::cachedFree(p, got, c->ctx.stream);
    });
}

int vrg_host_alloc(vrg_ctx_t c, unsigned long long bytes, void** out) {
    return guarded(c, [&] { VRG_CUDA(cudaMallocHost(out, bytes)); });
}

int vrg_host_free(vrg_ctx_t c, void* p) {
    return guarded(c, [&] { VRG_CUDA(cudaFreeHost(p)); });
}

int vrg_copy_h2d(vrg_ctx_t c, void* dst, const void* src, unsigned long long bytes) {
    return guarded(c, [&] {
        VRG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->ctx.stream));
        c->ctx.sync();
    });
}

int vrg_copy_d2h(vrg_ctx_t c, void* dst, const void* src, unsigned long long bytes) {
    return guarded(c, [&] {
        VRG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->ctx.stream));
        c->ctx.sync();
    });
}

int vrg_counters(vrg_ctx_t c, long long* ffts, long long* interps) {
    *ffts = c->ctx.ffts;
    *interps = c->ctx.interps;
    return VRG_OK;
}

int vrg_counters_reset(vrg_ctx_t c) {
    c->ctx.ffts = 0;
    c->ctx.interps = 0;
    return VRG_OK;
}

int vrg_launch_count(vrg_ctx_t c, long long* launches) {
    *launches = c->ctx.launches;
    return VRG_OK;
}

int vrg_profile(vrg_ctx_t c, int enable) {
    return guarded(c, [&] {
        c->ctx.sync();
        c->ctx.profOn = enable != 0;
        c->ctx.profRecs.clear();
        c->ctx.evNext = 0;
        c->ctx.profAcc.clear();
    });
}

int vrg_profile_dump(vrg_ctx_t c, char* buf, int cap) {
    return guarded(c, [&] {
        vrg::Ctx& ctx = c->ctx;
        ctx.profFlush();
        std::map<std::string, std::pair<long long, double>> acc;
        acc.swap(ctx.profAcc);
        std::string out;
        for (const auto& kv : acc) {
            char line[256];
            std::snprintf(line, sizeof line, "%s\t%lld\t%.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
            out += line;
        }
        ctx.profRecs.clear();
        ctx.evNext = 0;
        if (cap > 0) {
            std::strncpy(buf, out.c_str(), static_cast<std::size_t>(cap) - 1);
            buf[cap - 1] = '\0';
        }
    });
}

// ---- BLAS-1
int vrg_dot(vrg_ctx_t c, int n1, int n2, const double* a1, const double* a2, const double* b1, const double* b2,
            double* out) {
    return guarded(c, [&] { *out = vrg::dot(c->ctx, dims(n1, n2), a1, a2, b1, b2); });
}

int vrg_norm_linf(vrg_ctx_t c, int n1, int n2, const double* a1, const double* a2, double* out) {
    return guarded(c, [&] { *out = vrg::normLinf(c->ctx, dims(n1, n2).points(), a1, a2); });
}

int vrg_axpy(vrg_ctx_t c, unsigned long long n, double a, const double* x, double* y) {
    return guarded(c, [&] { vrg::axpby(c->ctx, n, a, x, 1.0, y); });
}

// ---- interp
int vrg_prefilter(vrg_ctx_t c, int n1, int n2, const double* u, double* coef) {
    return guarded(c, [&] {
        const auto g = dims(n1, n2);
        double* tmp = c->ctx.scratchBuf(30, sizeof(double) * 2 * g.points());
        double* padded = c->ctx.scratchBuf(33, sizeof(double) * vrg::paddedPoints(n1, n2));
        unsigned* flag = reinterpret_cast<unsigned*>(c->ctx.scratchBuf(31, 64));
        VRG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), c->ctx.stream));
        vrg::launchPrefilter(c->ctx, g, u, padded, tmp, flag);
        vrg::launchUnpad(c->ctx, g, padded, coef);
        unsigned h = 0;
        VRG_CUDA(cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, c->ctx.stream));
        c->ctx.sync();
        if (h) throw vrg::InvalidArgument("prefilter: non-finite value");
    });
}

int vrg_evaluate(vrg_ctx_t c, int n1, int n2, const double* coef, const double* x1, const double* x2, double* out) {
    return guarded(c, [&] {
        const auto g = dims(n1, n2);
        if (vrg::anyNonFinite(c->ctx, g.points(), x1, x2))
            throw vrg::InvalidArgument("evaluate: non-finite point coordinate");
        double* padded = c->ctx.scratchBuf(33, sizeof(double) * vrg::paddedPoints(n1, n2));
        vrg::launchPad(c->ctx, g, coef, padded);
        vrg::launchEvaluate<1>(c->ctx, g, vrg::CoeffSet<1>{{padded}}, x1, x2, vrg::EpiStore1{nullptr, out});
        c->ctx.interps += 1;
        c->ctx.sync();
    });
}

// ---- transport
int vrg_derive_steps(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, double cfl, int* nt) {
    return guarded(c, [&] { *nt = vrg::deriveSteps(c->ctx, dims(n1, n2), v1, v2, cfl); });
}

int vrg_trace(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, double ht, int direction, double* x1,
              double* x2) {
    return guarded(c, [&] {
        const auto g = dims(n1, n2);
        if (!(ht > 0.0)) throw vrg::InvalidArgument("traceCharacteristics: ht must be positive");
        if (vrg::anyNonFinite(c->ctx, g.points(), v1, v2))
            throw vrg::InvalidArgument("traceCharacteristics velocity: non-finite value");
        const std::size_t PN = vrg::paddedPoints(n1, n2);
        double* cv = c->ctx.scratchBuf(32, sizeof(double) * 2 * PN);
        double* tmp = c->ctx.scratchBuf(30, sizeof(double) * 2 * g.points());
        vrg::launchPrefilter(c->ctx, g, v1, cv, tmp, nullptr);
        vrg::launchPrefilter(c->ctx, g, v2, cv + PN, tmp, nullptr);
        vrg::launchTrace(c->ctx, g, v1, v2, cv, cv + PN, ht, direction, x1, x2);
        c->ctx.interps += 2;
        c->ctx.sync();
    });
}

int vrg_solver_create(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, int nt, vrg_solver_t* out) {
    *out = nullptr;
    return guarded(c, [&] {
        auto* h = new vrg_solver_s{c, vrg::Solver(c->ctx, dims(n1, n2), v1, v2, nt), nullptr, vrg::DBuf()};
        if (c->scheme != VRG_SCHEME_SL) {
            h->heun = std::make_unique<vrg::HeunTransport>(c->ctx, dims(n1, n2), v1, v2, nt,
                                                           c->scheme == VRG_SCHEME_RK2A);
            h->stages.alloc(sizeof(double) * nt * dims(n1, n2).points());
        }
        *out = h;
    });
}

int vrg_solver_create_ex(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, int nt, int scheme,
                         vrg_solver_t* out) {
    *out = nullptr;
    return guarded(c, [&] {
        if (scheme < VRG_SCHEME_SL || scheme > VRG_SCHEME_RK2A) throw vrg::InvalidArgument("unknown transport scheme");
        auto* h = new vrg_solver_s{c, vrg::Solver(c->ctx, dims(n1, n2), v1, v2, nt), nullptr, vrg::DBuf()};
        if (scheme != VRG_SCHEME_SL) {
            h->heun = std::make_unique<vrg::HeunTransport>(c->ctx, dims(n1, n2), v1, v2, nt,
                                                           scheme == VRG_SCHEME_RK2A);
            h->stages.alloc(sizeof(double) * nt * dims(n1, n2).points());
        }
        *out = h;
    });
}

int vrg_solver_stages(vrg_solver_t s, double* out) {
    return guarded(s->owner, [&] {
        if (!s->heun) throw vrg::NotSupported("Heun predictor fields exist for the RK2 / RK2A schemes only");
        vrg::copy(s->solver.ctx, static_cast<std::size_t>(s->solver.nt) * s->solver.g.points(), s->stages.d(), out);
        s->solver.ctx.sync();
    });
}

void vrg_solver_destroy(vrg_solver_t s) {
    if (!s) return;
    vrg::AllocStreamScope as_(s->owner->ctx.stream);  // stream-ordered release into the pool
    delete s;
}

int vrg_solver_state(vrg_solver_t s, const double* m0, double* traj) {
    return guarded(s->owner, [&] {
        if (s->heun)
            s->heun->forward(m0, traj, s->stages.d(), true);
        else
            s->solver.state(m0, traj, true);
    });
}

int vrg_solver_adjoint(vrg_solver_t s, const double* lam1, double* traj) {
    return guarded(s->owner, [&] {
        if (s->heun)
            s->heun->backward(lam1, traj, s->stages.d(), true);
        else
            s->solver.adjoint(lam1, traj, true);
    });
}

int vrg_solver_state_final(vrg_solver_t s, const double* m0, double* out) {
    return guarded(s->owner, [&] {
        if (s->heun)
            s->heun->stateFinal(m0, out);
        else
            s->solver.stateFinal(m0, out);
    });
}

int vrg_solver_adjoint_final(vrg_solver_t s, const double* lam1, double* out) {
    return guarded(s->owner, [&] {
        if (s->heun)
            s->heun->adjointFinal(lam1, out);
        else
            s->solver.adjointFinal(lam1, out);
    });
}

int vrg_solver_incstate(vrg_solver_t s, const double* vt1, const double* vt2, const double* state, double* traj) {
    return guarded(s->owner, [&] {
        if (s->heun) {  // the state's Heun predictors, recomputed from its nodes
            vrg::HeunTransport& H = *s->heun;
            const long long f0 = H.ctx.ffts;
            H.forwardStages(state, s->stages.d());
            H.ctx.ffts = f0;  // the reference holds them from the state solve
            H.incState(vt1, vt2, state, s->stages.d(), traj);
            H.ctx.sync();
        } else {
            s->solver.incState(vt1, vt2, state, traj);
        }
    });
}

int vrg_solver_incadjoint(vrg_solver_t s, const double* vt1, const double* vt2, const double* lt1,
                          const double* adjoint, int mode, double* traj) {
    return guarded(s->owner, [&] {
        if (mode == VRG_FULL_NEWTON) {
            if (!adjoint)
                throw vrg::InvalidArgument("solveIncAdjoint: full Newton mode requires the adjoint trajectory");
            if (s->heun) {
                vrg::HeunTransport& H = *s->heun;
                const long long f0 = H.ctx.ffts;
                H.backwardStages(adjoint, s->stages.d());
                H.ctx.ffts = f0;
                H.incAdjointFullNewton(vt1, vt2, lt1, adjoint, s->stages.d(), traj);
                H.ctx.sync();
                return;
            }
            vrg::Solver& S = s->solver;
            const std::size_t N = S.g.points();
            vrg::DBuf work(sizeof(double) * 5 * N), flag(64);
            VRG_CUDA(cudaMemsetAsync(flag.d(), 0, sizeof(unsigned), S.ctx.stream));
            S.incAdjointFullNewton(vt1, vt2, lt1, adjoint, traj, work.d(), flag.as<unsigned>());
            unsigned h = 0;
            VRG_CUDA(cudaMemcpyAsync(&h, flag.d(), sizeof h, cudaMemcpyDeviceToHost, S.ctx.stream));
            S.ctx.sync();
            if (h) throw vrg::InvalidArgument("prefilter: non-finite value");
            return;
        }
        // Gauss-Newton drops every term in lambda: same operator as the adjoint
        // (transport.cpp:392-397), unguarded.
        if (s->heun)
            s->heun->backward(lt1, traj, s->stages.d(), false);
        else
            s->solver.adjoint(lt1, traj, false);
    });
}

int vrg_solver_jacobian(vrg_solver_t s, double* out) {
    return guarded(s->owner, [&] {
        if (s->heun)
            s->heun->jacobian(out);
        else
            s->solver.jacobian(out);
    });
}

int vrg_solver_departure(vrg_solver_t s, int direction, double* x1, double* x2) {
    return guarded(s->owner, [&] {
        if (s->heun) throw vrg::NotSupported("departure points exist for the SL scheme only");
        const double* X = s->solver.departure(direction);
        const std::size_t N = s->solver.g.points();
        vrg::copy(s->solver.ctx, N, X, x1);
        vrg::copy(s->solver.ctx, N, X + N, x2);
        s->solver.ctx.sync();
    });
}

// ---- spectral
int vrg_gradient(vrg_ctx_t c, int n1, int n2, const double* u, double* g1, double* g2) {
    return guarded(c, [&] {
        vrg::gradient(c->ctx, dims(n1, n2), u, g1, g2);
        c->ctx.sync();
    });
}

int vrg_apply_helmholtz(vrg_ctx_t c, int n1, int n2, const double* u, double* out) {
    return guarded(c, [&] {
        vrg::applyHelmholtz(c->ctx, dims(n1, n2), u, out);
        c->ctx.sync();
    });
}

int vrg_body_force(vrg_ctx_t c, int n1, int n2, int nt, const double* state_traj, const double* adj_traj, double* b1,
                   double* b2) {
    return guarded(c, [&] {
        if (nt < 1) throw vrg::InvalidArgument("assembleBodyForce: trajectory length mismatch");
        vrg::bodyForce(c->ctx, dims(n1, n2), nt, state_traj, adj_traj, b1, b2);
        c->ctx.sync();
    });
}

int vrg_divergence(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, double* out) {
    return guarded(c, [&] {
        vrg::divergence(c->ctx, dims(n1, n2), v1, v2, out);
        c->ctx.sync();
    });
}

int vrg_apply_reg(vrg_ctx_t c, int n1, int n2, int norm, double beta, const double* v1, const double* v2, double* o1,
                  double* o2) {
    return guarded(c, [&] {
        if (beta <= 0.0) throw vrg::InvalidArgument("applyReg: beta must be positive");
        vrg::Weights w(dims(n1, n2), modelOf(norm, beta, 0).norm);
        vrg::applyRealSymbol(c->ctx, w.g, v1, v2, o1, o2, w.regSymbol(beta));
        c->ctx.sync();
    });
}

int vrg_apply_inv_reg(vrg_ctx_t c, int n1, int n2, int norm, double beta, double power, const double* v1,
                      const double* v2, double* o1, double* o2) {
    return guarded(c, [&] {
        if (beta <= 0.0) throw vrg::InvalidArgument("applyInvReg: beta must be positive");
        vrg::Weights w(dims(n1, n2), modelOf(norm, beta, 0).norm);
        vrg::applyRealSymbol(c->ctx, w.g, v1, v2, o1, o2, w.invRegSymbol(beta, power));
        c->ctx.sync();
    });
}

int vrg_project_div_free(vrg_ctx_t c, int n1, int n2, const double* b1, const double* b2, double* o1, double* o2) {
    return guarded(c, [&] {
        vrg::projectDivFree(c->ctx, dims(n1, n2), b1, b2, o1, o2);
        c->ctx.sync();
    });
}

int vrg_resample(vrg_ctx_t c, int n1, int n2, const double* u, int t1, int t2, double* out) {
    return guarded(c, [&] {
        vrg::resample(c->ctx, dims(n1, n2), u, dims(t1, t2), out);
        c->ctx.sync();
    });
}

int vrg_cutoff(vrg_ctx_t c, int n1, int n2, const double* u, int band, double* out) {
    return guarded(c, [&] {
        const auto g = dims(n1, n2);
        vrg::cutoff(c->ctx, g, u, band == VRG_BAND_LOW ? out : nullptr, band == VRG_BAND_LOW ? nullptr : out);
        c->ctx.sync();
    });
}

int vrg_gaussian_smooth(vrg_ctx_t c, int n1, int n2, const double* u, double sigma, double* out) {
    return guarded(c, [&] {
        vrg::gaussianSmooth(c->ctx, dims(n1, n2), u, sigma, out);
        c->ctx.sync();
    });
}

// ---- inverse
int vrg_hess_create(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                    const double* mT, int norm, double beta, int deformation, int nt, int mode, const double* state,
                    vrg_hess_t* out) {
    *out = nullptr;
    return guarded(c, [&] {
        if (mode != VRG_GAUSS_NEWTON && mode != VRG_FULL_NEWTON)
            throw vrg::InvalidArgument("HessianOperator: unknown Hessian mode");
        *out = new vrg_hess_s{c, vrg::Hessian(c->ctx, dims(n1, n2), v1, v2, mR, mT, modelOf(norm, beta, deformation),
                                              nt, state, mode == VRG_FULL_NEWTON ? 1 : 0),
                              vrg::DBuf()};
    });
}

int vrg_hess_create_batch(vrg_ctx_t c, int n1, int n2, int pairs, const double* v1, const double* v2, const double* mR,
                          const double* mT, int norm, double beta, int deformation, int nt, vrg_hess_t* out) {
    *out = nullptr;
    return guarded(c, [&] {
        if (pairs < 1) throw vrg::InvalidArgument("batched HessianOperator: pairs must be >= 1");
        dims(n1, n2);
        *out = new vrg_hess_s{c, vrg::Hessian(c->ctx, vrg::GridDims(n1, n2, pairs), v1, v2, mR, mT,
                                              modelOf(norm, beta, deformation), nt, nullptr, 0),
                              vrg::DBuf()};
    });
}

int vrg_hess_create_ex(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                       const double* mT, const vrg_model* model, int scheme, int nt, int mode, const double* state,
                       const double* adjoint, vrg_hess_t* out) {
    *out = nullptr;
    return guarded(c, [&] {
        if (mode != VRG_GAUSS_NEWTON && mode != VRG_FULL_NEWTON)
            throw vrg::InvalidArgument("HessianOperator: unknown Hessian mode");
        const vrg::Model m = modelEx(model, scheme);
        *out = new vrg_hess_s{c, vrg::Hessian(c->ctx, dims(n1, n2), v1, v2, mR, mT, m, nt, state,
                                              mode == VRG_FULL_NEWTON ? 1 : 0,
                                              mode == VRG_FULL_NEWTON ? adjoint : nullptr),
                              vrg::DBuf()};
    });
}

void vrg_hess_destroy(vrg_hess_t h) {
    if (!h) return;
    vrg::AllocStreamScope as_(h->owner->ctx.stream);  // stream-ordered release into the pool
    delete h;
}

int vrg_hess_apply(vrg_hess_t h, const double* vt1, const double* vt2, double* o1, double* o2) {
    return guarded(h->owner, [&] { h->hess.apply(vt1, vt2, o1, o2); });
}

int vrg_hess_apply_data(vrg_hess_t h, const double* vt1, const double* vt2, double* o1, double* o2) {
    return guarded(h->owner, [&] { h->hess.applyDataTerm(vt1, vt2, o1, o2); });
}

int vrg_hess_apply_split(vrg_hess_t h, const double* s1, const double* s2, double* o1, double* o2) {
    return guarded(h->owner, [&] { h->hess.applySplit(s1, s2, o1, o2); });
}

int vrg_hess_apply_host(vrg_hess_t h, const double* vt1, const double* vt2, double* o1, double* o2) {
    return guarded(h->owner, [&] {
        vrg::Ctx& ctx = h->hess.ctx;
        const std::size_t N = h->hess.g.points();
        if (!h->io) h->io.alloc(sizeof(double) * 4 * N);
        double* d = h->io.d();
        VRG_CUDA(cudaMemcpyAsync(d, vt1, sizeof(double) * N, cudaMemcpyHostToDevice, ctx.stream));
        VRG_CUDA(cudaMemcpyAsync(d + N, vt2, sizeof(double) * N, cudaMemcpyHostToDevice, ctx.stream));
        h->hess.apply(d, d + N, d + 2 * N, d + 3 * N);
        VRG_CUDA(cudaMemcpyAsync(o1, d + 2 * N, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx.stream));
        VRG_CUDA(cudaMemcpyAsync(o2, d + 3 * N, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
    });
}

// k independent matvecs from host buffers, copies overlapped with compute: two device slots;
// the H2D of matvec i+1 (copy stream `in`) and the D2H of matvec i-1 (copy stream `out`) run
// while matvec i computes on the context stream.  Each apply() still checks its guard before the
// next is issued, so errors surface at the matvec that raised them, as with apply_host.
int vrg_hess_apply_host_batch(vrg_hess_t h, int k, const double* const* vt1, const double* const* vt2,
                              double* const* o1, double* const* o2) {
    return guarded(h->owner, [&] {
        if (k < 0) throw vrg::InvalidArgument("apply_host_batch: negative count");
        if (k == 0) return;
        vrg::Ctx& ctx = h->hess.ctx;
        const std::size_t N = h->hess.g.points(), B = sizeof(double) * N;
        if (h->io.bytes() < 8 * B) h->io.alloc(8 * B);
        HostPipe& P = h->pipe;
        P.init();
        double* base = h->io.d();
        auto in = [&](int s) { return base + static_cast<std::size_t>(s) * 4 * N; };
        auto outp = [&](int s) { return in(s) + 2 * N; };
        VRG_CUDA(cudaEventRecord(P.start, ctx.stream));  // slots free of earlier work on the stream
        VRG_CUDA(cudaStreamWaitEvent(P.in, P.start, 0));
        VRG_CUDA(cudaStreamWaitEvent(P.out, P.start, 0));
        auto upload = [&](int i) {
            const int s = i & 1;
            if (i >= 2) VRG_CUDA(cudaStreamWaitEvent(P.in, P.evComp[s], 0));  // matvec i-2 read slot s
            VRG_CUDA(cudaMemcpyAsync(in(s), vt1[i], B, cudaMemcpyHostToDevice, P.in));
            VRG_CUDA(cudaMemcpyAsync(in(s) + N, vt2[i], B, cudaMemcpyHostToDevice, P.in));
            VRG_CUDA(cudaEventRecord(P.evIn[s], P.in));
        };
        // matvec j's result leaves only after its guard check passed (an error delivers nothing
        // from the failing matvec on)
        auto download = [&](int j) {
            const int s = j & 1;
            VRG_CUDA(cudaStreamWaitEvent(P.out, P.evComp[s], 0));
            VRG_CUDA(cudaMemcpyAsync(o1[j], outp(s), B, cudaMemcpyDeviceToHost, P.out));
            VRG_CUDA(cudaMemcpyAsync(o2[j], outp(s) + N, B, cudaMemcpyDeviceToHost, P.out));
            VRG_CUDA(cudaEventRecord(P.evOut[s], P.out));
        };
        try {
            upload(0);
            for (int i = 0; i < k; ++i) {
                const int s = i & 1;
                if (i + 1 < k) upload(i + 1);
                VRG_CUDA(cudaStreamWaitEvent(ctx.stream, P.evIn[s], 0));
                if (i >= 2) VRG_CUDA(cudaStreamWaitEvent(ctx.stream, P.evOut[s], 0));  // D2H i-2 read slot s
                h->hess.applyQueued(in(s), in(s) + N, outp(s), outp(s) + N, s);
                VRG_CUDA(cudaEventRecord(P.evComp[s], ctx.stream));
                if (i >= 1) {  // matvec i-1's guard, checked while matvec i runs
                    h->hess.checkQueued((i - 1) & 1);
                    download(i - 1);
                }
            }
            h->hess.checkQueued((k - 1) & 1);
            download(k - 1);
        } catch (...) {
            cudaStreamSynchronize(ctx.stream);  // nothing outlives the call
            cudaStreamSynchronize(P.in);
            cudaStreamSynchronize(P.out);
            throw;
        }
        VRG_CUDA(cudaStreamWaitEvent(ctx.stream, P.evIn[(k - 1) & 1], 0));
        VRG_CUDA(cudaStreamWaitEvent(ctx.stream, P.evOut[(k - 1) & 1], 0));
        if (k > 1) VRG_CUDA(cudaStreamWaitEvent(ctx.stream, P.evOut[k & 1], 0));
        ctx.sync();
    });
}

int vrg_hess_apply_batch(vrg_hess_t h, int k, const double* const* vt1, const double* const* vt2, double* const* o1,
                         double* const* o2) {
    return guarded(h->owner, [&] {
        if (k < 0) throw vrg::InvalidArgument("apply_batch: negative count");
        vrg::Hessian& H = h->hess;
        try {
            for (int i = 0; i < k; ++i) {
                H.applyQueued(vt1[i], vt2[i], o1[i], o2[i], i & 1);
                if (i >= 1) H.checkQueued((i - 1) & 1);  // matvec i-1's guard while matvec i runs
            }
            if (k > 0) H.checkQueued((k - 1) & 1);
        } catch (...) {
            cudaStreamSynchronize(H.ctx.stream);
            throw;
        }
    });
}

int vrg_hess_bench_kernel(vrg_hess_t h, int kernel, int iters, double* ms_per_launch) {
    return guarded(h->owner, [&] { *ms_per_launch = h->hess.benchKernel(kernel, iters); });
}

int vrg_band_mapping(int mode) {
    return vrg::g_bandMapping.exchange(mode < 0 || mode > 2 ? 0 : mode);
}

int vrg_hess_graph_info(vrg_hess_t h, int* info) {
    return guarded(h->owner, [&] {
        for (int i = 0; i < 3; ++i) info[i] = h->hess.graphInfo_[i];
    });
}

int vrg_hess_band_path(vrg_hess_t h, int* band) {
    return guarded(h->owner, [&] { *band = h->hess.bandPath() ? 1 : 0; });
}

int vrg_hess_buffers(vrg_hess_t h, const double** ptrs) {
    return guarded(h->owner, [&] {
        vrg::Hessian& H = h->hess;
        ptrs[0] = H.state();
        ptrs[1] = H.gradTraj();
        ptrs[2] = H.gradDepTraj();
        ptrs[3] = H.solver.departure(vrg::kForward);
        ptrs[4] = H.solver.departure(vrg::kBackward);
        ptrs[5] = H.solver.divVelocity();
        ptrs[6] = H.solver.divVelocityAtDeparture(vrg::kBackward);
    });
}

int vrg_prefilter_rows(vrg_ctx_t c, int n1, int n2, const double* u, double* rowFiltered, unsigned* nonfinite) {
    return guarded(c, [&] { vrg::launchPrefilterRows(c->ctx, dims(n1, n2), u, rowFiltered, nonfinite); });
}

int vrg_slab_cols(vrg_ctx_t c, int winRows, int n2, const double* inHalo, double* window) {
    return guarded(c, [&] { vrg::launchSlabCols(c->ctx, winRows, n2, inHalo, window); });
}

int vrg_slab_step(vrg_ctx_t c, int kind, int n1, int n2, int L, int winBase, int winRows, const double* coef,
                  const double* x1, const double* x2, const double* const* ops, int nops, double ht, double w,
                  double* rowOut, double* guardPartials, unsigned* nonfinite, unsigned* winErr) {
    return guarded(c, [&] {
        vrg::slabStep(c->ctx, kind, n1, n2, L, winBase, winRows, coef, x1, x2, ops, nops, ht, w, rowOut,
                      guardPartials, nonfinite, winErr);
    });
}

int vrg_hess_state(vrg_hess_t h, double* traj) {
    return guarded(h->owner, [&] {
        const std::size_t N = h->hess.g.points();
        vrg::copy(h->hess.ctx, (h->hess.nt + 1) * N, h->hess.state(), traj);
        h->hess.ctx.sync();
    });
}

int vrg_evaluate_gradient(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                          const double* mT, int norm, double beta, int deformation, int nt, double* g1, double* g2,
                          double* scalars) {
    return guarded(c, [&] {
        double sc[4];
        vrg::evaluateGradient(c->ctx, dims(n1, n2), v1, v2, mR, mT, modelOf(norm, beta, deformation), nt, g1, g2,
                              sc, nullptr, nullptr, nullptr);
        c->ctx.sync();
        std::copy(sc, sc + 3, scalars);
    });
}

int vrg_evaluate_objective(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                           const double* mT, int norm, double beta, int deformation, int nt, double* scalars) {
    return guarded(c, [&] {
        double sc[4];
        vrg::evaluateObjective(c->ctx, dims(n1, n2), v1, v2, mR, mT, modelOf(norm, beta, deformation), nt, sc,
                               nullptr);
        c->ctx.sync();
        std::copy(sc, sc + 3, scalars);
    });
}

int vrg_evaluate_gradient_ex(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                             const double* mT, const vrg_model* model, int scheme, int nt, const double* reuse_state,
                             double* g1, double* g2, double* body, double* state, double* state_stages,
                             double* adjoint, double* adjoint_stages, double* scalars) {
    return guarded(c, [&] {
        if (nt < 1) throw vrg::InvalidArgument("TimeGrid: nt must be >= 1");
        vrg::evaluateGradient(c->ctx, dims(n1, n2), v1, v2, mR, mT, modelEx(model, scheme), nt, g1, g2, scalars,
                              state, adjoint, reuse_state, nullptr, body, state_stages, adjoint_stages);
        c->ctx.sync();
    });
}

int vrg_evaluate_objective_ex(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                              const double* mT, const vrg_model* model, int scheme, int nt, double* state,
                              double* state_stages, double* scalars) {
    return guarded(c, [&] {
        if (nt < 1) throw vrg::InvalidArgument("TimeGrid: nt must be >= 1");
        vrg::evaluateObjective(c->ctx, dims(n1, n2), v1, v2, mR, mT, modelEx(model, scheme), nt, scalars, state,
                               state_stages);
        c->ctx.sync();
    });
}

}  // extern "C"

// ---- precond / newton (precond.hpp, newton.hpp)
struct vrg_coarse_s {
    vrg_ctx_s* owner;
    std::unique_ptr<vrg::CoarseOperator> op;
};

namespace {

vrg::PrecondChoice choiceOf(const int* pi, const double* pd) {
    vrg::PrecondChoice c;
    c.kind = pi[0] ? vrg::kPcTwoLevel : vrg::kPcReg;
    c.coarseSolver = pi[1] ? vrg::kCoarseCheb : vrg::kCoarsePcg;
    c.chebIters = pi[2];
    c.hasEig = pi[3] != 0;
    c.epsScale = pd[0];
    c.eMin = pd[1];
    c.eMax = pd[2];
    return c;
}

// Contiguous [c0 | c1] copy of a vector field given as two pointers.
const double* packed(vrg::Ctx& ctx, const vrg::GridDims& g, const double* a, const double* b, int slot) {
    if (b == a + g.points()) return a;
    double* p = ctx.scratchBuf(slot, sizeof(double) * 2 * g.points());
    vrg::copy(ctx, g.points(), a, p);
    vrg::copy(ctx, g.points(), b, p + g.points());
    return p;
}

}  // namespace

extern "C" {

int vrg_random_bandlimited_field(vrg_ctx_t c, int n1, int n2, unsigned long long seed, double* out) {
    return guarded(c, [&] {
        vrg::randomBandLimitedField(c->ctx, dims(n1, n2), seed, out);
        c->ctx.sync();
    });
}

int vrg_coarse_create(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                      const double* mT, int norm, double beta, int deformation, double coarse_cfl, vrg_coarse_t* out) {
    *out = nullptr;
    return guarded(c, [&] {
        const auto g = dims(n1, n2);
        const double* v = v1 ? packed(c->ctx, g, v1, v2, 40) : nullptr;
        auto op = std::make_unique<vrg::CoarseOperator>(c->ctx, g, v, mR, mT, modelOf(norm, beta, deformation),
                                                        coarse_cfl);
        *out = new vrg_coarse_s{c, std::move(op)};
    });
}

void vrg_coarse_destroy(vrg_coarse_t c) {
    if (!c) return;
    vrg::AllocStreamScope as_(c->owner->ctx.stream);  // stream-ordered release into the pool
    delete c;
}

int vrg_coarse_info(vrg_coarse_t c, int* n1c, int* n2c, int* nt) {
    *n1c = c->op->gc.n1;
    *n2c = c->op->gc.n2;
    *nt = c->op->nt;
    return VRG_OK;
}

int vrg_coarse_apply_split(vrg_coarse_t c, const double* s1, const double* s2, double* o1, double* o2) {
    return guarded(c->owner, [&] { c->op->hess->applySplit(s1, s2, o1, o2); });
}

int vrg_two_level_apply(vrg_coarse_t c, const double* r1, const double* r2, int coarse_solver, int cheb_iters,
                        double eps_scale, double outer_tol, double emin, double emax, double* o1, double* o2,
                        int* fallback) {
    return guarded(c->owner, [&] {
        vrg::Ctx& ctx = c->owner->ctx;
        const vrg::GridDims g = c->op->fine;
        vrg::PrecondChoice pc;
        pc.kind = vrg::kPcTwoLevel;
        pc.coarseSolver = coarse_solver ? vrg::kCoarseCheb : vrg::kCoarsePcg;
        pc.chebIters = cheb_iters;
        pc.epsScale = eps_scale;
        const double* r = packed(ctx, g, r1, r2, 41);
        double* o = ctx.scratchBuf(42, sizeof(double) * 2 * g.points());
        const bool ok = vrg::applyTwoLevel(ctx, g, r, *c->op, pc, outer_tol, emin, emax, o);
        vrg::copy(ctx, g.points(), o, o1);
        vrg::copy(ctx, g.points(), o + g.points(), o2);
        ctx.sync();
        if (fallback) *fallback = ok ? 0 : 1;
    });
}

int vrg_estimate_eigs(vrg_ctx_t c, int n1, int n2, const double* v1, const double* v2, const double* mR,
                      const double* mT, int norm, double beta, int deformation, double coarse_cfl,
                      unsigned long long seed, double* emin, double* emax) {
    return guarded(c, [&] {
        const auto g = dims(n1, n2);
        const double* v = v1 ? packed(c->ctx, g, v1, v2, 40) : nullptr;
        const auto e = vrg::estimateEigsAt(c->ctx, g, v, mR, mT, modelOf(norm, beta, deformation), coarse_cfl, seed);
        *emin = e.first;
        *emax = e.second;
    });
}

int vrg_solve_kkt(vrg_hess_t h, const double* rhs1, const double* rhs2, double tol, int max_iter, const int* pc_int,
                  const double* pc_dbl, const double* mR, const double* mT, const double* v1, const double* v2,
                  double coarse_cfl, double* sol1, double* sol2, double* result) {
    return guarded(h->owner, [&] {
        vrg::Ctx& ctx = h->hess.ctx;
        const vrg::GridDims g = h->hess.g;
        const double* rhs = packed(ctx, g, rhs1, rhs2, 41);
        const double* v = packed(ctx, g, v1, v2, 40);
        double* sol = ctx.scratchBuf(43, sizeof(double) * 2 * g.points());
        const auto r = vrg::solveKkt(ctx, h->hess, rhs, tol, max_iter, choiceOf(pc_int, pc_dbl), mR, mT, v,
                                     coarse_cfl, sol);
        vrg::copy(ctx, g.points(), sol, sol1);
        vrg::copy(ctx, g.points(), sol + g.points(), sol2);
        ctx.sync();
        result[0] = r.iterations;
        result[1] = r.converged;
        result[2] = r.negativeCurvature;
        result[3] = r.relResidual;
        result[4] = r.totalTimeSec;
        result[5] = r.precondTimeSec;
    });
}

int vrg_set_fine_operator(vrg_ctx_t c, vrg_fine_build_fn build, vrg_fine_data_term_fn data_term, void* user) {
    return guarded(c, [&] {
        if (!c) throw vrg::InvalidArgument("null context");
        if ((build == nullptr) != (data_term == nullptr))
            throw vrg::InvalidArgument("external fine operator: give both callbacks or neither");
        c->ctx.fine.build = build;
        c->ctx.fine.dataTerm = data_term;
        c->ctx.fine.gradient = nullptr;
        c->ctx.fine.objective = nullptr;
        c->ctx.fine.coarseBuild = nullptr;
        c->ctx.fine.twoLevel = nullptr;
        c->ctx.fine.coarseEmax = nullptr;
        c->ctx.fine.split = nullptr;
        c->ctx.fine.user = build ? user : nullptr;
    });
}

int vrg_set_external_ops(vrg_ctx_t c, const vrg_external_ops* ops) {
    return guarded(c, [&] {
        if (!c) throw vrg::InvalidArgument("null context");
        auto& f = c->ctx.fine;
        if (!ops) {
            f = {};
            return;
        }
        if (!ops->build || !ops->data_term || (ops->gradient == nullptr) != (ops->objective == nullptr) ||
            (ops->coarse_build == nullptr) != (ops->two_level == nullptr) ||
            (ops->coarse_build == nullptr) != (ops->coarse_emax == nullptr))
            throw vrg::InvalidArgument(
                "external operators: build + data_term, optionally gradient + objective and coarse_build + two_level "
                "+ coarse_emax");
        f.build = ops->build;
        f.dataTerm = ops->data_term;
        f.gradient = ops->gradient;
        f.objective = ops->objective;
        f.coarseBuild = ops->coarse_build;
        f.twoLevel = ops->two_level;
        f.coarseEmax = ops->coarse_emax;
        f.split = ops->split;
        f.user = ops->user;
    });
}

namespace {
void newtonToHost(vrg_ctx_s* c, int n1, int n2, const double* mR_host, const double* mT_host, const vrg::Model& model,
                  const vrg::NewtonConfig& cfg, const vrg::PrecondChoice& pc, double* v1_host, double* v2_host,
                  double* records, int records_cap, double* summary) {
    {
        vrg::Ctx& ctx = c->ctx;
        const auto g = dims(n1, n2);
        const std::size_t N = g.points();
        if (cfg.hessianMode != VRG_GAUSS_NEWTON && cfg.hessianMode != VRG_FULL_NEWTON)
            throw vrg::InvalidArgument("newtonSolve: unknown Hessian mode");
        vrg::DBuf img(sizeof(double) * 2 * N), v(sizeof(double) * 2 * N);
        VRG_CUDA(cudaMemcpyAsync(img.d(), mR_host, sizeof(double) * N, cudaMemcpyHostToDevice, ctx.stream));
        VRG_CUDA(cudaMemcpyAsync(img.d() + N, mT_host, sizeof(double) * N, cudaMemcpyHostToDevice, ctx.stream));
        const auto rep = vrg::newtonSolve(ctx, g, img.d(), img.d() + N, model, cfg, pc, v.d());
        VRG_CUDA(cudaMemcpyAsync(v1_host, v.d(), sizeof(double) * N, cudaMemcpyDeviceToHost, ctx.stream));
        VRG_CUDA(cudaMemcpyAsync(v2_host, v.d() + N, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        int k = 0;
        for (const auto& it : rep.iterations) {
            if (k >= records_cap) break;
            double* r = records + 12 * k++;
            r[0] = it.iter;
            r[1] = it.gradNormInf;
            r[2] = it.gradNormRel;
            r[3] = it.objective;
            r[4] = it.mismatch;
            r[5] = it.innerIterations;
            r[6] = it.lineSearchSteps;
            r[7] = it.stepLength;
            r[8] = it.searchDirDivRatio;
            r[9] = it.wallTimeSec;
            r[10] = static_cast<double>(it.ffts);
            r[11] = static_cast<double>(it.interps);
        }
        summary[0] = rep.status;
        summary[1] = static_cast<double>(rep.iterations.size());
        summary[2] = rep.finalGradNormRel;
        summary[3] = rep.finalResidualRel;
        summary[4] = rep.jacMin;
        summary[5] = rep.jacMax;
        summary[6] = rep.totalTimeSec;
    }
}
}  // namespace

int vrg_newton_solve_batch(vrg_ctx_t c, int n1, int n2, int pairs, const double* mR_host, const double* mT_host,
                           int norm, double beta, int deformation, const int* cfg_int, const double* cfg_dbl,
                           const int* pc_int, const double* pc_dbl, double* v1_host, double* v2_host, double* records,
                           int records_cap, double* summary, int* pair_status) {
    return guarded(c, [&] {
        vrg::NewtonConfig cfg;
        cfg.maxOuterIter = cfg_int[0];
        cfg.maxInnerIter = cfg_int[1];
        cfg.ntOverride = cfg_int[2];
        cfg.lsMaxSteps = cfg_int[3];
        cfg.hessianMode = cfg_int[4];
        cfg.tolRelGrad = cfg_dbl[0];
        cfg.tolAbsGrad = cfg_dbl[1];
        cfg.forcingCap = cfg_dbl[2];
        cfg.lsC1 = cfg_dbl[3];
        cfg.lsShrink = cfg_dbl[4];
        cfg.gradCfl = cfg_dbl[5];
        if (pairs < 1) throw vrg::InvalidArgument("batched newtonSolve: pairs must be >= 1");
        vrg::Ctx& ctx = c->ctx;
        const auto g1 = dims(n1, n2);
        const vrg::GridDims g(n1, n2, pairs);
        const std::size_t Np = g1.points(), N = g.points();
        vrg::DBuf img(sizeof(double) * 2 * N), v(sizeof(double) * 2 * N);
        VRG_CUDA(cudaMemcpyAsync(img.d(), mR_host, sizeof(double) * N, cudaMemcpyHostToDevice, ctx.stream));
        VRG_CUDA(cudaMemcpyAsync(img.d() + N, mT_host, sizeof(double) * N, cudaMemcpyHostToDevice, ctx.stream));
        std::vector<int> status;
        std::vector<std::string> errors;
        const auto reps = vrg::newtonSolveBatch(ctx, g, img.d(), img.d() + N, modelOf(norm, beta, deformation), cfg,
                                                choiceOf(pc_int, pc_dbl), v.d(), status, errors);
        VRG_CUDA(cudaMemcpyAsync(v1_host, v.d(), sizeof(double) * N, cudaMemcpyDeviceToHost, ctx.stream));
        VRG_CUDA(cudaMemcpyAsync(v2_host, v.d() + N, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        for (int k = 0; k < pairs; ++k) {
            const auto& rep = reps[k];
            int j = 0;
            for (const auto& it : rep.iterations) {
                if (j >= records_cap) break;
                double* r = records + (static_cast<std::size_t>(k) * records_cap + j++) * 12;
                r[0] = it.iter;
                r[1] = it.gradNormInf;
                r[2] = it.gradNormRel;
                r[3] = it.objective;
                r[4] = it.mismatch;
                r[5] = it.innerIterations;
                r[6] = it.lineSearchSteps;
                r[7] = it.stepLength;
                r[8] = it.searchDirDivRatio;
                r[9] = it.wallTimeSec;
                r[10] = static_cast<double>(it.ffts);
                r[11] = static_cast<double>(it.interps);
            }
            double* sm = summary + 7 * k;
            sm[0] = rep.status;
            sm[1] = static_cast<double>(rep.iterations.size());
            sm[2] = rep.finalGradNormRel;
            sm[3] = rep.finalResidualRel;
            sm[4] = rep.jacMin;
            sm[5] = rep.jacMax;
            sm[6] = rep.totalTimeSec;
            pair_status[k] = status[k];
            if (status[k]) std::fprintf(stderr, "batched newtonSolve: pair %d: %s\n", k, errors[k].c_str());
        }
        (void)Np;
    });
}

int vrg_newton_solve(vrg_ctx_t c, int n1, int n2, const double* mR_host, const double* mT_host, int norm, double beta,
                     int deformation, const int* cfg_int, const double* cfg_dbl, const int* pc_int,
                     const double* pc_dbl, double* v1_host, double* v2_host, double* records, int records_cap,
                     double* summary) {
    return guarded(c, [&] {
        vrg::NewtonConfig cfg;
        cfg.maxOuterIter = cfg_int[0];
        cfg.maxInnerIter = cfg_int[1];
        cfg.ntOverride = cfg_int[2];
        cfg.lsMaxSteps = cfg_int[3];
        cfg.hessianMode = cfg_int[4];
        cfg.tolRelGrad = cfg_dbl[0];
        cfg.tolAbsGrad = cfg_dbl[1];
        cfg.forcingCap = cfg_dbl[2];
        cfg.lsC1 = cfg_dbl[3];
        cfg.lsShrink = cfg_dbl[4];
        cfg.gradCfl = cfg_dbl[5];
        newtonToHost(c, n1, n2, mR_host, mT_host, modelOf(norm, beta, deformation), cfg, choiceOf(pc_int, pc_dbl),
                     v1_host, v2_host, records, records_cap, summary);
    });
}

int vrg_newton_solve_ex(vrg_ctx_t c, int n1, int n2, const double* mR_host, const double* mT_host,
                        const vrg_model* model, const vrg_newton_cfg* cfg, const vrg_precond_choice* pc,
                        double* v1_host, double* v2_host, double* records, int records_cap, double* summary) {
    return guarded(c, [&] {
        if (!cfg || !pc) throw vrg::InvalidArgument("null Newton or preconditioner configuration");
        const vrg_scheme_cfg& gs = cfg->grad_scheme;
        if (gs.nt_override < 0 || (cfg->has_hess_scheme && cfg->hess_scheme.nt_override < 0))
            throw vrg::InvalidArgument("TimeGrid: nt must be >= 1");
        vrg::NewtonConfig nc;
        nc.maxOuterIter = cfg->max_outer_iter;
        nc.tolRelGrad = cfg->tol_rel_grad;
        nc.tolAbsGrad = cfg->tol_abs_grad;
        nc.maxInnerIter = cfg->max_inner_iter;
        nc.forcingCap = cfg->forcing_cap;
        nc.lsC1 = cfg->ls_c1;
        nc.lsShrink = cfg->ls_shrink;
        nc.lsMaxSteps = cfg->ls_max_steps;
        nc.hessianMode = cfg->hessian_mode;
        nc.gradCfl = gs.cfl;
        nc.ntOverride = gs.nt_override;
        nc.hasHessScheme = cfg->has_hess_scheme != 0;
        if (nc.hasHessScheme) {
            const vrg_scheme_cfg& hs = cfg->hess_scheme;
            if (hs.scheme < VRG_SCHEME_SL || hs.scheme > VRG_SCHEME_RK2A)
                throw vrg::InvalidArgument("unknown transport scheme");
            nc.hessScheme = hs.scheme;
            nc.hessCfl = hs.cfl;
            nc.hessNtOverride = hs.nt_override;
        }
        vrg::PrecondChoice ch;
        ch.kind = pc->kind ? vrg::kPcTwoLevel : vrg::kPcReg;
        ch.coarseSolver = pc->coarse_solver ? vrg::kCoarseCheb : vrg::kCoarsePcg;
        ch.epsScale = pc->eps_scale;
        ch.chebIters = pc->cheb_iters;
        ch.hasEig = pc->has_eig != 0;
        ch.eMin = pc->emin;
        ch.eMax = pc->emax;
        ch.reestimateEachIteration = pc->reestimate_each_iteration != 0;
        newtonToHost(c, n1, n2, mR_host, mT_host, modelEx(model, gs.scheme), nc, ch, v1_host, v2_host, records,
                     records_cap, summary);
    });
}

}  // extern "C"
