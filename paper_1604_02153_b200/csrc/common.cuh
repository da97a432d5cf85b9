// Shared runtime pieces of libvrg: context, device buffers, errors, cuFFT plan cache.
//
// Layout in HBM: every scalar field is one contiguous fp64 array of
// n1*n2 values, row-major with axis 1 fastest, node (i1,i2) at (-pi+i1*h1, -pi+i2*h2) — the
// reference's Grid/ScalarField layout (include/veloreg/field.hpp:15-54).  Vector fields are two
// such arrays (SoA).  Trajectories are (nt+1) consecutive fields.  Half spectra are n1 x
// (n2/2+1) cufftDoubleComplex, the FFTW r2c layout of src/fft.cpp:57-78.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <cufft.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace vrg {

// NVTX range over a library operation, named after the reference API it implements (visible
// in Nsight Systems / ncu --nvtx; a no-op without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kBlowupFactor = 1e3;  // src/transport.cpp:14

// Status codes of the C ABI (include/vrg.h).
enum Status : int { kOk = 0, kInvalidArgument = 1, kBlowup = 2, kRuntime = 3, kNotSupported = 4 };

struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct BlowupError : std::runtime_error {  // transport::BlowupError (transport.hpp:35-38)
    using std::runtime_error::runtime_error;
};
struct NotSupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void throwCuda(cudaError_t e, const char* what, const char* file, int line);
void throwCufft(cufftResult r, const char* what, const char* file, int line);

#define VRG_CUDA(x)                                                              \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) ::vrg::throwCuda(e_, #x, __FILE__, __LINE__);     \
    } while (0)
#define VRG_CUFFT(x)                                                             \
    do {                                                                         \
        cufftResult r_ = (x);                                                    \
        if (r_ != CUFFT_SUCCESS) ::vrg::throwCufft(r_, #x, __FILE__, __LINE__);  \
    } while (0)
#define VRG_LAUNCH_CHECK() VRG_CUDA(cudaGetLastError())

// Stream of the library call in progress on this host thread (set by the C ABI entry points).
// Device buffers released during a call go to a per-stream cache of cudaMalloc blocks instead
// of cudaFree, and allocations on that stream reuse them (exact size): constructing operators
// and solvers inside a Newton iteration then costs no cudaMalloc/cudaFree device
// synchronisation.  Reuse is stream-ordered (a block only serves the stream that released it).
// Outside a library call (no stream set) buffers use cudaMalloc/cudaFree directly.
extern thread_local cudaStream_t g_allocStream;
extern thread_local bool g_allocStreamSet;
bool poolAllocations();  // VRG_POOL=0 disables the block cache
void* cachedAlloc(std::size_t bytes, cudaStream_t s, std::size_t* got);  // got: the block's true size
void cachedFree(void* p, std::size_t bytes, cudaStream_t s);
void releaseCachedBlocks(cudaStream_t s);

// Owning device allocation (RAII).
class DBuf {
public:
    DBuf() = default;
    explicit DBuf(std::size_t bytes) { alloc(bytes); }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p_(o.p_), bytes_(o.bytes_), cap_(o.cap_) { o.p_ = nullptr; o.bytes_ = o.cap_ = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p_ = o.p_; bytes_ = o.bytes_; cap_ = o.cap_; o.p_ = nullptr; o.bytes_ = o.cap_ = 0; }
        return *this;
    }
    void alloc(std::size_t bytes) {
        release();
        cap_ = bytes;
        if (bytes) {
            if (g_allocStreamSet)
                p_ = cachedAlloc(bytes, g_allocStream, &cap_);
            else
                VRG_CUDA(cudaMalloc(&p_, bytes));
        }
        bytes_ = bytes;
    }
    void release() {
        if (p_) {
            if (g_allocStreamSet)
                cachedFree(p_, cap_, g_allocStream);
            else
                cudaFree(p_);
        }
        p_ = nullptr;
        bytes_ = cap_ = 0;
    }
    template <typename T = double>
    T* as() const { return static_cast<T*>(p_); }
    double* d() const { return static_cast<double*>(p_); }
    std::size_t bytes() const { return bytes_; }
    explicit operator bool() const { return p_ != nullptr; }

private:
    void* p_ = nullptr;
    std::size_t bytes_ = 0;
    std::size_t cap_ = 0;  // size of the block behind p_ (>= bytes_ when it came from the cache)
};

// Sets the allocation stream for the duration of a library call (restores the previous one).
struct AllocStreamScope {
    cudaStream_t prev;
    bool prevSet;
    explicit AllocStreamScope(cudaStream_t s) : prev(g_allocStream), prevSet(g_allocStreamSet) {
        g_allocStream = s;
        g_allocStreamSet = poolAllocations();
    }
    ~AllocStreamScope() {
        g_allocStream = prev;
        g_allocStreamSet = prevSet;
    }
};

// An n1 x n2 periodic grid, or a batch of `pairs` independent image pairs on that grid stacked
// pair after pair: a field of a batch holds the pairs' n1 x n2 fields one after the other
// (pointsPer() apart), so element-wise work runs over points() = pairs * n1 * n2 values and
// every spatial kernel maps a row / node / mode to (pair, local index).  A vector field of a
// batch is [component 0 of all pairs | component 1 of all pairs].
struct GridDims {
    int n1 = 0, n2 = 0;
    int pairs = 1;
    GridDims() = default;
    GridDims(int a, int b, int p = 1) : n1(a), n2(b), pairs(p) {}
    std::size_t pointsPer() const { return static_cast<std::size_t>(n1) * n2; }
    std::size_t points() const { return pointsPer() * pairs; }
    int specCols() const { return n2 / 2 + 1; }
    std::size_t specPer() const { return static_cast<std::size_t>(n1) * specCols(); }
    std::size_t specPoints() const { return specPer() * pairs; }
    GridDims one() const { return GridDims(n1, n2); }
    double h1() const { return kTwoPi / n1; }
    double h2() const { return kTwoPi / n2; }
    bool operator==(const GridDims& o) const { return n1 == o.n1 && n2 == o.n2 && pairs == o.pairs; }
    bool operator!=(const GridDims& o) const { return !(*this == o); }
    bool operator<(const GridDims& o) const { return std::tie(n1, n2, pairs) < std::tie(o.n1, o.n2, o.pairs); }
};

// Grid::Grid validation (src/field.cpp:9-15).
void checkGrid(int n1, int n2);

// One context per (device, stream).  Not thread-safe across concurrent calls on the same
// context: one host thread drives one context (one per GPU for batched pairs).
struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool ownStream = false;
    std::string err;
    // Logical operation counters with the reference's semantics (src/counters.cpp): one FFT
    // per forward/inverse 2-D transform of one scalar field, one interp per scattered
    // evaluation of one scalar field.
    long long ffts = 0, interps = 0;
    int numSMs = 148;
    std::size_t l2Bytes = 0;

    struct PlanKey {
        int n1, n2, type, batch;
        cudaStream_t stream;  // plans are bound to the stream current at creation
        bool operator<(const PlanKey& o) const {
            return std::tie(n1, n2, type, batch, stream) < std::tie(o.n1, o.n2, o.type, o.batch, o.stream);
        }
    };
    std::map<PlanKey, cufftHandle> plans;
    // Scratch spectra / fields reused across calls (grown on demand, freed with the context).
    std::map<std::pair<int, std::size_t>, DBuf> scratch;
    DBuf reduce;  // reduction scratch (partials + results)
    DBuf reduceTickets;  // per-pair block counters of the fused two-stage reductions (self-resetting)
    double* hostScalars = nullptr;  // pinned staging for scalar reads
    // pinned staging of at least `bytes` for a synchronous readback (grown, never shrunk: the
    // buffer lives as long as the context, so no pinned allocation per operation)
    void* hostStage(std::size_t bytes);
    void* hostStage_ = nullptr;
    std::size_t hostStageBytes_ = 0;
    // External fine-level GN data term for newtonSolve (C ABI vrg_set_fine_operator): the
    // plug-in point of precond::LinOp (precond.hpp:25) that a slab-decomposed operator fills.
    // build(v, nt) is called once per Newton iterate, dataTerm(vt, b) per matvec (2N fields,
    // device pointers on this context's stream); nonzero return = failure.
    // gradient / objective (optional, C ABI vrg_set_external_ops) replace evaluateGradient and
    // the line search's evaluateObjective: gradient(v, nt, reuse, g, m1, scalars[4]) with reuse
    // = 1 when the state of the last objective call (the accepted trial) is to be reused;
    // objective(v, nt, m1, scalars[4]) returns 2 on a blow-up (BlowupError), other nonzero on
    // failure.  m1 = the final state m(1) (N doubles).
    struct FineHook {
        int (*build)(void* user, const double* v, int nt) = nullptr;
        int (*dataTerm)(void* user, const double* vt, double* b) = nullptr;
        int (*gradient)(void* user, const double* v, int nt, int reuse, double* g, double* m1, double* scalars) = nullptr;
        int (*objective)(void* user, const double* v, int nt, double* m1, double* scalars) = nullptr;
        // two-level CHEB preconditioner of solveKkt (precond.cpp:264-289, 319-331):
        // coarseBuild(v, &ntc) per solveKkt (the CoarseOperator), twoLevel(r, z, k, eMin,
        // eMaxInflated) per application (3 = the coarse solve diverged, z = r), coarseEmax(&eMax,
        // &applications) for the re-estimate after a breakdown (lanczosEmax, precond.cpp:338-347)
        int (*coarseBuild)(void* user, const double* v, int* ntc) = nullptr;
        int (*twoLevel)(void* user, const double* r, double* z, int chebIters, double eMin, double eMax) = nullptr;
        int (*coarseEmax)(void* user, double* eMax, int* applications) = nullptr;
        // the whole split matvec M^{-1/2} Q M^{-1/2} s + s (applySplitHessianOf, precond.cpp:20-26),
        // so the regularisation symbols are applied on the slabs too (nullable: data_term is used)
        int (*split)(void* user, const double* s, double* o) = nullptr;
        void* user = nullptr;
    } fine;

    // Kernel launches issued by this library (cuFFT's own kernels are not counted), and an
    // optional per-tag CUDA-event profile of every launch site (bench.py roofline).
    long long launches = 0;
    bool profOn = false;
    struct ProfRec {
        const char* tag;
        cudaEvent_t a, b;
    };
    std::vector<ProfRec> profRecs;
    std::vector<cudaEvent_t> evPool;
    std::size_t evNext = 0;
    std::map<std::string, std::pair<long long, double>> profAcc;  // tag -> (launches, ms)
    cudaEvent_t profEvent();
    // Reads the pending event pairs into profAcc (synchronises) and recycles the pool.
    void profFlush();
    void profAccumulate(const std::vector<ProfRec>& recs);
    // Enqueues a kernel that sleeps `us` microseconds, so the launches queued behind it run
    // back to back (profiling only; keeps host launch latency out of the event pairs).
    void profGate(int us);

    Ctx(int dev, cudaStream_t s);
    ~Ctx();
    cufftHandle plan(const GridDims& g, cufftType type, int batch);
    double* scratchBuf(int slot, std::size_t bytes);
    void sync();
};

// Runs the library's launches of a scope on another stream (ctx.stream swapped), e.g. an
// independent branch forked with events.
struct StreamSwap {
    Ctx& c;
    cudaStream_t old;
    StreamSwap(Ctx& ctx, cudaStream_t s) : c(ctx), old(ctx.stream) { c.stream = s; }
    ~StreamSwap() { c.stream = old; }
};

// Marks one kernel launch of this library; records a CUDA event pair around it when the
// context profile is on.  Construct immediately before the launch, destroy right after.
struct LaunchScope {
    Ctx& c;
    const char* tag;
    cudaEvent_t a = nullptr;
    LaunchScope(Ctx& ctx, const char* t, bool mine = true) : c(ctx), tag(t) {
        if (mine) ++c.launches;
        if (c.profOn) {
            a = c.profEvent();
            cudaEventRecord(a, c.stream);
        }
    }
    ~LaunchScope() {
        if (a) {
            cudaEvent_t b = c.profEvent();
            cudaEventRecord(b, c.stream);
            c.profRecs.push_back({tag, a, b});
        }
    }
};

inline dim3 grid1d(std::size_t n, int block) { return dim3(static_cast<unsigned>((n + block - 1) / block)); }

// Programmatic dependent launch (sm_90+).  Kernels of the time loops are launched with
// programmatic stream serialisation: each one runs its independent prologue (departure
// points, per-iterate fields), then pdlWait() until the predecessor grid has completed, then
// pdlTrigger() so the successor may launch and run its own prologue under this body.  Because
// every kernel waits before it triggers, at most two grids overlap and completion stays
// transitive along the stream.
__device__ __forceinline__ void pdlWait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdlTrigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Which kernel families get the PDL attribute (bit 0: evaluate/pointwise, bit 1: prefilter);
// the kernels' wait/trigger instructions are no-ops under a plain launch.  Both families: the
// band kernels and the column pass trigger their dependents only at their end, so an early
// launched successor never takes SM slots from the tail of the kernel it waits on (measured on
// B200 at 1024^2: SL state step 18.5 -> 16.4 us, column pass 6.2 -> 4.4 us back to back;
// triggering at the start instead, with both families, made the matvec 4% slower).
constexpr int kPdlMask = 3;

template <class... KArgs, class... Args>
void launchPdl(int family, void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t stream,
               Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (kPdlMask & family) ? 1 : 0;
    VRG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace vrg
