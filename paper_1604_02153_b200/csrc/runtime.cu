// Context, errors, cuFFT plan cache and BLAS-1 / reduction kernels (K9).
// BLAS-1 restates src/field.cpp:19-119: dot = h1*h2*sum(u*w) per component, normLinf = max|x|
// with NaN ignored (std::max semantics), axpy/scale.  Reductions are two-stage with a fixed
// block count and a fixed-order final pass (run by the last block of the same launch), so
// results are run-to-run deterministic.
#include <cstdlib>
#include <cstdint>
#include <map>
#include <set>
#include <mutex>
#include <cstdio>
#include <cstring>

#include "blas.cuh"

namespace vrg {

void throwCuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
                  file, line, what);
    throw std::runtime_error(buf);
}

void throwCufft(cufftResult r, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "cuFFT error %d at %s:%d: %s", static_cast<int>(r), file, line, what);
    throw std::runtime_error(buf);
}

void checkGrid(int n1, int n2) {
    if (n1 < 4 || n1 % 2 != 0 || n2 < 4 || n2 % 2 != 0)
        throw InvalidArgument("Grid: axis sizes must be even and >= 4");
}

thread_local cudaStream_t g_allocStream = nullptr;
thread_local bool g_allocStreamSet = false;

namespace {
// Per-stream block cache over the stream-ordered allocator.  A block is reused by the stream
// that freed it (best fit); misses come from cudaMallocAsync and blocks beyond the cache cap go
// back with cudaFreeAsync, so neither ever synchronises the device: a cudaFree there would
// serialise every concurrent lane of a process (measured: config-5b lanes fell from 229 to
// 83 pairs/s once an earlier 4096^2 registration had filled the cache up to its cap).
// Blocks allocated while their stream is being captured come from cudaMalloc (an allocation
// node inside a graph would change its lifetime) and are freed with cudaFree.
struct BlockCache {
    std::mutex mu;
    std::multimap<std::pair<cudaStream_t, std::size_t>, void*> blocks;
    std::set<void*> syncBlocks;  // from cudaMalloc (stream capture in progress)
    std::size_t held = 0;
};
BlockCache& blockCache() {
    static BlockCache* c = new BlockCache;  // leaked on purpose: outlives every context
    return *c;
}
constexpr std::size_t kCacheCap = std::size_t(48) << 30;  // beyond this, release (stream-ordered)
// The pool keeps what it holds (no trimming at synchronisation points: a trim unmaps memory the
// next allocation maps again, and the batched lanes synchronise constantly); an allocation that
// fails trims it explicitly (cachedAlloc).
constexpr std::uint64_t kPoolKeep = ~std::uint64_t(0);

bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return st != cudaStreamCaptureStatusNone;
}

void poolSetup() {
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    VRG_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(dev)) return;
    cudaMemPool_t pool;
    VRG_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    std::uint64_t keep = kPoolKeep;
    VRG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    done.insert(dev);
}

// Returns a block to the driver in stream order (no device-wide synchronisation).
void releaseBlock(BlockCache& c, void* p, cudaStream_t s) {
    auto it = c.syncBlocks.find(p);
    if (it != c.syncBlocks.end()) {
        c.syncBlocks.erase(it);
        cudaFree(p);
    } else {
        cudaFreeAsync(p, s);
    }
}
}  // namespace

void* cachedAlloc(std::size_t bytes, cudaStream_t s, std::size_t* got) {
    BlockCache& c = blockCache();
    {
        // best fit among the stream's blocks of bytes .. 2 x bytes (a batch that shrinks as its
        // pairs finish reuses the larger blocks instead of allocating)
        std::lock_guard<std::mutex> lock(c.mu);
        auto it = c.blocks.lower_bound({s, bytes});
        if (it != c.blocks.end() && it->first.first == s && it->first.second <= 2 * bytes) {
            void* p = it->second;
            *got = it->first.second;
            c.held -= it->first.second;
            c.blocks.erase(it);
            return p;
        }
    }
    *got = bytes;
    void* p = nullptr;
    const bool cap = capturing(s);
    auto allocate = [&] {
        if (cap) return cudaMalloc(&p, bytes);
        poolSetup();
        return cudaMallocAsync(&p, bytes, s);
    };
    cudaError_t e = allocate();
    if (e == cudaErrorMemoryAllocation) {  // drop the cache and retry once
        cudaGetLastError();
        std::lock_guard<std::mutex> lock(c.mu);
        for (auto& kv : c.blocks) releaseBlock(c, kv.second, kv.first.first);
        c.blocks.clear();
        c.held = 0;
        cudaDeviceSynchronize();
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
            cudaMemPoolTrimTo(pool, 0);
        e = allocate();
    }
    VRG_CUDA(e);
    if (cap) {
        std::lock_guard<std::mutex> lock(c.mu);
        c.syncBlocks.insert(p);
    }
    return p;
}

void cachedFree(void* p, std::size_t bytes, cudaStream_t s) {
    BlockCache& c = blockCache();
    std::lock_guard<std::mutex> lock(c.mu);
    if (c.held + bytes <= kCacheCap) {
        c.blocks.emplace(std::make_pair(s, bytes), p);
        c.held += bytes;
        return;
    }
    releaseBlock(c, p, s);
}

// Frees the cached blocks of a stream (its context is going away).
void releaseCachedBlocks(cudaStream_t s) {
    BlockCache& c = blockCache();
    std::lock_guard<std::mutex> lock(c.mu);
    for (auto it = c.blocks.begin(); it != c.blocks.end();) {
        if (it->first.first == s) {
            releaseBlock(c, it->second, s);
            c.held -= it->first.second;
            it = c.blocks.erase(it);
        } else {
            ++it;
        }
    }
}

bool poolAllocations() {
    static const bool on = [] {
        const char* e = std::getenv("VRG_POOL");
        return !(e && e[0] == '0');
    }();
    return on;
}

Ctx::Ctx(int dev, cudaStream_t s) : device(dev) {
    VRG_CUDA(cudaSetDevice(dev));
    VRG_CUDA(cudaFree(nullptr));
    if (s) {
        stream = s;
    } else {
        VRG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        ownStream = true;
    }
    VRG_CUDA(cudaDeviceGetAttribute(&numSMs, cudaDevAttrMultiProcessorCount, dev));
    int l2 = 0;
    VRG_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    l2Bytes = static_cast<std::size_t>(l2);
    reduce.alloc(sizeof(double) * (kReduceBlocks * 4 + 64));
    reduceTickets.alloc(sizeof(unsigned) * kReduceTicketSlots);
    VRG_CUDA(cudaMemsetAsync(reduceTickets.d(), 0, sizeof(unsigned) * kReduceTicketSlots, stream));
    VRG_CUDA(cudaMallocHost(&hostScalars, sizeof(double) * 64));
}

Ctx::~Ctx() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (auto& kv : plans) cufftDestroy(kv.second);
    for (cudaEvent_t e : evPool) cudaEventDestroy(e);
    plans.clear();
    scratch.clear();
    reduce.release();
    if (hostScalars) cudaFreeHost(hostScalars);
    if (hostStage_) cudaFreeHost(hostStage_);
    if (stream) releaseCachedBlocks(stream);
    if (ownStream && stream) cudaStreamDestroy(stream);
}

cufftHandle Ctx::plan(const GridDims& g, cufftType type, int batch) {
    // `batch` fields of the grid: batch * pairs 2-D transforms of one n1 x n2 field each
    const int transforms = batch * g.pairs;
    PlanKey key{g.n1, g.n2, static_cast<int>(type), transforms, stream};
    auto it = plans.find(key);
    if (it != plans.end()) return it->second;
    cufftHandle h;
    int n[2] = {g.n1, g.n2};
    VRG_CUFFT(cufftCreate(&h));
    std::size_t work = 0;
    if (type == CUFFT_D2Z) {
        VRG_CUFFT(cufftMakePlanMany(h, 2, n, nullptr, 1, static_cast<int>(g.pointsPer()), nullptr, 1,
                                    static_cast<int>(g.specPer()), CUFFT_D2Z, transforms, &work));
    } else {
        VRG_CUFFT(cufftMakePlanMany(h, 2, n, nullptr, 1, static_cast<int>(g.specPer()), nullptr, 1,
                                    static_cast<int>(g.pointsPer()), CUFFT_Z2D, transforms, &work));
    }
    VRG_CUFFT(cufftSetStream(h, stream));
    plans[key] = h;
    return h;
}

double* Ctx::scratchBuf(int slot, std::size_t bytes) {
    auto key = std::make_pair(slot, bytes);
    auto it = scratch.find(key);
    if (it != scratch.end()) return it->second.d();
    DBuf b(bytes);
    double* p = b.d();
    scratch.emplace(key, std::move(b));
    return p;
}

void Ctx::sync() { VRG_CUDA(cudaStreamSynchronize(stream)); }

cudaEvent_t Ctx::profEvent() {
    if (evNext == evPool.size()) {
        cudaEvent_t e;
        VRG_CUDA(cudaEventCreate(&e));
        evPool.push_back(e);
    }
    return evPool[evNext++];
}

void Ctx::profAccumulate(const std::vector<ProfRec>& recs) {
    for (const auto& r : recs) {
        float ms = 0.f;
        VRG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        auto& e = profAcc[r.tag];
        e.first += 1;
        e.second += ms;
    }
}

namespace {
__global__ void k_sleep(int us) {
    for (int i = 0; i < us; ++i) __nanosleep(1000);
}
}  // namespace

void Ctx::profGate(int us) {
    k_sleep<<<1, 1, 0, stream>>>(us);
    VRG_LAUNCH_CHECK();
}

void Ctx::profFlush() {
    sync();
    profAccumulate(profRecs);
    profRecs.clear();
    evNext = 0;
}

// ------------------------------------------------------------------------------ kernels
namespace {

__device__ __forceinline__ double warpSum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warpMax(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Fused final stage of the two-stage reductions: the last block of a reduction (per pair:
// blockIdx.y) to finish its partial takes a ticket and reduces the partials itself, with the
// arithmetic of the 1024-thread final kernels it replaces (one launch instead of two; the
// tickets reset themselves, so graph replays see them at 0).  "Virtual thread" i < 1024 holds
// partial i (nb <= kReduceBlocks < 1024) or the identity, virtual warp w reduces its 32 values
// with the xor butterfly, thread 0 then combines the 32 warp results in order.
__device__ __forceinline__ bool lastBlockOf(unsigned* ticket) {
    __shared__ bool last;
    __threadfence();  // this block's partial (written by thread 0) before its ticket
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

template <bool kMax>
__device__ __forceinline__ double finalOf(const double* partial, int nb, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = 0; k < 1024 / kReduceThreads; ++k) {
        const int i = k * kReduceThreads + threadIdx.x;
        double v = i < nb ? __ldcg(partial + i) : 0.0;
        v = kMax ? warpMax(v) : warpSum(v);
        if (lane == 0) red[k * (kReduceThreads / 32) + warp] = v;
    }
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < 32; ++w) t = kMax ? fmax(t, red[w]) : t + red[w];
    return t;
}

// Stage 1: per-block partial sums of sum_i a_i*b_i for up to two (a,b) pairs (kept separate).
__global__ void __launch_bounds__(kReduceThreads) k_dot_partial(const double* __restrict__ a0,
                                                                const double* __restrict__ b0,
                                                                const double* __restrict__ a1,
                                                                const double* __restrict__ b1, std::size_t n,
                                                                double* partial, unsigned* ticket, double scale,
                                                                double* out) {
    double s0 = 0.0, s1 = 0.0;
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        s0 += a0[i] * b0[i];
        if (a1) s1 += a1[i] * b1[i];
    }
    __shared__ double r0[kReduceThreads / 32], r1[kReduceThreads / 32];
    s0 = warpSum(s0);
    s1 = warpSum(s1);
    if ((threadIdx.x & 31) == 0) {
        r0[threadIdx.x >> 5] = s0;
        r1[threadIdx.x >> 5] = s1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < kReduceThreads / 32; ++w) {
            t0 += r0[w];
            t1 += r1[w];
        }
        partial[blockIdx.x] = t0;
        partial[kReduceBlocks + blockIdx.x] = t1;
    }
    if (!lastBlockOf(ticket)) return;
    __shared__ double f0[32], f1[32];
    const double t0 = finalOf<false>(partial, gridDim.x, f0);
    const double t1 = finalOf<false>(partial + kReduceBlocks, gridDim.x, f1);
    if (threadIdx.x == 0) {
        *out = scale * t0 + scale * t1;  // dot per component, then added (field.cpp:47-54)
        *ticket = 0;
    }
}

__global__ void __launch_bounds__(kReduceThreads) k_maxabs_partial(const double* __restrict__ a0,
                                                                   const double* __restrict__ a1, std::size_t n,
                                                                   double* partial, unsigned* ticket, double scale,
                                                                   double* out) {
    double m = 0.0;
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        m = fmax(m, fabs(a0[i]));  // fmax drops NaN like std::max(m, NaN) == m
        if (a1) m = fmax(m, fabs(a1[i]));
    }
    __shared__ double r[kReduceThreads / 32];
    m = warpMax(m);
    if ((threadIdx.x & 31) == 0) r[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kReduceThreads / 32; ++w) t = fmax(t, r[w]);
        partial[blockIdx.x] = t;
    }
    if (!lastBlockOf(ticket)) return;
    __shared__ double f[32];
    const double t = finalOf<true>(partial, gridDim.x, f);
    if (threadIdx.x == 0) {
        *out = scale * t;
        *ticket = 0;
    }
}


// Per-pair forms of the two-stage reductions (stacked pairs, GridDims::pairs): blockIdx.y = pair,
// each pair reduced over its own nPer values with the block partition and summation order of the
// single-field kernels above, so a pair's result is bit-identical to reducing it alone.
__global__ void __launch_bounds__(kReduceThreads) k_dot_partial_pairs(const double* __restrict__ a0,
                                                                      const double* __restrict__ b0,
                                                                      const double* __restrict__ a1,
                                                                      const double* __restrict__ b1, std::size_t nPer,
                                                                      double* partial, unsigned* tickets, double scale,
                                                                      double* out) {
    const std::size_t off = blockIdx.y * nPer;
    double s0 = 0.0, s1 = 0.0;
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nPer; i += stride) {
        s0 += a0[off + i] * b0[off + i];
        if (a1) s1 += a1[off + i] * b1[off + i];
    }
    __shared__ double r0[kReduceThreads / 32], r1[kReduceThreads / 32];
    s0 = warpSum(s0);
    s1 = warpSum(s1);
    if ((threadIdx.x & 31) == 0) {
        r0[threadIdx.x >> 5] = s0;
        r1[threadIdx.x >> 5] = s1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0;
        for (int w = 0; w < kReduceThreads / 32; ++w) {
            t0 += r0[w];
            t1 += r1[w];
        }
        partial[blockIdx.y * 2 * kReduceBlocks + blockIdx.x] = t0;
        partial[blockIdx.y * 2 * kReduceBlocks + kReduceBlocks + blockIdx.x] = t1;
    }
    unsigned* ticket = tickets + blockIdx.y;
    if (!lastBlockOf(ticket)) return;
    __shared__ double f0[32], f1[32];
    const double* pp = partial + blockIdx.y * 2 * kReduceBlocks;
    const double t0 = finalOf<false>(pp, gridDim.x, f0);
    const double t1 = finalOf<false>(pp + kReduceBlocks, gridDim.x, f1);
    if (threadIdx.x == 0) {
        out[blockIdx.y] = scale * t0 + scale * t1;
        *ticket = 0;
    }
}

__global__ void __launch_bounds__(kReduceThreads) k_maxabs_partial_pairs(const double* __restrict__ a0,
                                                                         const double* __restrict__ a1,
                                                                         std::size_t nPer, double* partial,
                                                                         unsigned* tickets, double* out) {
    const std::size_t off = blockIdx.y * nPer;
    double m = 0.0;
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nPer; i += stride) {
        m = fmax(m, fabs(a0[off + i]));
        if (a1) m = fmax(m, fabs(a1[off + i]));
    }
    __shared__ double r[kReduceThreads / 32];
    m = warpMax(m);
    if ((threadIdx.x & 31) == 0) r[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kReduceThreads / 32; ++w) t = fmax(t, r[w]);
        partial[blockIdx.y * 2 * kReduceBlocks + blockIdx.x] = t;
    }
    unsigned* ticket = tickets + blockIdx.y;
    if (!lastBlockOf(ticket)) return;
    __shared__ double f[32];
    const double t = finalOf<true>(partial + blockIdx.y * 2 * kReduceBlocks, gridDim.x, f);
    if (threadIdx.x == 0) {
        out[blockIdx.y] = t;
        *ticket = 0;
    }
}

__global__ void k_nonfinite(const double* __restrict__ a, std::size_t n, unsigned* flag) {
    bool bad = false;
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        bad |= !isfinite(a[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

__global__ void k_axpby(std::size_t n, double a, const double* __restrict__ x, double b, double* y) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        y[i] = b == 1.0 ? y[i] + a * x[i] : (b == 0.0 ? a * x[i] : b * y[i] + a * x[i]);
}

__global__ void k_axpy_negcoef(std::size_t n, const double* __restrict__ c, const double* __restrict__ x, double* y) {
    const double a = -c[0];
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        y[i] = y[i] + a * x[i];
}

__global__ void k_lincomb(std::size_t n, double a, const double* __restrict__ x, double b,
                          const double* __restrict__ y, double* out) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = a * x[i] + b * y[i];
}

__global__ void k_fill(std::size_t n, double v, double* y) {
    const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
    for (std::size_t i = static_cast<std::size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        y[i] = v;
}

}  // namespace

unsigned elemBlocks(const Ctx& ctx, std::size_t n) {
    const std::size_t want = (n + 255) / 256;
    const std::size_t cap = static_cast<std::size_t>(ctx.numSMs) * 8;
    return static_cast<unsigned>(std::max<std::size_t>(1, std::min(want, cap)));
}


double* launchDot(Ctx& ctx, std::size_t n, const double* a0, const double* b0, const double* a1, const double* b1,
                  double scale, int slot) {
    double* out = ctx.reduce.d() + 2 * kReduceBlocks + slot;
    launchDotInto(ctx, n, a0, b0, a1, b1, scale, out);
    return out;
}

void launchDotInto(Ctx& ctx, std::size_t n, const double* a0, const double* b0, const double* a1, const double* b1,
                   double scale, double* out) {
    double* partial = ctx.reduce.d();
    const int nb = static_cast<int>(std::min<std::size_t>(kReduceBlocks, (n + kReduceThreads - 1) / kReduceThreads));
    {
        LaunchScope ls_(ctx, "k_dot_partial");
        k_dot_partial<<<nb, kReduceThreads, 0, ctx.stream>>>(a0, b0, a1, b1, n, partial,
                                                             ctx.reduceTickets.as<unsigned>(), scale, out);
    }
    VRG_LAUNCH_CHECK();
}

double* launchMaxAbs(Ctx& ctx, std::size_t n, const double* a0, const double* a1, double scale, int slot) {
    double* partial = ctx.reduce.d();
    double* out = partial + 2 * kReduceBlocks + slot;
    const int nb = static_cast<int>(std::min<std::size_t>(kReduceBlocks, (n + kReduceThreads - 1) / kReduceThreads));
    {
        LaunchScope ls_(ctx, "k_maxabs_partial");
        k_maxabs_partial<<<nb, kReduceThreads, 0, ctx.stream>>>(a0, a1, n, partial, ctx.reduceTickets.as<unsigned>(),
                                                                scale, out);
    }
    VRG_LAUNCH_CHECK();
    return out;
}


double* launchDotPairs(Ctx& ctx, const GridDims& g, const double* a0, const double* b0, const double* a1,
                       const double* b1, double scale, int slot) {
    const std::size_t n = g.pointsPer();
    const int P = g.pairs;
    if (P > kReduceTicketSlots) throw NotSupported("reductions: more pairs than ticket slots");
    double* partial = ctx.scratchBuf(200, sizeof(double) * 2 * kReduceBlocks * P);
    double* out = ctx.scratchBuf(201 + slot, sizeof(double) * P);
    const int nb = static_cast<int>(std::min<std::size_t>(kReduceBlocks, (n + kReduceThreads - 1) / kReduceThreads));
    {
        LaunchScope ls_(ctx, "k_dot_partial");
        k_dot_partial_pairs<<<dim3(nb, P), kReduceThreads, 0, ctx.stream>>>(
            a0, b0, a1, b1, n, partial, ctx.reduceTickets.as<unsigned>(), scale, out);
    }
    VRG_LAUNCH_CHECK();
    return out;
}

double* launchMaxAbsPairs(Ctx& ctx, const GridDims& g, const double* a0, const double* a1, int slot) {
    const std::size_t n = g.pointsPer();
    const int P = g.pairs;
    if (P > kReduceTicketSlots) throw NotSupported("reductions: more pairs than ticket slots");
    double* partial = ctx.scratchBuf(200, sizeof(double) * 2 * kReduceBlocks * P);
    double* out = ctx.scratchBuf(201 + slot, sizeof(double) * P);
    const int nb = static_cast<int>(std::min<std::size_t>(kReduceBlocks, (n + kReduceThreads - 1) / kReduceThreads));
    {
        LaunchScope ls_(ctx, "k_maxabs_partial");
        k_maxabs_partial_pairs<<<dim3(nb, P), kReduceThreads, 0, ctx.stream>>>(
            a0, a1, n, partial, ctx.reduceTickets.as<unsigned>(), out);
    }
    VRG_LAUNCH_CHECK();
    return out;
}

void readPairs(Ctx& ctx, const double* dev, int P, double* host) {
    if (P <= 64) {  // through the context's pinned staging (a pageable copy stages synchronously)
        VRG_CUDA(cudaMemcpyAsync(ctx.hostScalars, dev, sizeof(double) * P, cudaMemcpyDeviceToHost, ctx.stream));
        ctx.sync();
        std::memcpy(host, ctx.hostScalars, sizeof(double) * P);
        return;
    }
    VRG_CUDA(cudaMemcpyAsync(host, dev, sizeof(double) * P, cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
}

void* Ctx::hostStage(std::size_t bytes) {
    if (bytes > hostStageBytes_) {
        if (hostStage_) {
            VRG_CUDA(cudaStreamSynchronize(stream));
            cudaFreeHost(hostStage_);
        }
        hostStage_ = nullptr;
        const std::size_t want = std::max<std::size_t>(bytes, 64 * 1024);
        VRG_CUDA(cudaMallocHost(&hostStage_, want));
        hostStageBytes_ = want;
    }
    return hostStage_;
}

double readScalar(Ctx& ctx, const double* dev) {
    VRG_CUDA(cudaMemcpyAsync(ctx.hostScalars, dev, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    return ctx.hostScalars[0];
}

double dot(Ctx& ctx, const GridDims& g, const double* a0, const double* a1, const double* b0, const double* b1) {
    return readScalar(ctx, launchDot(ctx, g.points(), a0, b0, a1, b1, g.h1() * g.h2(), 0));
}

double normLinf(Ctx& ctx, std::size_t n, const double* a0, const double* a1) {
    return readScalar(ctx, launchMaxAbs(ctx, n, a0, a1, 1.0, 0));
}

bool anyNonFinite(Ctx& ctx, std::size_t n, const double* a0, const double* a1) {
    unsigned* flag = reinterpret_cast<unsigned*>(ctx.reduce.d() + 2 * kReduceBlocks + 60);
    VRG_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), ctx.stream));
    {
        LaunchScope ls_(ctx, "k_nonfinite");
        k_nonfinite<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(a0, n, flag);
    }
    VRG_LAUNCH_CHECK();
    if (a1) {
        {
            LaunchScope ls_(ctx, "k_nonfinite");
            k_nonfinite<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(a1, n, flag);
        }
        VRG_LAUNCH_CHECK();
    }
    unsigned h = 0;
    VRG_CUDA(cudaMemcpyAsync(ctx.hostScalars, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx.stream));
    ctx.sync();
    std::memcpy(&h, ctx.hostScalars, sizeof(unsigned));
    return h != 0;
}

void axpby(Ctx& ctx, std::size_t n, double a, const double* x, double b, double* y) {
    {
        LaunchScope ls_(ctx, "k_axpby");
        k_axpby<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, a, x, b, y);
    }
    VRG_LAUNCH_CHECK();
}

void axpyNegDevCoef(Ctx& ctx, std::size_t n, const double* c, const double* x, double* y) {
    {
        LaunchScope ls_(ctx, "k_axpy_negcoef");
        k_axpy_negcoef<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, c, x, y);
    }
    VRG_LAUNCH_CHECK();
}

void lincomb(Ctx& ctx, std::size_t n, double a, const double* x, double b, const double* y, double* out) {
    {
        LaunchScope ls_(ctx, "k_lincomb");
        k_lincomb<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, a, x, b, y, out);
    }
    VRG_LAUNCH_CHECK();
}

void fill(Ctx& ctx, std::size_t n, double v, double* y) {
    {
        LaunchScope ls_(ctx, "k_fill");
        k_fill<<<elemBlocks(ctx, n), 256, 0, ctx.stream>>>(n, v, y);
    }
    VRG_LAUNCH_CHECK();
}

void copy(Ctx& ctx, std::size_t n, const double* src, double* dst) {
    if (src != dst) VRG_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
}

}  // namespace vrg
