// Does an L2 access-policy window keep a re-read 48 MB set resident while 32 MB of fresh
// data streams through each launch?  (models one SL step: X/vt/vtD reused, G/GD fresh)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(const double2* __restrict__ reuse, size_t nr, const double2* __restrict__ fresh, size_t nf,
                       double* out) {
    double s = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nr; i += stride) {
        double2 v = reuse[i];
        s += v.x + v.y;
    }
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nf; i += stride) {
        double2 v = __ldcs(fresh + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) out[0] = s;
}

int main() {
    int dev = 0, maxPersist = 0, maxWin = 0, l2 = 0, sms = 0;
    cudaDeviceGetAttribute(&maxPersist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxWin, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    printf("L2 %d MB, max persisting %d MB, max window %d MB\n", l2 >> 20, maxPersist >> 20, maxWin >> 20);
    const size_t reuseMB = 48, freshMB = 32, poolMB = 4096;
    double2 *reuse, *pool;
    double* out;
    cudaMalloc(&reuse, reuseMB << 20);
    cudaMalloc(&pool, poolMB << 20);
    cudaMalloc(&out, 8);
    cudaMemset(reuse, 0, reuseMB << 20);
    cudaMemset(pool, 0, poolMB << 20);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const size_t nr = (reuseMB << 20) / 16, nf = (freshMB << 20) / 16;
    const int iters = 100;
    for (int mode = 0; mode < 4; ++mode) {
        size_t persistBytes = 0;
        float hit = 1.0f;
        if (mode == 1) persistBytes = reuseMB << 20;
        if (mode == 2) { persistBytes = (size_t)maxPersist; hit = 1.0f; }
        if (mode == 3) { persistBytes = (size_t)maxPersist; hit = 0.75f; }
        if (persistBytes > (size_t)maxPersist) persistBytes = maxPersist;
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persistBytes);
        cudaStreamAttrValue v = {};
        if (mode > 0) {
            v.accessPolicyWindow.base_ptr = reuse;
            v.accessPolicyWindow.num_bytes = reuseMB << 20;
            v.accessPolicyWindow.hitRatio = hit;
            v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        }
        cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
        cudaCtxResetPersistingL2Cache();
        for (int w = 0; w < 5; ++w) k_step<<<sms * 8, 256, 0, st>>>(reuse, nr, pool + (size_t)w * nf, nf, out);
        cudaEventRecord(e0, st);
        for (int i = 0; i < iters; ++i)
            k_step<<<sms * 8, 256, 0, st>>>(reuse, nr, pool + (size_t)((i * nf) % ((poolMB << 20) / 16 - nf)), nf, out);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mode %d (persist %zu MB, hit %.2f): %.2f us/launch, %.0f GB/s of %zu MB\n", mode, persistBytes >> 20, hit,
               ms * 1e3 / iters, (double)((reuseMB + freshMB) << 20) * iters / (ms / 1e3) / 1e9, reuseMB + freshMB);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
