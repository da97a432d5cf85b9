// Read bandwidth vs working-set size (is a working set that fits the 126 MB L2 re-read
// faster than HBM across kernel launches?).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const double2* __restrict__ a, size_t n, double* out) {
    double s = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double2 v = __ldg(a + i);
        s += v.x + v.y;
    }
    if (s == 12345.678) out[0] = s;
}
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main() {
    size_t maxBytes = (size_t)2048 << 20;
    double2* a; double2* b; double* out;
    cudaMalloc(&a, maxBytes); cudaMalloc(&b, maxBytes); cudaMalloc(&out, 8);
    cudaMemset(a, 0, maxBytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t sizesMB[] = {8, 16, 24, 32, 48, 64, 80, 96, 112, 128, 192, 256, 512, 2048};
    for (size_t mb : sizesMB) {
        size_t n = (mb << 20) / sizeof(double2);
        int iters = 50;
        for (int w = 0; w < 3; ++w) k_read<<<sms * 8, 256>>>(a, n, out);
        cudaEventRecord(e0);
        for (int i = 0; i < iters; ++i) k_read<<<sms * 8, 256>>>(a, n, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double rd = (double)(mb << 20) * iters / (ms / 1e3) / 1e9;
        size_t nc = n / 2;
        for (int w = 0; w < 3; ++w) k_copy<<<sms * 8, 256>>>(a, b, nc);
        cudaEventRecord(e0);
        for (int i = 0; i < iters; ++i) k_copy<<<sms * 8, 256>>>(a, b, nc);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double cp = (double)(mb << 20) * iters / (ms / 1e3) / 1e9;  // read half + write half = mb per launch
        printf("%6zu MB  read %8.0f GB/s (%7.2f us/launch)   copy(rd+wr) %8.0f GB/s\n", mb, rd,
               (double)(mb << 20) / rd / 1e3, cp);
    }
    return 0;
}
