// gather_size_bench.cu -- random fp64 gather rate vs the footprint the gathers span.
// x has NX = 2e8 doubles (1.6 GB, C5's x); 1e8 gathers land uniformly in the first W
// doubles. W <= ~1.5e7 (L2-resident) vs W = 3.2e7 (256 MB: the TLB reach of 2 MB pages)
// vs W = 2e8 separates L2 capacity, TLB reach and random-DRAM effects.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_init(int* col, long long m, long long w) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
        col[i] = (int)(h % (unsigned long long)w);
    }
}
template <int SORTED>
__global__ void __launch_bounds__(256) k_g(const int* __restrict__ col, const double* __restrict__ x, long long m, double* out) {
    const int lane = threadIdx.x & 31;
    long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (long long c = w; c * 256 < m; c += W) {
        const long long b = c * 256 + lane;
        int cc[8]; double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) cc[u] = __ldcs(col + b + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (SORTED == 1) asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(xv[u]) : "l"(x + cc[u]));
            else if (SORTED == 2) asm volatile("ld.global.nc.L2::256B.f64 %0, [%1];" : "=d"(xv[u]) : "l"(x + cc[u]));
            else if (SORTED == 3) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(xv[u]) : "l"(x + cc[u]));
            else xv[u] = __ldg(x + cc[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += xv[u];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
    if (lane == 0) atomicAdd(out, acc);
}
int main(int argc, char** argv) {
    const long long NX = 200000000LL, m = 100000000LL;
    double* x; int* col; double* out; char* flush;
    CK(cudaMalloc(&x, NX * 8)); CK(cudaMalloc(&col, m * 4)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&flush, 256 << 20));
    CK(cudaMemset(x, 0, NX * 8));
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t gran = 0;
    if (argc > 1) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1])));
    CK(cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity));
    printf("cudaLimitMaxL2FetchGranularity = %zu\n", gran);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    long long ws[] = {4000000, 32000000, 200000000};
    for (int mode = 0; mode < 4; ++mode)
    for (long long w : ws) {
        k_init<<<4096, 256>>>(col, m, w);
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            CK(cudaMemset(flush, r, 256 << 20));
            cudaEventRecord(e0);
            if (mode == 0) k_g<0><<<sms * 4, 256>>>(col, x, m, out);
            if (mode == 1) k_g<1><<<sms * 4, 256>>>(col, x, m, out);
            if (mode == 2) k_g<2><<<sms * 4, 256>>>(col, x, m, out);
            if (mode == 3) k_g<3><<<sms * 4, 256>>>(col, x, m, out);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 1 && ms < best) best = ms;
        }
        printf("mode %d window %10lld doubles (%7.1f MB): %8.2f us  %6.1f Ggather/s\n", mode, w, w * 8 / 1e6, best * 1e3, m / (best * 1e-3) / 1e9);
    }
    return 0;
}
