// dsmem_bench.cu -- microbenchmark: random fp64 gathers from distributed shared memory.
// Each CTA of a cluster holds PER doubles of a "band"; 1e7 gathers with uniformly random band
// indices are served by ld.shared::cluster from the owning CTA. Compared with random gathers
// from local shared memory. nvcc -O3 -gencode arch=compute_100a,code=sm_100a dsmem_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned hsh(unsigned long long i) {
    unsigned long long h = i * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    return (unsigned)h;
}

template <int CL, int LOCAL>
__global__ void __launch_bounds__(512) k_ds(long long m, int per, double* out) {
    extern __shared__ double xs[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < per; i += blockDim.x) xs[i] = 1.0 + (i & 7);
    cl.sync();
    const unsigned band = (unsigned)per * CL;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long T = (long long)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (long long b = tid * 8; b < m; b += T * 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const unsigned idx = hsh(b + u) % (LOCAL ? (unsigned)per : band);
            if (LOCAL) {
                v[u] = xs[idx];
            } else {
                const unsigned r = idx / per, o = idx - r * per;
                const double* p = cl.map_shared_rank(xs, r);
                v[u] = p[o];
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    cl.sync();
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

template <int CL, int LOCAL>
void run(int per, int threads, long long m, double* out) {
    auto k = k_ds<CL, LOCAL>;
    const int smem = per * 8;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (CL > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = 0;
    cfg.gridDim = dim3(CL);
    CK(cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
    cfg.gridDim = dim3(CL * ncl);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0);
        CK(cudaLaunchKernelEx(&cfg, k, m, per, out));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 1 && ms < best) best = ms;
    }
    printf("cluster %2d %s per-CTA %6d doubles (%4d KB) threads %d clusters %3d (%3d SMs): %8.2f us  %7.1f Ggather/s  %.2f gathers/cyc/SM@1.9GHz\n",
           CL, LOCAL ? "LOCAL " : "DSMEM ", per, per * 8 / 1024, threads, ncl, ncl * CL, best * 1e3, m / (best * 1e-3) / 1e9,
           m / (best * 1e-3) / (ncl * CL) / 1.9e9);
}

int main() {
    double* out; CK(cudaMalloc(&out, 8));
    const long long m = 10000000;
    run<1, 1>(24576, 512, m, out);
    run<8, 0>(24576, 512, m, out);
    run<8, 0>(24576, 256, m, out);
    run<16, 0>(24576, 512, m, out);
    run<16, 0>(24576, 256, m, out);
    run<4, 0>(24576, 512, m, out);
    run<2, 0>(24576, 512, m, out);
    return 0;
}
