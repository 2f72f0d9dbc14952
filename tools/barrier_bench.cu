// barrier_bench.cu -- cost of a grid-wide barrier on B200: cooperative_groups grid.sync()
// vs a two-level counter barrier (CTAs arrive on one of G group counters, the last of a group
// arrives on the top counter; waiters spin on a generation word).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_cg(int iters, unsigned long long* sink) {
    cg::grid_group g = cg::this_grid();
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
    if (threadIdx.x == 0 && acc == 42) *sink = acc;
}

struct Bar { unsigned int cnt[64 * 32]; unsigned int top; unsigned int gen; };

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ void bar2(Bar* b, int groups, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const int G = gridDim.x;
        const int grp = blockIdx.x % groups;
        const int members = G / groups + (grp < G % groups);
        __threadfence();
        unsigned* c = &b->cnt[grp * 32];       // one 128-byte line per group
        if (atomicAdd(c, 1u) == (unsigned)members - 1) {
            *c = 0;
            __threadfence();
            if (atomicAdd(&b->top, 1u) == (unsigned)groups - 1) {
                b->top = 0;
                __threadfence();
                atomicAdd(&b->gen, 1u);
            }
        }
        while (ld_acq(&b->gen) == gen) {}
        ++gen;
    }
    __syncthreads();
}

__global__ void k_two(int iters, Bar* b, int groups, unsigned long long* sink) {
    unsigned gen = 0;
    if (threadIdx.x == 0) gen = ld_acq(&b->gen);
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) { acc += i; bar2(b, groups, gen); }
    if (threadIdx.x == 0 && acc == 42) *sink = acc;
}

int main() {
    unsigned long long* sink; Bar* b;
    CK(cudaMalloc(&sink, 8)); CK(cudaMalloc(&b, sizeof(Bar))); CK(cudaMemset(b, 0, sizeof(Bar)));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2000;
    for (int grid : {16, 64, 148, 196, 296}) {
        void* args[] = {(void*)&iters, (void*)&sink};
        float ms;
        CK(cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args, 0, 0));
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, args, 0, 0));
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %3d  cg grid.sync      %6.3f us\n", grid, ms * 1e3 / iters);
        for (int groups : {1, 8, 16}) {
            void* a2[] = {(void*)&iters, (void*)&b, (void*)&groups, (void*)&sink};
            CK(cudaLaunchCooperativeKernel((void*)k_two, grid, 256, a2, 0, 0));
            cudaEventRecord(e0);
            CK(cudaLaunchCooperativeKernel((void*)k_two, grid, 256, a2, 0, 0));
            cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
            printf("grid %3d  2-level groups=%2d %6.3f us\n", grid, groups, ms * 1e3 / iters);
        }
    }
    return 0;
}
