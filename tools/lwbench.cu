// Per-element cost of the table-building sims (lane_walk_threads over HARD threads) with 1 and 16
// busy warps: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -o tools/lwbench_bin tools/lwbench.cu
// lane_walk_threads cost: 16 warps, each walks 32 HARD threads x E products (a random walk
// through zero), lanes = 32 candidates near the start. cycles per element per warp.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1210_6412_b200/csrc/device.cuh"
using namespace mcr;
using namespace mcr::xd;
__global__ void k_lw(const double* p, int E, double* out, long long* cyc, int mode, int nwarps) {
    extern __shared__ __align__(16) unsigned char dyn[];
    Run* runs = (Run*)dyn;
    double* sp = (double*)(dyn + 512 * sizeof(Run));
    for (int k = threadIdx.x; k < 512 * E; k += blockDim.x) sp[k] = p[k];
    for (int k = threadIdx.x; k < 512; k += blockDim.x) { Run r = run_empty(); r.e = E_HARD; runs[k] = r; }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp >= nwarps) return;
    double v = fb(bt(1e-3) + lane), lo = -INFINITY, hi = INFINITY;
    int km = KM_NONE;
    long long t0 = clock64();
    if (mode == 0) lane_walk_threads(runs, sp, 512 * E, E, warp * 32, warp * 32 + 32, v, lo, hi, km, nullptr, false, 0.0);
    else if (mode == 1) lane_walk_threads(runs, sp, 512 * E, E, warp * 32, warp * 32 + 32, v, lo, hi, km, nullptr, true, 0.0);
    else if (mode == 2) lane_walk_threads(runs, sp, 512 * E, E, warp * 32, warp * 32 + 32, v, lo, hi, km, nullptr, false, quantum32(v));
    else { for (int t = warp * 32; t < warp * 32 + 32; ++t) for (int k = 0; k < E; ++k) sim_step(v, sp[t * E + k], lo, hi, km); }
    long long t1 = clock64();
    out[threadIdx.x] = v + lo + hi + km;
    if (lane == 0) cyc[warp] = t1 - t0;
}
int main() {
    const int E = 15, N = 512 * E;
    std::vector<double> h(N);
    srand(3);
    // a walk through zero: terms ~1e-3 with random signs, partial sums wander around 0
    for (int i = 0; i < N; ++i) h[i] = ((rand() / (double)RAND_MAX) - 0.5) * 2e-3;
    double *dp, *dout; long long* dc;
    cudaMalloc(&dp, N * 8); cudaMalloc(&dout, 512 * 8); cudaMalloc(&dc, 16 * 8);
    cudaMemcpy(dp, h.data(), N * 8, cudaMemcpyHostToDevice);
    const char* names[4] = {"sim_elems", "bare", "collapse", "sim_step"};
    for (int nw : {1, 16}) for (int mode = 0; mode < 4; ++mode) {
        long long c[16];
        size_t sm = 512 * sizeof(Run) + N * 8; cudaFuncSetAttribute(k_lw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int rep = 0; rep < 3; ++rep) k_lw<<<1, 512, sm>>>(dp, E, dout, dc, mode, nw);
        cudaMemcpy(c, dc, nw * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; for (int w = 0; w < nw; ++w) mx = c[w] > mx ? c[w] : mx;
        printf("warps %2d %-10s %.1f cycles per element (max warp)\n", nw, names[mode], (double)mx / (32 * E));
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
