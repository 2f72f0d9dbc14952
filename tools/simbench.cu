// Cycles per element of sim_elems / plain DADD chain / sim_step (one warp):
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -o tools/simbench_bin tools/simbench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1210_6412_b200/csrc/device.cuh"
using namespace mcr;
using namespace mcr::xd;
__global__ void k_sim(const double* p, int cnt, double* out, long long* cyc, int mode) {
    __shared__ double sp[1024];
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) sp[k] = p[k];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double v = 1.5 + lane * 1e-15, lo = -INFINITY, hi = INFINITY;
    int km = KM_NONE;
    long long t0 = clock64();
    if (mode == 0) sim_elems(sp, cnt, v, lo, hi, km);
    else if (mode == 1) { for (int k = 0; k < cnt; ++k) v = mcr::dadd(v, sp[k]); }
    else { for (int k = 0; k < cnt; ++k) sim_step(v, sp[k], lo, hi, km); }
    long long t1 = clock64();
    out[threadIdx.x] = v + lo + hi + km;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    const int cnt = 960;
    double* hp = new double[cnt];
    for (int i = 0; i < cnt; ++i) hp[i] = 1e-3 * ((i * 7919) % 1000) / 1000.0;
    double *dp, *dout; long long* dc;
    cudaMalloc(&dp, cnt * 8); cudaMalloc(&dout, 32 * 8); cudaMalloc(&dc, 8);
    cudaMemcpy(dp, hp, cnt * 8, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            k_sim<<<1, 32>>>(dp, cnt, dout, dc, mode);
            long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
            if (rep == 2) printf("mode %d: %.1f cycles/element\n", mode, (double)c / cnt);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
