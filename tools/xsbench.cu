// One-CTA reference-order dot (xd::cta_seqdots) microbenchmark with phase timings (MCR_XS_TIMING):
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -o tools/xsbench_t tools/xsbench.cu
// ./tools/xsbench_t n reps mode   (mode 0: signed products wandering through zero, 1: positive, 2: drift)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define MCR_XS_TIMING 1
#include "../paper_1210_6412_b200/csrc/device.cuh"
using namespace mcr;
__global__ void k_xs(const double* p, int n, double* out, int reps) {
    extern __shared__ __align__(16) unsigned char dyn[];
    double* buf = (double*)dyn;
    auto& D = *(xd::CtaDots<256, 1>*)(dyn + 2 * n * sizeof(double));
    for (int i = threadIdx.x; i < n; i += 256) buf[i] = p[i];
    __syncthreads();
    double r = 0;
    for (int q = 0; q < reps; ++q) { double res[1]; xd::cta_seqdots<256, 1>(buf, n, D, res); r += res[0]; }
    if (threadIdx.x == 0) out[0] = r;
}
int main(int argc, char** argv) {
    int n = argc > 1 ? atoi(argv[1]) : 2000;
    std::vector<double> h(n);
    srand(1);
    const int mode = argc > 3 ? atoi(argv[3]) : 0;
    for (int i = 0; i < n; ++i) {
        const double a = rand() / (double)RAND_MAX, b = rand() / (double)RAND_MAX;
        h[i] = mode == 1 ? a * b + 0.1 : (mode == 2 ? (a - 0.5) * b + 0.01 : (a - 0.5) * b);
    }
    double *dp, *dout;
    cudaMalloc(&dp, n * 8); cudaMalloc(&dout, 8);
    cudaMemcpy(dp, h.data(), n * 8, cudaMemcpyHostToDevice);
    size_t sm = 2 * n * 8 + sizeof(xd::CtaDots<256, 1>);
    cudaFuncSetAttribute(k_xs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int reps = argc > 2 ? atoi(argv[2]) : 1000;
    k_xs<<<1, 256, sm>>>(dp, n, dout, 4);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_xs<<<1, 256, sm>>>(dp, n, dout, reps);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("n=%d: %.3f us per call\n", n, ms * 1e3 / reps);
    k_xs<<<1, 256, sm>>>(dp, n, dout, 4);
    cudaDeviceSynchronize();
    double s = 0; for (int i = 0; i < n; ++i) s += h[i];
    double r; cudaMemcpy(&r, dout, 8, cudaMemcpyDeviceToHost);
    printf("n=%d result/4=%.17g serial=%.17g %s\n", n, r / 4, s, cudaGetErrorString(cudaGetLastError()));
}
