// Microbenchmark: cycles per dependent fp64 add (DADD) and per dependent LDS+DADD step, the two
// costs of the exact row-sum chain in the small-system kernels. nvcc -arch=sm_100a -o dadd_lat dadd_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const double* in, double* out, long long* cyc, int n) {
    __shared__ double sm[4096];
    for (int k = threadIdx.x; k < 4096; k += blockDim.x) sm[k] = in[k];
    __syncthreads();
    double acc = 0.0;
    long long t0 = clock64();
    for (int k = 0; k < n; ++k) acc = __dadd_rn(acc, in[4096]);  // register operand after first load
    long long t1 = clock64();
    double acc2 = 0.0;
#pragma unroll 16
    for (int k = 0; k < 4096; ++k) acc2 = __dadd_rn(acc2, sm[k]);
    long long t2 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
    out[threadIdx.x] = acc + acc2;
}

int main() {
    double *in, *out; long long* cyc;
    cudaMalloc(&in, 8 * 8192); cudaMalloc(&out, 8 * 1024); cudaMallocManaged(&cyc, 16);
    cudaMemset(in, 0, 8 * 8192);
    for (int rep = 0; rep < 3; ++rep) {
        chain<<<1, 32>>>(in, out, cyc, 4096);
        cudaDeviceSynchronize();
        printf("dependent DADD: %.2f cyc/op; LDS-fed DADD chain: %.2f cyc/op\n", cyc[0] / 4096.0, cyc[1] / 4096.0);
    }
    return 0;
}
