// Latency of one run_apply step in a dependent chain (one warp), with and without the 10
// shuffles that fetch the run from a lane: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -o tools/rabench_bin tools/rabench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1210_6412_b200/csrc/device.cuh"
using namespace mcr;
using namespace mcr::xd;
// a run step for the exact value only: the new value from the parity alone, the in-binade
// checks on the bit patterns (integer ops) off the value's dependency chain
__device__ __forceinline__ double run_step_fast(const Run& R, double v, bool& ok) {
    const unsigned long long b = bt(v);
    const bool odd = (b & 1ull) != 0;
    const double vn = mcr::dadd(v, odd ? R.d[1] : R.d[0]);
    const unsigned long long lb = bt(mcr::dadd(v, odd ? R.lo[1] : R.lo[0])), hb = bt(mcr::dadd(v, odd ? R.hi[1] : R.hi[0]));
    const unsigned long long top12 = ((unsigned long long)R.neg << 11) | (unsigned long long)R.e;
    // same sign and binade as the run, every partial sum one ulp clear of the binade's ends
    // (lb, hb bracket the partial sums; for a negative run the larger pattern is the smaller value)
    const unsigned long long lo_b = R.neg ? hb : lb, hi_b = R.neg ? lb : hb;
    ok = (b >> 52) == top12 && (lo_b >> 52) == top12 && (hi_b >> 52) == top12 && (lo_b & MANT) != 0ull &&
         (hi_b & MANT) != MANT;
    return vn;
}
template <int mode>
__global__ void k_ra(double* out, long long* cyc, int iters) {
    const int lane = threadIdx.x & 31;
    // a run of binade [1, 2): displacement 2^-40 per step, range small
    Run R;
    R.e = 1023; R.neg = 0;
    R.d[0] = R.d[1] = ldexp(1.0, -40);
    R.lo[0] = R.lo[1] = 0.0;
    R.hi[0] = R.hi[1] = ldexp(1.0, -40);
    double v = mode >= 5 ? 1.25 + lane * ldexp(1.0, -30) : 1.25;  // mode >= 5: a different value per lane
    bool allok = true;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if constexpr (mode >= 3) asm volatile("mov.b64 %0, %0;" : "+d"(v));  // keep v per-thread (not uniform)
        Run G = R;
        if constexpr (mode == 1) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                G.d[p] = __shfl_sync(FULL, R.d[p], i & 31);
                G.lo[p] = __shfl_sync(FULL, R.lo[p], i & 31);
                G.hi[p] = __shfl_sync(FULL, R.hi[p], i & 31);
            }
            G.e = __shfl_sync(FULL, R.e, i & 31);
            G.neg = __shfl_sync(FULL, R.neg, i & 31);
        }
        if constexpr (mode < 2 || mode == 3 || mode == 5) {
            double lo = -INFINITY, hi = INFINITY;
            int km = KM_NONE;
            if (!run_apply(G, v, lo, hi, km)) v = mcr::dadd(v, 1e-20);
        } else {  // speculative: the value advances through the parity alone, checks accumulate
            bool ok;
            v = run_step_fast(G, v, ok);
            allok &= ok;
        }
    }
    if (!allok) v = -v;
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* d; long long* c;
    cudaMalloc(&d, 32 * 8); cudaMalloc(&c, 8);
    auto run = [&](auto kern, int mode, const char* name) {
        for (int rep = 0; rep < 2; ++rep) kern<<<1, 32>>>(d, c, 1000);
        long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %.1f cycles per step\n", mode, name, h / 1000.0);
    };
    run(k_ra<0>, 0, "run_apply, register run");
    run(k_ra<1>, 1, "run_apply, shuffled run");
    run(k_ra<2>, 2, "speculative step");
    run(k_ra<3>, 3, "run_apply, asm-laundered v");
    run(k_ra<4>, 4, "speculative, asm-laundered v");
    run(k_ra<5>, 5, "run_apply, lane-varying v");
    run(k_ra<6>, 6, "speculative, lane-varying v");
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
