// gather_bench.cu -- microbenchmark: random fp64 gathers x[col[k]] on B200 by
//   (A) LDG from every lane (L1tex wavefront per distinct line),
//   (B) TMA tile::gather4 into shared memory (x viewed as [n/2][2] f64, 16-byte rows),
// over the C2 shape (n = 1e6, 1e7 uniformly random columns). Prints us and effective
// gathers/s. Standalone: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gb gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_init(int* col, double* val, double* x, long long m, int n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
        col[i] = (int)(h % (unsigned long long)n);
        val[i] = 1.0 + (double)(h & 7);
        if (i < n) x[i] = 0.5 + (double)(i % 13);
    }
}

// (A) lane per entry, coalesced col/val, LDG gather, warp sum.
__global__ void __launch_bounds__(256) k_ldg(const int* __restrict__ col, const double* __restrict__ val,
                                             const double* __restrict__ x, long long m, double* out) {
    const int lane = threadIdx.x & 31;
    long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (long long c = w; c * 256 < m; c += W) {
        const long long b = c * 256 + lane;
        int cc[8]; double vv[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { cc[u] = __ldcs(col + b + 32 * u); vv[u] = __ldcs(val + b + 32 * u); }
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = __ldg(x + cc[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += vv[u] * xv[u];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
    if (lane == 0) atomicAdd(out, acc);
}


// variants to locate the gather limiter
template <int MODE>
__global__ void __launch_bounds__(256) k_var(const int* __restrict__ col, const double* __restrict__ val,
                                             const double* __restrict__ x, long long m, int nx, double* out) {
    const int lane = threadIdx.x & 31;
    long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (long long c = w; c * 256 < m; c += W) {
        const long long b = c * 256 + lane;
        int cc[8]; double vv[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 3) {  // no stream: hash column in registers
                unsigned long long h = (unsigned long long)(b + 32 * u) * 0x9E3779B97F4A7C15ull; h ^= h >> 29;
                cc[u] = (int)(h % (unsigned long long)nx); vv[u] = 1.0;
            } else {
                cc[u] = __ldcs(col + b + 32 * u); vv[u] = __ldcs(val + b + 32 * u);
            }
            if (MODE == 2) cc[u] = cc[u] % nx;            // small x (L1-resident)
            if (MODE == 4) cc[u] = (cc[u] & ~1) | (lane & 1); // lane pairs share a 16-byte pair
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 1) { double t; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(t) : "l"(x + cc[u])); xv[u] = t; }
            else if (MODE == 5) { double t; asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(t) : "l"(x + cc[u])); xv[u] = t; }
            else xv[u] = __ldg(x + cc[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += vv[u] * xv[u];
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
    if (lane == 0) atomicAdd(out, acc);
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) { while (!mbar_try(b, ph)) {} }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int c0, int r0, int r1, int r2, int r3, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(su32(dst)), "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)) : "memory");
}

constexpr int CH = 1024;          // entries per stage
constexpr int STG = 4;
constexpr int SLOT = GSLOT;       // bytes of smem per gather4 (4 rows x 16 B = 64 B)
struct alignas(128) Stage {
    char xg[CH / 4 * SLOT];
    double val[CH];
    int col[CH];
};

// (B) producer warp: bulk-copies col/val of a chunk, then 32 lanes issue CH/4 gather4s.
template <int NCONS>
__global__ void __launch_bounds__(NCONS + 32) k_tma(const __grid_constant__ CUtensorMap xmap, const int* __restrict__ col,
                                                    const double* __restrict__ val, long long m, double* out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Stage* S = reinterpret_cast<Stage*>(raw);
    __shared__ __align__(8) uint64_t colbar[STG], full[STG], empty[STG];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long long nch = m / CH;
    if (tid == 0) {
        for (int s = 0; s < STG; ++s) { mbar_init(&colbar[s], 1); mbar_init(&full[s], 1); mbar_init(&empty[s], NCONS / 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc = 0.0;
    if (warp == NCONS / 32) {
        int i = 0;
        for (long long c = blockIdx.x; c < nch; c += gridDim.x, ++i) {
            const int s = i % STG;
            if (i >= STG) mbar_wait(&empty[s], ((i / STG) + 1) & 1);
            if (lane == 0) {
                mbar_expect_tx(&colbar[s], CH * 4);
                bulk_g2s(S[s].col, col + c * CH, CH * 4, &colbar[s]);
                mbar_expect_tx(&full[s], CH * 8 + CH * 16);
                bulk_g2s(S[s].val, val + c * CH, CH * 8, &full[s]);
            }
            mbar_wait(&colbar[s], (i / STG) & 1);
            __syncwarp();
            for (int g = lane; g < CH / 4; g += 32) {
                const int* cp = S[s].col + 4 * g;
                gather4(S[s].xg + g * SLOT, &xmap, 0, cp[0] >> 1, cp[1] >> 1, cp[2] >> 1, cp[3] >> 1, &full[s]);
            }
        }
    } else {
        int i = 0;
        for (long long c = blockIdx.x; c < nch; c += gridDim.x, ++i) {
            const int s = i % STG;
            mbar_wait(&full[s], (i / STG) & 1);
            for (int k = tid; k < CH; k += NCONS) {
                const int cc = S[s].col[k];
                const double* xr = reinterpret_cast<const double*>(S[s].xg + (k >> 2) * SLOT) + (k & 3) * 2;
                acc += S[s].val[k] * xr[cc & 1];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(~0u, acc, o);
        if (lane == 0) atomicAdd(out, acc);
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int n = 1000000;
    const long long m = 10000000;
    int* col; double *val, *x, *out;
    CK(cudaMalloc(&col, m * 4)); CK(cudaMalloc(&val, m * 8)); CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&out, 8));
    char* flush; CK(cudaMalloc(&flush, 512 << 20));
    k_init<<<2048, 256>>>(col, val, x, m, n);
    CK(cudaDeviceSynchronize());
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        double ref = 0; float best = 1e9;
        for (int r = 0; r < 8; ++r) {
            CK(cudaMemset(flush, r, 512 << 20));
            CK(cudaMemset(out, 0, 8));
            cudaEventRecord(e0); launch(); cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 2 && ms < best) best = ms;
            CK(cudaMemcpy(&ref, out, 8, cudaMemcpyDeviceToHost));
        }
        printf("%-28s %8.2f us  %6.2f Ggather/s  stream %6.0f GB/s  sum %.6e\n", name, best * 1e3, m / (best * 1e-3) / 1e9,
               m * 12.0 / (best * 1e-3) / 1e9, ref);
    };
    for (int per : {4, 8, 16}) {
        char nm[64]; snprintf(nm, 64, "ldg grid=%dx%d", sms, per);
        timeit(nm, [&] { k_ldg<<<sms * per, 256>>>(col, val, x, m, out); });
    }
    const char* vn[] = {"base", "nc.L1::no_allocate", "x%16384 (L1)", "no stream (hash cols)", "lane pairs same 16B", "ld.cg"};
    timeit("var0 base", [&] { k_var<0><<<sms * 4, 256>>>(col, val, x, m, n, out); });
    timeit("var1 no_allocate", [&] { k_var<1><<<sms * 4, 256>>>(col, val, x, m, n, out); });
    timeit("var2 x%16384", [&] { k_var<2><<<sms * 4, 256>>>(col, val, x, m, 16384, out); });
    timeit("var2 x%262144", [&] { k_var<2><<<sms * 4, 256>>>(col, val, x, m, 262144, out); });
    timeit("var3 no stream", [&] { k_var<3><<<sms * 4, 256>>>(col, val, x, m, n, out); });
    timeit("var4 lane pairs", [&] { k_var<4><<<sms * 4, 256>>>(col, val, x, m, n, out); });
    timeit("var5 ld.cg", [&] { k_var<5><<<sms * 4, 256>>>(col, val, x, m, n, out); });
    timeit("var3 no stream x=16K", [&] { k_var<3><<<sms * 4, 256>>>(col, val, x, m, 16384, out); });
    if (getenv("NO_TMA")) return 0;
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap map;
    cuuint64_t dims[2] = {2, (cuuint64_t)n / 2};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int smem = STG * sizeof(Stage);
    CK(cudaFuncSetAttribute(k_tma<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_tma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tma<256>, 288, smem));
    printf("tma stage %zu B, smem %d, occ %d\n", sizeof(Stage), smem, occ);
    for (int per = 1; per <= occ; ++per) {
        char nm[64]; snprintf(nm, 64, "tma-gather4 grid=%dx%d", sms, per);
        timeit(nm, [&] { k_tma<256><<<sms * per, 288, smem>>>(map, col, val, m, out); });
        CK(cudaGetLastError());
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
