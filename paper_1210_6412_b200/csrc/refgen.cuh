// refgen.cuh -- the reference's input generator on the device, same random stream.
//
// `generate_dd_matrix(GenSpec)` / `generate_rhs(n, seed)` (S/generator.py:77-132) draw from
// numpy's `default_rng(seed)`: PCG64 (128-bit LCG, XSL-RR output) through
// `Generator.integers`, whose bounded draws are Lemire's multiply-shift with rejection -- on
// the 64-bit outputs for ranges beyond 2^32 (the position codes), on 32-bit halves of them
// (low half first, the high half kept for the next 32-bit draw, across calls) for the small
// value ranges. Everything here is position-indexed so it runs in parallel and still consumes
// the stream exactly as the reference's loop does:
//
//   * raw output j = XSL-RR(state after j + 1 steps), state jumped ahead in O(log j);
//   * a draw is rejected exactly when its low product word is below Lemire's threshold, which
//     depends only on that output: accept flags, then a stream compaction, give the k-th
//     accepted draw and where the stream stands afterwards;
//   * `_sample_off_diagonal` keeps the first occurrence of each code in draw order until
//     `count` are chosen, drawing whole batches of max(1024, 2 * missing) codes: a stable
//     sort by code marks first occurrences, a compaction in draw order picks them.
//
// The initial PCG64 state (state, inc) comes from the host (numpy's SeedSequence seeding).
// The Python restatement oracle/pcg64.py is checked against numpy itself; the device output
// against the host generator, which is pinned to the reference's arrays (tests/golden).
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_reduce.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

namespace mcr {
namespace rg {

typedef unsigned __int128 u128;
constexpr u128 PCG_MULT = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

// state after `delta` more steps of s -> s * MULT + inc
__host__ __device__ inline u128 pcg_advance(u128 s, u128 inc, unsigned long long delta) {
    u128 am = 1, ap = 0, cm = PCG_MULT, cp = inc;
    while (delta) {
        if (delta & 1ull) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    return am * s + ap;
}
__host__ __device__ __forceinline__ uint64_t pcg_out(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned r = (unsigned)(s >> 122);
    return (x >> r) | (x << ((64u - r) & 63u));
}

constexpr int RAW_PER_THREAD = 64;

struct ToLL {
    __host__ __device__ long long operator()(unsigned char c) const { return (long long)c; }
};

// 64-bit Lemire draws for raw positions [j0, j0 + cnt): value (valid where accepted) and the
// accept flag. re = range size (rng + 1), th = (2^64 - re) % re.
__global__ void k_lemire64(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, unsigned long long j0,
                           long long cnt, uint64_t re, uint64_t th, uint64_t* val, unsigned char* ok) {
    const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * RAW_PER_THREAD;
    if (b >= cnt) return;
    const u128 inc = mk128(i_hi, i_lo);
    u128 s = pcg_advance(mk128(s_hi, s_lo), inc, j0 + (unsigned long long)b);
    const long long e = min(cnt, b + RAW_PER_THREAD);
    for (long long j = b; j < e; ++j) {
        s = s * PCG_MULT + inc;
        const uint64_t x = pcg_out(s);
        const u128 m = (u128)x * re;
        val[j] = (uint64_t)(m >> 64);
        ok[j] = (uint64_t)m >= th ? 1 : 0;
    }
}

// 32-bit Lemire draws on half-draws [h0, h0 + cnt) (half h = low (h even) / high (h odd) word
// of raw output h / 2): value lo + (h32 * re) >> 32 (as a double) and the accept flag.
__global__ void k_lemire32(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, unsigned long long h0,
                           long long cnt, uint32_t re, uint32_t th, double lo, double* val, unsigned char* ok) {
    const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * RAW_PER_THREAD;
    if (b >= cnt) return;
    const u128 inc = mk128(i_hi, i_lo);
    const unsigned long long hb = h0 + (unsigned long long)b;
    u128 s = pcg_advance(mk128(s_hi, s_lo), inc, hb >> 1);  // state before raw output hb / 2
    uint64_t x = 0;
    const long long e = min(cnt, b + RAW_PER_THREAD);
    for (long long j = b; j < e; ++j) {
        const unsigned long long h = h0 + (unsigned long long)j;
        if (j == b || (h & 1ull) == 0) {  // a new raw output
            s = s * PCG_MULT + inc;
            x = pcg_out(s);
        }
        const uint32_t w = (h & 1ull) ? (uint32_t)(x >> 32) : (uint32_t)x;
        if (re == 0u) {  // the full 2^32 range: the half itself, never rejected
            val[j] = lo + (double)w;
            ok[j] = 1;
            continue;
        }
        const uint64_t m = (uint64_t)w * re;
        val[j] = lo + (double)(uint32_t)(m >> 32);
        ok[j] = (uint32_t)m >= th ? 1 : 0;
    }
}

__global__ void k_iota64(uint64_t* p, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = (uint64_t)i;
}
__global__ void k_iota32(uint32_t* p, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}
// first occurrences: keys sorted (stable), vals = draw positions
__global__ void k_first(const uint64_t* keys, const uint32_t* pos, long long n, unsigned char* first) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        first[pos[i]] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}
// position of the rejected draws (flag 0), for the stream position bookkeeping
__global__ void k_not(const unsigned char* ok, long long n, unsigned char* rej) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        rej[i] = ok[i] ? 0 : 1;
}

__global__ void k_d2u(const double* in, long long n, uint64_t* out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (uint64_t)in[i];
}
__global__ void k_add(double* v, long long n, double a) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] += a;
}

// CSR pieces from the sorted chosen codes (row-major = CSR order off the diagonal)
__global__ void k_rows(const uint64_t* code, long long m, long long nm1, int* cnt_off, int* cnt_lt,
                       double* rowsum, const double* val) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const long long r = (long long)(code[i] / (uint64_t)nm1), off = (long long)(code[i] % (uint64_t)nm1);
        atomicAdd(cnt_off + r, 1);
        if (off < r) atomicAdd(cnt_lt + r, 1);
        atomicAdd(rowsum + r, fabs(val[i]));  // small integers: exact in any order
    }
}
__global__ void k_rowptr(const long long* offx, long long n, long long* rp) {  // rp[r] = offx[r] + r
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r <= n; r += (long long)gridDim.x * blockDim.x)
        rp[r] = offx[r] + r;
}
__global__ void k_scatter(const uint64_t* code, const double* val, long long m, long long nm1,
                          const long long* offx, const long long* rp, int* col, double* out) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const long long r = (long long)(code[i] / (uint64_t)nm1), off = (long long)(code[i] % (uint64_t)nm1);
        const long long c = off + (off >= r ? 1 : 0);
        const long long dst = rp[r] + (i - offx[r]) + (c > r ? 1 : 0);
        col[dst] = (int)c;
        out[dst] = val[i];
    }
}
__global__ void k_diag(long long n, const long long* rp, const int* cnt_lt, const double* rowsum,
                       const double* slack, int* col, double* out) {
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        const long long dst = rp[r] + cnt_lt[r];
        col[dst] = (int)r;
        out[dst] = rowsum[r] + slack[r];
    }
}

}  // namespace rg
}  // namespace mcr
