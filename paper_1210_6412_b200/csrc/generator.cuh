// generator.cuh -- row-keyed synthetic systems built directly in HBM (config C5).
//
// Same family as the reference generator (S/generator.py:100-132): strictly diagonally
// dominant, off-diagonal positions uniform over the other n-1 columns without replacement,
// values U{lo..hi}, diagonal = row sum of |values| + U{1..hi}, right-hand side U{1..10}. The
// reference draws all positions from one PCG64 stream (and needs ~141 B/nnz of host memory,
// infeasible at n = 2e8); here every row draws from its own counter-based stream keyed by
// (seed, global row), so any row range -- any shard of any world size -- is generated alone
// and identically:
//   k_i   = off-diagonal count ~ Poisson(mean) by inverse CDF against 64-bit thresholds
//           (capped at GEN_KMAX and at n-1),
//   cols  = draws u_a = U[0, n-1) for a = 0, 1, ... (stream COL), keeping first occurrences
//           until k_i are kept; sorted; c >= i shifted to c+1 (skip the diagonal),
//   vals  = lo + U[0, hi-lo] for sorted position j (stream VAL, counter j),
//   diag  = sum of vals (exact: small integers) + 1 + U[0, hi) (stream SLACK),
//   b_i   = 1 + U[0, 10) (stream RHS).
// U[0, m) of a 64-bit hash h is floor(h * m / 2^64). oracle/oracle.c (orc_generate) restates
// this bit for bit; tests compare the two.
#pragma once

#include <stdint.h>

namespace mcr {

constexpr int GEN_KMAX = 64;
enum GenStream : uint64_t { GS_COUNT = 1, GS_COL = 2, GS_VAL = 3, GS_SLACK = 4, GS_RHS = 5 };

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t gen_hash(uint64_t seed, uint64_t row, uint64_t stream,
                                                      uint64_t ctr) {
    return splitmix64(splitmix64(splitmix64(seed ^ (stream << 58)) + row) + ctr);
}

__device__ __forceinline__ uint64_t gen_below(uint64_t h, uint64_t m) { return __umul64hi(h, m); }

struct GenParams {
    uint64_t seed;
    long long n;          // global dimension
    long long row0;       // first global row generated
    int lo, hi;           // value range
    uint64_t thr[GEN_KMAX];  // Poisson inverse-CDF thresholds: k = #{j : u >= thr[j]}
};

__device__ __forceinline__ int gen_count(const GenParams& P, long long gi) {
    const uint64_t u = gen_hash(P.seed, (uint64_t)gi, GS_COUNT, 0);
    int k = 0;
    while (k < GEN_KMAX && u >= P.thr[k]) ++k;
    const long long cap = P.n - 1;
    return (int)(k < cap ? k : cap);
}

// Row lengths (off-diagonal count + the diagonal) into len[0..rows).
__global__ void k_gen_count(GenParams P, long long rows, long long* len) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
         i += (long long)gridDim.x * blockDim.x)
        len[i] = gen_count(P, P.row0 + i) + 1;
}

// One thread per row: sample, sort, shift past the diagonal, write columns and values.
__global__ void __launch_bounds__(128) k_gen_fill(GenParams P, long long rows,
                                                  const long long* __restrict__ rp, int* col,
                                                  double* val) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
         i += (long long)gridDim.x * blockDim.x) {
        const long long gi = P.row0 + i;
        const int k = gen_count(P, gi);
        long long c[GEN_KMAX];
        int cnt = 0;
        const uint64_t m = (uint64_t)(P.n - 1);
        for (uint64_t a = 0; cnt < k; ++a) {
            const long long v = (long long)gen_below(gen_hash(P.seed, (uint64_t)gi, GS_COL, a), m);
            bool dup = false;
            for (int j = 0; j < cnt; ++j) dup |= c[j] == v;
            if (!dup) c[cnt++] = v;
        }
        for (int j = 1; j < cnt; ++j) {  // insertion sort, ascending
            const long long v = c[j];
            int t = j - 1;
            while (t >= 0 && c[t] > v) { c[t + 1] = c[t]; --t; }
            c[t + 1] = v;
        }
        const uint64_t span = (uint64_t)(P.hi - P.lo + 1);
        long long e = rp[i];
        double sum = 0.0;
        bool diag_done = false;
        const double slack =
            1.0 + (double)gen_below(gen_hash(P.seed, (uint64_t)gi, GS_SLACK, 0), (uint64_t)P.hi);
        double vals[GEN_KMAX];
        for (int j = 0; j < cnt; ++j) {
            vals[j] = (double)(P.lo + (long long)gen_below(gen_hash(P.seed, (uint64_t)gi, GS_VAL, j), span));
            sum += fabs(vals[j]);
        }
        const double diag = sum + slack;
        for (int j = 0; j < cnt; ++j) {
            const long long cj = c[j] >= gi ? c[j] + 1 : c[j];
            if (!diag_done && cj > gi) {
                col[e] = (int)gi;
                val[e] = diag;
                ++e;
                diag_done = true;
            }
            col[e] = (int)cj;
            val[e] = vals[j];
            ++e;
        }
        if (!diag_done) {
            col[e] = (int)gi;
            val[e] = diag;
        }
    }
}

__global__ void k_gen_rhs(uint64_t seed, long long row0, long long rows, double* b) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows;
         i += (long long)gridDim.x * blockDim.x)
        b[i] = 1.0 + (double)gen_below(gen_hash(seed, (uint64_t)(row0 + i), GS_RHS, 0), 10ull);
}

}  // namespace mcr
