// upload.cuh -- upload-time kernels: column conversion and checks, diagonal, off-diagonal split, dense build (part of device.cuh).
#pragma once

#include "common.cuh"

namespace mcr {

// ---------------------------------------------------------------- upload helpers
__global__ void k_col64to32(const long long* __restrict__ in, int* __restrict__ out, long long m,
                            int n, int* bad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x) {
        const long long c = in[i];
        if (c < 0 || c >= n) atomicExch(bad, 1);
        out[i] = (int)c;
    }
}

// Rows must be sorted by column without duplicates (the reference's CsrMatrix invariant,
// sparse.py:101-118): the row sums are defined in that order.
// Row bounds are clamped to [0, nnz]: rstart is checked for monotonicity on the host while
// this runs, and a malformed one must not send the scan out of bounds.
__global__ void k_check_rows(const long long* __restrict__ rp, const int* __restrict__ col, int n,
                             long long nnz, int* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (long long e = max(rp[i], 0ll) + 1, end = min(rp[i + 1], nnz); e < end; ++e)
            if (col[e] <= col[e - 1]) {
                atomicExch(bad, 1);
                break;
            }
}

// Stored diagonal per row (0.0 if absent; rows sorted -> binary search), the off-diagonal
// row length, and the first row whose diagonal is 0 (ZeroDiagonal). Row i of the handle is
// global row roff + i (row shards keep global column indices).
__global__ void k_diag(const long long* __restrict__ rp, const int* __restrict__ col,
                       const double* __restrict__ val, int n, long long roff, double* d,
                       long long* offlen, unsigned long long* first_zero,
                       unsigned long long* ndiag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        long long lo = rp[i], hi = rp[i + 1];
        const long long len = hi - lo;
        const long long gi = roff + i;
        double dv = 0.0;
        int has = 0;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            const long long c = col[mid];
            if (c == gi) { dv = val[mid]; has = 1; break; }
            if (c < gi) lo = mid + 1; else hi = mid;
        }
        d[i] = dv;
        if (offlen) offlen[i] = len - has;
        if (dv == 0.0) atomicMin(first_zero, (unsigned long long)i);
        const unsigned act = __activemask(), hb = __ballot_sync(act, has);  // one atomic per warp
        if (ndiag && (threadIdx.x & 31) == __ffs(act) - 1 && hb)
            atomicAdd(ndiag, (unsigned long long)__popc(hb));
    }
}

// Off-diagonal copy R (without_diagonal, sparse.py:227-231): order of the kept entries is
// unchanged. One warp per row.
__global__ void k_split_offdiag(const long long* __restrict__ rp, const int* __restrict__ col,
                                const double* __restrict__ val, int n, long long roff,
                                const long long* __restrict__ rrp, int* rcol, double* rval) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const long long b = rp[i], e = rp[i + 1];
        long long out = rrp[i];
        for (long long k0 = b; k0 < e; k0 += 32) {
            const long long k = k0 + lane;
            const bool inr = k < e;
            const int c = inr ? col[k] : -1;
            const bool keep = inr && (long long)c != roff + i;
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const long long pos = out + __popc(msk & ((1u << lane) - 1u));
                rcol[pos] = c;
                rval[pos] = val[k];
            }
            out += __popc(msk);
        }
    }
}

// Dense slab build: zero-filled beforehand; one CTA per row scatters its entries into
// [column pair][row][2] slabs of npad (even) columns.
__global__ void k_dense_build(const long long* __restrict__ rp, const int* __restrict__ col,
                              const double* __restrict__ val, int n, int npad, double* A) {
    const int i = blockIdx.x;
    const size_t slab = (size_t)(i / DSLAB), r = (size_t)(i % DSLAB);
    double* S = A + slab * (size_t)npad * DSLAB;
    for (long long k = rp[i] + threadIdx.x; k < rp[i + 1]; k += blockDim.x) {
        const size_t j = (size_t)col[k];
        S[((j >> 1) * DSLAB + r) * 2 + (j & 1)] = val[k];
    }
}

}  // namespace mcr
