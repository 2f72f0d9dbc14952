// dense.cuh -- dense slab GEMV (part of device.cuh).
#pragma once

#include "common.cuh"

namespace mcr {

// ---------------------------------------------------------------- dense slab GEMV (TMA bulk)
// One warp per 32-row slab. Lane r owns row 32*slab + r and adds a_rj * x_j for j = 0..n-1
// strictly in order (skipping stored zeros exactly like CSR skips absent entries, and the
// diagonal for Jacobi). A slab is stored as [column pair][row][2] (512 B per pair) and streams
// HBM -> shared memory through a DSTAGES-deep ring of cp.async.bulk copies completed on
// mbarriers. Per 16 columns the lane first forms all 16 products (LDS.128 of its two entries
// per pair, x broadcast from shared memory), then runs the 16 dependent adds back to back, so
// the serial chain is pure DADD latency. A skipped entry contributes +0.0: the running sum
// starts at +0.0 and can never become -0.0 under round-to-nearest, so acc + 0.0 == acc
// exactly and the result is bit-identical to the CSR row sum.
template <int EPI>
__global__ void __launch_bounds__(32) k_dense(const double* __restrict__ A, int n, int npad,
                                              const double* __restrict__ x, Vecs V,
                                              SolveState* st) {
    extern __shared__ __align__(128) double dsm[];
    __shared__ __align__(8) uint64_t bars[DSTAGES];
    __shared__ __align__(16) double xs[DCOLS];
    __shared__ int s_flag;
    griddep_wait();
    griddep_launch();
    if constexpr (epi_checks_stop<EPI>()) {
        if (st->stop) return;
    }
    const double* xin = jacobi_select<EPI>(x, V, st);
    const int lane = threadIdx.x;
    const int slab = blockIdx.x;
    const int row = slab * DSLAB + lane;
    const double* src = A + (size_t)slab * (size_t)npad * DSLAB;
    const int nchunks = (npad + DCOLS - 1) / DCOLS;
    if (lane == 0) {
        for (int s = 0; s < DSTAGES; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
        for (int c = 0; c < DSTAGES && c < nchunks; ++c) {
            const int cols = min(DCOLS, npad - c * DCOLS);
            const uint32_t bytes = (uint32_t)(cols * DSLAB * sizeof(double));
            mbar_expect_tx(&bars[c], bytes);
            bulk_g2s_hint(dsm + c * DCOLS * DSLAB, src + (size_t)c * DCOLS * DSLAB, bytes, &bars[c],
                          l2_evict_first());
        }
    }
    __syncwarp();
    EpiIn in{0.0, 0.0, 0.0};
    if (row < n) in = epi_load<EPI>(V, row);
    double acc = 0.0;
    // x of chunk c: lane holds columns j0 + lane and j0 + 32 + lane
    double xa = lane < n ? __ldg(xin + lane) : 0.0;
    double xb = lane + 32 < n ? __ldg(xin + lane + 32) : 0.0;
    for (int c = 0; c < nchunks; ++c) {
        const int stage = c % DSTAGES;
        const uint32_t parity = (uint32_t)((c / DSTAGES) & 1);
        const int j0 = c * DCOLS;
        const int jn = j0 + DCOLS;  // prefetch next chunk's x
        const double nxa = jn + lane < n ? __ldg(xin + jn + lane) : 0.0;
        const double nxb = jn + 32 + lane < n ? __ldg(xin + jn + 32 + lane) : 0.0;
        xs[lane] = xa;
        xs[lane + 32] = xb;
        __syncwarp();
        mbar_wait(&bars[stage], parity);
        const double2* tile = reinterpret_cast<const double2*>(dsm + stage * DCOLS * DSLAB);
        const double2* xs2 = reinterpret_cast<const double2*>(xs);
        const int pairs = min(DCOLS, npad - j0) / 2;
#pragma unroll
        for (int kb = 0; kb < DCOLS / 2; kb += 8) {
            if (kb < pairs) {  // pairs is a multiple of 8 except in the last chunk
                double pr[16];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int kk = kb + u;
                    double2 a = make_double2(0.0, 0.0), xv = make_double2(0.0, 0.0);
                    if (kk < pairs) {
                        a = tile[kk * DSLAB + lane];
                        xv = xs2[kk];
                    }
                    bool u0 = a.x != 0.0, u1 = a.y != 0.0;
                    if constexpr (EPI == EPI_JACOBI) {
                        const int j = j0 + 2 * kk;
                        u0 = u0 && j != row;
                        u1 = u1 && j + 1 != row;
                    }
                    pr[2 * u] = u0 ? dmul(a.x, xv.x) : 0.0;
                    pr[2 * u + 1] = u1 ? dmul(a.y, xv.y) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 16; ++u) acc = dadd(acc, pr[u]);
            }
        }
        __syncwarp();
        if (lane == 0 && c + DSTAGES < nchunks) {
            fence_proxy_async();
            const int cn = c + DSTAGES;
            const int cc = min(DCOLS, npad - cn * DCOLS);
            const uint32_t bytes = (uint32_t)(cc * DSLAB * sizeof(double));
            mbar_expect_tx(&bars[stage], bytes);
            bulk_g2s_hint(dsm + stage * DCOLS * DSLAB, src + (size_t)cn * DCOLS * DSLAB, bytes,
                          &bars[stage], l2_evict_first());
        }
        xa = nxa;
        xb = nxb;
    }
    double p1 = 0.0, p2 = 0.0;
    unsigned long long mb = 0;
    if (row < n) epi_store<EPI>(V, row, acc, in, p1, p2, mb);
    if constexpr (epi_has_dot<EPI>()) {
        p1 = group_sum<1, 0>(p1, nullptr);
        if (lane == 0) V.P1[slab] = p1;
        if constexpr (EPI == EPI_T) {
            p2 = group_sum<1, 0>(p2, nullptr);
            if (lane == 0) V.P2[slab] = p2;
        }
    }
    kernel_finish<32, EPI>(V, st, gridDim.x, mb, nullptr, nullptr, &s_flag);
}

}  // namespace mcr
