// spmv.cuh -- CSR SpMV: the persistent TMA-pipelined tile kernel with fused epilogues, and SELL-32-sigma (part of device.cuh).
#pragma once

#include "common.cuh"

namespace mcr {

// ---------------------------------------------------------------- CSR SpMV (persistent)
// One stage of the tile pipeline: a tile's row pointers, columns and values, copied from HBM
// by 16-byte aligned TMA bulk copies. Columns and values are both copied from the same base
// entry (e0 rounded down to a multiple of 4), so position j of either array is entry base+j.
struct alignas(16) SpStage {
    double val[TILE_NNZ + 8];
    int col[TILE_NNZ + 8];
    long long rp[TILE_ROWS + 4];
};
constexpr size_t SP_SMEM = sizeof(SpStage) * SP_STAGES;
// Tiles whose mean row holds more than this many entries gather cooperatively (all 256
// threads) before the per-row sums; shorter rows are summed thread-per-row straight from the
// staged columns and values.
constexpr int SP_COOP_ROWLEN = 32;
#ifndef MCR_SP_BATCH
#define MCR_SP_BATCH 8
#endif
#ifndef MCR_SP_MINB
#define MCR_SP_MINB 3
#endif
constexpr int SP_BATCH = MCR_SP_BATCH;  // gathers in flight per thread in the row loop

// Persistent, warp-specialised CSR SpMV with a fused epilogue.
//   producer warp: walks a static tile schedule (tile t -> CTA t mod grid), prefetches the
//                  next tile descriptor, and streams each tile into a free stage with three
//                  cp.async.bulk copies (rowptr, col, val) completed on a full mbarrier;
//   256 consumer threads: thread r owns tile row r and accumulates a_rj * x_j over the row's
//                  staged entries left to right (scipy's order, bit-identical); rows of
//                  long-row tiles are first gathered cooperatively into shared memory.
// While the consumers work on one tile, the next tile is already in flight.
template <int EPI>
__global__ void __launch_bounds__(SP_THREADS, MCR_SP_MINB) k_spmv(Csr A, const double* __restrict__ x, Vecs V,
                                                     SolveState* st) {
    extern __shared__ __align__(128) unsigned char sp_raw[];
    SpStage* stg = reinterpret_cast<SpStage*>(sp_raw);
    __shared__ __align__(8) uint64_t full_bar[SP_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[SP_STAGES];
    __shared__ TileDesc s_desc[SP_STAGES];
    __shared__ int s_tile[SP_STAGES];
    __shared__ double s_red[SP_THREADS / 32];
    __shared__ unsigned long long s_redu[SP_THREADS / 32];
    __shared__ int s_flag;
    // The matrix does not depend on the previous kernel: the producer fills the first stages
    // before waiting for it (with PDL this overlaps the previous kernel's tail); everything
    // that reads vectors or the solver state waits first.
    griddep_launch();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < SP_STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], SP_CONSUMERS / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    unsigned long long mb = 0;
    const int G = gridDim.x;
    // dot partials: each consumer thread adds its rows' terms over ALL its tiles (the static
    // schedule t = blockIdx.x + i*G fixes the order), one CTA tree at the end -> P[blockIdx.x]
    double acc1 = 0.0, acc2 = 0.0;

    if (warp == SP_CONSUMERS / 32) {
        // ------------------------------------------------------------ producer warp
        if (lane == 0) {
            const uint64_t pol = l2_evict_first();
            int t = blockIdx.x;
            TileDesc dn{};
            if (t < A.ntiles) dn = A.desc[t];
            bool stopped = false;
            for (int i = 0;; ++i, t += G) {
                const int s = i % SP_STAGES;
                const TileDesc d = dn;
                if (t + G < A.ntiles) dn = A.desc[t + G];  // prefetch the next descriptor
                if (i == SP_STAGES) {  // first stages issued: now the stop flag is needed
                    griddep_wait();
                    if constexpr (epi_checks_stop<EPI>()) stopped = ld_state(&st->stop) != 0;
                }
                if (i >= SP_STAGES) mbar_wait(&empty_bar[s], (uint32_t)(((i / SP_STAGES) + 1) & 1));
                if (t >= A.ntiles || stopped) {
                    s_tile[s] = -1;
                    mbar_arrive(&full_bar[s]);
                    break;
                }
                s_tile[s] = t;
                s_desc[s] = d;
                if (d.e1 - d.e0 > TILE_NNZ) {  // one long row: consumers stream it from HBM
                    mbar_arrive(&full_bar[s]);
                    continue;
                }
                const long long ra = d.r0 & ~1ll, base = d.e0 & ~3ll;
                const uint32_t rb = (uint32_t)(((d.r1 + 1 - ra) * 8 + 15) & ~15ll);
                const uint32_t vb = d.e1 > d.e0 ? (uint32_t)(((d.e1 - base) * 8 + 15) & ~15ll) : 0u;
                const uint32_t cb = d.e1 > d.e0 ? (uint32_t)(((d.e1 - base) * 4 + 15) & ~15ll) : 0u;
                mbar_expect_tx(&full_bar[s], rb + vb + cb);
                bulk_g2s_hint(stg[s].rp, A.rp + ra, rb, &full_bar[s], pol);
                if (vb) {
                    bulk_g2s_hint(stg[s].val, A.val + base, vb, &full_bar[s], pol);
                    bulk_g2s_hint(stg[s].col, A.col + base, cb, &full_bar[s], pol);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ consumer warps
        griddep_wait();
        bool stopped = false;
        if constexpr (epi_checks_stop<EPI>()) stopped = ld_state(&st->stop) != 0;
        const double* xin = jacobi_select<EPI>(x, V, st);
        for (int i = 0;; ++i) {
            const int s = i % SP_STAGES;
            mbar_wait(&full_bar[s], (uint32_t)((i / SP_STAGES) & 1));
            TileDesc d;
            const int t = stage_tile(s_tile, s_desc, s, d);
            if (t < 0) break;
            if (stopped) {  // the solve has stopped: only release the prefetched stages
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
                continue;
            }
            const int nrows = d.r1 - d.r0;
            const int row = d.r0 + tid;
            EpiIn in{0.0, 0.0, 0.0};
            if (tid < nrows) in = epi_load<EPI>(V, row);
            SpStage& S = stg[s];
            const long long len = d.e1 - d.e0;
            double acc = 0.0;
            if (len > TILE_NNZ) {
                // single row longer than a tile: stream it through this stage's buffer
                double a = 0.0;
                for (long long b0 = d.e0; b0 < d.e1; b0 += TILE_NNZ) {
                    const int clen = (int)((d.e1 - b0) < TILE_NNZ ? (d.e1 - b0) : TILE_NNZ);
                    for (int k = tid; k < clen; k += SP_CONSUMERS)
                        S.val[k] = dmul(__ldcs(A.val + b0 + k), __ldg(xin + __ldcs(A.col + b0 + k)));
                    named_sync(1, SP_CONSUMERS);
                    if (tid == 0)
                        for (int k = 0; k < clen; ++k) a = dadd(a, S.val[k]);
                    fence_proxy_async();
                    named_sync(1, SP_CONSUMERS);
                }
                acc = a;
            } else {
                const long long base = d.e0 & ~3ll;
                const int ro = d.r0 & 1;                      // rowptr r0 sits at S.rp[ro]
                if (len > (long long)SP_COOP_ROWLEN * nrows) {
                    // long rows: all threads gather + multiply in place, then row sums
                    const int j0 = (int)(d.e0 - base), j1 = (int)(d.e1 - base);
                    for (int j = j0 + tid; j < j1; j += SP_CONSUMERS)
                        S.val[j] = dmul(S.val[j], __ldg(xin + S.col[j]));
                    named_sync(1, SP_CONSUMERS);
                    if (tid < nrows) {
                        const int b = (int)(S.rp[ro + tid] - base), e = (int)(S.rp[ro + tid + 1] - base);
                        double a = 0.0;
                        for (int k = b; k < e; ++k) a = dadd(a, S.val[k]);
                        acc = a;
                    }
                    fence_proxy_async();  // in-place products (generic) before the next refill
                    named_sync(1, SP_CONSUMERS);
                } else if (tid < nrows) {
                    // short rows: thread-per-row, SP_BATCH gathers in flight per thread
                    int k = (int)(S.rp[ro + tid] - base);
                    const int e = (int)(S.rp[ro + tid + 1] - base);
                    double a = 0.0;
                    while (k < e) {
                        const int cnt = min(SP_BATCH, e - k);
                        double xv[SP_BATCH];
#pragma unroll
                        for (int u = 0; u < SP_BATCH; ++u)
                            if (u < cnt) xv[u] = __ldg(xin + S.col[k + u]);
#pragma unroll
                        for (int u = 0; u < SP_BATCH; ++u)
                            if (u < cnt) a = dadd(a, dmul(S.val[k + u], xv[u]));
                        k += cnt;
                    }
                    acc = a;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);  // stage free for the producer
            double p1 = 0.0, p2 = 0.0;
            if (tid < nrows) {
                epi_store<EPI>(V, row, acc, in, p1, p2, mb);
                if constexpr (epi_has_dot<EPI>()) {
                    acc1 = dadd(acc1, p1);
                    if constexpr (EPI == EPI_T) acc2 = dadd(acc2, p2);
                }
            }
        }
        if constexpr (epi_has_dot<EPI>()) {
            acc1 = group_sum<SP_CONSUMERS / 32, 1>(acc1, s_red);
            if (tid == 0) V.P1[blockIdx.x] = acc1;
            if constexpr (EPI == EPI_T) {
                acc2 = group_sum<SP_CONSUMERS / 32, 1>(acc2, s_red);
                if (tid == 0) V.P2[blockIdx.x] = acc2;
            }
        }
    }
    griddep_wait();  // (the producer lane may have ended before its wait)
    if constexpr (epi_checks_stop<EPI>()) {
        if (ld_state(&st->stop)) return;  // stopped before this kernel: no partials, no step
    }
    if constexpr (EPI == EPI_JACOBI) {
        if (V.peers) __threadfence_system();  // peer stores performed before the grid retires
    }
    kernel_finish<SP_THREADS, EPI, true>(V, st, G, mb, s_red, s_redu, &s_flag);
}

// Descriptors of the off-diagonal copy's tiles (same row ranges, entry ranges from rrp).
__global__ void k_tile_desc(const long long* __restrict__ rp, const int* __restrict__ tile_row,
                            int ntiles, TileDesc* desc) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        const int r0 = tile_row[t], r1 = tile_row[t + 1];
        desc[t] = TileDesc{rp[r0], rp[r1], r0, r1};
    }
}

// ---------------------------------------------------------------- SELL-32-sigma SpMV
// Short-row matrices (mean row <= SELL_MAX_MEAN entries) are re-laid out at upload as
// SELL-C-sigma with C = 32, sigma = 256: inside each window of 256 rows the rows are ordered by
// length (descending, stable), every slice of 32 consecutive ordered rows is stored
// column-major ([k][lane], padded to the slice's longest row with col = -1), so at step k a
// warp loads 32 consecutive values (256 B) and columns (128 B) straight from HBM -- coalesced,
// no shared-memory staging. Lane l still owns one row and adds its entries in their original
// ascending column order, so the row sums stay bit-identical to scipy.
constexpr int SELL_C = 32;
constexpr int SELL_W = 256;              // rows per window = threads per CTA
constexpr int SELL_SLICES = SELL_W / SELL_C;
constexpr int SELL_UNROLL = 8;           // entries in flight per lane
#ifndef MCR_SELL_CTA
#define MCR_SELL_CTA 256
#endif
constexpr int SELL_CTA = MCR_SELL_CTA;   // threads per SpMV CTA: slices of similar width
constexpr int SELL_MAX_MEAN = 32;

struct Sell {
    const long long* sptr;   // [nslices + 1] slot offset of each slice
    const int* perm;         // [nwin * 256] original row of each slot row (-1 = padding)
    const int* col;          // [slots] column, -1 for padding
    const double* val;       // [slots]
    int nwin;
};

template <int EPI>
__global__ void __launch_bounds__(SELL_CTA) k_sell(Sell A, const double* __restrict__ x, Vecs V,
                                                   SolveState* st) {
    __shared__ double s_red[SELL_CTA / 32];
    __shared__ unsigned long long s_redu[SELL_CTA / 32];
    __shared__ int s_flag;
    griddep_wait();
    griddep_launch();
    if constexpr (epi_checks_stop<EPI>()) {
        if (st->stop) return;
    }
    const double* xin = jacobi_select<EPI>(x, V, st);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int slice = blockIdx.x * (SELL_CTA / 32) + warp;
    const long long b0 = __ldg(A.sptr + slice);
    const int width = (int)((__ldg(A.sptr + slice + 1) - b0) / SELL_C);
    const int row = __ldg(A.perm + slice * SELL_C + lane);
    EpiIn in{0.0, 0.0, 0.0};
    if (row >= 0) in = epi_load<EPI>(V, row);
    const int* cp = A.col + b0 + lane;
    const double* vp = A.val + b0 + lane;
    double acc = 0.0;
    for (int k0 = 0; k0 < width; k0 += SELL_UNROLL) {
        int c[SELL_UNROLL];
        double v[SELL_UNROLL], xv[SELL_UNROLL];
#pragma unroll
        for (int u = 0; u < SELL_UNROLL; ++u) {
            const bool ok = k0 + u < width;
            c[u] = ok ? __ldcs(cp + (size_t)(k0 + u) * SELL_C) : -1;
            v[u] = ok ? __ldcs(vp + (size_t)(k0 + u) * SELL_C) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < SELL_UNROLL; ++u) xv[u] = c[u] >= 0 ? __ldg(xin + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < SELL_UNROLL; ++u)
            if (c[u] >= 0) acc = dadd(acc, dmul(v[u], xv[u]));
    }
    double p1 = 0.0, p2 = 0.0;
    unsigned long long mb = 0;
    if (row >= 0) epi_store<EPI>(V, row, acc, in, p1, p2, mb);
    if constexpr (epi_has_dot<EPI>()) {
        p1 = group_sum<SELL_CTA / 32, 0>(p1, s_red);
        if (threadIdx.x == 0) V.P1[blockIdx.x] = p1;
        if constexpr (EPI == EPI_T) {
            p2 = group_sum<SELL_CTA / 32, 0>(p2, s_red);
            if (threadIdx.x == 0) V.P2[blockIdx.x] = p2;
        }
    }
    kernel_finish<SELL_CTA, EPI>(V, st, gridDim.x, mb, s_red, s_redu, &s_flag);
}

// SELL build 1/2: per window, order rows by (length desc, index asc); record each slice's
// width (its first row's length). `offdiag` drops the stored diagonal (Jacobi's R).
__global__ void __launch_bounds__(SELL_W) k_sell_rank(const long long* __restrict__ rp,
                                                      const long long* __restrict__ offlen,
                                                      int n, int offdiag, int* perm,
                                                      long long* swidth) {
    __shared__ int lens[SELL_W];
    const int i = blockIdx.x * SELL_W + threadIdx.x;
    const int len = i < n ? (int)(offdiag ? offlen[i] : rp[i + 1] - rp[i]) : -1;
    lens[threadIdx.x] = len;
    __syncthreads();
    int rank = 0;
    for (int j = 0; j < SELL_W; ++j) {
        const int lj = lens[j];
        rank += (lj > len) || (lj == len && j < (int)threadIdx.x);
    }
    perm[blockIdx.x * SELL_W + rank] = i < n ? i : -1;
    __syncthreads();
    lens[rank] = len;  // lengths in slot order
    __syncthreads();
    if (threadIdx.x < SELL_SLICES) {
        int l = 0;
        for (int k = 0; k < SELL_C; ++k) l = max(l, lens[threadIdx.x * SELL_C + k]);
        swidth[blockIdx.x * SELL_SLICES + threadIdx.x] = (long long)l * SELL_C;
    }
}

// SELL build 2/2: one thread per slot row copies its row's entries (optionally skipping the
// diagonal) into the slice, column-major, padding with col = -1.
__global__ void k_sell_fill(const long long* __restrict__ rp, const int* __restrict__ col,
                            const double* __restrict__ val, const long long* __restrict__ sptr,
                            const int* __restrict__ perm, int nslots_rows, int offdiag,
                            int* scol, double* sval) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nslots_rows) return;
    const int slice = r / SELL_C, lane = r % SELL_C;
    const long long b0 = sptr[slice];
    const int width = (int)((sptr[slice + 1] - b0) / SELL_C);
    const int row = perm[r];
    long long k = row >= 0 ? rp[row] : 0;
    const long long e = row >= 0 ? rp[row + 1] : 0;
    for (int j = 0; j < width; ++j) {
        if (offdiag)
            while (k < e && col[k] == row) ++k;
        const size_t slot = (size_t)b0 + (size_t)j * SELL_C + lane;
        if (k < e) {
            scol[slot] = col[k];
            sval[slot] = val[k];
            ++k;
        } else {
            scol[slot] = -1;
            sval[slot] = 0.0;
        }
    }
}

}  // namespace mcr
