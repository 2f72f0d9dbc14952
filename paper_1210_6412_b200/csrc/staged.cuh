// staged.cuh -- band-staged SpMV for systems whose x is far larger than L2 (part of device.cuh).
//
// A CSR SpMV over a matrix with uniformly random columns gathers x at random. Once x no longer
// fits in L2 (C5: 1.6 GB of x against 126 MB of L2) every gather is a random HBM access, and
// HBM serves only ~40 G of those per second. The staged layout splits the SpMV in two passes
// whose memory traffic is all sequential or L2-resident:
//
//   pass 1 (k_stage_products): the entries are stored in (column band, row tile, CSR order)
//       order; band b covers columns [b*band, (b+1)*band), sized so the band's slice of x
//       stays in L2. The whole grid walks the entries in storage order, so at any moment it
//       gathers from one L2-resident band, and writes the product a_ij * x_j of every entry
//       to a product array in the same order (coalesced streams in and out).
//   pass 2 (k_spmv_staged): for each row tile, the tile's products sit in one contiguous
//       segment per band; the producer warp copies those segments into shared memory with TMA
//       bulk copies (one per band), plus the tile's row pointers and a 2-byte local index per
//       entry (CSR order -> position in the staged products). Consumers then add each row's
//       products in CSR order straight from shared memory and run the usual epilogue.
//
// Exactness: the product of each entry is the same __dmul_rn as in k_spmv, and every row sum
// adds its products from +0.0 in ascending column order (CSR order) with __dadd_rn, so both
// passes together are bit-identical to k_spmv and to scipy. Jacobi's off-diagonal sum skips
// the stored diagonal, flagged in bit 15 of its local index (the kept terms keep their order,
// as in without_diagonal, sparse.py:227-231), so one staged copy serves every epilogue.
//
// Segments are padded to an even number of entries (16-byte aligned bulk copies); a padding
// slot holds value 0 and a column inside its band and is never referenced by a local index.
#pragma once

#include "common.cuh"

namespace mcr {

constexpr int STG_NB_MAX = 128;                 // bands per system (segments per tile)
constexpr int STG_CAP = TILE_NNZ + STG_NB_MAX;  // staged products per tile, padding included
constexpr unsigned short STG_DIAG = 0x8000;     // local-index flag: stored diagonal entry
constexpr int STG_P1_NT = 256;                  // pass-1 threads per CTA
constexpr int STG_BUILD_WARPS = 8;              // build kernels: one warp per tile

// seg[t * nb + b] = (P offset of tile t's band-b segment) << 32 | (its offset inside the
// tile's staged block) << 16 | (padded entry count)
__host__ __device__ inline unsigned long long seg_pack(long long off, int loff, int cnt) {
    return ((unsigned long long)off << 32) | ((unsigned long long)(unsigned)loff << 16) |
           (unsigned long long)(unsigned)cnt;
}

struct Staged {
    const long long* rp;         // CSR row starts (the full matrix)
    const unsigned short* lidx;  // [nnz] local index of each CSR entry (| STG_DIAG)
    const unsigned long long* seg;  // [ntiles * nb] segment table, tile-major
    const double* pval;          // [npos] values in staged order
    const int* pcol;             // [npos] columns in staged order
    double* prod;                // [npos] pass-1 products
    const TileDesc* desc;
    long long npos;              // even
    int ntiles, nb;
    int early;                   // bit 0 / 1: pass 1 / pass 2 lets its dependent launch at entry
};

struct alignas(16) StgStage {
    double prod[STG_CAP];
    unsigned short lidx[TILE_NNZ + 16];
    long long rp[TILE_ROWS + 4];
};
#ifndef MCR_STG_STAGES
#define MCR_STG_STAGES 2
#endif
constexpr int STG_STAGES = MCR_STG_STAGES;  // tiles in flight per pass-2 CTA
constexpr size_t STG_SMEM = sizeof(StgStage) * STG_STAGES;
constexpr int STG_DIAG_COL = (int)0x80000000;  // pcol flag: stored diagonal (Jacobi skips it)

// ---------------------------------------------------------------- pass 1
// prod[k] = pval[k] * x[pcol[k]] over the staged order. CTAs take chunks of STG_P1_CHUNK
// entries in storage order from a ticket counter (the next ticket is fetched while the current
// chunk is processed), so all chunks in flight lie within ~CTAs x chunk entries of each other
// and the gathers stay inside one or two L2-resident bands of x. (A grid-stride loop lets the
// CTAs drift apart over a long array until the gathers span all of x again: measured L2 hit
// rate 30%.) Matrix streams and products are evict-first so the band keeps its L2 lines.
constexpr int STG_P1_U = 4;                                 // double2 per thread per chunk
constexpr int STG_P1_CHUNK = 2 * STG_P1_U * STG_P1_NT;       // entries per ticket

// x_c for a staged entry; the stored diagonal (flagged) is not gathered by a Jacobi sweep,
// whose row sums skip it (its product slot is never read)
template <int EPI>
__device__ __forceinline__ double stage_gather(const double* __restrict__ xin, int c) {
    if constexpr (EPI == EPI_JACOBI) {
        if (c < 0) return 0.0;
    }
    return __ldg(xin + (c & 0x7fffffff));
}

template <int EPI>
__global__ void __launch_bounds__(STG_P1_NT) k_stage_products(Staged A, const double* x, Vecs V,
                                                              SolveState* st) {
    __shared__ long long s_ticket[2];
    griddep_wait();
    if (A.early & 1) griddep_launch();
    if constexpr (epi_checks_stop<EPI>()) {
        if (st->stop) return;
    }
    const double* __restrict__ xin = jacobi_select<EPI>(x, V, st);
    const int2* __restrict__ pc = reinterpret_cast<const int2*>(A.pcol);
    const double2* __restrict__ pv = reinterpret_cast<const double2*>(A.pval);
    double2* __restrict__ out = reinterpret_cast<double2*>(A.prod);
    const long long n2 = A.npos >> 1;
    const long long nchunks = (n2 + STG_P1_CHUNK / 2 - 1) / (STG_P1_CHUNK / 2);
    if (threadIdx.x == 0) s_ticket[0] = (long long)atomicAdd(&st->p1_ctr, 1ull);
    __syncthreads();
    for (int k = 0;; ++k) {
        const long long c = s_ticket[k & 1];
        if (c >= nchunks) break;
        if (threadIdx.x == 0) s_ticket[(k + 1) & 1] = (long long)atomicAdd(&st->p1_ctr, 1ull);
        const long long i0 = c * (STG_P1_CHUNK / 2) + threadIdx.x;
        if (i0 + (STG_P1_U - 1) * STG_P1_NT < n2) {
            int2 cc[STG_P1_U];
            double2 v[STG_P1_U], g[STG_P1_U];
#pragma unroll
            for (int u = 0; u < STG_P1_U; ++u) {
                cc[u] = __ldcs(pc + i0 + u * STG_P1_NT);
                v[u] = __ldcs(pv + i0 + u * STG_P1_NT);
            }
#pragma unroll
            for (int u = 0; u < STG_P1_U; ++u) {
                g[u].x = stage_gather<EPI>(xin, cc[u].x);
                g[u].y = stage_gather<EPI>(xin, cc[u].y);
            }
#pragma unroll
            for (int u = 0; u < STG_P1_U; ++u)
                __stcs(out + i0 + u * STG_P1_NT,
                       make_double2(dmul(v[u].x, g[u].x), dmul(v[u].y, g[u].y)));
        } else {
            for (long long i = i0; i < n2; i += STG_P1_NT) {
                const int2 c2 = __ldcs(pc + i);
                const double2 v2 = __ldcs(pv + i);
                __stcs(out + i, make_double2(dmul(v2.x, stage_gather<EPI>(xin, c2.x)),
                                             dmul(v2.y, stage_gather<EPI>(xin, c2.y))));
            }
        }
        __syncthreads();  // next ticket visible; this one's slot free for reuse
    }
    // the dependent pass 2 is let in only as this pass drains: its CTAs, resident early, would
    // hold SM slots the gathers need (measured: 16.7 vs 12.5 ms per C5 sweep)
    griddep_launch();
}

// ---------------------------------------------------------------- pass 2
// Persistent, warp-specialised like k_spmv: the producer warp fills a stage per tile (row
// pointers, local indices and the tile's product segments, all by cp.async.bulk on one
// mbarrier); consumer thread r sums tile row r from shared memory and runs the epilogue.
template <int EPI>
__global__ void __launch_bounds__(SP_THREADS, MCR_SP_MINB) k_spmv_staged(Staged A, Vecs V,
                                                                          SolveState* st) {
    extern __shared__ __align__(128) unsigned char stg_raw[];
    StgStage* stg = reinterpret_cast<StgStage*>(stg_raw);
    __shared__ __align__(8) uint64_t full_bar[STG_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[STG_STAGES];
    __shared__ TileDesc s_desc[STG_STAGES];
    __shared__ int s_tile[STG_STAGES];
    __shared__ double s_red[SP_THREADS / 32];
    __shared__ unsigned long long s_redu[SP_THREADS / 32];
    __shared__ int s_flag;
    griddep_wait();
    if (A.early & 2) griddep_launch();
    if constexpr (epi_checks_stop<EPI>()) {
        if (st->stop) return;
    }
    jacobi_select<EPI>(nullptr, V, st);  // xcur / xnext of this sweep
    if (blockIdx.x == 0 && threadIdx.x == 0) st->p1_ctr = 0;  // pass 1 has completed
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STG_STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], SP_CONSUMERS / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    unsigned long long mb = 0;
    const int G = gridDim.x;
    double acc1 = 0.0, acc2 = 0.0;

    if (warp == SP_CONSUMERS / 32) {
        // ------------------------------------------------------------ producer warp
        // the next tile's descriptor and segment table are loaded before waiting for a free
        // stage, so their HBM latency overlaps the consumers' work
        const int nb = A.nb;
        int t = blockIdx.x;
        TileDesc dn{};
        unsigned long long sn[STG_NB_MAX / 32];
        auto fetch = [&](int tt) {
            if (tt < A.ntiles) dn = A.desc[tt];
#pragma unroll
            for (int j = 0; j < STG_NB_MAX / 32; ++j) {
                const int b = lane + 32 * j;
                sn[j] = (tt < A.ntiles && b < nb) ? __ldg(A.seg + (size_t)tt * nb + b) : 0ull;
            }
        };
        fetch(t);
        for (int i = 0;; ++i, t += G) {
            const int s = i % STG_STAGES;
            const TileDesc d = dn;
            unsigned long long sg[STG_NB_MAX / 32];
#pragma unroll
            for (int j = 0; j < STG_NB_MAX / 32; ++j) sg[j] = sn[j];
            if (t < A.ntiles) fetch(t + G);
            if (i >= STG_STAGES) mbar_wait(&empty_bar[s], (uint32_t)(((i / STG_STAGES) + 1) & 1));
            if (t >= A.ntiles) {
                if (lane == 0) {
                    s_tile[s] = -1;
                    mbar_arrive(&full_bar[s]);
                }
                break;
            }
            uint32_t bytes = 0;
#pragma unroll
            for (int j = 0; j < STG_NB_MAX / 32; ++j) bytes += (uint32_t)(sg[j] & 0xffffu) * 8u;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, off);
            if (lane == 0) {
                s_tile[s] = t;
                s_desc[s] = d;
                const long long ra = d.r0 & ~1ll, lb0 = d.e0 & ~7ll;
                const uint32_t rb = (uint32_t)(((d.r1 + 1 - ra) * 8 + 15) & ~15ll);
                const uint32_t lb = d.e1 > d.e0 ? (uint32_t)(((d.e1 - lb0) * 2 + 15) & ~15ll) : 0u;
                mbar_expect_tx(&full_bar[s], rb + lb + bytes);
                bulk_g2s(stg[s].rp, A.rp + ra, rb, &full_bar[s]);
                if (lb) bulk_g2s(stg[s].lidx, A.lidx + lb0, lb, &full_bar[s]);
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < STG_NB_MAX / 32; ++j) {
                const uint32_t cnt = (uint32_t)(sg[j] & 0xffffu);
                if (cnt) {
                    const int loff = (int)((sg[j] >> 16) & 0xffffu);
                    const long long off = (long long)(sg[j] >> 32);
                    bulk_g2s(stg[s].prod + loff, A.prod + off, cnt * 8u, &full_bar[s]);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ consumer warps
        for (int i = 0;; ++i) {
            const int s = i % STG_STAGES;
            mbar_wait(&full_bar[s], (uint32_t)((i / STG_STAGES) & 1));
            TileDesc d;
            const int t = stage_tile(s_tile, s_desc, s, d);
            if (t < 0) break;
            const int nrows = d.r1 - d.r0;
            const int row = d.r0 + tid;
            EpiIn in{0.0, 0.0, 0.0};
            if (tid < nrows) in = epi_load<EPI>(V, row);
            const StgStage& S = stg[s];
            double acc = 0.0;
            if (tid < nrows) {
                const long long lb0 = d.e0 & ~7ll;
                const int ro = d.r0 & 1;
                int k = (int)(S.rp[ro + tid] - lb0);
                const int e = (int)(S.rp[ro + tid + 1] - lb0);
                double a = 0.0;
                for (; k < e; ++k) {
                    const unsigned li = S.lidx[k];
                    if constexpr (EPI == EPI_JACOBI) {
                        if (li & STG_DIAG) continue;  // R = M without its diagonal
                    }
                    a = dadd(a, S.prod[li & 0x7fffu]);
                }
                acc = a;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);
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
    if constexpr (EPI == EPI_JACOBI) {
        if (V.peers) __threadfence_system();
    }
    griddep_launch();  // late, as in pass 1
    kernel_finish<SP_THREADS, EPI, true>(V, st, G, mb, s_red, s_redu, &s_flag);
}

// ---------------------------------------------------------------- build
// 1/2: padded entry count of every (band, tile) segment, band-major (the scan order).
__global__ void __launch_bounds__(STG_BUILD_WARPS * 32) k_stage_count(
    const int* __restrict__ col, const TileDesc* __restrict__ desc, int ntiles, int band, int nb,
    long long* counts) {
    __shared__ int hist[STG_BUILD_WARPS][STG_NB_MAX];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * STG_BUILD_WARPS + w;
    for (int b = lane; b < STG_NB_MAX; b += 32) hist[w][b] = 0;
    __syncwarp();
    if (t >= ntiles) return;
    const TileDesc d = desc[t];
    for (long long e = d.e0 + lane; e < d.e1; e += 32) atomicAdd(&hist[w][col[e] / band], 1);
    __syncwarp();
    for (int b = lane; b < nb; b += 32) counts[(size_t)b * ntiles + t] = (hist[w][b] + 1) & ~1;
}

// 2/2: place every entry. Within a (band, tile) segment entries keep CSR order (a warp walks
// the tile 32 entries at a time; lanes of the same band are ranked with __match_any_sync).
__global__ void __launch_bounds__(STG_BUILD_WARPS * 32) k_stage_fill(
    const long long* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
    const TileDesc* __restrict__ desc, int ntiles, int band, int nb, long long roff,
    const long long* __restrict__ offs, double* pval, int* pcol, unsigned short* lidx,
    unsigned long long* seg) {
    __shared__ int run[STG_BUILD_WARPS][STG_NB_MAX];
    __shared__ int loc[STG_BUILD_WARPS][STG_NB_MAX];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * STG_BUILD_WARPS + w;
    if (t >= ntiles) return;
    const TileDesc d = desc[t];
    if (lane == 0) {
        int acc = 0;
        for (int b = 0; b < nb; ++b) {
            const size_t k = (size_t)b * ntiles + t;
            const int cnt = (int)(offs[k + 1] - offs[k]);
            loc[w][b] = acc;
            run[w][b] = 0;
            seg[(size_t)t * nb + b] = seg_pack(offs[k], acc, cnt);
            acc += cnt;
        }
    }
    __syncwarp();
    for (long long e0 = d.e0; e0 < d.e1; e0 += 32) {
        const long long e = e0 + lane;
        const bool act = e < d.e1;
        const unsigned amask = __ballot_sync(0xffffffffu, act);
        if (act) {
            const int c = col[e];
            const int b = c / band;
            const unsigned peers = __match_any_sync(amask, b);
            const int rank = run[w][b] + __popc(peers & ((1u << lane) - 1u));
            // row of entry e: last row r of the tile with rp[r] <= e
            int lo = d.r0, hi = d.r1 - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (rp[mid] <= e) lo = mid; else hi = mid - 1;
            }
            const long long pos = offs[(size_t)b * ntiles + t] + rank;
            const bool diag = (long long)c == roff + lo;
            pval[pos] = val[e];
            pcol[pos] = diag ? (c | STG_DIAG_COL) : c;
            lidx[e] = (unsigned short)(loc[w][b] + rank) | (diag ? STG_DIAG : (unsigned short)0);
            __syncwarp(amask);
            if (lane == __ffs(peers) - 1) run[w][b] += __popc(peers);
        }
        __syncwarp();
    }
    // padding slot of every odd segment
    for (int b = lane; b < nb; b += 32) {
        const size_t k = (size_t)b * ntiles + t;
        const int cnt = (int)(offs[k + 1] - offs[k]);
        if (cnt > run[w][b]) {
            pval[offs[k] + cnt - 1] = 0.0;
            pcol[offs[k] + cnt - 1] = b * band;
        }
    }
}

}  // namespace mcr
