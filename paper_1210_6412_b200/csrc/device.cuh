// device.cuh -- sm_100a kernels of the reachability solver.
//
// Arithmetic contract: every row sum of M x is accumulated from +0.0
// in ascending column order with separately rounded products and sums (no FMA), so SpMV,
// the Jacobi sweep and the residual are bit-identical to scipy's csr_matvec + numpy as used by
// the reference (sparse.py:191, solvers.py:219-225). Element-wise BiCGStab updates use the
// exact evaluation order of the reference's numpy expressions (solvers.py:298-305). Inner
// products are either deterministic fixed-shape trees (per-tile block trees, then a
// fixed-order reduction over tiles; default) or the reference's own strictly sequential
// order (k_seqdot, bit-exact, slow).
//
// Storage (HBM):
//   CSR:   rowptr int64[n+1], col int32[nnz], val f64[nnz] (each padded by 16 B so 16-byte
//          aligned bulk copies may round up); rows cut into tiles of at most TILE_ROWS rows
//          and TILE_NNZ entries (a longer single row is a tile of its own).
//   Dense: slab layout, slab s holds rows 32s..32s+31 as [col j][row r] (256 B per column),
//          so one warp streams a contiguous slab with TMA bulk copies and every thread keeps
//          its row's strictly sequential sum.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mcr {

#ifndef MCR_TILE_NNZ
#define MCR_TILE_NNZ 2048
#endif
constexpr int TILE_ROWS = 256;   // rows per tile = consumer threads per SpMV CTA
constexpr int TILE_NNZ = MCR_TILE_NNZ;  // entries staged in shared memory per tile
constexpr int SP_CONSUMERS = TILE_ROWS;
constexpr int SP_THREADS = SP_CONSUMERS + 32;  // + one producer warp
#ifndef MCR_SP_STAGES
#define MCR_SP_STAGES 2
#endif
constexpr int SP_STAGES = MCR_SP_STAGES;  // tiles in flight per CTA
constexpr int CHUNK_NT = 256;    // threads per element-wise CTA
constexpr int CHUNK_PER = 4;     // rows per thread
constexpr int CHUNK_ROWS = CHUNK_NT * CHUNK_PER;
constexpr int DSLAB = 32;        // dense rows per slab (one warp)
constexpr int DCOLS = 64;        // dense columns per pipeline stage (16 KB)
constexpr int DSTAGES = 3;       // dense TMA pipeline depth
constexpr size_t DENSE_SMEM = sizeof(double) * DSTAGES * DCOLS * DSLAB;
constexpr int CSR_PAD = 4;       // extra elements allocated behind rowptr / col / val

constexpr double TINY = 1e-300;  // solvers.py:40

enum Stop : int { RUNNING = 0, CONVERGED = 1, NOTCONV = 2, BREAKDOWN = 3 };
constexpr int SEND_SLOTS = 4;    // doubles each rank contributes per reduction point

// Device-resident solver state: all control flow of a solve lives here, so an iteration never
// needs the host. Written only by the "last CTA" of a kernel (after every other CTA of that
// kernel has published its partials) and read by the next kernel.
struct SolveState {
    int stop;
    int which;
    long long it;        // completed sweeps / iterations
    long long bd_it;
    long long max_it;
    double tol;
    unsigned long long maxbits;  // atomicMax of |.| bit patterns (non-negative doubles order as u64)
    unsigned int done;           // last-CTA counter
    unsigned int tile_ctr;       // dynamic tile scheduler of k_spmv
    double y, a, w, beta, qv, tt, ts, resid;
    int small;
    int seqdots;  // 1: inner products by k_seqdot (reference order, bit-exact), not the tree
    int sharded;  // 1: row shard of a multi-GPU system -- reduction kernels publish their local
                  //    partials in send[] instead of finalising; k_finalize finishes after the
                  //    per-rank exchange
    double send[SEND_SLOTS];  // {dot 1, dot 2, max|.| as bits, unused} of this rank
};

// Entry range [e0, e1) and row range [r0, r1) of one tile.
struct TileDesc {
    long long e0, e1;
    int r0, r1;
};

struct Csr {
    const long long* rp;
    const int* col;
    const double* val;
    const TileDesc* desc;
    int ntiles;
    int n;
};

// Pointers an epilogue may touch. Unused ones are null.
struct Vecs {
    const double* b;
    const double* d;
    const double* xcur;  // Jacobi: iterate read by this sweep
    double* xnext;       // Jacobi: iterate written by this sweep
    double* y;           // plain SpMV output
    double* x;
    double* r;
    double* q;
    double* p;
    double* v;
    double* s;
    double* t;
    double* P1;          // per-unit partials
    double* P2;
    double* x_jac0;      // Jacobi double buffer (for sweep parity); full length when sharded
    double* x_jac1;
    long long roff;      // first global row of this shard (0 on one GPU): own slice of x_jac*
    // Fused exchange (row shards in peer-to-peer mode): peers[slot * world + q] is rank q's
    // copy of full vector `slot` (FV_X, FV_X1, FV_P, FV_S), mapped into this device's address
    // space; the producer of an own-row value also stores it into every peer's copy, so the
    // "allgather" rides NVLink while the kernel computes. Null when not in that mode.
    double* const* peers;
    int world, rank;
    int xnext_slot;      // FV_X / FV_X1: which Jacobi buffer this sweep writes (set per launch)
};
enum FullVec : int { FV_X = 0, FV_X1 = 1, FV_P = 2, FV_S = 3 };

// Store an own-row value of full vector `slot` (global index g) into every peer's copy.
__device__ __forceinline__ void peer_store(const Vecs& V, int slot, long long g, double v) {
    if (!V.peers) return;
    for (int q = 0; q < V.world; ++q)
        if (q != V.rank) V.peers[slot * V.world + q][g] = v;
}

enum Epi : int { EPI_Y = 0, EPI_RESID = 1, EPI_JACOBI = 2, EPI_S0 = 3, EPI_V = 4, EPI_T = 5 };
enum Phase : int { PH_A = 0, PH_C = 1, PH_E = 2 };

template <int EPI> __host__ __device__ constexpr bool epi_checks_stop() { return EPI != EPI_Y && EPI != EPI_RESID; }
template <int EPI> __host__ __device__ constexpr bool epi_has_max() {
    return EPI == EPI_RESID || EPI == EPI_JACOBI || EPI == EPI_S0;
}
template <int EPI> __host__ __device__ constexpr bool epi_has_dot() {
    return EPI == EPI_S0 || EPI == EPI_V || EPI == EPI_T;
}

// ---------------------------------------------------------------- scalar helpers
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ unsigned long long absbits(double v) {
    return (unsigned long long)__double_as_longlong(fabs(v));
}
__device__ __forceinline__ double bits2d(unsigned long long b) {
    return __longlong_as_double((long long)b);
}
__device__ __forceinline__ unsigned long long umax(unsigned long long a, unsigned long long b) {
    return a > b ? a : b;
}
__device__ __forceinline__ bool tiny(double v) { return v == 0.0 || fabs(v) < TINY; }
// Ordered loads (asm volatile keeps their issue order): streaming vector loads first, then the
// solver state, so the state's L2 round trip overlaps the stream instead of gating it.
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_state(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_state(const int* p) {
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// ---------------------------------------------------------------- mbarrier / bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// 1-D TMA bulk copy global -> shared, completion counted in bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Programmatic dependent launch: solve kernels are launched with the PDL attribute, so the
// next kernel's CTAs can be scheduled while this grid drains; griddep_wait() blocks until the
// previous grid has completed and its writes are visible, griddep_launch() lets the next one
// start launching. Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Named barrier among the first `count` threads (count multiple of 32).
__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---------------------------------------------------------------- group reductions
// Fixed-shape trees: the same inputs in the same slots always give the same bits.
// NW warps participate (threads 0 .. 32*NW-1); BAR 0 = whole-CTA __syncthreads, else a named
// barrier over the NW warps. Result valid in thread 0.
template <int NW, int BAR>
__device__ __forceinline__ void group_sync() {
    if constexpr (BAR == 0) __syncthreads();
    else named_sync(BAR, NW * 32);
}

template <int NW, int BAR>
__device__ __forceinline__ double group_sum(double v, double* s_red) {
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = dadd(v, __shfl_down_sync(full, v, off));
    if constexpr (NW > 1) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) s_red[warp] = v;
        group_sync<NW, BAR>();
        if (warp == 0) {
            v = lane < NW ? s_red[lane] : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v = dadd(v, __shfl_down_sync(full, v, off));
        }
        group_sync<NW, BAR>();
    }
    return v;
}

template <int NW, int BAR>
__device__ __forceinline__ unsigned long long group_max(unsigned long long v,
                                                        unsigned long long* s_red) {
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = umax(v, __shfl_down_sync(full, v, off));
    if constexpr (NW > 1) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) s_red[warp] = v;
        group_sync<NW, BAR>();
        if (warp == 0) {
            v = lane < NW ? s_red[lane] : 0ull;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v = umax(v, __shfl_down_sync(full, v, off));
        }
        group_sync<NW, BAR>();
    }
    return v;
}

// Fixed-order reduction of count partials by one CTA: thread t sums slots t, t+NT, ...
// sequentially, then a CTA tree. Partials were written by other CTAs: read through L2.
template <int NT>
__device__ double reduce_partials(const double* P, int count, double* s_red) {
    double acc = 0.0;
    for (int k = threadIdx.x; k < count; k += NT) acc = dadd(acc, __ldcg(P + k));
    return group_sum<NT / 32, 0>(acc, s_red);
}

// "Last CTA" detection: every CTA publishes its writes, then bumps a counter; the CTA that
// sees gridDim-1 runs the kernel's finalisation with all partials visible.
__device__ __forceinline__ bool last_cta(unsigned int* ctr, int* s_flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned prev = atomicAdd(ctr, 1u);
        *s_flag = (prev == gridDim.x - 1);
    }
    __syncthreads();
    const bool last = *s_flag != 0;
    if (last) __threadfence();
    return last;
}

// ---------------------------------------------------------------- BiCGStab scalar steps
// y_prev = y; y = q.r; breakdown on y_prev*w; beta = (y*a)/(y_prev*w) (solvers.py:462-467).
__device__ __forceinline__ void bicg_prepare(SolveState* st, double qr, long long next_it) {
    const double y_prev = st->y;
    const double denom = dmul(y_prev, st->w);
    st->y = qr;
    if (tiny(denom)) {
        st->stop = BREAKDOWN;
        st->which = 1;
        st->bd_it = next_it;
        return;
    }
    st->beta = ddiv(dmul(qr, st->a), denom);
}

// Finalisation of each BiCGStab reduction point (thread 0 of one CTA). Shared by the tree
// path (last CTA of the producing kernel) and the sequential path (k_seqdot).
__device__ __forceinline__ void fin_s0(SolveState* st, double qr) {
    const double mr = bits2d(atomicExch(&st->maxbits, 0ull));
    st->it = 0;
    if (mr <= st->tol) {                            // solvers.py:453-454
        st->stop = CONVERGED;
    } else {
        st->y = 1.0; st->a = 1.0; st->w = 1.0;      // solvers.py:456
        bicg_prepare(st, qr, 1);
    }
}
__device__ __forceinline__ void fin_v(SolveState* st, double qv) {
    st->qv = qv;
    if (tiny(qv)) {                                 // solvers.py:470-472
        st->stop = BREAKDOWN; st->which = 2; st->bd_it = st->it + 1;
    } else {
        st->a = ddiv(st->y, qv);                    // solvers.py:473
    }
}
__device__ __forceinline__ void fin_t(SolveState* st, double tt, double ts) {
    const double ms = bits2d(atomicExch(&st->maxbits, 0ull));
    const int small = ms <= st->tol;                // solvers.py:476
    st->small = small;
    st->tt = tt;
    st->ts = ts;
    if (tiny(tt)) {                                 // solvers.py:478-483
        if (!small) { st->stop = BREAKDOWN; st->which = 3; st->bd_it = st->it + 1; }
        else st->w = 0.0;
    } else {
        st->w = ddiv(ts, tt);                       // solvers.py:485
    }
}
__device__ __forceinline__ void fin_e(SolveState* st, double qr) {
    const long long it = st->it + 1;                // solvers.py:486-490
    st->it = it;
    if (st->small) st->stop = CONVERGED;
    else if (it >= st->max_it) st->stop = NOTCONV;
    else bicg_prepare(st, qr, it + 1);
}

// ---------------------------------------------------------------- row epilogues
// Operands of a row's epilogue, loaded before the row sum is known so their latency hides
// behind the gather.
struct EpiIn {
    double a, b, c;
};

template <int EPI>
__device__ __forceinline__ EpiIn epi_load(const Vecs& V, int row) {
    EpiIn in{0.0, 0.0, 0.0};
    if constexpr (EPI == EPI_RESID || EPI == EPI_S0) {
        in.a = __ldg(V.b + row);
    } else if constexpr (EPI == EPI_JACOBI) {
        in.a = __ldg(V.b + row);
        in.b = __ldg(V.d + row);
        in.c = V.xcur[row];
    } else if constexpr (EPI == EPI_V) {
        in.a = V.q[row];
    } else if constexpr (EPI == EPI_T) {
        in.a = V.s[row];
    }
    return in;
}

// Per-row work after the row sum s; p1/p2 feed the unit's dot partials, mb the running max.
template <int EPI>
__device__ __forceinline__ void epi_store(const Vecs& V, int row, double s, const EpiIn& in,
                                          double& p1, double& p2, unsigned long long& mb) {
    if constexpr (EPI == EPI_Y) {
        V.y[row] = s;
    } else if constexpr (EPI == EPI_RESID) {
        mb = umax(mb, absbits(dsub(in.a, s)));                // |b - M x|
    } else if constexpr (EPI == EPI_JACOBI) {
        const double xn = ddiv(dsub(in.a, s), in.b);          // (b - R x) / d
        V.xnext[row] = xn;
        peer_store(V, V.xnext_slot, V.roff + row, xn);
        mb = umax(mb, absbits(dsub(xn, in.c)));               // |x' - x|
    } else if constexpr (EPI == EPI_S0) {
        const double r = dsub(in.a, dmul(1.0, s));            // r = b - 1.0 * (M x)
        V.r[row] = r;
        V.q[row] = r;
        V.p[row] = 0.0;
        V.v[row] = 0.0;
        mb = umax(mb, absbits(r));
        p1 = dmul(r, r);                                      // q . r with q = r
    } else if constexpr (EPI == EPI_V) {
        V.v[row] = s;                                         // v = M p
        p1 = dmul(in.a, s);                                   // q . v
    } else if constexpr (EPI == EPI_T) {
        V.t[row] = s;                                         // t = M s
        p1 = dmul(s, s);                                      // t . t
        p2 = dmul(s, in.a);                                   // t . s
    }
}

// End of an SpMV-family kernel (all NT threads): fold the running max into the state, then
// the last CTA finalises the kernel's scalars from the per-unit partials.
template <int NT, int EPI, bool PERSISTENT = false>
__device__ __forceinline__ void kernel_finish(const Vecs& V, SolveState* st, int nunits,
                                              unsigned long long mb, double* s_red,
                                              unsigned long long* s_redu, int* s_flag) {
    if constexpr (epi_has_max<EPI>()) {
        mb = group_max<NT / 32, 0>(mb, s_redu);
        if (threadIdx.x == 0 && mb) atomicMax(&st->maxbits, mb);
    }
    if constexpr (EPI == EPI_Y && !PERSISTENT) return;  // nothing to finalise
    if (!last_cta(&st->done, s_flag)) return;
    if (st->sharded) {  // publish this rank's partials; k_finalize runs after the exchange
        double r1 = 0.0, r2 = 0.0;
        if constexpr (epi_has_dot<EPI>()) r1 = reduce_partials<NT>(V.P1, nunits, s_red);
        if constexpr (EPI == EPI_T) r2 = reduce_partials<NT>(V.P2, nunits, s_red);
        if (threadIdx.x == 0) {
            st->send[0] = r1;
            st->send[1] = r2;
            st->send[2] = bits2d(atomicExch(&st->maxbits, 0ull));
            st->send[3] = 0.0;
            st->done = 0;
            st->tile_ctr = 0;
        }
        return;
    }
    if constexpr (epi_has_dot<EPI>()) {
        if (st->seqdots) {  // k_seqdot runs the reference-order dots and finalises
            if (threadIdx.x == 0) { st->done = 0; st->tile_ctr = 0; }
            return;
        }
    }
    double r1 = 0.0, r2 = 0.0;
    if constexpr (epi_has_dot<EPI>()) r1 = reduce_partials<NT>(V.P1, nunits, s_red);
    if constexpr (EPI == EPI_T) r2 = reduce_partials<NT>(V.P2, nunits, s_red);
    if (threadIdx.x != 0) return;
    st->done = 0;
    st->tile_ctr = 0;
    if constexpr (EPI == EPI_RESID) {
        st->resid = bits2d(atomicExch(&st->maxbits, 0ull));
    } else if constexpr (EPI == EPI_JACOBI) {
        const double md = bits2d(atomicExch(&st->maxbits, 0ull));
        const long long it = st->it + 1;
        st->it = it;
        if (md <= st->tol) st->stop = CONVERGED;       // NaN compares false: keep going
        else if (it >= st->max_it) st->stop = NOTCONV;
    } else if constexpr (EPI == EPI_S0) {
        fin_s0(st, r1);
    } else if constexpr (EPI == EPI_V) {
        fin_v(st, r1);
    } else if constexpr (EPI == EPI_T) {
        fin_t(st, r1, r2);
    }
}

template <int EPI>
__device__ __forceinline__ const double* jacobi_select(const double* x, Vecs& V, SolveState* st) {
    if constexpr (EPI == EPI_JACOBI) {
        const long long it = st->it + 1;  // sweep it reads buffer (it+1)&1, writes it&1
        const double* cur = (it & 1) ? V.x_jac0 : V.x_jac1;
        V.xcur = cur + V.roff;          // own rows (the whole vector on one GPU)
        V.xnext = ((it & 1) ? V.x_jac1 : V.x_jac0) + V.roff;
        V.xnext_slot = (it & 1) ? FV_X1 : FV_X;
        return cur;                     // gathers read the full (allgathered) iterate
    }
    return x;
}

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
    griddep_wait();
    griddep_launch();
    if constexpr (epi_checks_stop<EPI>()) {
        if (st->stop) return;
    }
    const double* xin = jacobi_select<EPI>(x, V, st);
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
            int t = blockIdx.x;
            TileDesc dn{};
            if (t < A.ntiles) dn = A.desc[t];
            for (int i = 0;; ++i, t += G) {
                const int s = i % SP_STAGES;
                const TileDesc d = dn;
                if (t + G < A.ntiles) dn = A.desc[t + G];  // prefetch the next descriptor
                if (i >= SP_STAGES) mbar_wait(&empty_bar[s], (uint32_t)(((i / SP_STAGES) + 1) & 1));
                if (t >= A.ntiles) {
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
                bulk_g2s(stg[s].rp, A.rp + ra, rb, &full_bar[s]);
                if (vb) {
                    bulk_g2s(stg[s].val, A.val + base, vb, &full_bar[s]);
                    bulk_g2s(stg[s].col, A.col + base, cb, &full_bar[s]);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ consumer warps
        for (int i = 0;; ++i) {
            const int s = i % SP_STAGES;
            mbar_wait(&full_bar[s], (uint32_t)((i / SP_STAGES) & 1));
            const int t = s_tile[s];
            if (t < 0) break;
            const TileDesc d = s_desc[s];
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

// ---------------------------------------------------------------- persistent small-system solvers
// For systems whose tiles all fit on the GPU at once (ntiles <= co-resident CTAs, e.g. C1 and
// the Table-1 shapes) one cooperative kernel runs the whole solve: sweeps / iterations are
// separated by grid barriers instead of kernel launches, and every CTA reduces the per-tile
// partials itself in the same fixed order, so all CTAs hold bit-identical scalars without a
// round trip through global state.
namespace cg = cooperative_groups;
constexpr int SM_NT = TILE_ROWS;

struct SmallSmem {
    double val[TILE_NNZ];      // this CTA's tile, loaded once per solve
    int col[TILE_NNZ];
    double prod[TILE_NNZ];
    int rp[TILE_ROWS + 1];
    double red[SM_NT / 32];
    unsigned long long redu[SM_NT / 32];
    long long e0, e1;
    int nrows, r0, cached;
};

// One tile per CTA (grid == ntiles): its row pointers, columns and values move to shared
// memory once per solve; a single row longer than a tile stays in HBM and is streamed.
__device__ __forceinline__ void load_tile(const Csr& A, int t, SmallSmem& sm) {
    if (threadIdx.x == 0) {
        const TileDesc d = A.desc[t];
        sm.e0 = d.e0;
        sm.e1 = d.e1;
        sm.nrows = d.r1 - d.r0;
        sm.r0 = d.r0;
        sm.cached = (d.e1 - d.e0) <= TILE_NNZ;
    }
    __syncthreads();
    if (sm.cached) {
        const int len = (int)(sm.e1 - sm.e0);
        for (int k = threadIdx.x; k < len; k += SM_NT) {
            sm.val[k] = A.val[sm.e0 + k];
            sm.col[k] = A.col[sm.e0 + k];
        }
        for (int k = threadIdx.x; k <= sm.nrows; k += SM_NT)
            sm.rp[k] = (int)(A.rp[sm.r0 + k] - sm.e0);
    }
    __syncthreads();
}

// Row sums of the CTA's tile against x_j = G(j): products (one rounding each) for all entries
// at once, then thread r adds its row left to right. G uses plain (L1-cached) loads: within a
// phase the gathered vectors are read-only, and the grid barrier between phases is a
// gpu-scope fence, which invalidates L1 (so the next phase never sees a stale line).
template <class Gather>
__device__ __forceinline__ double tile_rowsum(const Csr& A, SmallSmem& sm, Gather G) {
    const int tid = threadIdx.x;
    double acc = 0.0;
    if (sm.cached) {
        const int len = (int)(sm.e1 - sm.e0);
        for (int k = tid; k < len; k += SM_NT) sm.prod[k] = dmul(sm.val[k], G(sm.col[k]));
        __syncthreads();
        if (tid < sm.nrows) {
            const int b = sm.rp[tid], e = sm.rp[tid + 1];
            for (int k = b; k < e; ++k) acc = dadd(acc, sm.prod[k]);
        }
        __syncthreads();
    } else {  // one long row
        double a = 0.0;
        for (long long b0 = sm.e0; b0 < sm.e1; b0 += TILE_NNZ) {
            const int clen = (int)((sm.e1 - b0) < TILE_NNZ ? (sm.e1 - b0) : TILE_NNZ);
            for (int k = tid; k < clen; k += SM_NT)
                sm.prod[k] = dmul(A.val[b0 + k], G(A.col[b0 + k]));
            __syncthreads();
            if (tid == 0)
                for (int k = 0; k < clen; ++k) a = dadd(a, sm.prod[k]);
            __syncthreads();
        }
        acc = a;
    }
    return acc;
}

// Same fixed-order reduction as reduce_partials, run by every CTA (L2 reads: the partials
// were just written by other CTAs).
__device__ __forceinline__ double all_reduce_partials(const double* P, int count, double* red) {
    double acc = 0.0;
    for (int k = threadIdx.x; k < count; k += SM_NT) acc = dadd(acc, __ldcg(P + k));
    acc = group_sum<SM_NT / 32, 0>(acc, red);
    if (threadIdx.x == 0) red[0] = acc;
    __syncthreads();
    acc = red[0];
    __syncthreads();
    return acc;
}

__device__ __forceinline__ double read_max(unsigned long long* slot) {
    return bits2d(__ldcg(slot));
}

// Jacobi, all sweeps in one launch. maxslot[3] are zero on entry. Each thread keeps its row's
// b, d and current iterate in registers; per sweep only the gathers, the x' store and one
// grid barrier remain.
__global__ void __launch_bounds__(SM_NT) k_jacobi_small(Csr R, Vecs V, SolveState* st,
                                                        unsigned long long* maxslot) {
    __shared__ SmallSmem sm;
    cg::grid_group grid = cg::this_grid();
    const double tol = st->tol;
    const long long max_it = st->max_it;
    load_tile(R, blockIdx.x, sm);
    const int row = threadIdx.x < sm.nrows ? sm.r0 + (int)threadIdx.x : -1;
    double bi = 0.0, di = 1.0, xi = 0.0;
    if (row >= 0) { bi = V.b[row]; di = V.d[row]; xi = V.x_jac0[row]; }
    long long it = 0;
    int stop = RUNNING;
    while (stop == RUNNING) {
        ++it;
        const double* xin = (it & 1) ? V.x_jac0 : V.x_jac1;
        double* xout = (it & 1) ? V.x_jac1 : V.x_jac0;
        const double s = tile_rowsum(R, sm, [&](int c) { return xin[c]; });
        unsigned long long mb = 0;
        if (row >= 0) {
            const double xn = ddiv(dsub(bi, s), di);   // (b - R x) / d
            xout[row] = xn;
            mb = absbits(dsub(xn, xi));
            xi = xn;
        }
        mb = group_max<SM_NT / 32, 0>(mb, sm.redu);
        if (threadIdx.x == 0 && mb) atomicMax(&maxslot[it % 3], mb);
        // slot (it+1)%3 was last read before the previous barrier by every CTA: clear it for
        // the next sweep before this barrier, so no CTA can add to it before it is cleared
        if (blockIdx.x == 0 && threadIdx.x == 0) maxslot[(it + 1) % 3] = 0ull;
        grid.sync();
        const double md = read_max(&maxslot[it % 3]);
        if (md <= tol) stop = CONVERGED;
        else if (it >= max_it) stop = NOTCONV;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->it = it;
        st->stop = stop;
    }
}

// BiCGStab, whole solve in one launch (solvers.py:450-491), three grid barriers per iteration.
// Each thread keeps its row's r, p, v, x, q in registers. The vectors other CTAs gather are
// recomputed on the fly from global copies instead of being materialised by extra phases:
//   v = M p   gathers p_j = r_j + beta (p_j - w v_j) from r, p_prev, v_prev (phase A fused),
//   t = M s   gathers s_j = r_j - a v_j from r, v (phase C fused),
// with exactly the reference's expressions, so every value is bit-identical to the phased
// kernels. p and v are double-buffered by iteration parity (V.p/V.s, V.v/V.t): other CTAs
// still read the previous pair while this iteration's is written. Partials live in four
// separate slots (parts + k*pstride: q.v, t.t, t.s, q.r) because no barrier separates a
// slot's all-reduce from the next slot's writes. maxslot[2] zero on entry.
__global__ void __launch_bounds__(SM_NT) k_bicg_small(Csr A, Vecs V, SolveState* st,
                                                      unsigned long long* maxslot, double* parts,
                                                      int pstride) {
    __shared__ SmallSmem sm;
    cg::grid_group grid = cg::this_grid();
    const double tol = st->tol;
    const long long max_it = st->max_it;
    const int nt = A.ntiles;
    double* Pqv = parts;
    double* Ptt = parts + pstride;
    double* Pts = parts + 2 * pstride;
    double* Pqr = parts + 3 * pstride;
    double* Rg = V.r;
    load_tile(A, blockIdx.x, sm);
    const int tid = threadIdx.x;
    const int row = tid < sm.nrows ? sm.r0 + tid : -1;
    double xi = 0.0, bi = 0.0;
    if (row >= 0) { xi = V.x[row]; bi = V.b[row]; }
    // setup: r = b - 1.0 * M x0, q = r, p = v = 0
    const double* X = V.x;
    const double s0 = tile_rowsum(A, sm, [&](int c) { return X[c]; });
    double ri = 0.0, qi = 0.0, pi = 0.0, vi = 0.0;
    unsigned long long mb = 0;
    double p1 = 0.0;
    if (row >= 0) {
        ri = dsub(bi, dmul(1.0, s0));
        qi = ri;
        Rg[row] = ri;
        V.p[row] = 0.0;  // buffer 0 of the (p, v) pair read by iteration 1
        V.v[row] = 0.0;
        mb = absbits(ri);
        p1 = dmul(ri, ri);
    }
    p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
    if (tid == 0) Pqr[blockIdx.x] = p1;
    mb = group_max<SM_NT / 32, 0>(mb, sm.redu);
    if (tid == 0 && mb) atomicMax(&maxslot[0], mb);
    grid.sync();
    int stop = RUNNING, which = 0;
    long long it = 0, bd_it = 0;
    double y = 1.0, a = 1.0, w = 1.0, beta = 0.0;
    {
        const double mr = read_max(&maxslot[0]);
        const double qr = all_reduce_partials(Pqr, nt, sm.red);
        if (mr <= tol) {
            stop = CONVERGED;
        } else {
            const double denom = dmul(y, w);
            y = qr;
            if (tiny(denom)) { stop = BREAKDOWN; which = 1; bd_it = 1; }
            else beta = ddiv(dmul(qr, a), denom);
        }
    }
    while (stop == RUNNING) {
        const long long cur = it + 1;
        const bool odd = (cur & 1) != 0;          // odd iterations read pair 0, write pair 1
        const double* Pold = odd ? V.p : V.s;
        const double* Vold = odd ? V.v : V.t;
        double* Pnew = odd ? V.s : V.p;
        double* Vnew = odd ? V.t : V.v;
        // v = M p with p = r + beta (p - w v) formed at each gathered column
        const double sv = tile_rowsum(A, sm, [&](int c) {
            return dadd(Rg[c], dmul(beta, dsub(Pold[c], dmul(w, Vold[c]))));
        });
        p1 = 0.0;
        if (row >= 0) {
            pi = dadd(ri, dmul(beta, dsub(pi, dmul(w, vi))));
            vi = sv;
            Pnew[row] = pi;
            Vnew[row] = vi;
            p1 = dmul(qi, vi);
        }
        p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
        if (tid == 0) Pqv[blockIdx.x] = p1;
        if (blockIdx.x == 0 && tid == 0) maxslot[1] = 0ull;
        grid.sync();
        const double qv = all_reduce_partials(Pqv, nt, sm.red);
        if (tiny(qv)) { stop = BREAKDOWN; which = 2; bd_it = cur; break; }
        a = ddiv(y, qv);
        // t = M s with s = r - a v formed at each gathered column; s, max|s| for own rows
        const double st_ = tile_rowsum(A, sm, [&](int c) {
            return dsub(Rg[c], dmul(a, Vnew[c]));
        });
        double si = 0.0, ti = 0.0, p2 = 0.0;
        p1 = 0.0;
        mb = 0;
        if (row >= 0) {
            si = dsub(ri, dmul(a, vi));
            ti = st_;
            mb = absbits(si);
            p1 = dmul(ti, ti);
            p2 = dmul(ti, si);
        }
        mb = group_max<SM_NT / 32, 0>(mb, sm.redu);
        if (tid == 0 && mb) atomicMax(&maxslot[1], mb);
        p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
        p2 = group_sum<SM_NT / 32, 0>(p2, sm.red);
        if (tid == 0) { Ptt[blockIdx.x] = p1; Pts[blockIdx.x] = p2; }
        grid.sync();
        const bool small = read_max(&maxslot[1]) <= tol;
        const double tt = all_reduce_partials(Ptt, nt, sm.red);
        const double ts = all_reduce_partials(Pts, nt, sm.red);
        if (tiny(tt)) {
            if (!small) { stop = BREAKDOWN; which = 3; bd_it = cur; break; }
            w = 0.0;
        } else {
            w = ddiv(ts, tt);
        }
        // x += a p + w s, r = s - w t, q.r
        p1 = 0.0;
        if (row >= 0) {
            xi = dadd(dadd(xi, dmul(a, pi)), dmul(w, si));
            ri = dsub(si, dmul(w, ti));
            Rg[row] = ri;
            p1 = dmul(qi, ri);
        }
        p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
        if (tid == 0) Pqr[blockIdx.x] = p1;
        grid.sync();
        it = cur;
        if (small) { stop = CONVERGED; break; }
        if (it >= max_it) { stop = NOTCONV; break; }
        const double qr = all_reduce_partials(Pqr, nt, sm.red);
        const double denom = dmul(y, w);
        y = qr;
        if (tiny(denom)) { stop = BREAKDOWN; which = 1; bd_it = it + 1; break; }
        beta = ddiv(dmul(qr, a), denom);
    }
    if (row >= 0) V.x[row] = xi;  // final iterate, or the snapshot before a breakdown
    if (blockIdx.x == 0 && tid == 0) {
        st->it = it;
        st->stop = stop;
        st->which = which;
        st->bd_it = bd_it;
    }
}

// ---------------------------------------------------------------- element-wise phases
// BiCGStab vector updates, CHUNK_PER rows per thread (rows strided by CHUNK_NT: coalesced).
// No phase branches on the stop flag before its loads: a branch would gate the whole stream on
// the state's L2 round trip (ptxas hoists early exits above side-effect-free loads). Instead a
// stopped solve is made harmless: p and s are dead once the solve has stopped (only x and the
// state are read afterwards), so A and C write them unconditionally and C adds to the running
// max only while live; E rewrites x with its old value and skips its scalar step.
template <int PH>
__global__ void __launch_bounds__(CHUNK_NT) k_phase(Vecs V, int n, SolveState* st) {
    __shared__ double s_red[CHUNK_NT / 32];
    __shared__ unsigned long long s_redu[CHUNK_NT / 32];
    __shared__ int s_flag;
    griddep_wait();
    griddep_launch();
    const int base = blockIdx.x * CHUNK_ROWS + threadIdx.x;
    if constexpr (PH == PH_A) {
        const double beta = st->beta, w = st->w;
        double r[CHUNK_PER], p[CHUNK_PER], v[CHUNK_PER];
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) { r[u] = __ldcs(V.r + i); p[u] = __ldcs(V.p + i); v[u] = __ldcs(V.v + i); }
        }
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) {
                const double pn = dadd(r[u], dmul(beta, dsub(p[u], dmul(w, v[u]))));  // r + beta (p - w v)
                V.p[i] = pn;
                peer_store(V, FV_P, V.roff + i, pn);
            }
        }
        if (V.peers) __threadfence_system();
    } else if constexpr (PH == PH_C) {
        const double a = st->a;
        const int stop = st->stop;
        double r[CHUNK_PER], v[CHUNK_PER];
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) { r[u] = __ldcs(V.r + i); v[u] = __ldcs(V.v + i); }
        }
        unsigned long long mb = 0;
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) {
                const double sv = dsub(r[u], dmul(a, v[u]));   // s = r - a v
                V.s[i] = sv;
                peer_store(V, FV_S, V.roff + i, sv);
                mb = umax(mb, absbits(sv));
            }
        }
        if (V.peers) __threadfence_system();
        mb = group_max<CHUNK_NT / 32, 0>(mb, s_redu);
        if (threadIdx.x == 0 && mb && !stop) atomicMax(&st->maxbits, mb);
    } else {
        const double a = st->a, w = st->w;
        const int stop = st->stop;
        double xv[CHUNK_PER], p[CHUNK_PER], s[CHUNK_PER], t[CHUNK_PER], q[CHUNK_PER];
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) {
                xv[u] = V.x[i]; p[u] = __ldcs(V.p + i); s[u] = __ldcs(V.s + i);
                t[u] = __ldcs(V.t + i); q[u] = __ldg(V.q + i);
            }
        }
        double part = 0.0;
        const long long keep = stop ? -1ll : 0ll;  // bit select, not a branch (see above)
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) {
                const double xn = dadd(dadd(xv[u], dmul(a, p[u])), dmul(w, s[u]));  // x + a p + w s
                V.x[i] = __longlong_as_double((__double_as_longlong(xn) & ~keep) |
                                              (__double_as_longlong(xv[u]) & keep));
                const double rv = dsub(s[u], dmul(w, t[u]));                      // r = s - w t
                V.r[i] = rv;
                part = dadd(part, dmul(q[u], rv));                                 // q . r
            }
        }
        part = group_sum<CHUNK_NT / 32, 0>(part, s_red);
        if (threadIdx.x == 0) V.P1[blockIdx.x] = part;
        if (!last_cta(&st->done, &s_flag)) return;
        if (st->seqdots || stop) {
            if (threadIdx.x == 0) st->done = 0;
            return;
        }
        const double qr = reduce_partials<CHUNK_NT>(V.P1, gridDim.x, s_red);
        if (threadIdx.x != 0) return;
        st->done = 0;
        if (st->sharded) {
            st->send[0] = qr;
            st->send[1] = 0.0;
            st->send[2] = 0.0;
            st->send[3] = 0.0;
            return;
        }
        fin_e(st, qr);
    }
}

// ---------------------------------------------------------------- reference-order dots
// Bit-exact _dot_ascending (solvers.py:136-141): acc = u0*v0, then acc = acc + ui*vi strictly
// in index order. The chain is inherently serial (one dependent add per element); warps 2..7
// stream the next block of products into shared memory while thread 0 (and thread 32 for the
// second chain t.s) adds the current block. Used when SolveState.seqdots is set.
enum SeqWhich : int { SQ_S0 = 0, SQ_V = 1, SQ_T = 2, SQ_E = 3 };
constexpr int SEQ_NT = 256;
constexpr int SEQ_BLK = 1024;

template <int W>
__global__ void __launch_bounds__(SEQ_NT) k_seqdot(Vecs V, int n, SolveState* st) {
    __shared__ double buf[2][2][SEQ_BLK];
    __shared__ double s_acc2;
    griddep_wait();
    griddep_launch();
    if (st->stop) return;
    const double* u1 = (W == SQ_T) ? V.t : V.q;
    const double* v1 = (W == SQ_S0 || W == SQ_E) ? V.r : (W == SQ_V ? V.v : V.t);
    const double* u2 = V.t;
    const double* v2 = V.s;
    constexpr int NCH = (W == SQ_T) ? 2 : 1;
    const int tid = threadIdx.x;
    const int nblk = (n + SEQ_BLK - 1) / SEQ_BLK;
    auto fill = [&](int blk, int slot, int t0, int nt) {
        const int b0 = blk * SEQ_BLK;
        for (int k = tid - t0; k < SEQ_BLK; k += nt) {
            const int i = b0 + k;
            if (i < n) {
                buf[0][slot][k] = dmul(u1[i], v1[i]);
                if (NCH == 2) buf[1][slot][k] = dmul(u2[i], v2[i]);
            }
        }
    };
    fill(0, 0, 0, SEQ_NT);
    __syncthreads();
    double acc = 0.0;
    for (int blk = 0; blk < nblk; ++blk) {
        const int cur = blk & 1;
        const int len = min(SEQ_BLK, n - blk * SEQ_BLK);
        if (tid == 0 || (NCH == 2 && tid == 32)) {
            const double* p = buf[tid == 0 ? 0 : 1][cur];
            int k = 0;
            if (blk == 0) { acc = p[0]; k = 1; }
#pragma unroll 8
            for (; k < len; ++k) acc = dadd(acc, p[k]);
        } else if (tid >= 64 && blk + 1 < nblk) {
            fill(blk + 1, cur ^ 1, 64, SEQ_NT - 64);
        }
        __syncthreads();
    }
    if (NCH == 2 && tid == 32) s_acc2 = acc;
    __syncthreads();
    if (tid != 0) return;
    if constexpr (W == SQ_S0) fin_s0(st, acc);
    else if constexpr (W == SQ_V) fin_v(st, acc);
    else if constexpr (W == SQ_T) fin_t(st, acc, s_acc2);
    else fin_e(st, acc);
}

// ---------------------------------------------------------------- multi-GPU reduction points
// After the per-rank exchange every rank holds the same `world` x SEND_SLOTS partials; one
// thread sums the dots in ascending rank order and takes the max, then runs the same scalar
// step as the single-GPU path. Identical inputs -> identical bits -> every rank takes the same
// stop / breakdown decision with no further communication.
enum FinWhich : int { FIN_JACOBI = 0, FIN_RESID = 1, FIN_S0 = 2, FIN_V = 3, FIN_T = 4, FIN_E = 5 };

template <int W>
__global__ void k_finalize(SolveState* st, const double* __restrict__ recv, int world) {
    griddep_wait();
    griddep_launch();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (W != FIN_RESID && st->stop) return;
    double d1 = 0.0, d2 = 0.0;
    unsigned long long mb = 0;
    for (int r = 0; r < world; ++r) {
        d1 = dadd(d1, recv[r * SEND_SLOTS + 0]);
        d2 = dadd(d2, recv[r * SEND_SLOTS + 1]);
        mb = umax(mb, (unsigned long long)__double_as_longlong(recv[r * SEND_SLOTS + 2]));
    }
    if constexpr (W == FIN_JACOBI) {
        const double md = bits2d(mb);
        const long long it = st->it + 1;
        st->it = it;
        if (md <= st->tol) st->stop = CONVERGED;
        else if (it >= st->max_it) st->stop = NOTCONV;
    } else if constexpr (W == FIN_RESID) {
        st->resid = bits2d(mb);
    } else {
        st->maxbits = mb;  // read (and cleared) by fin_s0 / fin_t
        if constexpr (W == FIN_S0) fin_s0(st, d1);
        else if constexpr (W == FIN_V) fin_v(st, d1);
        else if constexpr (W == FIN_T) fin_t(st, d1, d2);
        else fin_e(st, d1);
        st->maxbits = 0ull;
    }
}

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
            bulk_g2s(dsm + c * DCOLS * DSLAB, src + (size_t)c * DCOLS * DSLAB, bytes, &bars[c]);
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
            bulk_g2s(dsm + stage * DCOLS * DSLAB, src + (size_t)cn * DCOLS * DSLAB, bytes,
                     &bars[stage]);
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
__global__ void k_check_rows(const long long* __restrict__ rp, const int* __restrict__ col, int n,
                             int* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (long long e = rp[i] + 1; e < rp[i + 1]; ++e)
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
                       long long* offlen, unsigned long long* first_zero) {
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
