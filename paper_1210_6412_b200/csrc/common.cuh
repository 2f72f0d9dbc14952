// common.cuh -- shared pieces of the sm_100a kernels: layout structs, solver state, scalar and
// reduction helpers, mbarrier / bulk-copy / PDL wrappers, BiCGStab scalar steps and the row
// epilogues of the SpMV family. (Included by every kernel header; device.cuh includes them all.)
//
// Arithmetic contract: every row sum of M x is accumulated from +0.0
// in ascending column order with separately rounded products and sums (no FMA), so SpMV,
// the Jacobi sweep and the residual are bit-identical to scipy's csr_matvec + numpy as used by
// the reference (sparse.py:191, solvers.py:219-225). Element-wise BiCGStab updates use the
// exact evaluation order of the reference's numpy expressions (solvers.py:298-305). Inner
// products are either deterministic trees (each thread over its statically assigned rows,
// then a CTA tree, then a fixed-order sum over CTAs; default) or the reference's own strictly
// sequential order (k_seqdot, bit-exact, slow).
//
// Storage (HBM):
//   CSR:   rowptr int64[n+1], col int32[nnz], val f64[nnz] (each padded by 16 B so 16-byte
//          aligned bulk copies may round up); rows cut into tiles of at most TILE_ROWS rows
//          and TILE_NNZ entries (a longer single row is a tile of its own).
//   Dense: slabs of 32 rows stored [column pair][row][2] (512 B per pair), streamed by one
//          warp with TMA bulk copies; every lane keeps its row's strictly sequential sum.
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
    unsigned long long p1_ctr;   // chunk tickets of the staged products pass (staged.cuh)
    double y, a, w, beta, qv, tt, ts, resid;
    unsigned long long cond;  // graph mode: the while-node's conditional handle (0 = none);
                              // the kernel that decides the stop clears it
    double last;         // convergence measure of the latest sweep / iteration (Jacobi max|x'-x|,
                         // BiCGStab max|s|): the host sizes its batches from its decay
    int small;
    int seqdots;  // 1: inner products by k_seqdot (reference order, bit-exact), not the tree
    int sharded;  // 1: row shard of a multi-GPU system -- reduction kernels publish their local
                  //    partials in send[] instead of finalising; k_finalize finishes after the
                  //    per-rank exchange
    double send[SEND_SLOTS];  // {dot 1, dot 2, max|.| as bits, unused} of this rank
    double xd[2];             // row shard, reference-order dots: k_xdot's sums of the whole
                              // gathered vectors (identical on every rank), read by k_finalize
};

// Entry range [e0, e1) and row range [r0, r1) of one tile.
struct TileDesc {
    long long e0, e1;
    int r0, r1;
};

// The stage's tile id and descriptor as read by lane 0 and broadcast: only the thread that
// releases the stage (lane 0's mbarrier arrive) reads the producer-written slots, so the
// producer's next write of them is ordered after that read by the arrive/wait pair alone.
__device__ __forceinline__ int stage_tile(const int* s_tile, const TileDesc* s_desc, int s,
                                          TileDesc& d) {
    const unsigned full = 0xffffffffu;
    int t = 0;
    long long e0 = 0, e1 = 0;
    int r0 = 0, r1 = 0;
    if ((threadIdx.x & 31) == 0) {
        t = s_tile[s];
        if (t >= 0) { e0 = s_desc[s].e0; e1 = s_desc[s].e1; r0 = s_desc[s].r0; r1 = s_desc[s].r1; }
    }
    t = __shfl_sync(full, t, 0);
    d.e0 = __shfl_sync(full, e0, 0);
    d.e1 = __shfl_sync(full, e1, 0);
    d.r0 = __shfl_sync(full, r0, 0);
    d.r1 = __shfl_sync(full, r1, 0);
    return t;
}

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
enum Phase : int { PH_A = 0, PH_C = 1, PH_E = 2, PH_EX = 3 };  // PH_EX: E without the tree q.r

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
// Solver-state loads through L2 (asm volatile keeps their place in the issue order).
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
// Same, with an L2 eviction-priority hint (policy from l2_evict_first()).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// L2 policy for data read once per pass (the matrix streams): evicted before anything else,
// so the solver's vectors stay L2-resident across the SpMV.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
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

// Graph mode (solve.cuh): the solve loop is a CUDA-graph while node; the kernel that takes
// the stop decision keeps it running (1) or ends it (0). Thread 0 of the deciding CTA.
__device__ __forceinline__ void graph_continue(SolveState* st) {
    if (st->cond) cudaGraphSetConditional((cudaGraphConditionalHandle)st->cond, st->stop == RUNNING ? 1u : 0u);
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
    st->last = ms;
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
        }
        return;
    }
    if constexpr (epi_has_dot<EPI>()) {
        if (st->seqdots) {  // k_seqdot runs the reference-order dots and finalises
            if (threadIdx.x == 0) st->done = 0;
            return;
        }
    }
    double r1 = 0.0, r2 = 0.0;
    if constexpr (epi_has_dot<EPI>()) r1 = reduce_partials<NT>(V.P1, nunits, s_red);
    if constexpr (EPI == EPI_T) r2 = reduce_partials<NT>(V.P2, nunits, s_red);
    if (threadIdx.x != 0) return;
    st->done = 0;
    if constexpr (EPI == EPI_RESID) {
        st->resid = bits2d(atomicExch(&st->maxbits, 0ull));
    } else if constexpr (EPI == EPI_JACOBI) {
        const double md = bits2d(atomicExch(&st->maxbits, 0ull));
        const long long it = st->it + 1;
        st->it = it;
        st->last = md;
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

}  // namespace mcr
