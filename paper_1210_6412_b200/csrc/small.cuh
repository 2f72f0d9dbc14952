// small.cuh -- whole-solve cooperative kernels for systems whose tiles all fit on the GPU at once (part of device.cuh).
#pragma once

#include "common.cuh"

namespace mcr {

// ---------------------------------------------------------------- persistent small-system solvers
// For systems whose tiles all fit on the GPU at once (ntiles <= co-resident CTAs, e.g. C1 and
// the Table-1 shapes) one cooperative kernel runs the whole solve: sweeps / iterations are
// separated by grid barriers instead of kernel launches, and every CTA reduces the per-tile
// partials itself in the same fixed order, so all CTAs hold bit-identical scalars without a
// round trip through global state.
namespace cg = cooperative_groups;
constexpr int SM_NT = TILE_ROWS;
constexpr int SMALL_CLUSTER_MAX = 16;  // CTAs of the cluster variant (non-portable above 8)

struct SmallSmem {
    double val[TILE_NNZ];      // this CTA's tile, loaded once per solve
    int col[TILE_NNZ];
    double prod[TILE_NNZ];
    int rp[TILE_ROWS + 1];
    double red[SM_NT / 32];
    unsigned long long redu[SM_NT / 32];
    double part[4];                 // cluster variant: this CTA's dot partials (q.v, t.t, t.s, q.r)
    unsigned long long mx[3];       // cluster variant: this CTA's max|.| bits per slot
    long long e0, e1;
    int nrows, r0, cached;
};

// ---------------------------------------------------------------- barrier / exchange policy
// CL = false: one cooperative grid, grid.sync() between phases, partials and maxima through
// global memory. CL = true: the whole grid is ONE thread-block cluster (<= 16 CTAs, one per SM):
// the hardware cluster barrier replaces the grid barrier and every CTA reads the others'
// partials and maxima straight from their shared memory (DSMEM), which removes the global
// round trips that dominate an iteration of these latency-bound systems. Vectors written by
// other CTAs are then gathered through L2 (ld.global.cg): a cluster barrier orders memory but
// does not clean this SM's L1.
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class T>
__device__ __forceinline__ T dsmem_load(const T* p, int rank);
template <>
__device__ __forceinline__ double dsmem_load<double>(const double* p, int rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
    return v;
}
template <>
__device__ __forceinline__ unsigned long long dsmem_load<unsigned long long>(const unsigned long long* p,
                                                                             int rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
    unsigned long long v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
    return v;
}

// A one-CTA system needs no cross-SM ordering at all: __syncthreads orders its global
// accesses for the whole block, the L1 stays coherent, and no release fence is paid.
template <bool CL>
struct SmallSync {
    __device__ __forceinline__ void sync() {
        if constexpr (CL) {
            if (gridDim.x == 1) __syncthreads();
            else cluster_barrier();
        } else {
            cg::this_grid().sync();
        }
    }
    template <class T>
    __device__ __forceinline__ T gather(const T* p) const {
        if constexpr (CL) return gridDim.x == 1 ? *p : __ldcg(p);
        else return *p;
    }
    __device__ __forceinline__ void exit_sync() {  // no CTA leaves while others read its slots
        if constexpr (CL) {
            if (gridDim.x > 1) cluster_barrier();
        }
    }
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
// tile_products issues all of a thread's gathers before the first product (one L2 round trip
// per phase instead of one per unrolled group); the caller syncs the CTA before tile_chain.
constexpr int SM_PER = (TILE_NNZ + SM_NT - 1) / SM_NT;  // entries per thread of a cached tile

template <class Gather>
__device__ __forceinline__ void tile_products(SmallSmem& sm, Gather G) {
    const int tid = threadIdx.x;
    const int len = (int)(sm.e1 - sm.e0);
    if (len <= SM_NT * (SM_PER / 2)) {  // short tile (Table-1 shapes): the plain loop is cheaper
        for (int k = tid; k < len; k += SM_NT) sm.prod[k] = dmul(sm.val[k], G(sm.col[k]));
        return;
    }
    double g[SM_PER];
#pragma unroll
    for (int u = 0; u < SM_PER; ++u) {
        const int k = tid + u * SM_NT;
        g[u] = k < len ? G(sm.col[k]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < SM_PER; ++u) {
        const int k = tid + u * SM_NT;
        if (k < len) sm.prod[k] = dmul(sm.val[k], g[u]);
    }
}

__device__ __forceinline__ double tile_chain(const SmallSmem& sm) {
    const int tid = threadIdx.x;
    double acc = 0.0;
    if (tid < sm.nrows) {
        const int b = sm.rp[tid], e = sm.rp[tid + 1];
        for (int k = b; k < e; ++k) acc = dadd(acc, sm.prod[k]);
    }
    return acc;
}

// Streamed row longer than a tile (sm.cached == 0): thread 0 adds it chunk by chunk.
template <class Gather>
__device__ __forceinline__ double long_row_sum(const Csr& A, SmallSmem& sm, Gather G) {
    const int tid = threadIdx.x;
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
    return a;
}

// (BiCGStab's gathers read three vectors each: the plain loop keeps fewer loads in flight but
// measured faster there than tile_products, C4 -3..-8%)
template <class Gather>
__device__ __forceinline__ double tile_rowsum(const Csr& A, SmallSmem& sm, Gather G) {
    if (!sm.cached) return long_row_sum(A, sm, G);
    const int len = (int)(sm.e1 - sm.e0);
    for (int k = threadIdx.x; k < len; k += SM_NT) sm.prod[k] = dmul(sm.val[k], G(sm.col[k]));
    __syncthreads();
    const double acc = tile_chain(sm);
    __syncthreads();
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

// The same value for count <= 32 without the CTA tree or any __syncthreads: every warp loads
// the partials into lanes 0..count-1 and runs group_sum's warp tree. In group_sum those lanes
// of warp 0 are the only nonzero inputs; the other warps' sums are +0.0 and the second-level
// tree adds them to warp 0's sum, which is never -0.0 (each input is 0.0 + P, and a sum of
// values other than -0.0 is never -0.0 in round-to-nearest), so adding them changes nothing:
// same bits as all_reduce_partials (the grid variant) over the CTAs' shared-memory slots.
// One CTA: the tree of a single nonzero input is 0.0 + P itself.
__device__ __forceinline__ double cluster_allreduce(const double* slot, int count) {
    if (count == 1) return dadd(0.0, *slot);
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    double v = lane < count ? dadd(0.0, dsmem_load(slot, lane)) : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = dadd(v, __shfl_down_sync(full, v, off));
    return __shfl_sync(full, v, 0);
}
__device__ __forceinline__ double cluster_read_max(const unsigned long long* slot, int count) {
    unsigned long long m = 0;
    for (int k = 0; k < count; ++k) m = umax(m, dsmem_load(slot, k));
    return bits2d(m);
}

// Jacobi, all sweeps in one launch. maxslot[3] are zero on entry (grid variant). Each thread
// keeps its row's b, d and current iterate in registers; per sweep only the gathers, the x'
// store and one barrier remain.
template <bool CL>
__global__ void __launch_bounds__(SM_NT) k_jacobi_small(Csr R, Vecs V, SolveState* st,
                                                        unsigned long long* maxslot) {
    __shared__ SmallSmem sm;
    SmallSync<CL> bar;
    const double tol = st->tol;
    const long long max_it = st->max_it;
    load_tile(R, blockIdx.x, sm);
    const int row = threadIdx.x < sm.nrows ? sm.r0 + (int)threadIdx.x : -1;
    double bi = 0.0, di = 1.0, xi = 0.0;
    if (row >= 0) { bi = V.b[row]; di = V.d[row]; xi = V.x_jac0[row]; }
    long long it = 0;
    int stop = RUNNING;
    const bool cached = sm.cached;
    // products of sweep 1 (x0 buffer); from then on the next sweep's products are formed right
    // after each barrier, while the stop test's max is still in flight (speculative: a sweep
    // that is never run only wrote shared memory)
    if (cached) tile_products(sm, [&](int c) { return bar.gather(V.x_jac0 + c); });
    while (stop == RUNNING) {
        ++it;
        const double* xin = (it & 1) ? V.x_jac0 : V.x_jac1;
        double* xout = (it & 1) ? V.x_jac1 : V.x_jac0;
        double s;
        if (cached) {
            __syncthreads();
            s = tile_chain(sm);
        } else {
            s = long_row_sum(R, sm, [&](int c) { return bar.gather(xin + c); });
        }
        unsigned long long mb = 0;
        if (row >= 0) {
            const double xn = ddiv(dsub(bi, s), di);   // (b - R x) / d
            xout[row] = xn;
            mb = absbits(dsub(xn, xi));
            xi = xn;
        }
        mb = group_max<SM_NT / 32, 0>(mb, sm.redu);  // (its barrier also ends the chains' reads)
        unsigned long long mraw;
        if constexpr (CL) {
            // slot it&1 is rewritten two sweeps later, after every CTA has passed the barrier
            // that follows its reads
            if (threadIdx.x == 0) sm.mx[it & 1] = mb;
            bar.sync();
            mraw = 0;
            for (int k = 0; k < (int)gridDim.x; ++k) mraw = umax(mraw, dsmem_load(&sm.mx[it & 1], k));
        } else {
            if (threadIdx.x == 0 && mb) atomicMax(&maxslot[it % 3], mb);
            // slot (it+1)%3 was last read before the previous barrier by every CTA: clear it for
            // the next sweep before this barrier, so no CTA can add to it before it is cleared
            if (blockIdx.x == 0 && threadIdx.x == 0) maxslot[(it + 1) % 3] = 0ull;
            bar.sync();
            mraw = __ldcg(&maxslot[it % 3]);
        }
        if (cached) tile_products(sm, [&](int c) { return bar.gather(xout + c); });
        const double md = bits2d(mraw);
        if (md <= tol) stop = CONVERGED;
        else if (it >= max_it) stop = NOTCONV;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->it = it;
        st->stop = stop;
    }
    bar.exit_sync();
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
//
// XD (the default, reference-order dots): the four inner products are the reference's
// left-to-right sums (solvers.py:136-141) instead of tile partials + a fixed tree. Each row's
// product goes to a global slot (xprod + k*n; in shared memory directly when the grid is one
// CTA) before the barrier the partials used; after it every CTA stages the slot in shared
// memory and computes the same sum with xd::cta_seqdots (all CTAs get identical bits, so no
// broadcast barrier). Dynamic shared memory: 2n doubles + xd::CtaDots<SM_NT, 2>.
constexpr int XS_MAX_N = 8192;  // largest system the XD variant takes (2n doubles staged)
using SmallDots = xd::CtaDots<SM_NT, 2>;
inline size_t small_xd_smem(long long n) { return (size_t)2 * (size_t)n * sizeof(double) + sizeof(SmallDots); }

template <bool CL, bool XD>
__global__ void __launch_bounds__(SM_NT, XD ? 2 : 1) k_bicg_small(Csr A, Vecs V, SolveState* st,
                                                      unsigned long long* maxslot, double* parts,
                                                      int pstride, double* xprod) {
    __shared__ SmallSmem sm;
    extern __shared__ __align__(16) unsigned char xs_dyn[];
    double* xbuf = (double*)xs_dyn;  // XD: [2][n]
    const int n = A.n;
    SmallDots& xdd = *(SmallDots*)(xs_dyn + (size_t)2 * n * sizeof(double));
    SmallSync<CL> bar;
    const double tol = st->tol;
    const long long max_it = st->max_it;
    const int nt = A.ntiles;
    double* Pqv = parts;
    double* Ptt = parts + pstride;
    double* Pts = parts + 2 * pstride;
    double* Pqr = parts + 3 * pstride;
    enum { S_QV = 0, S_TT = 1, S_TS = 2, S_QR = 3 };
    // publish this CTA's partial of slot k (thread 0 holds it), then (after a barrier) the
    // fixed-order all-reduce over the CTAs
    auto publish = [&](int k, double* gslot, double v) {
        if (threadIdx.x == 0) {
            if constexpr (CL) sm.part[k] = v;
            else gslot[blockIdx.x] = v;
        }
    };
    auto allreduce = [&](int k, const double* gslot) {
        if constexpr (CL) return cluster_allreduce(&sm.part[k], nt);  // nt <= 16
        else return all_reduce_partials(gslot, nt, sm.red);
    };
    auto publish_max = [&](int k, unsigned long long m) {  // m valid in thread 0
        if (threadIdx.x == 0) {
            if constexpr (CL) sm.mx[k] = m;
            else if (m) atomicMax(&maxslot[k], m);
        }
    };
    auto read_maxk = [&](int k) {
        if constexpr (CL) return cluster_read_max(&sm.mx[k], nt);
        else return read_max(&maxslot[k]);
    };
    // XD: row product of slot k (j = its place in the next cta_seqdots call); after the barrier,
    // the K consecutive slots from k0 are staged and summed in the reference's order
    auto put = [&](int k, int j, int r, double p) {
        if (gridDim.x == 1) xbuf[(size_t)j * n + r] = p;
        else xprod[(size_t)k * n + r] = p;
    };
    auto seqdots = [&](int k0, auto kk, double* res) {
        constexpr int K = decltype(kk)::value;
        if (gridDim.x > 1) {
            for (int i = threadIdx.x; i < K * n; i += SM_NT) xbuf[i] = __ldcg(xprod + (size_t)k0 * n + i);
            __syncthreads();
        }
        xd::cta_seqdots<SM_NT, K>(xbuf, n, *(xd::CtaDots<SM_NT, K>*)&xdd, res);
    };
    using One = std::integral_constant<int, 1>;
    using Two = std::integral_constant<int, 2>;
    double* Rg = V.r;
    load_tile(A, blockIdx.x, sm);
    const int tid = threadIdx.x;
    const int row = tid < sm.nrows ? sm.r0 + tid : -1;
    double xi = 0.0, bi = 0.0;
    if (row >= 0) { xi = V.x[row]; bi = V.b[row]; }
    // setup: r = b - 1.0 * M x0, q = r, p = v = 0
    const double* X = V.x;
    const double s0 = tile_rowsum(A, sm, [&](int c) { return bar.gather(X + c); });
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
        if constexpr (XD) put(S_QR, 0, row, p1);
    }
    if constexpr (!XD) {
        p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
        publish(S_QR, Pqr, p1);
    }
    mb = group_max<SM_NT / 32, 0>(mb, sm.redu);
    publish_max(0, mb);
    bar.sync();
    int stop = RUNNING, which = 0;
    long long it = 0, bd_it = 0;
    double y = 1.0, a = 1.0, w = 1.0, beta = 0.0;
    {
        const double mr = read_maxk(0);
        double qr;
        if constexpr (XD) seqdots(S_QR, One{}, &qr);
        else qr = allreduce(S_QR, Pqr);
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
            return dadd(bar.gather(Rg + c), dmul(beta, dsub(bar.gather(Pold + c), dmul(w, bar.gather(Vold + c)))));
        });
        p1 = 0.0;
        if (row >= 0) {
            pi = dadd(ri, dmul(beta, dsub(pi, dmul(w, vi))));
            vi = sv;
            Pnew[row] = pi;
            Vnew[row] = vi;
            p1 = dmul(qi, vi);
            if constexpr (XD) put(S_QV, 0, row, p1);
        }
        if constexpr (!XD) {
            p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
            publish(S_QV, Pqv, p1);
        }
        if constexpr (!CL) {
            if (blockIdx.x == 0 && tid == 0) maxslot[1] = 0ull;
        }
        bar.sync();
        double qv;
        if constexpr (XD) seqdots(S_QV, One{}, &qv);
        else qv = allreduce(S_QV, Pqv);
        if (tiny(qv)) { stop = BREAKDOWN; which = 2; bd_it = cur; break; }
        a = ddiv(y, qv);
        // t = M s with s = r - a v formed at each gathered column; s, max|s| for own rows
        const double st_ = tile_rowsum(A, sm, [&](int c) {
            return dsub(bar.gather(Rg + c), dmul(a, bar.gather(Vnew + c)));
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
            if constexpr (XD) {
                put(S_TT, 0, row, p1);
                put(S_TS, 1, row, p2);
            }
        }
        mb = group_max<SM_NT / 32, 0>(mb, sm.redu);
        publish_max(1, mb);
        if constexpr (!XD) {
            p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
            p2 = group_sum<SM_NT / 32, 0>(p2, sm.red);
            publish(S_TT, Ptt, p1);
            publish(S_TS, Pts, p2);
        }
        bar.sync();
        const bool small = read_maxk(1) <= tol;
        double tt, ts;
        if constexpr (XD) {
            double r2[2];
            seqdots(S_TT, Two{}, r2);  // slots TT, TS are consecutive
            tt = r2[0];
            ts = r2[1];
        } else {
            tt = allreduce(S_TT, Ptt);
            ts = allreduce(S_TS, Pts);
        }
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
            if constexpr (XD) put(S_QR, 0, row, p1);
        }
        if constexpr (!XD) {
            p1 = group_sum<SM_NT / 32, 0>(p1, sm.red);
            publish(S_QR, Pqr, p1);
        }
        bar.sync();
        it = cur;
        if (small) { stop = CONVERGED; break; }
        if (it >= max_it) { stop = NOTCONV; break; }
        double qr;
        if constexpr (XD) seqdots(S_QR, One{}, &qr);
        else qr = allreduce(S_QR, Pqr);
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
    bar.exit_sync();
}

// The one-CTA reference-order dot of the small whole-solve kernels (xd::cta_seqdots, the path
// k_bicg_small<*, true> takes), stand-alone: k = 1 or 2 dots of length n <= XS_MAX_N in one
// launch (the second pair may alias the first). Test entry point (mcr_xdot_cta).
template <int K>
__global__ void __launch_bounds__(SM_NT) k_xdot_cta(const double* u0, const double* v0, const double* u1,
                                                    const double* v1, int n, double* out) {
    extern __shared__ __align__(16) unsigned char dyn[];
    double* buf = (double*)dyn;
    auto& D = *(xd::CtaDots<SM_NT, K>*)(dyn + (size_t)2 * n * sizeof(double));
    for (int i = threadIdx.x; i < n; i += SM_NT) {
        buf[i] = dmul(u0[i], v0[i]);
        if (K == 2) buf[n + i] = dmul(u1[i], v1[i]);
    }
    __syncthreads();
    double res[K];
    xd::cta_seqdots<SM_NT, K>(buf, n, D, res);
    if (threadIdx.x < K) out[threadIdx.x] = res[threadIdx.x];
}


}  // namespace mcr
