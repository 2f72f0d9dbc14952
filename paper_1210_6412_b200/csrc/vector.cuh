// vector.cuh -- BiCGStab vector phases, reference-order dots, multi-GPU reduction points (part of device.cuh).
#pragma once

#include "common.cuh"

namespace mcr {

// ---------------------------------------------------------------- element-wise phases
// BiCGStab vector updates, CHUNK_PER rows per thread (rows strided by CHUNK_NT: coalesced).
// No phase branches on the stop flag before its loads: a branch would gate the whole stream on
// the state's L2 round trip (ptxas hoists early exits above side-effect-free loads). Instead a
// stopped solve is made harmless: p and s are dead once the solve has stopped (only x and the
// state are read afterwards), so A and C write them unconditionally and C adds to the running
// max only while live; E rewrites x with its old value and skips its scalar step.
// Rows per thread: A and C (no inner product, so no summation order to keep) take
// MCR_PHASE_PER_AC rows so their grid fits in one wave of co-resident CTAs; E keeps CHUNK_PER
// because its per-CTA q.r partials fix the dot order.
#ifndef MCR_PHASE_PER_AC
#define MCR_PHASE_PER_AC 8
#endif
template <int PH>
__host__ __device__ constexpr int phase_per() { return PH == PH_E ? CHUNK_PER : MCR_PHASE_PER_AC; }

template <int PH>
__global__ void __launch_bounds__(CHUNK_NT) k_phase(Vecs V, int n, SolveState* st) {
    constexpr int CHUNK_PER = phase_per<PH>();
    __shared__ double s_red[CHUNK_NT / 32];
    __shared__ unsigned long long s_redu[CHUNK_NT / 32];
    __shared__ int s_flag;
    griddep_wait();
    griddep_launch();
    const int base = blockIdx.x * (CHUNK_NT * CHUNK_PER) + threadIdx.x;
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
    } else if constexpr (PH == PH_EX) {
        // E with the reference-order dots on one device: the x and r updates alone (q.r is
        // k_xdot's), A/C-sized chunks, no partials; a stopped solve ends the graph loop here
        const double a = st->a, w = st->w;
        const int stop = st->stop;
        double xv[CHUNK_PER], p[CHUNK_PER], s[CHUNK_PER], t[CHUNK_PER];
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) {
                xv[u] = V.x[i]; p[u] = __ldcs(V.p + i); s[u] = __ldcs(V.s + i); t[u] = __ldcs(V.t + i);
            }
        }
        const long long keep = stop ? -1ll : 0ll;  // bit select, not a branch (see above)
#pragma unroll
        for (int u = 0; u < CHUNK_PER; ++u) {
            const int i = base + u * CHUNK_NT;
            if (i < n) {
                const double xn = dadd(dadd(xv[u], dmul(a, p[u])), dmul(w, s[u]));  // x + a p + w s
                V.x[i] = __longlong_as_double((__double_as_longlong(xn) & ~keep) |
                                              (__double_as_longlong(xv[u]) & keep));
                V.r[i] = dsub(s[u], dmul(w, t[u]));                               // r = s - w t
            }
        }
        if (stop && blockIdx.x == 0 && threadIdx.x == 0) graph_continue(st);  // stopped earlier
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
            if (threadIdx.x == 0) {
                st->done = 0;
                if (stop) graph_continue(st);  // stopped earlier in this iteration
            }
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
        graph_continue(st);
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
        st->last = md;
        if (md <= st->tol) st->stop = CONVERGED;
        else if (it >= st->max_it) st->stop = NOTCONV;
    } else if constexpr (W == FIN_RESID) {
        st->resid = bits2d(mb);
    } else {
        if (st->seqdots) {  // reference-order dots of the whole gathered vectors (k_xdot)
            d1 = st->xd[0];
            d2 = st->xd[1];
        }
        st->maxbits = mb;  // read (and cleared) by fin_s0 / fin_t
        if constexpr (W == FIN_S0) fin_s0(st, d1);
        else if constexpr (W == FIN_V) fin_v(st, d1);
        else if constexpr (W == FIN_T) fin_t(st, d1, d2);
        else fin_e(st, d1);
        st->maxbits = 0ull;
    }
}

}  // namespace mcr
