// xdot.cuh -- the reference's strictly sequential inner product, bit-exact, on the whole GPU.
//
// `_dot_ascending(u, v) = np.cumsum(u * v)[-1]` (solvers.py:136-141): s_0 = p_0,
// s_k = fl(s_{k-1} + p_k) with p_k = fl(u_k v_k). The chain of roundings is what makes
// BiCGStab's stopping iteration match the reference (a tree sum stops 3 iterations later on
// C2). One dependent add per element (8.3 cycles) would cost 4.4 ms per dot at n = 1e6; this
// file computes the SAME bits in a few microseconds. The idea:
//
// * Inside one binade (sign, exponent e; grid u = ulp) every partial sum is an integer
//   multiple of u and a step is a TRANSLATION: fl(s + p) = s + D(p, parity of s/u), where
//   the parity only matters for exact ties (round half to even). So a stretch of elements
//   whose partial sums stay inside one binade (a "run") is summarised by two displacements
//   d0 / d1 (start index even / odd) and an excursion bound x: for ANY start s in that
//   binade with |s| - x and |s| + x still inside it, the stretch ends at s + d[parity(s)].
//   Two runs of the same binade compose associatively. d0, d1 come from summing the stretch
//   from two reference starts in the middle of the binade (plain DADD chains, exact).
// * Where the sum changes binade (crossings, passes near zero) a "table" describes the
//   stretch as a function of its start: 32 consecutive candidate starts (doubles around a
//   predicted start) are carried through the stretch exactly (runs applied per candidate,
//   anything else added element by element), and each candidate keeps the range [lo, hi] of
//   start shifts delta that leave every partial sum inside its binade with one ulp of margin
//   plus the coarsest grid 2^km it passed. A start s = cand_k + delta in cand_k's binade
//   with delta in [lo, hi] and delta = 0 mod 2^km (k = the candidate congruent to s mod 32
//   ulps) ends at out_k + delta: every rounding step commutes with such a shift.
// * Tables compose (evaluate the second at the first's outputs) — that is how warps, CTAs
//   and the whole vector are stitched together. Predicted starts come from a plain
//   (non-exact) prefix sum of the products; a prediction only has to land in the right
//   binade for runs and within the translation range for tables. Nothing is ever assumed:
//   every use of a run or table is checked, and a failed check falls back to the finer
//   level (CTA -> warp pieces -> thread pieces -> element-by-element), so the result is the
//   reference's bits for every input (NaN/Inf/overflow/-0.0 included); only the time
//   depends on how often a fallback is needed.
//
// One launch per reduction point: a CTA owns NT*E consecutive elements of one sequence
// (thread t owns E consecutive ones, E odd so the shared-memory reads are conflict free),
// builds thread runs -> warp pieces -> a CTA piece, publishes it; the last CTA of the
// sequence composes the CTA pieces (8 warps on 8 consecutive groups, then a scalar walk of
// the true value from 0.0) and runs the BiCGStab scalar step. Sequences: one per dot, or one
// per row block when the reference's parallel_dot_products mode is on (solvers.py:384-396:
// each block summed sequentially, block results added in ascending order from 0.0).
#pragma once

#include "common.cuh"

namespace mcr {
namespace xd {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int EMAX = 63;
constexpr unsigned long long MANT = 0x000FFFFFFFFFFFFFull;
constexpr unsigned long long SGN = 0x8000000000000000ull;
constexpr int KM_NONE = -4096;
constexpr int E_HARD = 0;       // not a run: summed element by element
constexpr int E_EMPTY = 0x800;  // no elements: identity
constexpr int RUN_MIN_E = 64;   // runs only where the grid u is a normal number
constexpr unsigned FULL = 0xffffffffu;
enum Kind : int { K_RUN = 0, K_TABLE = 1 };
enum Stat : int { ST_HARD = 0, ST_WARP_TABLE, ST_CTA_TABLE, ST_GROUP_FB, ST_CTA_FB, ST_WARP_FB,
                  ST_CHUNK_FB, ST_SERIAL,
                  // MCR_XDOT_DEBUG builds: self-checks of every piece against element-by-element sums
                  ST_DBG_RUN, ST_DBG_RUN_BAD, ST_DBG_TAB, ST_DBG_TAB_BAD, ST_DBG_TR, ST_DBG_TR_BAD,
                  ST_DBG_LEVEL_BAD, ST_COUNT };

struct Run {        // 32 B
    double d0, d1;  // displacement for a start of even / odd index
    double x;       // excursion bound
    int e, neg;     // binade; e = E_HARD (not a run) or E_EMPTY (identity)
};
struct Lane {       // 32 B: one candidate of a table
    double out, lo, hi;
    int km, hole;
};
struct Hdr {        // 64 B
    int kind, neg, e, pad;
    unsigned long long mb0;  // table: magnitude bits of candidate 0
    double d0, d1, x;        // run
    double pred;             // predicted start of the piece (window of later tables)
    double pad2;
};
struct Desc {       // 1088 B
    Hdr h;
    Lane l[32];
};

// One sequence: sum_{i=a}^{b-1} u[i] v[i] in index order. CTAs [cta0, cta0 + ncta).
struct Seq {
    const double* u;
    const double* v;
    long long a, b;
    int cta0, ncta;
};

// Scratch (device memory owned by the plan).
struct Scratch {
    Desc* cta;             // [grid]
    Desc* warp;            // [grid * NW]
    Run* runs;             // [grid * NT]
    double* lb_val;        // [grid] look-back: CTA totals (predictions only)
    int* lb_flag;          // [grid]
    unsigned* ticket;      // [nseq]
    unsigned* done;        // [nseq]
    unsigned* flags;       // [nseq]: bit 0 = some product is not -0.0, bit 1 = non-finite product
    double* result;        // [nseq]
    unsigned* all_done;    // [1]
    unsigned long long* stats;  // [ST_COUNT] or null
};

struct Args {
    const Seq* seqs;
    int nseq;
    int nseq0;      // sequences of the first dot; the rest belong to the second
    int ndot;       // 1 or 2
    int pardots;    // combine the sequences of a dot as the reference's block partials
    int E;
    Scratch S;
    double* out;    // test mode: the dot results go here (no solver state)
};

__device__ __forceinline__ unsigned long long bt(double v) { return (unsigned long long)__double_as_longlong(v); }
__device__ __forceinline__ double fb(unsigned long long b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ int dexp(unsigned long long b) { return (int)((b >> 52) & 0x7ff); }
__device__ __forceinline__ void stat(const Scratch& S, int k) {
    if (S.stats) atomicAdd(S.stats + k, 1ull);
}

// parity of D/u for a displacement D that is a multiple of u = ulp(binade e) (e >= RUN_MIN_E,
// so a non-zero D is a normal number): the bit of D's significand that has weight u
__device__ __forceinline__ int disp_parity(double D, int e) {
    const unsigned long long b = bt(D);
    const int sh = e - dexp(b);
    if (D == 0.0 || sh < 0 || sh > 52) return 0;
    return (int)((((b & MANT) | (1ull << 52)) >> sh) & 1ull);
}

// a then b (same binade, or either empty)
__device__ __forceinline__ Run run_merge(const Run& a, const Run& b) {
    if (a.e == E_EMPTY) return b;
    if (b.e == E_EMPTY) return a;
    Run r;
    r.e = a.e;
    r.neg = a.neg;
    r.d0 = dadd(a.d0, disp_parity(a.d0, a.e) ? b.d1 : b.d0);        // start index even
    r.d1 = dadd(a.d1, (1 ^ disp_parity(a.d1, a.e)) ? b.d1 : b.d0);  // start index odd
    r.x = __dadd_ru(a.x, b.x);
    return r;
}

// Does the run R apply to a start v? If so v advances and the start-shift constraints of the
// carried piece (lo, hi, km) tighten.
__device__ __forceinline__ bool run_apply(const Run& R, double& v, double& lo, double& hi, int& km) {
    if (R.e == E_EMPTY) return true;
    const unsigned long long b = bt(v);
    const int ng = (int)(b >> 63);
    if (R.e == E_HARD || dexp(b) != R.e || ng != R.neg) return false;
    const double lowlim = __dadd_ru(fb(((unsigned long long)R.e << 52) | 1ull), R.x);     // 2^e + u + x
    const double highlim = __dsub_rd(fb(((unsigned long long)R.e << 52) | MANT), R.x);    // 2^(e+1) - u - x
    const double av = fabs(v);
    if (!(av >= lowlim && av <= highlim)) return false;
    double a, c;
    if (!ng) { a = __dsub_ru(lowlim, v); c = __dsub_rd(highlim, v); }
    else { a = __dsub_ru(-highlim, v); c = __dsub_rd(-lowlim, v); }
    lo = fmax(lo, a);
    hi = fmin(hi, c);
    km = max(km, R.e - 1074);
    v = dadd(v, (b & 1ull) ? R.d1 : R.d0);  // exact: stays on the grid of the binade
    return true;
}

// The value v (a partial sum of the carried piece) must stay in its binade, one ulp clear of
// its ends, under the start shift; zero / subnormal / non-finite: no shift at all.
__device__ __forceinline__ void value_slack(double v, double& lo, double& hi, int& km) {
    const unsigned long long b = bt(v);
    const int ex = dexp(b);
    if (ex == 0 || ex == 0x7ff) {
        lo = fmax(lo, 0.0);
        hi = fmin(hi, 0.0);
        return;
    }
    const double top = fb(b | MANT), bot = fb((b & ~MANT) | 1ull);  // +-(2^(e+1) - u), +-(2^e + u)
    lo = fmax(lo, dsub(fmin(top, bot), v));  // exact (same binade)
    hi = fmin(hi, dsub(fmax(top, bot), v));
    km = max(km, ex - 1074);
}

__device__ __forceinline__ void sim_step(double& v, double p, double& lo, double& hi, int& km) {
    v = dadd(v, p);
    value_slack(v, lo, hi, km);
}

// Warp-collective: evaluate the table (this lane holds entry `lane`; mb0/tneg uniform) at
// this lane's s. On success out = the table's value at s and lo/hi/km tighten.
__device__ __forceinline__ bool table_eval(unsigned long long mb0, int tneg, const Lane& T, double s,
                                           double& out, double& lo, double& hi, int& km) {
    const unsigned long long b = bt(s);
    const unsigned long long mb = b & ~SGN;
    const long long d = (long long)(mb - mb0);
    const int k = (int)(d & 31);
    double o = __shfl_sync(FULL, T.out, k);
    const double l = __shfl_sync(FULL, T.lo, k);
    const double h = __shfl_sync(FULL, T.hi, k);
    const int kmk = __shfl_sync(FULL, T.km, k);
    const int hole = __shfl_sync(FULL, T.hole, k);
    if (hole || (int)(b >> 63) != tneg) return false;
    double dl = 0.0;
    if (!(d >= 0 && d < 32)) {
        const unsigned long long cb = mb0 + (unsigned long long)k;
        const int ce = dexp(cb), se = dexp(mb);
        if (ce != se || se == 0 || se == 0x7ff) return false;
        dl = dsub(s, fb(cb | ((unsigned long long)tneg << 63)));  // exact
        if (!(dl >= l && dl <= h)) return false;
        const int sh = kmk - (ce - 1075);
        if (sh > 5 && (sh >= 63 || ((d - k) & ((1ll << sh) - 1)))) return false;
        o = dadd(o, dl);  // exact
    }
    lo = fmax(lo, __dsub_ru(l, dl));
    hi = fmin(hi, __dsub_rd(h, dl));
    km = max(km, kmk);
    out = o;
    return true;
}

// Same for a uniform scalar s (every lane gets the result).
__device__ __forceinline__ bool table_eval_scalar(unsigned long long mb0, int tneg, const Lane& T, double& s) {
    double lo = -INFINITY, hi = INFINITY, out = 0.0;
    int km = KM_NONE;
    const bool ok = table_eval(mb0, tneg, T, s, out, lo, hi, km);
    if (ok) s = out;
    return ok;
}

__device__ __forceinline__ unsigned long long window_mb0(double pred) {
    const unsigned long long mb = bt(pred) & ~SGN;
    unsigned long long m0 = mb > 16 ? mb - 16 : 0;
    const unsigned long long lim = (0x7feull << 52) | MANT;  // largest finite
    if (m0 + 31 > lim) m0 = lim - 31;
    return m0;
}
__device__ __forceinline__ int window_neg(double pred) { return (int)(bt(pred) >> 63); }
__device__ __forceinline__ double cand(unsigned long long mb0, int neg, int j) {
    return fb((mb0 + (unsigned long long)j) | ((unsigned long long)neg << 63));
}

__device__ __forceinline__ Run hdr_run(const Hdr& h) {
    Run r;
    r.d0 = h.d0; r.d1 = h.d1; r.x = h.x; r.e = h.e; r.neg = h.neg;
    return r;
}
__device__ __forceinline__ void hdr_set_run(Hdr& h, const Run& r, double pred) {
    h.kind = K_RUN; h.e = r.e; h.neg = r.neg; h.d0 = r.d0; h.d1 = r.d1; h.x = r.x;
    h.pred = pred; h.mb0 = 0; h.pad = 0; h.pad2 = 0.0;
}
__device__ __forceinline__ bool runs_compatible(const Run& a, const Run& b) {
    return a.e == E_EMPTY || b.e == E_EMPTY || (a.e != E_HARD && a.e == b.e && a.neg == b.neg);
}

// Warp-collective: carry this lane's value (lo/hi/km) through one piece (run or table).
// A table piece's entries are read from `D` (shared or global memory).
__device__ __forceinline__ bool piece_apply(const Desc* D, double& v, double& lo, double& hi, int& km) {
    const int lane = threadIdx.x & 31;
    const int kind = D->h.kind;
    if (kind == K_RUN) {
        const Run R = hdr_run(D->h);
        return run_apply(R, v, lo, hi, km);
    }
    const Lane T = D->l[lane];
    value_slack(v, lo, hi, km);
    double out;
    const bool ok = table_eval(D->h.mb0, D->h.neg, T, v, out, lo, hi, km);
    if (ok) v = out;
    return ok;
}

// ---------------------------------------------------------------- scalar walks (fallbacks)
// Uniform across the warp: every lane carries the same value.
__device__ bool piece_scalar(const Desc* D, double& v) {
    if (D->h.kind == K_RUN) {
        double lo = -INFINITY, hi = INFINITY;
        int km = KM_NONE;
        return run_apply(hdr_run(D->h), v, lo, hi, km);
    }
    const Lane T = D->l[threadIdx.x & 31];
    return table_eval_scalar(D->h.mb0, D->h.neg, T, v);
}

__device__ void walk_chunk(const Args& A, const Seq& q, int slot, int ci, int t, double& v) {
    const Run R = A.S.runs[(size_t)slot * NT + t];
    double lo = -INFINITY, hi = INFINITY;
    int km = KM_NONE;
    if (R.e == E_EMPTY || run_apply(R, v, lo, hi, km)) return;
    stat(A.S, ST_CHUNK_FB);
    const long long c0 = q.a + (long long)ci * NT * A.E;
    const long long i0 = c0 + (long long)t * A.E;
    const long long i1 = min(min(q.b, c0 + (long long)NT * A.E), i0 + A.E);
    for (long long i = i0; i < i1; ++i) v = dadd(v, dmul(__ldcg(q.u + i), __ldcg(q.v + i)));
}

__device__ void walk_warp(const Args& A, const Seq& q, int slot, int ci, int w, double& v) {
    if (piece_scalar(A.S.warp + (size_t)slot * NW + w, v)) return;
    stat(A.S, ST_WARP_FB);
    for (int c = 0; c < 32; ++c) walk_chunk(A, q, slot, ci, w * 32 + c, v);
}

__device__ void walk_cta(const Args& A, const Seq& q, int ci, double& v) {
    const int slot = q.cta0 + ci;
    if (piece_scalar(A.S.cta + slot, v)) return;
    stat(A.S, ST_CTA_FB);
    for (int w = 0; w < NW; ++w) walk_warp(A, q, slot, ci, w, v);
}

#ifdef MCR_XDOT_DEBUG
__device__ double dbg_serial(const Seq& q, long long i0, long long i1, double v) {
    for (long long i = i0; i < i1; ++i) v = dadd(v, dmul(__ldcg(q.u + i), __ldcg(q.v + i)));
    return v;
}
__device__ __forceinline__ bool same_bits(double a, double b) { return bt(a) == bt(b); }
// this lane's table entry (start cand) over elements [i0, i1): exact value, and one translation
__device__ void dbg_check_lane(const Scratch& S, const Seq& q, long long i0, long long i1, double c,
                               const Lane& Lx, int level) {
    if (Lx.hole) return;
    const double want = dbg_serial(q, i0, i1, c);
    stat(S, ST_DBG_TAB);
    if (!same_bits(want, Lx.out)) {
        stat(S, ST_DBG_TAB_BAD);
        if (S.stats) printf("xdot dbg: level %d table lane value c=%a want=%a got=%a [%lld,%lld)\n", level, c, want, Lx.out, i0, i1);
        return;
    }
    const unsigned long long cb = bt(c);
    const int ce = dexp(cb);
    if (ce == 0 || ce == 0x7ff) return;
    const int ex = max(Lx.km, ce - 1075 + 5);
    for (int sgn = -1; sgn <= 1; sgn += 2) {
        const double dl = sgn * fb((unsigned long long)(ex + 1023) << 52);  // 2^ex
        if (!(dl >= Lx.lo && dl <= Lx.hi)) continue;
        const double c2 = dadd(c, dl);
        if (dexp(bt(c2)) != ce) continue;
        stat(S, ST_DBG_TR);
        const double w2 = dbg_serial(q, i0, i1, c2);
        if (!same_bits(w2, dadd(Lx.out, dl))) {
            stat(S, ST_DBG_TR_BAD);
            if (S.stats) printf("xdot dbg: level %d translation c=%a dl=%a km=%d lo=%a hi=%a want=%a got=%a\n", level, c, dl, Lx.km, Lx.lo, Lx.hi, w2, dadd(Lx.out, dl));
        }
    }
}
#endif

// ---------------------------------------------------------------- the kernel pieces
// Phase 1-3 of a CTA: products -> thread runs -> warp pieces -> CTA piece (published).
// Returns the CTA's local index (its ticket) in the sequence.
__device__ int build_cta(const Args& A, const Seq& q, int si, double* sp, Run* s_runs, Desc* s_wd,
                         double* s_red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const Scratch& S = A.S;
    const int E = A.E;
    __shared__ int s_tk;
    __shared__ unsigned s_fl;
    __shared__ double s_pred;
    if (tid == 0) {
        s_tk = (int)atomicAdd(S.ticket + si, 1u);
        s_fl = 0u;
    }
    __syncthreads();
    const int ci = s_tk;
    const int slot = q.cta0 + ci;
    const long long c0 = q.a + (long long)ci * NT * E;
    const long long c1 = min(q.b, c0 + (long long)NT * E);
    const int len = (int)max(0ll, c1 - c0);
    // products, coalesced, into shared memory
    unsigned fl = 0u;
    for (int k = tid; k < len; k += NT) {
        const double p = dmul(__ldcg(q.u + c0 + k), __ldcg(q.v + c0 + k));
        const unsigned long long pb = bt(p);
        fl |= (pb != SGN) ? 1u : 0u;
        fl |= (dexp(pb) == 0x7ff) ? 2u : 0u;
        sp[k] = p;
    }
    if (fl) atomicOr(&s_fl, fl);
    __syncthreads();
    // pass 1 over this thread's elements: plain sum (prediction) and sum of |p|
    const int t0 = tid * E;
    const int tl = max(0, min(E, len - t0));
    double ts = 0.0, ta = 0.0;
    for (int k = 0; k < tl; ++k) {
        const double p = sp[t0 + k];
        ts = dadd(ts, p);
        ta = __dadd_ru(ta, fabs(p));
    }
    // block exclusive scan of ts
    double inc = ts;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double o = __shfl_up_sync(FULL, inc, off);
        if (lane >= off) inc = dadd(inc, o);
    }
    double exc = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) exc = 0.0;
    if (lane == 31) s_red[warp] = inc;
    __syncthreads();
    double wexc = 0.0, total = 0.0;
    for (int w = 0; w < NW; ++w) {
        if (w < warp) wexc = dadd(wexc, s_red[w]);
        total = dadd(total, s_red[w]);
    }
    // look-back: publish this CTA's total, collect the totals of the CTAs before it
    if (tid == 0) {
        S.lb_val[slot] = total;
        __threadfence();
        atomicExch(S.lb_flag + slot, 1);
        if (s_fl) atomicOr(S.flags + si, s_fl);
    }
    double acc = 0.0;
    for (int j = tid; j < ci; j += NT) {
        volatile int* f = S.lb_flag + q.cta0 + j;
        while (*f == 0) {
        }
        __threadfence();
        acc = dadd(acc, __ldcg(S.lb_val + q.cta0 + j));
    }
    __syncthreads();  // s_red reuse
    acc = group_sum<NW, 0>(acc, s_red);
    if (tid == 0) s_pred = acc;
    __syncthreads();
    const double pred_cta = s_pred;
    const double pred = dadd(pred_cta, dadd(wexc, exc));  // predicted start of this thread's elements
    // pass 2: this thread's run
    Run R;
    R.d0 = R.d1 = R.x = 0.0;
    R.neg = 0;
    if (tl == 0) {
        R.e = E_EMPTY;
    } else {
        R.e = E_HARD;
        const unsigned long long pb = bt(pred);
        const int e = dexp(pb);
        const int ng = (int)(pb >> 63);
        if (e >= RUN_MIN_E && e <= 0x7f0 && !(s_fl & 2u)) {
            const double u = fb((unsigned long long)(e - 52) << 52);
            const double X = __dadd_ru(ta, __dmul_ru((double)tl, u));
            const double quarter = fb((unsigned long long)(e - 2) << 52);
            const double margin = fb((unsigned long long)(e - 24) << 52);
            const double lowlim = dadd(fb(((unsigned long long)e << 52) | 1ull), X);
            const double highlim = dsub(fb(((unsigned long long)e << 52) | MANT), X);
            const double ap = fabs(pred);
            if (X < quarter && ap >= dadd(lowlim, margin) && ap <= dsub(highlim, margin)) {
                const double ref0 = fb(((unsigned long long)ng << 63) | ((unsigned long long)e << 52) | (1ull << 51));
                const double ref1 = fb(bt(ref0) + 1ull);
                double s0 = ref0, s1 = ref1;
                for (int k = 0; k < tl; ++k) {
                    const double p = sp[t0 + k];
                    s0 = dadd(s0, p);
                    s1 = dadd(s1, p);
                }
                R.d0 = dsub(s0, ref0);
                R.d1 = dsub(s1, ref1);
                R.x = X;
                R.e = e;
                R.neg = ng;
            }
        }
    }
    s_runs[tid] = R;
    S.runs[(size_t)slot * NT + tid] = R;
#ifdef MCR_XDOT_DEBUG
    if (R.e != E_HARD && R.e != E_EMPTY) {
        for (int t = 0; t < 3; ++t) {
            double v = t == 0 ? pred : (t == 1 ? fb(bt(pred) + 1ull) : fb(bt(pred) + 2ull));
            double lo = -INFINITY, hi = INFINITY, v0 = v;
            int km = KM_NONE;
            if (!run_apply(R, v, lo, hi, km)) continue;
            stat(S, ST_DBG_RUN);
            const double want = dbg_serial(q, c0 + t0, c0 + t0 + tl, v0);
            if (!same_bits(want, v)) {
                stat(S, ST_DBG_RUN_BAD);
                if (S.stats) printf("xdot dbg: run e=%d neg=%d d0=%a d1=%a x=%a start=%a want=%a got=%a\n", R.e, R.neg, R.d0, R.d1, R.x, v0, want, v);
            }
        }
    }
#endif
    if (R.e == E_HARD && tl > 0 && S.stats) stat(S, ST_HARD);
    __syncwarp();
    // warp piece: one merged run when all 32 thread runs share a binade, else a table
    const int first = __ffs(__ballot_sync(FULL, R.e != E_EMPTY)) - 1;
    const int e0 = __shfl_sync(FULL, R.e, max(first, 0));
    const int n0 = __shfl_sync(FULL, R.neg, max(first, 0));
    const bool same = R.e == E_EMPTY || (R.e != E_HARD && R.e == e0 && R.neg == n0);
    const double wpred = __shfl_sync(FULL, pred, 0);
    Desc* WD = s_wd + warp;
    if (__all_sync(FULL, same)) {
        Run M = R;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            Run o;
            o.d0 = __shfl_down_sync(FULL, M.d0, off);
            o.d1 = __shfl_down_sync(FULL, M.d1, off);
            o.x = __shfl_down_sync(FULL, M.x, off);
            o.e = __shfl_down_sync(FULL, M.e, off);
            o.neg = __shfl_down_sync(FULL, M.neg, off);
            if ((lane & (2 * off - 1)) == 0) M = run_merge(M, o);
        }
        if (lane == 0) hdr_set_run(WD->h, M, wpred);
    } else {
        if (S.stats && lane == 0) stat(S, ST_WARP_TABLE);
        const unsigned long long mb0 = window_mb0(wpred);
        const int wn = window_neg(wpred);
        double v = cand(mb0, wn, lane), lo = -INFINITY, hi = INFINITY;
        int km = KM_NONE;
        for (int c = 0; c < 32; ++c) {
            const Run Rc = s_runs[warp * 32 + c];
            if (run_apply(Rc, v, lo, hi, km)) continue;
            const int b0 = (warp * 32 + c) * E;
            const int bl = max(0, min(E, len - b0));
            for (int k = 0; k < bl; ++k) sim_step(v, sp[b0 + k], lo, hi, km);
        }
        Lane Lx;
        Lx.out = v; Lx.lo = lo; Lx.hi = hi; Lx.km = km;
        Lx.hole = dexp(bt(v)) == 0x7ff ? 1 : 0;
        WD->l[lane] = Lx;
#ifdef MCR_XDOT_DEBUG
        dbg_check_lane(S, q, c0 + warp * 32 * E, min(c1, c0 + (long long)(warp + 1) * 32 * E), cand(mb0, wn, lane), Lx, 1);
#endif
        if (lane == 0) {
            WD->h.kind = K_TABLE; WD->h.neg = wn; WD->h.e = 0; WD->h.mb0 = mb0; WD->h.pred = wpred;
            WD->h.d0 = WD->h.d1 = WD->h.x = 0.0; WD->h.pad = 0; WD->h.pad2 = 0.0;
        }
    }
    __syncthreads();
    // global copies of the warp pieces (fallback walks)
    {
        const int words = (int)(sizeof(Desc) / sizeof(double)) * NW;
        const double* src = (const double*)s_wd;
        double* dst = (double*)(S.warp + (size_t)slot * NW);
        for (int k = tid; k < words; k += NT) dst[k] = src[k];
    }
    // CTA piece (warp 0)
    if (warp == 0) {
        bool allrun = true;
        Run M;
        M.e = E_EMPTY; M.neg = 0; M.d0 = M.d1 = M.x = 0.0;
        for (int w = 0; w < NW; ++w) {
            const Hdr& h = s_wd[w].h;
            if (h.kind != K_RUN) { allrun = false; break; }
            const Run r = hdr_run(h);
            if (!runs_compatible(M, r)) { allrun = false; break; }
            M = run_merge(M, r);
        }
        Desc* CD = S.cta + slot;
        if (allrun) {
            if (lane == 0) hdr_set_run(CD->h, M, pred_cta);
        } else {
            if (S.stats && lane == 0) stat(S, ST_CTA_TABLE);
            const unsigned long long mb0 = window_mb0(pred_cta);
            const int cn = window_neg(pred_cta);
            double v = cand(mb0, cn, lane), lo = -INFINITY, hi = INFINITY;
            int km = KM_NONE;
            int hole = 0;
            for (int w = 0; w < NW; ++w) {
                const bool ok = piece_apply(s_wd + w, v, lo, hi, km);  // collective
                hole |= ok ? 0 : 1;
            }
            Lane Lx;
            Lx.out = v; Lx.lo = lo; Lx.hi = hi; Lx.km = km;
            Lx.hole = (hole || dexp(bt(v)) == 0x7ff) ? 1 : 0;
            CD->l[lane] = Lx;
#ifdef MCR_XDOT_DEBUG
            dbg_check_lane(S, q, c0, c1, cand(mb0, cn, lane), Lx, 2);
#endif
            if (lane == 0) {
                CD->h.kind = K_TABLE; CD->h.neg = cn; CD->h.e = 0; CD->h.mb0 = mb0; CD->h.pred = pred_cta;
                CD->h.d0 = CD->h.d1 = CD->h.x = 0.0; CD->h.pad = 0; CD->h.pad2 = 0.0;
            }
        }
    }
    return ci;
}

// The last CTA of a sequence: compose the CTA pieces and walk the true value from 0.0.
__device__ double root(const Args& A, const Seq& q, int si, Desc* s_gd) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Scratch& S = A.S;
    const int n = q.ncta;
    const int Q = (n + NW - 1) / NW;
    __shared__ double s_v;
    __shared__ int s_nf;
    if (threadIdx.x == 0) s_nf = (int)((__ldcg((const int*)S.flags + si) >> 1) & 1);
    __syncthreads();
    if (s_nf) {  // a non-finite product: the reference's IEEE chain, element by element
        if (warp == 0) {
            stat(S, ST_SERIAL);
            double v = 0.0;
            for (long long i = q.a; i < q.b; ++i) v = dadd(v, dmul(__ldcg(q.u + i), __ldcg(q.v + i)));
            if (lane == 0) s_v = v;
        }
        __syncthreads();
        return s_v;
    }
    // groups 1..NW-1: tables over Q consecutive CTA pieces
    if (warp > 0) {
        const int g0 = warp * Q, g1 = min(n, g0 + Q);
        Desc* G = s_gd + warp;
        if (g0 < g1) {
            const double gp = __ldcg(&S.cta[q.cta0 + g0].h.pred);
            const unsigned long long mb0 = window_mb0(gp);
            const int gn = window_neg(gp);
            double v = cand(mb0, gn, lane), lo = -INFINITY, hi = INFINITY;
            int km = KM_NONE, hole = 0;
            for (int c = g0; c < g1; ++c) {
                const bool ok = piece_apply(S.cta + q.cta0 + c, v, lo, hi, km);
                hole |= ok ? 0 : 1;
            }
            Lane Lx;
            Lx.out = v; Lx.lo = lo; Lx.hi = hi; Lx.km = km;
            Lx.hole = (hole || dexp(bt(v)) == 0x7ff) ? 1 : 0;
            G->l[lane] = Lx;
#ifdef MCR_XDOT_DEBUG
            dbg_check_lane(S, q, q.a + (long long)g0 * NT * A.E, min(q.b, q.a + (long long)g1 * NT * A.E), cand(mb0, gn, lane), Lx, 3);
#endif
            if (lane == 0) {
                G->h.kind = K_TABLE; G->h.neg = gn; G->h.e = 0; G->h.mb0 = mb0; G->h.pred = gp;
            }
        }
    } else {
        // group 0 from the exact start
        double v = 0.0;
        for (int c = 0; c < min(n, Q); ++c) walk_cta(A, q, c, v);
        if (lane == 0) s_v = v;
    }
    __syncthreads();
    if (warp == 0) {
        double v = s_v;
        for (int g = 1; g < NW; ++g) {
            const int g0 = g * Q, g1 = min(n, g0 + Q);
            if (g0 >= g1) break;
            if (piece_scalar(s_gd + g, v)) continue;
            stat(S, ST_GROUP_FB);
            for (int c = g0; c < g1; ++c) walk_cta(A, q, c, v);
        }
        // cumsum starts from p_0 itself: -0.0 survives only when every product is -0.0
        if (v == 0.0 && q.b > q.a && !(__ldcg((const int*)S.flags + si) & 1)) v = -0.0;
        if (lane == 0) s_v = v;
    }
    __syncthreads();
    return s_v;
}

// Reset the sequence's counters and look-back flags for the next launch (the root only).
__device__ void reset_seq(const Args& A, const Seq& q, int si) {
    for (int j = threadIdx.x; j < q.ncta; j += NT) A.S.lb_flag[q.cta0 + j] = 0;
    if (threadIdx.x == 0) {
        A.S.ticket[si] = 0u;
        A.S.done[si] = 0u;
        A.S.flags[si] = 0u;
    }
}

__device__ __forceinline__ int find_seq(const Seq* seqs, int nseq, int cta) {
    int lo = 0, hi = nseq - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (seqs[mid].cta0 <= cta) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Shared memory: NT*E products, NT thread runs, NW warp pieces (also the root's group tables).
__host__ __device__ constexpr size_t smem_bytes(int E) {
    return sizeof(double) * (size_t)NT * (size_t)E + sizeof(Run) * NT + sizeof(Desc) * NW;
}

// Per-launch body. Returns true in the one CTA that finished the last sequence, with the
// dots (block partials combined when pardots) in d[0], d[1]; thread 0 only.
__device__ bool xdot_body(const Args& A, double* d) {
    extern __shared__ __align__(16) unsigned char xsm[];
    double* sp = (double*)xsm;
    Run* s_runs = (Run*)(xsm + sizeof(double) * (size_t)NT * (size_t)A.E);
    Desc* s_wd = (Desc*)(s_runs + NT);
    __shared__ double s_red[NW];
    __shared__ int s_flag;
    const int si = find_seq(A.seqs, A.nseq, blockIdx.x);
    const Seq q = A.seqs[si];
    build_cta(A, q, si, sp, s_runs, s_wd, s_red);
    // the last CTA of the sequence composes it
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_flag = atomicAdd(A.S.done + si, 1u) == (unsigned)(q.ncta - 1);
    __syncthreads();
    if (!s_flag) return false;
    __threadfence();
    const double r = root(A, q, si, s_wd);
    if (threadIdx.x == 0) A.S.result[si] = r;
    reset_seq(A, q, si);
    // the last sequence combines
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_flag = atomicAdd(A.S.all_done, 1u) == (unsigned)(A.nseq - 1);
    __syncthreads();
    if (!s_flag || threadIdx.x != 0) return false;
    __threadfence();
    *A.S.all_done = 0u;
    for (int k = 0; k < 2; ++k) {
        const int s0 = k == 0 ? 0 : A.nseq0, s1 = k == 0 ? A.nseq0 : A.nseq;
        double acc = 0.0;
        if (k < A.ndot) {
            if (!A.pardots) {
                acc = __ldcg(A.S.result + s0);
            } else {  // solvers.py:392-396: acc = 0.0; acc += part, ascending block order
                for (int s = s0; s < s1; ++s) acc = dadd(acc, __ldcg(A.S.result + s));
            }
        }
        d[k] = acc;
    }
    if (A.out) {
        A.out[0] = d[0];
        A.out[1] = d[1];
        for (int s = 0; s < A.nseq; ++s) A.out[2 + s] = __ldcg(A.S.result + s);
    }
    return true;
}

}  // namespace xd
}  // namespace mcr

namespace mcr {

// Reference-order dots of one BiCGStab reduction point (W = SQ_S0 / SQ_V / SQ_T / SQ_E), or
// the test entry (W = SQ_TEST: results to A.out, no solver state).
enum : int { SQ_TEST = 4 };
template <int W>
__global__ void __launch_bounds__(xd::NT) k_xdot(xd::Args A, SolveState* st) {
    griddep_wait();
    griddep_launch();
    if (W != SQ_TEST && st->stop) return;  // stopped earlier in this iteration (uniform)
    double d[2];
    if (!xd::xdot_body(A, d)) return;
    if constexpr (W == SQ_S0) fin_s0(st, d[0]);
    else if constexpr (W == SQ_V) fin_v(st, d[0]);
    else if constexpr (W == SQ_T) fin_t(st, d[0], d[1]);
    else if constexpr (W == SQ_E) {
        fin_e(st, d[0]);
        graph_continue(st);
    }
}

}  // namespace mcr
