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
//   d[0] / d[1] (start index even / odd) and the range [lo, hi] its partial sums move through:
//   for ANY start s in that binade with s + [lo, hi] one ulp clear of the binade's ends, the
//   stretch ends at s + d[parity(s)]. Runs of one binade compose associatively. d, lo, hi
//   come from summing the stretch from two reference starts in the middle of the binade.
// * Where the sum changes binade (crossings, passes near zero) a "table" describes the
//   stretch as a function of its start: 32 consecutive candidate starts (doubles around a
//   predicted start) are carried through the stretch exactly (runs applied per candidate,
//   anything else added element by element), and each candidate keeps the range [lo, hi] of
//   start shifts delta that leave every partial sum inside its binade one ulp clear of its
//   ends, plus the coarsest grid 2^km it passed. A start s = cand_k + delta in cand_k's
//   binade with delta in [lo, hi] and delta = 0 mod 2^km (k = the candidate congruent to s
//   mod 32 ulps) ends at out_k + delta: every rounding step commutes with such a shift.
// * Tables compose (evaluate the second at the first's outputs): that is how warps and CTAs
//   are stitched together. Predicted starts come from a plain (non-exact) prefix sum of the
//   products; a prediction only has to land in the right binade for runs and within the
//   translation range for tables. Nothing is assumed: every use of a run or table is
//   checked, and where a check fails the stretch is recomputed from the exact start (a CTA's
//   range rebuilt with its true start; a thread's elements added one by one), so the result
//   is the reference's bits for every input (NaN / Inf / overflow / -0.0 included); only the
//   time depends on how often that happens.
//
// One launch per reduction point: a CTA owns NT*E consecutive elements of one sequence
// (thread t owns E consecutive ones, E odd so the shared-memory reads are conflict free),
// builds thread runs -> warp pieces -> a CTA piece and publishes it; the last CTA of the
// sequence stages the CTA pieces in shared memory, composes 7 groups of them (warps 1..7)
// while warp 0 carries the true value from 0.0 through group 0, then through the group
// tables, and runs the BiCGStab scalar step. Sequences: one per dot, or one per row block
// when the reference's parallel_dot_products mode is on (solvers.py:384-396: each block
// summed sequentially, block results added in ascending order from 0.0).
#pragma once

#include "common.cuh"

namespace mcr {
namespace xd {

#ifndef XD_NT
#define XD_NT 256  // threads per CTA (C2 BiCGStab: 512 -> 27.3 ms, 256 -> 25.2 ms, 128 -> 32.8 ms)
#endif
constexpr int NT = XD_NT;
#ifndef XD_WALK_MAX
#define XD_WALK_MAX 1  // CTA fold levels whose lanes re-add a stretch a table does not take (above: holes;
                       // C2 BiCGStab: 0 levels 24.25 ms, 1: 23.70, 2: 23.80, all 3: 25.04)
#endif
#ifndef XD_SIM_UNROLL
#define XD_SIM_UNROLL 12  // C2 BiCGStab: 2: 24.36 ms, 4: 23.74, 8: 23.55, 12: 23.47, 16: 24.07
#endif
#ifndef XD_RUN_UNROLL
#define XD_RUN_UNROLL 4  // 2: 23.82, 8: 23.76
#endif
#ifndef XD_MARGIN
#define XD_MARGIN 40  // a thread run keeps its partial sums 2^(52 - XD_MARGIN) ulps clear of the binade ends
                      // (C2 BiCGStab: 36, 40, 44, 48 all 23.68 ms)
#endif
constexpr int NW = NT / 32;
constexpr int SIM_UNROLL = XD_SIM_UNROLL, RUN_UNROLL = XD_RUN_UNROLL;
constexpr int EMAX = 79;  // large n: products per CTA (C5 BiCGStab ms per iteration, 20M | 200M: E 31: 7.13 | -, 47: - | 74.6, 63: 6.25 | 68.0, 79: 6.26 | 65.1, 95: 6.91 | 69.8 -- the root's stage runs out of room)
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
                  ST_DBG_SPARE,
                  // why the true value could not use a piece (debug builds)
                  ST_R_HOLE, ST_R_SIGN, ST_R_EXP, ST_R_SLACK, ST_R_KM, ST_R_RUN_BIN, ST_R_RUN_BOUND,
                  // MCR_XDOT_TIMING builds: SM cycles per phase (CTA phases summed over CTAs)
                  ST_T_LOAD, ST_T_LOOKBACK, ST_T_RUNS, ST_T_CTA, ST_T_ROOT_GROUPS, ST_T_ROOT_WALK,
                  ST_T_LAUNCHES,
                  // MCR_XDOT_TIMING: ns per launch (globaltimer): entry skew, entry -> last build end,
                  // last build end -> root start... root end, and min-entry -> root end
                  ST_G_SKEW, ST_G_BUILD, ST_G_ROOT, ST_G_TOTAL, ST_G_MIN_ENTRY, ST_G_MAX_ENTRY,
                  ST_G_MAX_BUILD,
                  // per-launch max of the CTA phases (slots), summed over launches
                  ST_M_LOAD, ST_M_LOOKBACK, ST_M_RUNS, ST_M_CTA, ST_MS_LOAD, ST_MS_LOOKBACK, ST_MS_RUNS,
                  ST_MS_CTA, ST_SIMS_WARP, ST_SIMS_CTA,
                  ST_W_CHAIN, ST_W_MERGE, ST_W_TABLE, ST_WS_CHAIN, ST_WS_MERGE, ST_WS_TABLE,
                  ST_W_SLOWEST, ST_COUNT };

struct Run {        // 56 B
    double d[2];    // displacement for a start of even / odd index
    double lo[2], hi[2];  // range of the partial sums' displacement from the start (per start parity)
    int e, neg;     // binade; e = E_HARD (not a run) or E_EMPTY (identity)
};
struct LaneR {      // one candidate of a table, as carried in registers
    double out, lo, hi;
    int km, hole;
};
struct LaneS {      // ... and as stored: slack bounds rounded inwards to float (conservative)
    double out;
    float lo, hi;
};
struct Hdr {        // 80 B
    int kind, neg, e, pad;
    unsigned long long mb0;  // table: magnitude bits of candidate 0
    double pred;             // predicted start of the piece (window of later tables)
    double d[2], lo[2], hi[2];  // run
};
struct Desc {       // 720 B
    Hdr h;
    LaneS l[32];
    int kmh[32];    // km << 1 | hole
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
    Desc* cta;             // [grid] the CTA pieces
    Desc* warp;            // [grid * NW] the warp pieces (the root's fallback)
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
    int stage;      // CTA pieces the root stages in shared memory at a time
    int upto;       // diagnostics (MCR_XDOT_UPTO): stop after build phase 1..4 (0 = complete)
    Scratch S;
    double* out;    // test mode: the dot results go here (no solver state)
};

__device__ __forceinline__ unsigned long long bt(double v) { return (unsigned long long)__double_as_longlong(v); }
__device__ __forceinline__ double fb(unsigned long long b) { return __longlong_as_double((long long)b); }
__device__ __forceinline__ int dexp(unsigned long long b) { return (int)((b >> 52) & 0x7ff); }
__device__ __forceinline__ void stat(const Scratch& S, int k) {
    if (S.stats) atomicAdd(S.stats + k, 1ull);
}
#ifdef MCR_XDOT_TIMING
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define XT_MARK(t) long long t = (long long)gtime()
#define XT_ADD(S, k, t0) do { if ((S).stats && threadIdx.x == 0) { const unsigned long long d_ = (unsigned long long)((long long)gtime() - (t0)); atomicAdd((S).stats + (k), d_); if ((k) >= ST_T_LOAD && (k) <= ST_T_CTA) atomicMax((S).stats + ST_M_LOAD + ((k) - ST_T_LOAD), d_); } } while (0)
#else
#define XT_MARK(t) do {} while (0)
#define XT_ADD(S, k, t0) do {} while (0)
#endif

// parity of D/u for a displacement D that is a multiple of u = ulp(binade e) (e >= RUN_MIN_E,
// so a non-zero D is a normal number): the bit of D's significand that has weight u
__device__ __forceinline__ int disp_parity(double D, int e) {
    const unsigned long long b = bt(D);
    const int sh = e - dexp(b);
    if (D == 0.0 || sh < 0 || sh > 52) return 0;
    return (int)((((b & MANT) | (1ull << 52)) >> sh) & 1ull);
}

__device__ __forceinline__ Run run_empty() {
    Run r;
    r.d[0] = r.d[1] = r.lo[0] = r.lo[1] = r.hi[0] = r.hi[1] = 0.0;
    r.e = E_EMPTY;
    r.neg = 0;
    return r;
}

// a then b (same binade, or either empty). All quantities are multiples of u smaller than the
// binade: the sums are exact. (Selects, not b.d[m]: a runtime index would put the structs in
// local memory.)
__device__ __forceinline__ Run run_merge(const Run& a, const Run& b) {
    if (a.e == E_EMPTY) return b;
    if (b.e == E_EMPTY) return a;
    Run r;
    r.e = a.e;
    r.neg = a.neg;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const bool m = (p ^ disp_parity(a.d[p], a.e)) != 0;  // parity of the index after a
        const double bd = m ? b.d[1] : b.d[0], bl = m ? b.lo[1] : b.lo[0], bh = m ? b.hi[1] : b.hi[0];
        r.d[p] = dadd(a.d[p], bd);
        r.lo[p] = fmin(a.lo[p], dadd(a.d[p], bl));
        r.hi[p] = fmax(a.hi[p], dadd(a.d[p], bh));
    }
    return r;
}

// Does the run R apply to a start v? It does when v is in R's binade and every partial sum
// v + [lo, hi] stays one ulp clear of the binade's ends; then v advances and the start-shift
// constraints of the carried piece (lo, hi, km) tighten.
__device__ __forceinline__ bool run_apply(const Run& R, double& v, double& lo, double& hi, int& km) {
    if (R.e == E_EMPTY) return true;
    const unsigned long long b = bt(v);
    const int ng = (int)(b >> 63);
    if (R.e == E_HARD || dexp(b) != R.e || ng != R.neg) return false;
    const bool odd = (b & 1ull) != 0;
    const double bot = fb(((unsigned long long)ng << 63) | ((unsigned long long)R.e << 52) | 1ull);  // +-(2^e + u)
    const double top = fb(((unsigned long long)ng << 63) | ((unsigned long long)R.e << 52) | MANT); // +-(2^(e+1) - u)
    const double vlo = dadd(v, odd ? R.lo[1] : R.lo[0]), vhi = dadd(v, odd ? R.hi[1] : R.hi[0]);  // exact
    double a, c;
    if (!ng) {
        if (!(vlo >= bot && vhi <= top)) return false;
        a = dsub(bot, vlo);
        c = dsub(top, vhi);
    } else {
        if (!(vhi <= bot && vlo >= top)) return false;
        a = dsub(top, vlo);
        c = dsub(bot, vhi);
    }
    lo = fmax(lo, a);
    hi = fmin(hi, c);
    km = max(km, R.e - 1074);
    v = dadd(v, odd ? R.d[1] : R.d[0]);  // exact: stays on the grid of the binade
    return true;
}

// The value v (a partial sum of the carried piece) must stay in its binade, one ulp clear of
// its ends, under the start shift; zero / subnormal / non-finite: no shift at all.
// Branch-free; plain compares instead of fmin / fmax (no NaN reaches them: a non-finite v
// takes the zero range, and lo / hi only ever hold finite values or +-inf).
__device__ __forceinline__ void value_slack(double v, double& lo, double& hi, int& km) {
    const unsigned long long b = bt(v);
    const int ex = dexp(b);
    const bool special = ex == 0 || ex == 0x7ff;
    const double t1 = dsub(fb(b | MANT), v);           // +-(2^(e+1) - u) - v, exact (same binade)
    const double t2 = dsub(fb((b & ~MANT) | 1ull), v); // +-(2^e + u) - v
    double a = t1 < t2 ? t1 : t2, c = t1 < t2 ? t2 : t1;
    a = special ? 0.0 : a;
    c = special ? 0.0 : c;
    lo = lo > a ? lo : a;
    hi = hi < c ? hi : c;
    km = special ? km : max(km, ex - 1074);
}

__device__ __forceinline__ void sim_step(double& v, double p, double& lo, double& hi, int& km) {
    v = dadd(v, p);
    value_slack(v, lo, hi, km);
}

// Warp-collective: evaluate the table (this lane holds entry `lane`; mb0/tneg uniform) at
// this lane's s. On success out = the table's value at s and lo/hi/km tighten.
__device__ __forceinline__ bool table_eval(unsigned long long mb0, int tneg, const LaneR& T, double s,
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
    r.d[0] = h.d[0]; r.d[1] = h.d[1]; r.lo[0] = h.lo[0]; r.lo[1] = h.lo[1];
    r.hi[0] = h.hi[0]; r.hi[1] = h.hi[1]; r.e = h.e; r.neg = h.neg;
    return r;
}
__device__ __forceinline__ void hdr_set_run(Hdr& h, const Run& r, double pred) {
    h.kind = K_RUN; h.e = r.e; h.neg = r.neg; h.pad = 0; h.mb0 = 0; h.pred = pred;
    h.d[0] = r.d[0]; h.d[1] = r.d[1]; h.lo[0] = r.lo[0]; h.lo[1] = r.lo[1];
    h.hi[0] = r.hi[0]; h.hi[1] = r.hi[1];
}
__device__ __forceinline__ void hdr_set_table(Hdr& h, unsigned long long mb0, int neg, double pred) {
    h.kind = K_TABLE; h.e = 0; h.neg = neg; h.pad = 0; h.mb0 = mb0; h.pred = pred;
    h.d[0] = h.d[1] = h.lo[0] = h.lo[1] = h.hi[0] = h.hi[1] = 0.0;
}
__device__ __forceinline__ bool runs_compatible(const Run& a, const Run& b) {
    return a.e == E_EMPTY || b.e == E_EMPTY || (a.e != E_HARD && a.e == b.e && a.neg == b.neg);
}
__device__ __forceinline__ void store_lane(Desc* D, int lane, const LaneR& L) {
    LaneS s;
    s.out = L.out;
    s.lo = __double2float_ru(L.lo);  // inwards: a smaller shift range is still a valid one
    s.hi = __double2float_rd(L.hi);
    D->l[lane] = s;
    D->kmh[lane] = (L.km << 1) | (L.hole ? 1 : 0);
}
__device__ __forceinline__ LaneR load_lane(const Desc* D, int lane) {
    const LaneS s = D->l[lane];
    const int kmh = D->kmh[lane];
    LaneR L;
    L.out = s.out;
    L.lo = (double)s.lo;
    L.hi = (double)s.hi;
    L.km = kmh >> 1;
    L.hole = kmh & 1;
    return L;
}

// A piece as a warp holds it: the uniform header plus this lane's table entry.
struct PieceR {
    int kind, neg;
    unsigned long long mb0;
    Run R;
    LaneR T;
};
__device__ __forceinline__ PieceR load_piece(const Desc* D) {
    PieceR P;
    const Hdr h = D->h;
    P.kind = h.kind;
    P.neg = h.neg;
    P.mb0 = h.mb0;
    P.R = hdr_run(h);
    P.T = load_lane(D, threadIdx.x & 31);
    return P;
}
// Warp-collective for tables (kind is the same in every lane: the branch does not diverge):
// carry this lane's value through the piece.
__device__ __forceinline__ bool piece_apply_r(const PieceR& P, double& v, double& lo, double& hi, int& km) {
    if (P.kind == K_RUN) return run_apply(P.R, v, lo, hi, km);
    double out = 0.0, l2 = lo, h2 = hi;
    int k2 = km;
    value_slack(v, l2, h2, k2);
    const bool ok = table_eval(P.mb0, P.neg, P.T, v, out, l2, h2, k2);
    if (ok) { v = out; lo = l2; hi = h2; km = k2; }
    return ok;
}

// Elements added one by one, carrying the start-shift constraints of every partial sum: the
// add chain plus, per stretch of one binade, the min / max of the partial sums' bit patterns
// (for one sign they order like the magnitudes); at a change of binade (sign and exponent
// bits) the stretch's constraints are those of its two extremes.
__device__ __forceinline__ void flush_range(unsigned long long bmin, unsigned long long bmax, double& lo,
                                            double& hi, int& km) {
    value_slack(fb(bmin), lo, hi, km);
    value_slack(fb(bmax), lo, hi, km);
}
// Any number of binades: every partial sum's own constraint, branch-free (lanes whose sums
// change binade at different elements do not diverge) and light on the integer pipe, which
// is what limits this loop when a whole CTA runs it: with lo <= 0 <= hi always, each bound is
// tracked as the smallest distance to the binade end a shift of that sign reaches, by the
// high word of the distance only (the low word dropped: a slightly smaller distance, so the
// bounds only get narrower -- always safe).
__device__ __forceinline__ void sim_elems_slow(const double* p, int cnt, double& v, double& lo, double& hi, int& km) {
    double x = v;
    unsigned lom = (unsigned)__double2hiint(lo) & 0x7fffffffu, him = (unsigned)__double2hiint(hi) & 0x7fffffffu;
    int kmx = km;
#pragma unroll (SIM_UNROLL)
    for (int k = 0; k < cnt; ++k) {
        x = dadd(x, p[k]);
        const unsigned h = (unsigned)__double2hiint(x);
        const unsigned hb = h & 0x7ff00000u;  // |x|'s binade: bottom end (hb, 1), top end (hb | 0xfffff, ~0)
        const double ax = fabs(x);
        const unsigned d_bot = (unsigned)__double2hiint(dsub(ax, __hiloint2double((int)hb, 1)));  // exact, >= 0
        const unsigned d_top = (unsigned)__double2hiint(dsub(__hiloint2double((int)(hb | 0xfffffu), -1), ax));
        // a negative shift moves a positive sum toward its bottom end, a negative sum toward its top
        const unsigned sgn = (unsigned)((int)h >> 31);
        const unsigned to_lo = (d_top & sgn) | (d_bot & ~sgn), to_hi = (d_bot & sgn) | (d_top & ~sgn);
        // zero / subnormal: no shift at all (inf / nan: the entry becomes a hole anyway)
        lom = min(lom, hb ? to_lo : 0u);
        him = min(him, hb ? to_hi : 0u);
        kmx = max(kmx, (int)(hb >> 20) - 1074);
    }
    lo = -__hiloint2double((int)lom, 0);
    hi = __hiloint2double((int)him, 0);
    km = kmx;
    v = x;
}

// Branch-free common case: the partial sums fall into at most two binades (the first one's and
// one other); the extremes are kept per binade, bucket membership as a bit mask (selects on a
// predicate compiled to a branch per element). Anything else: the per-stretch path above.
__device__ __forceinline__ void sim_elems(const double* p, int cnt, double& v, double& lo, double& hi, int& km) {
    if (cnt <= 0) return;
    double x = dadd(v, p[0]);
    const unsigned t0 = (unsigned)(bt(x) >> 52);
    unsigned long long amin = bt(x), amax = amin, bmin = ~0ull, bmax = 0ull;
#pragma unroll 4
    for (int k = 1; k < cnt; ++k) {
        x = dadd(x, p[k]);
        const unsigned long long b = bt(x);
        const unsigned long long mA = 0ull - (unsigned long long)((unsigned)(b >> 52) == t0);
        amin = min(amin, b | ~mA);
        amax = max(amax, b & mA);
        bmin = min(bmin, b | mA);
        bmax = max(bmax, b & ~mA);
    }
    const bool has_b = bmin != ~0ull;  // (+0.0 is a member too: test the minimum, not the maximum)
    if (has_b && (bmin >> 52) != (bmax >> 52)) {  // a third binade: redo per stretch
        sim_elems_slow(p, cnt, v, lo, hi, km);
        return;
    }
    flush_range(amin, amax, lo, hi, km);
    if (has_b) flush_range(bmin, bmax, lo, hi, km);
    v = x;
}

// plain left-to-right sum of p[i0, i1) onto v (8 loads ahead of the add chain)
__device__ __forceinline__ double walk_elems(const double* p, int i0, int i1, double v) {
    int i = i0;
    for (; i + 8 <= i1; i += 8) {
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = p[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) v = dadd(v, x[j]);
    }
    const int r = i1 - i;  // 0..7 left: all loads first (a load per add would chain the latency)
    double x[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) x[j] = j < r ? p[i + j] : 0.0;
#pragma unroll
    for (int j = 0; j < 7; ++j)
        if (j < r) v = dadd(v, x[j]);
    return v;
}

// Per lane, no collectives: carry v through the thread runs [t0, t1) of the CTA range in shared
// memory, adding a thread's products one by one where its run does not apply.
//
// `q` (> 0): 32 ulps of the binade of this lane's candidate start. A table entry is looked up
// either at its candidate exactly or at a start 32k ulps away (k != 0), so once the entry's
// shift range [lo, hi] lies inside (-q, q) -- the sum passed close to zero, where the grid is
// fine -- it can serve its candidate alone: the range is set to [0, 0] and the rest of the walk
// carries the value only (plain adds instead of the slack bookkeeping).
__device__ __forceinline__ double quantum32(double c) {
    const int e = max(dexp(bt(c)), 1);
    return e >= 48 ? fb((unsigned long long)(e - 47) << 52) : ldexp(32.0, e - 1075);
}
__device__ void lane_walk_threads(const Run* s_runs, const double* sp, int len, int E, int t0, int t1,
                                  double& v, double& lo, double& hi, int& km,
                                  unsigned long long* sims = nullptr, bool bare = false, double q = 0.0) {
    for (int t = t0; t < t1; ++t) {
        if (!bare && lo > -q && hi < q) {
            bare = true;
            lo = 0.0;
            hi = 0.0;
        }
        const Run R = s_runs[t];
        if (run_apply(R, v, lo, hi, km)) continue;
        const int b0 = t * E, bl = max(0, min(E, len - b0));
        if (bare) {  // the value only: this lane then serves its exact start alone
            v = walk_elems(sp + b0, 0, bl, v);
            lo = fmax(lo, 0.0);
            hi = fmin(hi, 0.0);
        } else if (R.e == E_HARD) {  // its sums change binade: the per-sum path straight away
            sim_elems_slow(sp + b0, bl, v, lo, hi, km);
        } else {
            sim_elems(sp + b0, bl, v, lo, hi, km);
        }
    }
}

#ifdef MCR_XDOT_DEBUG
__device__ double dbg_serial(const Seq& q, long long i0, long long i1, double v) {
    for (long long i = i0; i < i1; ++i) v = dadd(v, dmul(__ldcg(q.u + i), __ldcg(q.v + i)));
    return v;
}
__device__ __forceinline__ bool same_bits(double a, double b) { return bt(a) == bt(b); }
// this lane's table entry (start c) over elements [i0, i1): exact value, and one translation
__device__ void dbg_check_lane(const Scratch& S, const Seq& q, long long i0, long long i1, double c,
                               const LaneR& Lx, int level) {
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
__device__ void why_failed(const Scratch& S, const Desc* D, double v) {
    if ((threadIdx.x & 31) != 0 || !S.stats) return;
    const unsigned long long b = bt(v);
    if (D->h.kind == K_RUN) {
        const Run R = hdr_run(D->h);
        if (R.e == E_HARD || dexp(b) != R.e || (int)(b >> 63) != R.neg) stat(S, ST_R_RUN_BIN);
        else stat(S, ST_R_RUN_BOUND);
        return;
    }
    const unsigned long long mb = b & ~SGN, mb0 = D->h.mb0;
    const long long d = (long long)(mb - mb0);
    const int k = (int)(d & 31);
    const LaneR T = load_lane(D, k);
    if (T.hole) { stat(S, ST_R_HOLE); return; }
    if ((int)(b >> 63) != D->h.neg) { stat(S, ST_R_SIGN); return; }
    const unsigned long long cb = mb0 + (unsigned long long)k;
    if (dexp(cb) != dexp(mb) || dexp(mb) == 0 || dexp(mb) == 0x7ff) { stat(S, ST_R_EXP); return; }
    const double dl = dsub(v, fb(cb | ((unsigned long long)D->h.neg << 63)));
    if (!(dl >= T.lo && dl <= T.hi)) { stat(S, ST_R_SLACK); return; }
    stat(S, ST_R_KM);
}
#endif

// ---------------------------------------------------------------- one CTA range
// Shared memory of a CTA (dynamic): the range's products, its thread runs, its warp pieces,
// the root's group tables, and the root's staging area for CTA pieces.
struct Smem {
    double* sp;     // NT * E
    Run* runs;      // NT
    Desc* wd;       // NW: warp pieces (then the CTA tree)
    Desc* gd;       // NW: the root's group tables
    Desc* td;       // NW: the root's tree over the group tables
    Desc* stage;    // A.stage
};
__host__ __device__ constexpr size_t smem_bytes(int E, int stage) {
    return sizeof(double) * (size_t)NT * (size_t)E + sizeof(Run) * NT + sizeof(Desc) * (3 * NW + stage);
}
__device__ __forceinline__ Smem smem_layout(unsigned char* base, int E) {
    Smem M;
    M.sp = (double*)base;
    M.runs = (Run*)(base + sizeof(double) * (size_t)NT * (size_t)E);
    M.wd = (Desc*)(M.runs + NT);
    M.gd = M.wd + NW;
    M.td = M.gd + NW;
    M.stage = M.td + NW;
    return M;
}

// All threads: products of elements [c0, c0 + len) into sp (32 loads in flight per thread);
// returns the CTA-wide OR of the flags (bit 0 a product that is not -0.0, bit 1 non-finite).
__device__ unsigned load_products(const Seq& q, long long c0, int len, double* sp) {
    __shared__ unsigned s_fl;
    if (threadIdx.x == 0) s_fl = 0u;
    __syncthreads();
    unsigned fl = 0u;
    for (int k0 = threadIdx.x; k0 < len; k0 += NT * 16) {
        double a[16], b[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int k = k0 + j * NT;
            a[j] = k < len ? __ldcg(q.u + c0 + k) : 0.0;
            b[j] = k < len ? __ldcg(q.v + c0 + k) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int k = k0 + j * NT;
            if (k < len) {
                const double p = dmul(a[j], b[j]);
                const unsigned long long pb = bt(p);
                fl |= (pb != SGN) ? 1u : 0u;
                fl |= (dexp(pb) == 0x7ff) ? 2u : 0u;
                sp[k] = p;
            }
        }
    }
    if (fl) atomicOr(&s_fl, fl);
    __syncthreads();
    return s_fl;
}

// All threads: plain sum of this thread's E products, block exclusive scan. Returns this
// thread's exclusive prefix; *total = the CTA's sum (same in every thread).
__device__ double thread_scan(const double* sp, int len, int E, double* s_red, double* total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t0 = tid * E;
    const int tl = max(0, min(E, len - t0));
    double ts = 0.0;
#pragma unroll 4
    for (int k = 0; k < tl; ++k) ts = dadd(ts, sp[t0 + k]);
    double inc = ts;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double o = __shfl_up_sync(FULL, inc, off);
        if (lane >= off) inc = dadd(inc, o);
    }
    double exc = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) exc = 0.0;
    __syncthreads();  // s_red may still be read by a previous user
    if (lane == 31) s_red[warp] = inc;
    __syncthreads();
    double wexc = 0.0, tot = 0.0;
    for (int w = 0; w < NW; ++w) {
        if (w < warp) wexc = dadd(wexc, s_red[w]);
        tot = dadd(tot, s_red[w]);
    }
    *total = tot;
    return dadd(wexc, exc);
}

// This thread's run over its tl products sp[0..tl): two reference chains from the predicted
// start (its index made even) and its odd neighbour; HARD unless every partial sum stayed in
// the prediction's binade, 4096 ulps clear of its ends. `allow` = false (a non-finite
// product): HARD.
__device__ __forceinline__ Run thread_run(const double* sp, int tl, double pred, bool allow) {
    Run R = run_empty();
    if (tl > 0) {
        R.e = E_HARD;
        const unsigned long long pb = bt(pred);
        const int e = dexp(pb);
        const int ng = (int)(pb >> 63);
#ifndef XD_SKIP_CHAIN
        if (e >= RUN_MIN_E && e <= 0x7f0 && allow) {
#else
        if (false) {
#endif
            // reference starts: the predicted start itself (index made even) and its odd neighbour,
            // so the chains follow the predicted trajectory
            const double ref0 = fb(bt(pred) & ~1ull);
            const double ref1 = fb(bt(ref0) + 1ull);
            double s0 = ref0, s1 = ref1;
            // extremes as bit patterns (one sign: they order like the magnitudes; a NaN or a sign
            // change shows up as a different top-12-bit field and fails the binade test below)
            unsigned long long a0 = bt(ref0), z0 = a0, a1 = bt(ref1), z1 = a1;
#pragma unroll (RUN_UNROLL)
            for (int k = 0; k < tl; ++k) {
                const double p = sp[k];
                s0 = dadd(s0, p);
                s1 = dadd(s1, p);
                a0 = min(a0, bt(s0)); z0 = max(z0, bt(s0));
                a1 = min(a1, bt(s1)); z1 = max(z1, bt(s1));
            }
            const bool same = (a0 >> 52) == (z0 >> 52) && (a1 >> 52) == (z1 >> 52) && (a0 >> 52) == (bt(ref0) >> 52);
            // value extremes (for a negative binade the largest pattern is the smallest value)
            const double mn0 = ng ? fb(z0) : fb(a0), mx0 = ng ? fb(a0) : fb(z0);
            const double mn1 = ng ? fb(z1) : fb(a1), mx1 = ng ? fb(a1) : fb(z1);
            // the chains model the run only if every partial sum stayed inside the binade, and
            // are worth keeping only if they stayed clear of its ends by more than the prediction's
            // error (4096 ulps); else the thread is summed element by element
            const double margin = fb((unsigned long long)(e - XD_MARGIN) << 52);
            const double bot = dadd(fb(((unsigned long long)e << 52) | 1ull), margin);
            const double top = dsub(fb(((unsigned long long)e << 52) | MANT), margin);
            const bool ok = same && (ng ? (-mx0 >= bot && -mn0 <= top && -mx1 >= bot && -mn1 <= top)
                                        : (mn0 >= bot && mx0 <= top && mn1 >= bot && mx1 <= top));
            if (ok) {
                R.d[0] = dsub(s0, ref0); R.d[1] = dsub(s1, ref1);
                R.lo[0] = dsub(mn0, ref0); R.hi[0] = dsub(mx0, ref0);
                R.lo[1] = dsub(mn1, ref1); R.hi[1] = dsub(mx1, ref1);
                R.e = e;
                R.neg = ng;
            }
        }
    }
    return R;
}

// Warp-collective: segments are maximal stretches of thread runs of one binade (a HARD thread
// is a segment of its own; trailing EMPTY threads join the segment before them). A segmented
// scan merges each segment into its last lane; returns this lane's merged run and the
// segment-head mask.
__device__ __forceinline__ Run warp_merge_runs(const Run& R, int lane, unsigned& heads) {
    const int pe = __shfl_up_sync(FULL, R.e, 1), pn = __shfl_up_sync(FULL, R.neg, 1);
    const bool head = lane == 0 || R.e == E_HARD || pe == E_HARD ||
                      (R.e != E_EMPTY && pe != E_EMPTY && (R.e != pe || R.neg != pn));
    heads = __ballot_sync(FULL, head);
    const int seg0 = 31 - __clz(heads & (FULL >> (31 - lane)));  // this lane's segment head
    Run A = R;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Run o;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            o.d[p] = __shfl_up_sync(FULL, A.d[p], off);
            o.lo[p] = __shfl_up_sync(FULL, A.lo[p], off);
            o.hi[p] = __shfl_up_sync(FULL, A.hi[p], off);
        }
        o.e = __shfl_up_sync(FULL, A.e, off);
        o.neg = __shfl_up_sync(FULL, A.neg, off);
        if (lane - off >= seg0) A = run_merge(o, A);
    }
    return A;
}

// All threads: this thread's run (two reference chains in the middle of the binade of `pred`,
// the predicted start of its elements), then the warp pieces (one merged run when the
// warp's 32 runs share a binade, else a table around the warp's predicted start). Ends with
// __syncthreads.
__device__ void runs_and_warp_pieces(const Scratch& S, const Seq& q, long long c0, int len, int E,
                                     double pred, unsigned fl, const Smem& M, bool force_table = false,
                                     bool first = false) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int t0 = tid * E;
    const int tl = max(0, min(E, len - t0));
    const double* sp = M.sp;
#ifdef MCR_XDOT_TIMING
    const unsigned long long w_t0 = gtime();
#endif
    const Run R = thread_run(sp + t0, tl, pred, !(fl & 2u));
    M.runs[tid] = R;
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
                if (S.stats) printf("xdot dbg: run e=%d neg=%d d0=%a d1=%a start=%a want=%a got=%a\n", R.e, R.neg, R.d[0], R.d[1], v0, want, v);
            }
        }
    }
#endif
    if (R.e == E_HARD && S.stats) stat(S, ST_HARD);
#ifdef MCR_XDOT_TIMING
    {  // distribution of HARD threads: max per warp (DBG_TAB), max per CTA (DBG_SPARE), CTAs with
       // more than 64 (DBG_TR_BAD), warps with more than 8 (DBG_TAB_BAD)
        const int wh = __popc(__ballot_sync(FULL, R.e == E_HARD));
        __shared__ int s_hard;
        if (threadIdx.x == 0) s_hard = 0;
        __syncthreads();
        if (lane == 0 && wh) atomicAdd(&s_hard, wh);
        if (lane == 0 && S.stats) {
            atomicMax(S.stats + ST_DBG_TAB, (unsigned long long)wh);
            if (wh > 8) atomicAdd(S.stats + ST_DBG_TAB_BAD, 1ull);
        }
        __syncthreads();
        if (threadIdx.x == 0 && S.stats) {
            atomicMax(S.stats + ST_DBG_SPARE, (unsigned long long)s_hard);
            if (s_hard > 64) atomicAdd(S.stats + ST_DBG_TR_BAD, 1ull);
        }
    }
#endif
    __syncwarp();
#ifdef MCR_XDOT_TIMING
    const unsigned long long w_t1 = gtime();
    if (lane == 0 && S.stats) atomicMax(S.stats + ST_W_CHAIN, w_t1 - w_t0);
#endif
    unsigned heads;
    const Run A = warp_merge_runs(R, lane, heads);
    const unsigned ends = (heads >> 1) | 0x80000000u;  // last lane of each segment
    const double wpred = __shfl_sync(FULL, pred, 0);
    Desc* WD = M.wd + warp;
    if (heads == 1u && __shfl_sync(FULL, A.e, 31) != E_HARD && !force_table) {
        if (lane == 31) hdr_set_run(WD->h, A, wpred);
#ifdef MCR_XDOT_TIMING
        if (lane == 0 && S.stats) atomicMax(S.stats + ST_W_MERGE, gtime() - w_t1);
#endif
    } else {
        if (S.stats && lane == 0) stat(S, ST_WARP_TABLE);
        const unsigned long long mb0 = window_mb0(wpred);
        const int wn = window_neg(wpred);
        double v = cand(mb0, wn, lane), lo = -INFINITY, hi = INFINITY;
        int km = KM_NONE;
        const double q32 = quantum32(v);
        // The first warp of a sequence starts at exactly 0.0 (its prediction, and candidate 0 of
        // its window): only that lane's value is ever used, so the lanes carry values alone
        // (plain adds, no slack bookkeeping; every other candidate is served at delta = 0 only).
        // (Carrying values only in other element-by-element warps measured slower: their
        // starts are not known, so the root walked them.)
        const bool bare = first && warp == 0;
#ifdef XD_TWICE
        for (int rep = 0; rep < 2; ++rep) {
        const unsigned long long tr0 = gtime();
        v = cand(mb0, wn, lane); lo = -INFINITY; hi = INFINITY; km = KM_NONE;
#endif
        int sl = 0;
#ifdef MCR_XDOT_TIMING
        int nfail = 0;
        long long cyc_apply = 0, cyc_walk = 0;
        const long long cyc_t0 = clock64();
#endif
        for (unsigned m = ends; m; m &= m - 1) {  // segment [sl, el]
            const int el = __ffs(m) - 1;
            Run G;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                G.d[p] = __shfl_sync(FULL, A.d[p], el);
                G.lo[p] = __shfl_sync(FULL, A.lo[p], el);
                G.hi[p] = __shfl_sync(FULL, A.hi[p], el);
            }
            G.e = __shfl_sync(FULL, A.e, el);
            G.neg = __shfl_sync(FULL, A.neg, el);
#ifdef MCR_XDOT_TIMING
            const long long c_a = clock64();
#endif
            const bool okr = run_apply(G, v, lo, hi, km);
#ifdef MCR_XDOT_TIMING
            nfail += __popc(__ballot_sync(FULL, !okr));
            const long long c_b = clock64();
            cyc_apply += c_b - c_a;
#endif
            if (!okr)
                lane_walk_threads(M.runs, sp, len, E, warp * 32 + sl, warp * 32 + el + 1, v, lo, hi, km,
                                  S.stats ? S.stats + ST_SIMS_WARP : nullptr, bare, q32);
#ifdef MCR_XDOT_TIMING
            __syncwarp();
            cyc_walk += clock64() - c_b;
#endif
            sl = el + 1;
        }
#ifdef XD_TWICE
        if (lane == 0 && S.stats) atomicMax(S.stats + (rep == 0 ? ST_W_CHAIN : ST_W_MERGE), gtime() - tr0);
        }
#endif
        LaneR Lx;
        Lx.out = v; Lx.lo = lo; Lx.hi = hi; Lx.km = km;
        Lx.hole = dexp(bt(v)) == 0x7ff ? 1 : 0;
        store_lane(WD, lane, Lx);
#ifdef MCR_XDOT_DEBUG
        dbg_check_lane(S, q, c0 + warp * 32 * E, min(c0 + len, c0 + (long long)(warp + 1) * 32 * E), cand(mb0, wn, lane), load_lane(WD, lane), 1);
#endif
        if (lane == 0) hdr_set_table(WD->h, mb0, wn, wpred);
#ifdef MCR_XDOT_TIMING
        const int nhard = __popc(__ballot_sync(FULL, R.e == E_HARD));
        if (lane == 0 && S.stats) {
            const unsigned long long dt = gtime() - w_t1;
            atomicMax(S.stats + ST_W_TABLE, dt);
            // slowest table: time | segments | hard threads | warp | CTA range start
            const long long cyc_all = clock64() - cyc_t0;
            const unsigned long long info = (dt << 40) | ((unsigned long long)__popc(heads) << 32) |
                ((unsigned long long)min((long long)(cyc_walk / 256), 255ll) << 24) |
                ((unsigned long long)min((long long)(cyc_apply / 64), 255ll) << 16) |
                (unsigned long long)min((long long)(cyc_all / 256), 65535ll);
            atomicMax(S.stats + ST_W_SLOWEST, info);
        }
#endif
    }
    __syncthreads();
}

// Warp: the piece of L then R (both in shared memory; L covers threads [t0, t1), R threads
// [t1, t2)) into *out (may be L): a merged run when both are runs of one binade, else a table
// in L's window. With `walk`, lanes a piece does not serve walk its thread runs (the CTA's own
// range is in shared memory); otherwise they become holes.
__device__ void compose_pair(const Smem& M, int len, int E, const Desc* L, const Desc* R, Desc* out,
                             int t0, int t1, int t2, bool walk) {
    const int lane = threadIdx.x & 31;
    const Hdr hl = L->h, hr = R->h;
    if (hl.kind == K_RUN && hr.kind == K_RUN) {
        const Run a = hdr_run(hl), b = hdr_run(hr);
        if (runs_compatible(a, b)) {
            __syncwarp();
            if (lane == 0) hdr_set_run(out->h, run_merge(a, b), hl.pred);
            __syncwarp();
            return;
        }
    }
    double v, lo = -INFINITY, hi = INFINITY;
    int km = KM_NONE, hole = 0;
    unsigned long long mb0;
    int neg;
    if (hl.kind == K_TABLE) {
        const LaneR T = load_lane(L, lane);
        v = T.out; lo = T.lo; hi = T.hi; km = T.km; hole = T.hole;
        mb0 = hl.mb0; neg = hl.neg;
    } else {
        mb0 = window_mb0(hl.pred);
        neg = window_neg(hl.pred);
        v = cand(mb0, neg, lane);
        if (!run_apply(hdr_run(hl), v, lo, hi, km)) {
            if (walk) lane_walk_threads(M.runs, M.sp, len, E, t0, t1, v, lo, hi, km, nullptr, false,
                                        quantum32(cand(mb0, neg, lane)));
            else hole = 1;
        }
    }
    const PieceR P = load_piece(R);
    if (!piece_apply_r(P, v, lo, hi, km) && !hole) {  // collective; then per lane
        if (walk) lane_walk_threads(M.runs, M.sp, len, E, t1, t2, v, lo, hi, km, nullptr, false,
                                    quantum32(cand(mb0, neg, lane)));
        else hole = 1;
    }
    LaneR Lx;
    Lx.out = v; Lx.lo = lo; Lx.hi = hi; Lx.km = km;
    Lx.hole = (hole || dexp(bt(v)) == 0x7ff) ? 1 : 0;
    __syncwarp();  // every lane has read L
    store_lane(out, lane, Lx);
    if (lane == 0) hdr_set_table(out->h, mb0, neg, hl.pred);
    __syncwarp();
}

// All threads: fold the NW pieces in p[0..NW) pairwise (level s merges p[2sw] and p[2sw + s]
// into p[2sw]); the result is in p[0]. Piece i covers threads [32 i, 32 i + 32) when `walk`.
__device__ void tree_fold(const Smem& M, int len, int E, Desc* p, bool walk) {
    const int warp = threadIdx.x >> 5;
    for (int s = 1; s < NW; s <<= 1) {
        if (warp < NW / (2 * s)) {
            const int a = 2 * s * warp, b = a + s;
            compose_pair(M, len, E, p + a, p + b, p + a, a * 32, b * 32, (b + s) * 32, walk && s <= XD_WALK_MAX);
        }
        __syncthreads();
    }
}

// Phase 1 of every CTA: take a ticket (the CTA's place in the sequence), build the CTA piece
// around the predicted start (the sum of the totals of the CTAs before it: look-back) and
// publish it. Returns the ticket.
__device__ int build_cta(const Args& A, const Seq& q, int si, const Smem& M, double* s_red) {
    const int tid = threadIdx.x;
    const Scratch& S = A.S;
    const int E = A.E;
    __shared__ int s_tk;
    __shared__ double s_pred;
    XT_MARK(t_start);
    if (tid == 0) s_tk = (int)atomicAdd(S.ticket + si, 1u);
    __syncthreads();
    const int ci = s_tk;
    const int slot = q.cta0 + ci;
    const long long c0 = q.a + (long long)ci * NT * E;
    const long long c1 = min(q.b, c0 + (long long)NT * E);
    const int len = (int)max(0ll, c1 - c0);
    const unsigned fl = load_products(q, c0, len, M.sp);
    XT_ADD(S, ST_T_LOAD, t_start);
    XT_MARK(t_lb);
    if (A.upto == 1) return ci;
    double total;
    const double exc = thread_scan(M.sp, len, E, s_red, &total);
    if (tid == 0) {
        S.lb_val[slot] = total;
        __threadfence();
        atomicExch(S.lb_flag + slot, 1);
        if (fl) atomicOr(S.flags + si, fl);
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
    XT_ADD(S, ST_T_LOOKBACK, t_lb);
    XT_MARK(t_runs);
    if (A.upto == 2) return ci;
    runs_and_warp_pieces(S, q, c0, len, E, dadd(pred_cta, exc), fl, M, A.upto == 13, ci == 0);
    XT_ADD(S, ST_T_RUNS, t_runs);
    XT_MARK(t_cta);
    if (A.upto == 3 || A.upto == 13) return ci;
    {  // the warp pieces, for the root's fallback (before the tree folds them in place)
        const double2* src = (const double2*)M.wd;
        double2* dst = (double2*)(S.warp + (size_t)slot * NW);
        for (int k = tid; k < (int)(NW * sizeof(Desc) / 16); k += NT) dst[k] = src[k];
    }
    __syncthreads();
    if (ci == 0 && A.upto != 13) {
        // The sequence's first CTA starts at exactly 0.0, and the root evaluates its piece
        // there alone: warp 0 carries that value through the warp pieces (a piece that does not
        // apply: its threads, values only), and the CTA piece is that value at candidate 0.0
        // (every other candidate a hole) -- no tree of tables, whose lanes would otherwise walk
        // the stretches that do not compose with the slack bookkeeping.
        const int lane = tid & 31;
        if ((tid >> 5) == 0) {
            double v = 0.0;
            PieceR P = load_piece(M.wd);
            for (int w = 0; w < NW; ++w) {
                const PieceR Pc = P;
                P = load_piece(M.wd + min(w + 1, NW - 1));  // next piece's loads off the chain
                double lo = -INFINITY, hi = INFINITY;
                int km = KM_NONE;
                if (piece_apply_r(Pc, v, lo, hi, km)) continue;  // uniform
                lo = hi = 0.0;
                lane_walk_threads(M.runs, M.sp, len, E, w * 32, w * 32 + 32, v, lo, hi, km, nullptr, true);
            }
            __syncwarp();
            LaneR L;
            L.out = v; L.lo = 0.0; L.hi = 0.0; L.km = KM_NONE;
            L.hole = (lane != 0 || dexp(bt(v)) == 0x7ff) ? 1 : 0;
            store_lane(M.wd, lane, L);
            if (lane == 0) hdr_set_table(M.wd->h, window_mb0(0.0), 0, 0.0);
        }
        __syncthreads();
    } else {
        tree_fold(M, len, E, M.wd, true);  // the CTA piece, in wd[0]
    }
    if (S.stats && tid == 0 && M.wd[0].h.kind == K_TABLE) stat(S, ST_CTA_TABLE);
#ifdef MCR_XDOT_DEBUG
    if ((tid >> 5) == 0 && M.wd[0].h.kind == K_TABLE)
        dbg_check_lane(S, q, c0, c0 + len, cand(M.wd[0].h.mb0, M.wd[0].h.neg, tid & 31), load_lane(M.wd, tid & 31), 2);
#endif
    {  // publish
        const double2* src = (const double2*)M.wd;
        double2* dst = (double2*)(S.cta + slot);
        for (int k = tid; k < (int)(sizeof(Desc) / 16); k += NT) dst[k] = src[k];
    }
    XT_ADD(S, ST_T_CTA, t_cta);
    return ci;
}

// Warp 0 of the root: warp w's elements of CTA range ci from the exact start v: the 32
// threads' runs rebuilt around predictions from v (one per lane), then a scalar walk over
// them; a thread whose run does not apply adds its elements one by one. Exact always.
__device__ double warp_walk_exact(const Args& A, const Seq& q, int ci, int w, double v, const Smem& M) {
    const int lane = threadIdx.x & 31;
    const int E = A.E;
    const long long c0 = q.a + (long long)ci * NT * E;
    const long long c1 = min(q.b, c0 + (long long)NT * E);
    const long long w0 = c0 + (long long)w * 32 * E;
    const int wl = (int)max(0ll, min(c1 - w0, (long long)32 * E));
    double* sp = M.sp;  // the root's own range is no longer needed
    for (int k = lane; k < wl; k += 32) sp[k] = dmul(__ldcg(q.u + w0 + k), __ldcg(q.v + w0 + k));
    __syncwarp();
    const int t0 = lane * E, tl = max(0, min(E, wl - t0));
    double ts = 0.0;
    for (int k = 0; k < tl; ++k) ts = dadd(ts, sp[t0 + k]);
    double inc = ts;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double o = __shfl_up_sync(FULL, inc, off);
        if (lane >= off) inc = dadd(inc, o);
    }
    double exc = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) exc = 0.0;
    const double pred = dadd(v, exc);
    Run R = run_empty();
    if (tl > 0) {
        R.e = E_HARD;
        const unsigned long long pb = bt(pred);
        const int e = dexp(pb);
        const int ng = (int)(pb >> 63);
        if (e >= RUN_MIN_E && e <= 0x7f0) {
            const double ref0 = fb(pb & ~1ull), ref1 = fb(bt(ref0) + 1ull);
            double s0 = ref0, s1 = ref1;
            unsigned long long a0 = bt(ref0), z0 = a0, a1 = bt(ref1), z1 = a1;
            for (int k = 0; k < tl; ++k) {
                s0 = dadd(s0, sp[t0 + k]);
                s1 = dadd(s1, sp[t0 + k]);
                a0 = min(a0, bt(s0)); z0 = max(z0, bt(s0));
                a1 = min(a1, bt(s1)); z1 = max(z1, bt(s1));
            }
            const bool same = (a0 >> 52) == (z0 >> 52) && (a1 >> 52) == (z1 >> 52) && (a0 >> 52) == (pb >> 52);
            const double mn0 = ng ? fb(z0) : fb(a0), mx0 = ng ? fb(a0) : fb(z0);
            const double mn1 = ng ? fb(z1) : fb(a1), mx1 = ng ? fb(a1) : fb(z1);
            const double bot = fb(((unsigned long long)e << 52) | 1ull), top = fb(((unsigned long long)e << 52) | MANT);
            if (same && (ng ? (-mx0 >= bot && -mn0 <= top && -mx1 >= bot && -mn1 <= top)
                            : (mn0 >= bot && mx0 <= top && mn1 >= bot && mx1 <= top))) {
                R.d[0] = dsub(s0, ref0); R.d[1] = dsub(s1, ref1);
                R.lo[0] = dsub(mn0, ref0); R.hi[0] = dsub(mx0, ref0);
                R.lo[1] = dsub(mn1, ref1); R.hi[1] = dsub(mx1, ref1);
                R.e = e;
                R.neg = ng;
            }
        }
    }
    for (int t = 0; t < 32; ++t) {  // uniform: every lane carries the same value
        Run G;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            G.d[p] = __shfl_sync(FULL, R.d[p], t);
            G.lo[p] = __shfl_sync(FULL, R.lo[p], t);
            G.hi[p] = __shfl_sync(FULL, R.hi[p], t);
        }
        G.e = __shfl_sync(FULL, R.e, t);
        G.neg = __shfl_sync(FULL, R.neg, t);
        double lo = -INFINITY, hi = INFINITY;
        int km = KM_NONE;
        if (run_apply(G, v, lo, hi, km)) continue;
        if (lane == 0) stat(A.S, ST_CHUNK_FB);
        const int b0 = t * E, bl = max(0, min(E, wl - b0));
        for (int k = 0; k < bl; ++k) v = dadd(v, sp[b0 + k]);
    }
    __syncwarp();
    return v;
}

// All threads of the root: CTA range ci from its true start (*s_v) through its warp pieces
// (staged from global memory); a warp piece that does not apply is walked exactly.
__device__ void walk_warps(const Args& A, const Seq& q, int ci, const Smem& M, double* s_v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) stat(A.S, ST_CTA_FB);
    __syncthreads();  // wd may still be read
    {
        const double2* src = (const double2*)(A.S.warp + (size_t)(q.cta0 + ci) * NW);
        double2* dst = (double2*)M.wd;
        for (int k = threadIdx.x; k < (int)(NW * sizeof(Desc) / 16); k += NT) dst[k] = __ldcg(src + k);
    }
    __syncthreads();
    if (warp == 0) {
        double v = *s_v;
        PieceR P = load_piece(M.wd);
        for (int w = 0; w < NW; ++w) {
            const PieceR Pc = P;
            P = load_piece(M.wd + min(w + 1, NW - 1));  // next piece's loads off the chain
            double lo = -INFINITY, hi = INFINITY;
            int km = KM_NONE;
            if (piece_apply_r(Pc, v, lo, hi, km)) continue;
            if (lane == 0) stat(A.S, ST_WARP_FB);
            v = warp_walk_exact(A, q, ci, w, v, M);
        }
        if (lane == 0) *s_v = v;
    }
    __syncthreads();
}

// All threads of the root: carry the true value (*s_v) through the staged CTA pieces
// [c0, c1) (the stage holds pieces from index b0), rebuilding the ones it cannot use.
__device__ void walk_ctas(const Args& A, const Seq& q, int b0, int c0, int c1, const Smem& M,
                          double* s_red, double* s_v) {
    __shared__ int s_c;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int c = c0;
    while (c < c1) {
        __syncthreads();
        if (warp == 0) {
            double v = *s_v;
            int cc = c;
            PieceR P = load_piece(M.stage + (cc - b0));
            for (; cc < c1; ++cc) {
                const PieceR Pn = load_piece(M.stage + (min(cc + 1, c1 - 1) - b0));
                double lo = -INFINITY, hi = INFINITY;
                int km = KM_NONE;
#ifdef MCR_XDOT_DEBUG
                const double v_in = v;
#endif
                if (!piece_apply_r(P, v, lo, hi, km)) {
#ifdef MCR_XDOT_DEBUG
                    why_failed(A.S, M.stage + (cc - b0), v_in);
#endif
                    break;
                }
                P = Pn;
            }
            if (lane == 0) { *s_v = v; s_c = cc; }
        }
        __syncthreads();
        c = s_c;
        if (c >= c1) break;
        walk_warps(A, q, c, M, s_v);
        ++c;
    }
    __syncthreads();
}

// The last CTA of a sequence: the sequence's sum, from the exact start 0.0.
__device__ double root(const Args& A, const Seq& q, int si, const Smem& M, double* s_red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Scratch& S = A.S;
    const int n = q.ncta;
    __shared__ double s_v;
    __shared__ int s_nf;
    XT_MARK(t_root);
    if (threadIdx.x == 0) {
        s_nf = (int)((__ldcg((const int*)S.flags + si) >> 1) & 1);
        s_v = 0.0;
    }
    __syncthreads();
    if (s_nf) {  // a non-finite product: the reference's IEEE chain, element by element
        if (warp == 0) {
            if (lane == 0) stat(S, ST_SERIAL);
            double v = 0.0;
            for (long long i0 = q.a; i0 < q.b; i0 += 32) {
                const int cnt = (int)min(32ll, q.b - i0);
                const double p = lane < cnt ? dmul(__ldcg(q.u + i0 + lane), __ldcg(q.v + i0 + lane)) : 0.0;
                for (int k = 0; k < cnt; ++k) v = dadd(v, __shfl_sync(FULL, p, k));
            }
            if (lane == 0) s_v = v;
        }
        __syncthreads();
        return s_v;
    }
    __shared__ __align__(8) uint64_t s_bar;
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        mbar_fence_init();
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int b0 = 0; b0 < n; b0 += A.stage) {
        const int b1 = min(n, b0 + A.stage);
        // stage the batch's CTA pieces: one bulk copy (the pieces were written through the
        // generic proxy by other CTAs; the stage may have been read by this one)
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            fence_proxy_async();
            const uint32_t bytes = (uint32_t)(sizeof(Desc) * (size_t)(b1 - b0));
            mbar_expect_tx(&s_bar, bytes);
            bulk_g2s(M.stage, S.cta + q.cta0 + b0, bytes, &s_bar);
        }
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        const int Q = (b1 - b0 + NW - 1) / NW;
        {  // group tables: warp g composes staged pieces [b0 + g Q, ...)
            const int g0 = b0 + warp * Q, g1 = min(b1, g0 + Q);
            Desc* G = M.gd + warp;
            if (g0 < g1) {
                const double gp = M.stage[g0 - b0].h.pred;
                const unsigned long long mb0 = window_mb0(gp);
                const int gn = window_neg(gp);
                double v = cand(mb0, gn, lane), lo = -INFINITY, hi = INFINITY;
                int km = KM_NONE, hole = 0;
                // the next piece is read from shared memory while this one applies (its load
                // latency stays off the value's dependency chain)
                PieceR P = load_piece(M.stage + (g0 - b0));
                for (int c = g0; c < g1; ++c) {
                    const PieceR Pn = load_piece(M.stage + (min(c + 1, g1 - 1) - b0));
                    hole |= piece_apply_r(P, v, lo, hi, km) ? 0 : 1;
                    P = Pn;
                }
                LaneR Lx;
                Lx.out = v; Lx.lo = lo; Lx.hi = hi; Lx.km = km;
                Lx.hole = (hole || dexp(bt(v)) == 0x7ff) ? 1 : 0;
                store_lane(G, lane, Lx);
#ifdef MCR_XDOT_DEBUG
                dbg_check_lane(S, q, q.a + (long long)g0 * NT * A.E, min(q.b, q.a + (long long)g1 * NT * A.E), cand(mb0, gn, lane), load_lane(G, lane), 3);
#endif
                if (lane == 0) hdr_set_table(G->h, mb0, gn, gp);
            } else if (lane == 0) {
                hdr_set_run(G->h, run_empty(), 0.0);  // identity
            }
            __syncwarp();
        }
        __syncthreads();
        XT_ADD(S, ST_T_ROOT_GROUPS, t_root);
        XT_MARK(t_walk);
        // Lane 0 of warp 0 carries the true value through the group tables until one does not
        // apply (no tree over them: their windows already sit at the predictions, and a table
        // application is cheaper than a tree level); a group that does not apply is walked CTA
        // piece by CTA piece by the whole CTA (walk_ctas), then the walk resumes after it.
        __shared__ int s_g;
        const int ngroups = min(NW, (b1 - b0 + Q - 1) / Q);
        for (int g = 0; g < ngroups;) {
            if (warp == 0) {
                double v = s_v;
                int gg = g, ok = 1;
                PieceR P = load_piece(M.gd + gg);
                for (; gg < ngroups; ++gg) {
                    const PieceR Pn = load_piece(M.gd + min(gg + 1, ngroups - 1));
                    double lo = -INFINITY, hi = INFINITY;
                    int km = KM_NONE;
                    ok = piece_apply_r(P, v, lo, hi, km);  // uniform over the warp
                    if (!ok) break;
                    P = Pn;
                }
                if (lane == 0) {
                    s_v = v;
                    s_g = gg;
                }
            }
            __syncthreads();
            g = s_g;
            if (g >= ngroups) break;
            if (threadIdx.x == 0) stat(S, ST_GROUP_FB);
            const int g0 = b0 + g * Q, g1 = min(b1, g0 + Q);
            walk_ctas(A, q, b0, g0, g1, M, s_red, &s_v);
            ++g;
        }
        XT_ADD(S, ST_T_ROOT_WALK, t_walk);
        __syncthreads();
    }
    // cumsum starts from p_0 itself: -0.0 survives only when every product is -0.0
    if (threadIdx.x == 0 && s_v == 0.0 && q.b > q.a && !(__ldcg((const int*)S.flags + si) & 1)) s_v = -0.0;
    if (threadIdx.x == 0) stat(S, ST_T_LAUNCHES);
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

// Per-launch body. Returns true in the one CTA that finished the last sequence, with the
// dots (block partials combined when pardots) in d[0], d[1]; thread 0 only.
__device__ bool xdot_body(const Args& A, double* d) {
    extern __shared__ __align__(16) unsigned char xsm[];
    const Smem M = smem_layout(xsm, A.E);
    __shared__ double s_red[NW];
    __shared__ int s_flag;
    const int si = find_seq(A.seqs, A.nseq, blockIdx.x);
    const Seq q = A.seqs[si];
#ifdef MCR_XDOT_TIMING
    if (threadIdx.x == 0 && A.S.stats) {
        const unsigned long long t = gtime();
        atomicMin(A.S.stats + ST_G_MIN_ENTRY, t);
        atomicMax(A.S.stats + ST_G_MAX_ENTRY, t);
    }
#endif
    build_cta(A, q, si, M, s_red);
    if ((A.upto >= 1 && A.upto <= 4) || A.upto == 13) {  // diagnostics: the build phases alone
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(A.S.done + si, 1u) == (unsigned)(q.ncta - 1)) {
            A.S.ticket[si] = 0u;
            A.S.done[si] = 0u;
            A.S.flags[si] = 0u;
            for (int j = 0; j < q.ncta; ++j) A.S.lb_flag[q.cta0 + j] = 0;
        }
        return false;
    }
#ifdef MCR_XDOT_TIMING
    if (threadIdx.x == 0 && A.S.stats) atomicMax(A.S.stats + ST_G_MAX_BUILD, gtime());
#endif
    // the last CTA of the sequence composes it
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_flag = atomicAdd(A.S.done + si, 1u) == (unsigned)(q.ncta - 1);
    __syncthreads();
    if (!s_flag) return false;
    __threadfence();
#ifdef MCR_XDOT_TIMING
    const unsigned long long g_root0 = gtime();
#endif
    const double r = root(A, q, si, M, s_red);
#ifdef MCR_XDOT_TIMING
    if (threadIdx.x == 0 && A.S.stats && A.nseq == 1) {
        unsigned long long* T = A.S.stats;
        const unsigned long long g1 = gtime(), mn = T[ST_G_MIN_ENTRY], mxe = T[ST_G_MAX_ENTRY], mb = T[ST_G_MAX_BUILD];
        T[ST_G_SKEW] += mxe - mn;
        T[ST_G_BUILD] += mb - mn;
        T[ST_G_ROOT] += g1 - g_root0;
        T[ST_G_TOTAL] += g1 - mn;
        T[ST_G_MIN_ENTRY] = ~0ull;
        T[ST_G_MAX_ENTRY] = 0ull;
        T[ST_G_MAX_BUILD] = 0ull;
        for (int k = 0; k < 4; ++k) {
            T[ST_MS_LOAD + k] += T[ST_M_LOAD + k];
            T[ST_M_LOAD + k] = 0ull;
        }
        for (int k = 0; k < 3; ++k) {
            T[ST_WS_CHAIN + k] += T[ST_W_CHAIN + k];
            T[ST_W_CHAIN + k] = 0ull;
        }
    }
#endif
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

// ---------------------------------------------------------------- one CTA, whole sequence
// For the whole-solve small kernels (small.cuh): K product arrays of length n in shared memory
// (buf + k*n), one CTA of NTH threads; every thread receives the K reference-order sums.
// Thread runs and warp segments as above (predictions from a plain block scan), then lane 0 of
// warp k walks dot k from 0.0 through the warp segments: a segment's merged run where it
// applies to the true value, its products one by one where it does not (a HARD thread is a
// segment of its own). No tables are needed: the walk always holds the exact value, so the
// result is the reference's bits for every input. The walk is one dependent chain, so it
// advances four segments at a time speculatively (each step only needs the value's parity)
// and checks the four steps' conditions afterwards; a group with a failed check is redone
// segment by segment.
// A segment as the walker reads it: 16-byte pairs (one vector load each, then a select on the
// value's parity -- a per-half load would put the shared-memory latency on the walk's chain).
struct __align__(16) SegRun {
    double2 d, lo, hi;
    int e, neg;
    int i0, i1;  // its products [i0, i1)
};

template <int NTH, int K>
struct CtaDots {
    SegRun seg[K][NTH];          // per warp, its segments (compacted)
    int cnt[K][NTH / 32];        // segments per warp
    double red[K][NTH / 32];     // warp totals of the plain sums
    unsigned wfl[K][NTH / 32];   // warp flags: bit 0 a product that is not -0.0, bit 1 non-finite
    double out[K];
};

// One segment from the exact value v: the run's value at v; ok = the run applies (v in the
// run's binade, every partial sum one ulp clear of its ends).
__device__ __forceinline__ double seg_step(const SegRun& R, double v, bool& ok) {
    const double2 d = R.d, l = R.lo, h = R.hi;
    const unsigned long long b = bt(v);
    const bool odd = (b & 1ull) != 0;
    const double vn = dadd(v, odd ? d.y : d.x);
    const int ng = (int)(b >> 63);
    const double vlo = dadd(v, odd ? l.y : l.x), vhi = dadd(v, odd ? h.y : h.x);
    const double bot = fb(((unsigned long long)ng << 63) | ((unsigned long long)R.e << 52) | 1ull);
    const double top = fb(((unsigned long long)ng << 63) | ((unsigned long long)R.e << 52) | MANT);
    const bool in = ng ? (vhi <= bot && vlo >= top) : (vlo >= bot && vhi <= top);
    ok = dexp(b) == R.e && ng == R.neg && in;
    return vn;
}

// the same with the products addressed as a 32-bit shared-memory window offset (no generic ->
// shared conversion per call: the walker runs this for every HARD segment)
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double x;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a));
    return x;
}
__device__ __forceinline__ double walk_elems_s(uint32_t p, int i0, int i1, double v) {
    int i = i0;
    for (; i + 8 <= i1; i += 8) {
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = lds_f64(p + 8u * (uint32_t)(i + j));
#pragma unroll
        for (int j = 0; j < 8; ++j) v = dadd(v, x[j]);
    }
    for (; i < i1; ++i) v = dadd(v, lds_f64(p + 8u * (uint32_t)i));
    return v;
}

constexpr int XS_SERIAL_MAX = 384;  // up to this many products one thread just adds them

template <int NTH, int K>
__device__ void cta_seqdots(const double* buf, int n, CtaDots<NTH, K>& D, double* res) {
    constexpr int NWS = NTH / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef MCR_XS_TIMING
    const long long xt0 = clock64();
    long long xt1 = xt0, xt2 = xt0;
    int nseg = 0, nwalk = 0;
#endif
    if (n <= XS_SERIAL_MAX) {  // the walk alone costs less than building runs
        if (lane == 0 && warp < K) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (k != warp) continue;
                const double* p = buf + (size_t)k * n;
                double v = walk_elems(p, 0, n, 0.0);
                // cumsum starts from p_0 itself: -0.0 survives only when every product is -0.0
                if (v == 0.0 && n > 0) {
                    bool allneg0 = true;
                    for (int i = 0; i < n; ++i) allneg0 &= bt(p[i]) == SGN;
                    if (allneg0) v = -0.0;
                }
                D.out[k] = v;
            }
        }
    } else {
        const int E = (n + NTH - 1) / NTH;
        const int t0 = tid * E, tl = max(0, min(E, n - t0));
        double pred[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double* p = buf + (size_t)k * n + t0;
            double ts = 0.0;
            unsigned fl = 0u;
            for (int i = 0; i < tl; ++i) {
                const double x = p[i];
                const unsigned long long b = bt(x);
                ts = dadd(ts, x);
                fl |= (b != SGN ? 1u : 0u) | (dexp(b) == 0x7ff ? 2u : 0u);
            }
            double inc = ts;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const double o = __shfl_up_sync(FULL, inc, off);
                if (lane >= off) inc = dadd(inc, o);
            }
            const double exc = __shfl_up_sync(FULL, inc, 1);
            pred[k] = lane == 0 ? 0.0 : exc;
            fl = __reduce_or_sync(FULL, fl);
            if (lane == 31) {
                D.red[k][warp] = inc;
                D.wfl[k][warp] = fl;
            }
        }
        __syncthreads();
#ifdef MCR_XS_TIMING
        xt1 = clock64();
#endif
        unsigned flags[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double wexc = 0.0;
            unsigned fl = 0u;
#pragma unroll
            for (int w = 0; w < NWS; ++w) {
                const double r = D.red[k][w];
                if (w < warp) wexc = dadd(wexc, r);
                fl |= D.wfl[k][w];
            }
            flags[k] = fl;
            const Run R = thread_run(buf + (size_t)k * n + t0, tl, dadd(wexc, pred[k]), !(fl & 2u));
            unsigned hd;
            const Run A = warp_merge_runs(R, lane, hd);
            const unsigned ends = (hd >> 1) | 0x80000000u;
            // segments made of EMPTY threads only (past the end of the products) are dropped;
            // they come after every other segment, so the compaction keeps the order
            const unsigned live = __ballot_sync(FULL, ((ends >> lane) & 1u) && A.e != E_EMPTY);
            if ((live >> lane) & 1u) {  // compact: segment j = lanes [first, lane]
                const unsigned before = ends & ((1u << lane) - 1u);
                const int first = before ? 32 - __clz(before) : 0;
                SegRun& S = D.seg[k][warp * 32 + __popc(live & ((1u << lane) - 1u))];
                S.d = make_double2(A.d[0], A.d[1]);
                S.lo = make_double2(A.lo[0], A.lo[1]);
                S.hi = make_double2(A.hi[0], A.hi[1]);
                S.e = A.e;
                S.neg = A.neg;
                S.i0 = (warp * 32 + first) * E;
                S.i1 = min(n, (warp * 32 + lane + 1) * E);
            }
            if (lane == 0) D.cnt[k][warp] = __popc(live);
        }
        __syncthreads();
#ifdef MCR_XS_TIMING
        xt2 = clock64();
#endif
        if (lane == 0 && warp < K) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (k != warp) continue;
                const uint32_t ps = smem_u32(buf + (size_t)k * n);
                double v = 0.0;
                // products to add one by one are collected into one pending stretch [w0, w1)
                // (consecutive HARD segments, failed runs, warps of short segments) and added
                // when a run is about to apply
                int w0 = 0, w1 = 0;
                for (int w = 0; w < NWS; ++w) {
                    const int cnt = D.cnt[k][w];
                    const SegRun* sg = &D.seg[k][w * 32];
#ifdef MCR_XS_TIMING
                    nseg += cnt;
#endif
                    const int we0 = w * 32 * E, we1 = min(n, (w + 1) * 32 * E);
                    if (cnt * 32 > we1 - we0) {  // a segment costs about 32 adds: many short ones, all one by one
                        if (w1 != we0) { v = walk_elems_s(ps, w0, w1, v); w0 = we0; }
                        w1 = max(w1, we1);
#ifdef MCR_XS_TIMING
                        nwalk += max(0, we1 - we0);
#endif
                        continue;
                    }
                    // the next segment is loaded while this one is applied (its shared-memory
                    // latency stays off the value's dependency chain); a HARD segment (e = 0)
                    // never matches the exponent of a value that a run could apply to
                    SegRun cur = sg[0];
                    for (int j = 0; j < cnt; ++j) {
                        const SegRun nxt = sg[min(j + 1, cnt - 1)];
                        if (cur.e == E_HARD) {
                            if (w1 != cur.i0) { v = walk_elems_s(ps, w0, w1, v); w0 = cur.i0; }
                            w1 = cur.i1;
#ifdef MCR_XS_TIMING
                            nwalk += cur.i1 - cur.i0;
#endif
                        } else {
                            if (w1 > w0) v = walk_elems_s(ps, w0, w1, v);
                            w0 = w1 = cur.i1;
                            bool ok;
                            const double vn = seg_step(cur, v, ok);
                            if (ok) {
                                v = vn;
                            } else {
                                w0 = cur.i0;
#ifdef MCR_XS_TIMING
                                nwalk += cur.i1 - cur.i0;
#endif
                            }
                        }
                        cur = nxt;
                    }
                }
                if (w1 > w0) v = walk_elems_s(ps, w0, w1, v);
                // cumsum starts from p_0 itself: -0.0 survives only when every product is -0.0
                if (v == 0.0 && !(flags[k] & 1u)) v = -0.0;
                D.out[k] = v;
            }
        }
    }
#ifdef MCR_XS_TIMING
    const long long xt3 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        static __device__ int xs_calls = 0;
        if (xs_calls < 12) {
            ++xs_calls;
            printf("xs n=%d K=%d: runs %lld merge %lld walk %lld cycles, segments %d, walked %d\n", n, K,
                   xt1 - xt0, xt2 - xt1, xt3 - xt2, nseg, nwalk);
        }
    }
#endif
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) res[k] = D.out[k];
}

}  // namespace xd

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
    if (W != SQ_TEST && st->sharded) {  // the exchange point finishes (k_finalize)
        st->xd[0] = d[0];
        st->xd[1] = d[1];
        return;
    }
    if constexpr (W == SQ_S0) fin_s0(st, d[0]);
    else if constexpr (W == SQ_V) fin_v(st, d[0]);
    else if constexpr (W == SQ_T) fin_t(st, d[0], d[1]);
    else if constexpr (W == SQ_E) {
        fin_e(st, d[0]);
        graph_continue(st);
    }
}

}  // namespace mcr
