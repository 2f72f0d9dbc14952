// chain.cuh -- the reduced reachability system of a Markov chain, built on the device
// (build_system, mcreach/markov.py:152-256, sparse.py:208-224).
//
//   reversed digraph     one edge t <- s for every stored transition s -> t (_reversed_adjacency,
//                        markov.py:152-159); adjacency order is irrelevant to the closures
//   two closures         states that reach the goals (markov.py:196), then, on paths that avoid
//                        the goals, states that reach the zero-probability set (:198-201); a
//                        level-synchronous BFS in ONE cooperative launch (grid barrier per level)
//   uncertain states     neither zero nor one, ascending; remap = exclusive scan of the flags
//   M = I - A            over the uncertain states: off-diagonal entries negated, diagonal
//                        1 - a_ss (or 1 when no self-loop), dropped when exactly zero
//                        (identity_minus, sparse.py:208-224); columns stay ascending because
//                        the remap is monotone
//   rhs                  one-step goal probability, summed exactly like numpy's float64
//                        np.sum over the row's goal entries (pairwise blocks of 8 accumulators,
//                        markov.py:228-231) -- bit-identical
#pragma once

#include <cooperative_groups.h>
#include <stdint.h>

namespace mcr {

__global__ void k_rev_count(const long long* __restrict__ rp, const int* __restrict__ col,
                            long long nnz, unsigned long long* cnt) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
         e += (long long)gridDim.x * blockDim.x)
        atomicAdd(cnt + col[e], 1ull);
}

__global__ void k_rev_fill(const long long* __restrict__ rp, const int* __restrict__ col, int n,
                           const unsigned long long* __restrict__ rev_rp,
                           unsigned long long* cursor, int* rev_src) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x)
        for (long long e = rp[s]; e < rp[s + 1]; ++e) {
            const int t = col[e];
            rev_src[rev_rp[t] + atomicAdd(cursor + t, 1ull)] = s;
        }
}

// Seeds: states with flag[s] == want (goal mask for the first closure, "zero" for the second).
__global__ void k_seed(const unsigned char* __restrict__ flag, unsigned char want, int n,
                       int* seen, int* frontier, unsigned* len) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x)
        if (flag[s] == want) {
            seen[s] = 1;
            frontier[atomicAdd(len, 1u)] = s;
        }
}

// Backward closure from the seeded frontier; states with blocked[t] != 0 are never entered.
// len[3] rotate as in k_jacobi_small: level L reads len[L%3], pushes into len[(L+1)%3] and
// clears len[(L+2)%3] (read before the previous barrier, written only after the next).
__global__ void k_closure(const unsigned long long* __restrict__ rev_rp,
                          const int* __restrict__ rev_src, const unsigned char* __restrict__ blocked,
                          int* seen, int* fa, int* fb, unsigned* len) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const unsigned T = gridDim.x * blockDim.x;
    const unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
    int* cur = fa;
    int* nxt = fb;
    for (int level = 0;; ++level) {
        const unsigned ncur = *(volatile unsigned*)(len + level % 3);
        if (ncur == 0) break;
        if (tid == 0) len[(level + 2) % 3] = 0u;
        for (unsigned i = tid; i < ncur; i += T) {
            const int s = cur[i];
            for (unsigned long long e = rev_rp[s]; e < rev_rp[s + 1]; ++e) {
                const int t = rev_src[e];
                if (blocked && blocked[t]) continue;
                if (*(volatile int*)(seen + t)) continue;
                if (atomicCAS(seen + t, 0, 1) == 0) nxt[atomicAdd(len + (level + 1) % 3, 1u)] = t;
            }
        }
        grid.sync();
        int* tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
}

__global__ void k_zero_flag(const int* __restrict__ reach_goal, int n, unsigned char* zero) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x)
        zero[s] = reach_goal[s] == 0;
}

// class: 0 = probability zero, 1 = probability one, 2 = uncertain; flag for the scan.
__global__ void k_classes(const int* __restrict__ reach_goal, const int* __restrict__ reach_zero,
                          int n, signed char* cls, long long* unc) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        const signed char c = !reach_goal[s] ? 0 : (!reach_zero[s] ? 1 : 2);
        cls[s] = c;
        unc[s] = c == 2;
    }
}

// After the exclusive scan: remap[s] (in place over the scanned flags) and the ascending list.
__global__ void k_uncertain_list(const signed char* __restrict__ cls, int n, long long* remap,
                                 long long* list) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        if (cls[s] == 2) list[remap[s]] = s;
        else remap[s] = -1;
    }
}

// Row lengths of M and the counts of goal entries (rhs terms), per uncertain row.
__global__ void k_m_count(const long long* __restrict__ rp, const int* __restrict__ col,
                          const double* __restrict__ val, const long long* __restrict__ list,
                          long long k, const long long* __restrict__ remap,
                          const unsigned char* __restrict__ goal, long long* mlen, long long* glen) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < k;
         i += (long long)gridDim.x * blockDim.x) {
        const long long s = list[i];
        long long cnt = 0, g = 0;
        double d = 1.0;
        for (long long e = rp[s]; e < rp[s + 1]; ++e) {
            const int t = col[e];
            if (goal[t]) ++g;
            if (remap[t] < 0) continue;
            if (t == s) d = __dsub_rn(1.0, val[e]);
            else ++cnt;
        }
        mlen[i] = cnt + (d != 0.0);
        glen[i] = g;
    }
}

__global__ void k_m_fill(const long long* __restrict__ rp, const int* __restrict__ col,
                         const double* __restrict__ val, const long long* __restrict__ list,
                         long long k, const long long* __restrict__ remap,
                         const unsigned char* __restrict__ goal,
                         const long long* __restrict__ mrp, int* mcol, double* mval,
                         const long long* __restrict__ goff, double* gsel) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < k;
         i += (long long)gridDim.x * blockDim.x) {
        const long long s = list[i];
        double d = 1.0;
        for (long long e = rp[s]; e < rp[s + 1]; ++e)
            if (col[e] == s) d = __dsub_rn(1.0, val[e]);
        long long o = mrp[i], go = goff[i];
        bool placed = d == 0.0;  // a zero diagonal is dropped (_assemble keeps vals != 0)
        for (long long e = rp[s]; e < rp[s + 1]; ++e) {
            const int t = col[e];
            if (goal[t]) gsel[go++] = val[e];
            const long long rt = remap[t];
            if (rt < 0 || t == s) continue;
            if (!placed && rt > i) {
                mcol[o] = (int)i;
                mval[o++] = d;
                placed = true;
            }
            mcol[o] = (int)rt;
            mval[o++] = -val[e];
        }
        if (!placed) {
            mcol[o] = (int)i;
            mval[o] = d;
        }
    }
}

// numpy's float64 pairwise summation (umath loops_utils pairwise_sum, PW_BLOCKSIZE 128).
__device__ double np_pairwise(const double* a, long long n) {
    if (n < 8) {
        double res = -0.0;
        for (long long i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        long long i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

// rhs_i = np.sum(goal entries of row s) = 0.0 + pairwise(...) (the reduction starts from the
// additive identity, which only matters for a -0.0 result).
__global__ void k_rhs(const long long* __restrict__ goff, long long k, const double* __restrict__ gsel,
                      double* rhs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < k;
         i += (long long)gridDim.x * blockDim.x)
        rhs[i] = __dadd_rn(0.0, np_pairwise(gsel + goff[i], goff[i + 1] - goff[i]));
}

// reachability_probabilities (markov.py:283-293): certain states exact, solved ones clipped.
__global__ void k_scatter_x(const signed char* __restrict__ cls, const long long* __restrict__ remap,
                            const double* __restrict__ xs, int n, double* x) {
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        const signed char c = cls[s];
        double v = c == 1 ? 1.0 : 0.0;
        if (c == 2) {
            v = xs[remap[s]];
            if (v < 0.0) v = 0.0;        // np.clip: NaN and -0.0 pass through
            else if (v > 1.0) v = 1.0;
        }
        x[s] = v;
    }
}

}  // namespace mcr
