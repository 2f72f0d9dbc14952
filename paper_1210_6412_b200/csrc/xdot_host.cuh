// xdot_host.cuh -- launch plans and scratch of the bit-exact sequential dots (xdot.cuh).
// Part of the single translation unit mcr.cu (after handle.h, before solve.cuh).
#pragma once

namespace {

// Scratch + one plan per reduction point (SQ_S0, SQ_V, SQ_T, SQ_E, SQ_TEST).
struct XdotCtx {
    int grid_cap = 0, nseq_cap = 0;
    void* blk = nullptr;
    size_t blk_bytes = 0;
    xd::Scratch S{};
    struct Plan {
        xd::Seq* d_seqs = nullptr;
        int nseq = 0, nseq0 = 0, ndot = 1, pardots = 0, grid = 0, E = 1, nblocks = 1;
        const double* key[4] = {nullptr, nullptr, nullptr, nullptr};
        size_t smem = 0;
        int stage = 1;
        int64_t n = -1;
    } plan[5];
    std::vector<void*> seq_bufs;
    unsigned long long* stats = nullptr;  // MCR_XDOT_STATS=1: fallback counters (diagnostics)
};

// solvers.py:159-168 _row_blocks: base + 1 rows for the first n % k blocks
inline void row_blocks(int64_t n, int k, std::vector<int64_t>& lo, std::vector<int64_t>& hi) {
    lo.clear();
    hi.clear();
    const int64_t base = n / k, extra = n % k;
    int64_t start = 0;
    for (int i = 0; i < k; ++i) {
        const int64_t size = base + (i < extra ? 1 : 0);
        lo.push_back(start);
        hi.push_back(start + size);
        start += size;
    }
}

// dynamic shared memory a k_xdot CTA may use: the opt-in maximum less the kernel's static part
inline int xdot_smem_max() {
    static int v = 0;
    if (v) return v;
    int dev = 0, optin = 227 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    int stat_bytes = 1024;
    if (cudaFuncGetAttributes(&fa, k_xdot<SQ_TEST>) == cudaSuccess) stat_bytes = (int)fa.sharedSizeBytes;
    v = optin - stat_bytes - 256;
    return v;
}

// resident k_xdot CTAs per SM the plans are sized for (MCR_XDOT_CPS, tuning; default 1) and the
// dynamic shared memory each may then use
inline int xdot_cps() {
    static int v = 0;
    if (!v) {
        const char* env = std::getenv("MCR_XDOT_CPS");
        v = env ? std::max(1, std::min(4, std::atoi(env))) : 1;
    }
    return v;
}
inline size_t xdot_smem_budget() {
    const int cps = xdot_cps();
    if (cps == 1) return (size_t)xdot_smem_max();
    int dev = 0, per_sm = 228 * 1024, rsv = 1024, optin = 227 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int stat_bytes = optin - 256 - xdot_smem_max();
    return (size_t)std::min(xdot_smem_max(), per_sm / cps - rsv - stat_bytes - 256);
}

inline int sm_count(int device) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    return nsm > 0 ? nsm : 148;
}

template <int W>
int xdot_smem_attr() {
    static int done = 0;
    if (done) return MCR_OK;
    CK(cudaFuncSetAttribute(k_xdot<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, xdot_smem_max()));
    done = 1;
    return MCR_OK;
}

// (Re)build plan `w`: ndot dots over n elements, pairs (u0, v0) and (u1, v1), each split into
// `nblocks` row blocks when nblocks > 1 (parallel_dot_products).
int xdot_plan(XdotCtx& X, int w, cudaStream_t s, int device, int64_t n, int ndot, int nblocks,
              const double* u0, const double* v0, const double* u1, const double* v1) {
    auto& P = X.plan[w];
    const double* key[4] = {u0, v0, u1, v1};
    if (P.d_seqs && P.n == n && P.ndot == ndot && P.nblocks == nblocks &&
        std::equal(key, key + 4, P.key))
        return MCR_OK;
    const int nb = std::max(1, nblocks);
    std::vector<int64_t> lo, hi;
    row_blocks(n, nb, lo, hi);
    const int nsm = sm_count(device) * xdot_cps();  // CTA slots
    const int64_t total = (int64_t)ndot * n;
    // one CTA per SM (the shared memory is sized for that): the smallest odd E whose grid fits
    int64_t E = (total + (int64_t)xd::NT * nsm - 1) / ((int64_t)xd::NT * nsm);
    E = std::max<int64_t>(1, std::min<int64_t>(E, xd::EMAX)) | 1;
    auto grid_of = [&](int64_t e) {
        int64_t g = 0;
        for (int k = 0; k < ndot; ++k)
            for (int b = 0; b < nb; ++b)
                g += std::max<int64_t>(1, (hi[b] - lo[b] + (int64_t)xd::NT * e - 1) / ((int64_t)xd::NT * e));
        return g;
    };
    while (E + 2 <= xd::EMAX && grid_of(E) > nsm) E += 2;
    // q.v and q.r (the V and E points): one step smaller ranges per CTA pay even with a few
    // CTAs in a second wave (C2, 256 threads: V 27 -> 25, 157 CTAs on 148 SMs, BiCGStab
    // 24.73 -> 24.38 ms; E 27 -> 25 neutral; a bigger second wave, E 23: 28.4 ms). The T point
    // (two dots) fills the SMs at E = 53 (31: 25.32 ms, 45: 25.45, 63: 28.27).
    if ((w == SQ_E || w == SQ_V) && E >= 3 && grid_of(E - 2) <= nsm + nsm / 16) E -= 2;
    if (const char* env = std::getenv("MCR_XDOT_E")) E = std::max(1, std::min(xd::EMAX, std::atoi(env))) | 1;
    {  // per reduction point (tuning): MCR_XDOT_E0 .. MCR_XDOT_E3 for S0, V, T, E
        char name[16];
        std::snprintf(name, sizeof(name), "MCR_XDOT_E%d", w);
        if (const char* env = std::getenv(name)) E = std::max(1, std::min(xd::EMAX, std::atoi(env))) | 1;
    }
    const int64_t per = (int64_t)xd::NT * E;
    std::vector<xd::Seq> seqs;
    int grid = 0;
    for (int k = 0; k < ndot; ++k) {
        for (int b = 0; b < nb; ++b) {
            xd::Seq q{};
            q.u = k == 0 ? u0 : u1;
            q.v = k == 0 ? v0 : v1;
            q.a = lo[b];
            q.b = hi[b];
            q.cta0 = grid;
            q.ncta = (int)std::max<int64_t>(1, (hi[b] - lo[b] + per - 1) / per);
            grid += q.ncta;
            seqs.push_back(q);
        }
    }
    const int nseq = (int)seqs.size();
    if (grid > X.grid_cap || nseq > X.nseq_cap) {
        const int gc = std::max(grid, X.grid_cap), sc = std::max(nseq, X.nseq_cap);
        const size_t bytes = sizeof(xd::Desc) * (size_t)gc * (1 + xd::NW) + sizeof(double) * (size_t)gc +
                             sizeof(int) * (size_t)gc + sizeof(double) * (size_t)sc +
                             sizeof(unsigned) * (size_t)(3 * sc + 1) + 256;
        if (X.blk) CK(cudaFreeAsync(X.blk, s));
        CK(cudaMallocAsync(&X.blk, bytes, s));
        CK(cudaMemsetAsync(X.blk, 0, bytes, s));
        X.blk_bytes = bytes;
        char* p = (char*)X.blk;
        auto take = [&](size_t b) { char* r = p; p += (b + 15) & ~(size_t)15; return r; };
        X.S.cta = (xd::Desc*)take(sizeof(xd::Desc) * (size_t)gc);
        X.S.warp = (xd::Desc*)take(sizeof(xd::Desc) * (size_t)gc * xd::NW);
        X.S.lb_val = (double*)take(sizeof(double) * (size_t)gc);
        X.S.result = (double*)take(sizeof(double) * (size_t)sc);
        X.S.lb_flag = (int*)take(sizeof(int) * (size_t)gc);
        X.S.ticket = (unsigned*)take(sizeof(unsigned) * (size_t)sc);
        X.S.done = (unsigned*)take(sizeof(unsigned) * (size_t)sc);
        X.S.flags = (unsigned*)take(sizeof(unsigned) * (size_t)sc);
        X.S.all_done = (unsigned*)take(sizeof(unsigned));
        X.grid_cap = gc;
        X.nseq_cap = sc;
    }
    if (!X.stats && std::getenv("MCR_XDOT_STATS")) {
        CK(cudaMallocAsync((void**)&X.stats, sizeof(unsigned long long) * xd::ST_COUNT, s));
        CK(cudaMemsetAsync(X.stats, 0, sizeof(unsigned long long) * xd::ST_COUNT, s));
        const unsigned long long big = ~0ull;
        CK(cudaMemcpyAsync(X.stats + xd::ST_G_MIN_ENTRY, &big, sizeof(big), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    X.S.stats = X.stats;
    if (P.d_seqs) CK(cudaFreeAsync(P.d_seqs, s));
    CK(cudaMallocAsync((void**)&P.d_seqs, sizeof(xd::Seq) * seqs.size(), s));
    CK(cudaMemcpyAsync(P.d_seqs, seqs.data(), sizeof(xd::Seq) * seqs.size(), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // the host vector dies here
    P.nseq = nseq;
    P.nseq0 = nb;
    P.ndot = ndot;
    P.pardots = nb > 1 ? 1 : 0;
    P.nblocks = nblocks;
    P.grid = grid;
    P.E = (int)E;
    // the root stages its sequence's CTA pieces in shared memory (in batches if they do not fit)
    int maxc = 1;
    for (const auto& q : seqs) maxc = std::max(maxc, q.ncta);
    size_t budget = xdot_smem_budget();
    if (budget < xd::smem_bytes((int)E, 1)) budget = (size_t)xdot_smem_max();  // E too large for the cap
    const int room = (int)((budget - xd::smem_bytes((int)E, 0)) / sizeof(xd::Desc));
    P.stage = std::max(1, std::min(maxc, room));
    P.smem = xd::smem_bytes((int)E, P.stage);
    P.n = n;
    std::copy(key, key + 4, P.key);
    return MCR_OK;
}

xd::Args xdot_args(const XdotCtx& X, int w, double* out) {
    const auto& P = X.plan[w];
    xd::Args A{};
    A.seqs = P.d_seqs;
    A.nseq = P.nseq;
    A.nseq0 = P.nseq0;
    A.ndot = P.ndot;
    A.pardots = P.pardots;
    A.E = P.E;
    A.stage = P.stage;
    static const int upto = std::getenv("MCR_XDOT_UPTO") ? std::atoi(std::getenv("MCR_XDOT_UPTO")) : 0;
    A.upto = upto;
    A.S = X.S;
    A.out = out;
    return A;
}

void xdot_free(XdotCtx* X, cudaStream_t s) {
    if (!X) return;
    for (auto& P : X->plan)
        if (P.d_seqs) cudaFreeAsync(P.d_seqs, s);
    if (X->blk) cudaFreeAsync(X->blk, s);
    if (X->stats) cudaFreeAsync(X->stats, s);
    delete X;
}

}  // namespace
