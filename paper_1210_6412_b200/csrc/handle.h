// handle.h -- host-side state of libmcr.so: error plumbing, the matrix / communicator / chain
// handles, device allocation helpers and the work-vector layout. Part of the single
// translation unit mcr.cu (included in order: handle.h, storage.cuh, solve.cuh, chain_host.cuh).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_scan.cuh>
#include <nvtx3/nvToolsExt.h>  // header-only: ranges cost nothing unless a tool attaches

#include "comm.h"
#include "device.cuh"
#include "chain.cuh"
#include "generator.cuh"
#include "mcr.h"

using namespace mcr;

namespace {

thread_local std::string g_err;

// NVTX range for the lifetime of a scope ("mcr.jacobi", "mcr.create", ...), visible in
// Nsight Systems / Compute timelines.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// MCR_TRACE=1: host timestamps of the create / solve stages on stderr (profiling aid).
struct Trace {
    bool on = std::getenv("MCR_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[mcr] %-28s %8.3f ms\n", what, ms);
    }
};

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(MCR_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// First failed kernel launch of this thread since the last launch_check(): launch_pdl records it
// (cudaLaunchKernelEx's status) so a launch failure surfaces at the next check even when the
// launcher itself has no status to return (graph bodies, batch loops).
thread_local cudaError_t g_launch_err = cudaSuccess;

inline void note_launch(cudaError_t e) {
    if (e != cudaSuccess && g_launch_err == cudaSuccess) g_launch_err = e;
}

inline int launch_check() {
    cudaError_t e = g_launch_err;
    g_launch_err = cudaSuccess;
    const cudaError_t last = cudaGetLastError();
    if (e == cudaSuccess) e = last;
    if (e != cudaSuccess) return fail(MCR_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
    return MCR_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Work vectors. FULL ones are gather inputs of the SpMV and span the whole system when the
// matrix is a row shard (world * chunk entries, indexed by global row); the others hold this
// handle's rows only. On one GPU both kinds are n long.
enum { V_X = 0, V_X1, V_P, V_S, V_R, V_Q, V_V, V_T, V_FULL_COUNT, V_B = V_FULL_COUNT, V_COUNT };

}  // namespace

struct mcr_matrix;
namespace {
struct XdotCtx;  // xdot_host.cuh
}

// A Markov chain with its goal set and the reduced system built from it (chain.cuh).
struct mcr_chain {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t n = 0, nnz = 0, k = 0, m_nnz = 0, nzero = 0, none = 0;
    long long* rp = nullptr;
    int* col = nullptr;
    double* val = nullptr;
    unsigned char* goal = nullptr;
    signed char* cls = nullptr;
    long long* remap = nullptr;
    long long* list = nullptr;
    long long* mrp = nullptr;
    int* mcol = nullptr;
    double* mval = nullptr;
    double* rhs = nullptr;
    double* xs = nullptr;
    double* xfull = nullptr;
    mcr_matrix* M = nullptr;  // solve-ready handle of M (created on first use)
    std::vector<void*> owned;
    std::mutex mu;
};

// Communicator of a row-sharded solve (comm.h): NCCL, or the in-process local group.
struct mcr_comm {
    std::shared_ptr<mcr::Transport> t;
};

struct mcr_matrix {
    int device = 0;
    int64_t n = 0, nnz = 0;           // rows (and entries) held by this handle
    // row sharding: this handle holds rows [roff, roff + n) of an n_global system; every rank
    // holds `chunk` = ceil(n_global / world) rows except the last
    int world = 1, rank = 0;
    int64_t n_global = 0, roff = 0, chunk = 0;
    std::shared_ptr<Transport> comm;
    double* recv = nullptr;           // world * SEND_SLOTS exchanged partials
    // peer-to-peer mode (mcr_shard_enable_p2p): the full vectors live in `fullblk` (cudaMalloc,
    // IPC-exportable); d_peers[slot * world + q] = rank q's copy, mapped here
    int p2p = 0;
    double* fullblk = nullptr;
    double** d_peers = nullptr;
    std::vector<void*> ipc_opened;
    int storage = MCR_STORAGE_CSR;
    cudaStream_t own_stream = nullptr, stream = nullptr;
    // full matrix, CSR
    long long* rp = nullptr;
    int* col = nullptr;
    double* val = nullptr;
    int* tile_row = nullptr;
    TileDesc* desc = nullptr;     // tiles of the full matrix
    TileDesc* rdesc = nullptr;    // tiles of the off-diagonal copy
    int ntiles = 0;
    // off-diagonal copy for Jacobi (lazy)
    long long* offlen = nullptr;
    long long* rrp = nullptr;
    int* rcol = nullptr;
    double* rval = nullptr;
    bool r_ready = false;
    // SELL-32-sigma copies (short-row matrices): full matrix and off-diagonal R
    struct SellDev {
        long long* sptr = nullptr;
        int* perm = nullptr;
        int* col = nullptr;
        double* val = nullptr;
        long long* swidth = nullptr;
        int nwin = 0;
        long long slots = 0;
    } sell, rsell;
    bool use_sell = false;
    // band-staged copy (staged.cuh): systems whose x is far larger than L2
    struct StagedDev {
        double* pval = nullptr;
        int* pcol = nullptr;
        unsigned short* lidx = nullptr;
        double* prod = nullptr;
        unsigned long long* seg = nullptr;
        long long npos = 0;
        int nb = 0, band = 0;
        int p1_grid = 1, grid = 1;  // pass-1 / pass-2 CTAs
    } stg;
    bool use_staged = false;
    // dense slabs
    double* dense = nullptr;
    int nslabs = 0;
    // diagonal + facts
    double* d = nullptr;
    long long first_zero = -1;
    unsigned long long fz_host[2] = {~0ull, 0ull};  // D2H target: first zero-diagonal row,
                                                    // count of stored diagonal entries
    int64_t nnz_off = 0;                            // entries of Jacobi's off-diagonal copy
    int bad_host[2] = {0, 0};            // D2H target of the upload checks
    long long max_row = 0;
    // workspace
    double* work = nullptr;
    double* P = nullptr;
    int nunits = 0;
    SolveState* st = nullptr;
    SolveState h_state{};
    SolveState* h_st = &h_state;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t bytes = 0;
    int seqdots = 0;       // 0 tree dots, 1 reference order (k_xdot), 2 reference order, serial
    int dot_blocks = 1;    // > 1: parallel_dot_products over that many row blocks
    XdotCtx* xdot = nullptr;
    // graph mode (solve.cuh): the whole iteration loop as one CUDA graph with a while node
    struct GraphLoop {
        cudaGraphExec_t exec = nullptr;
        cudaGraph_t graph = nullptr;
        unsigned long long cond = 0;
        int unroll = 1;
        bool failed = false;
        long long key = -1;  // dot mode and blocks the body was captured with
    } gl_bicg;
    int bicg_solves = 0;
    int spmv_grid = 1;
    int small_grid = 0;                     // > 0: whole solve in one cooperative launch
    bool small_cluster = false;             // ... launched as one thread-block cluster
    bool small_xd = false;                  // ... and its reference-order-dot variant fits too
    double* xsprod = nullptr;               // that variant's product slots (4n)
    unsigned long long* maxslot = nullptr;  // 3 slots for the persistent solvers
    std::mutex mu;

    int64_t n_full() const { return comm ? chunk * world : n; }
    double* vec(int k) const {
        if (k < V_FULL_COUNT && fullblk) return fullblk + (size_t)k * (size_t)n_full();
        return k < V_FULL_COUNT ? work + (size_t)k * (size_t)n_full()
                                : work + (size_t)V_FULL_COUNT * (size_t)n_full() +
                                      (size_t)(k - V_FULL_COUNT) * (size_t)n;
    }
    // a row shard (mcr_shard_create) runs the exchange points even at world 1, so the NCCL
    // transport is exercised end to end on a one-GPU box
    bool sharded() const { return comm != nullptr; }
    int nchunks() const { return (int)((n + CHUNK_ROWS - 1) / CHUNK_ROWS); }
};

namespace {

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync) with the
// release threshold lifted, so creating and destroying handles (the end-to-end path uploads a
// matrix per solve) recycles memory instead of paying cudaMalloc/cudaFree each time.
template <class T>
int dalloc(mcr_matrix* h, T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    CK(cudaMallocAsync((void**)p, sizeof(T) * count, h->stream));
    h->bytes += (int64_t)(sizeof(T) * count);
    return MCR_OK;
}

template <class T>
void dfree(mcr_matrix* h, T*& p, size_t count) {
    if (p) {
        cudaFreeAsync(p, h->stream);
        h->bytes -= (int64_t)(sizeof(T) * (count ? count : 1));
        p = nullptr;
    }
}

int keep_pool_memory(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return MCR_OK;
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done.push_back(device);
    return MCR_OK;
}

#define TRY(x)                   \
    do {                         \
        int rc_ = (x);           \
        if (rc_ != MCR_OK) return rc_; \
    } while (0)

Csr csr_full(const mcr_matrix* h) {
    return Csr{h->rp, h->col, h->val, h->desc, h->ntiles, (int)h->n};
}
Staged staged_view(const mcr_matrix* h) {
    const auto& S = h->stg;
    static const int early = std::getenv("MCR_STAGED_PDL") ? std::atoi(std::getenv("MCR_STAGED_PDL")) : 0;
    return Staged{h->rp, S.lidx, S.seg, S.pval, S.pcol, S.prod, h->desc, S.npos, h->ntiles, S.nb, early};
}
Csr csr_off(const mcr_matrix* h) {
    return Csr{h->rrp, h->rcol, h->rval, h->rdesc, h->ntiles, (int)h->n};
}

// Own-row views (x, p, s point at this rank's slice of the full vectors).
Vecs base_vecs(const mcr_matrix* h) {
    Vecs V{};
    V.b = h->vec(V_B);
    V.d = h->d;
    V.x = h->vec(V_X) + h->roff;
    // r, q, v, t are full length too: on a row shard with reference-order dots they are
    // gathered and every rank sums the whole vectors (sharded xdot_prepare)
    V.r = h->vec(V_R) + h->roff;
    V.q = h->vec(V_Q) + h->roff;
    V.p = h->vec(V_P) + h->roff;
    V.v = h->vec(V_V) + h->roff;
    V.s = h->vec(V_S) + h->roff;
    V.t = h->vec(V_T) + h->roff;
    V.P1 = h->P;
    V.P2 = h->P + h->nunits;
    V.x_jac0 = h->vec(V_X);
    V.x_jac1 = h->vec(V_X1);
    V.roff = h->roff;
    V.peers = h->p2p ? h->d_peers : nullptr;
    V.world = h->world;
    V.rank = h->rank;
    V.xnext_slot = FV_X;
    return V;
}

int ensure_work(mcr_matrix* h) {
    if (h->work) return MCR_OK;
    const size_t words = (size_t)V_FULL_COUNT * (size_t)h->n_full() +
                         (size_t)(V_COUNT - V_FULL_COUNT) * (size_t)h->n;
    TRY(dalloc(h, &h->work, words));
    // full vectors start zeroed: blocks past the last rank's rows are gathered but never read
    if (h->sharded())
        CK(cudaMemsetAsync(h->work, 0, sizeof(double) * (size_t)V_FULL_COUNT * (size_t)h->n_full(),
                           h->stream));
    h->nunits = std::max({h->ntiles, h->nchunks(), h->nslabs, h->sell.nwin * (SELL_W / SELL_CTA), 1});
    TRY(dalloc(h, &h->P, (size_t)4 * h->nunits));  // P1, P2 (+ 2 more slots: k_bicg_small)
    if (h->sharded()) TRY(dalloc(h, &h->recv, (size_t)h->world * SEND_SLOTS));
    return MCR_OK;
}

}  // namespace
