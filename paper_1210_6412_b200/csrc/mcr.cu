// mcr.cu -- host side of libmcr.so: device storage, solve drivers and the C ABI (include/mcr.h).
//
// A handle uploads the reference's CSR once (sparse.py:71-98 keeps a cached scipy handle the
// same way), derives the diagonal and the first zero-diagonal row on the device, cuts the
// rows into shared-memory tiles, and (for >= 2/3-full matrices) re-lays the matrix out as
// dense 32-row slabs. The Jacobi off-diagonal copy (without_diagonal, sparse.py:227-231) is
// built on the device the first time Jacobi runs on the handle. Solves run entirely on the
// device: every kernel reads the solver state (iteration, scalars, stop flag) from device
// memory, so the host only enqueues batches of iterations and polls the stop flag once per
// batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "comm.h"
#include "device.cuh"
#include "chain.cuh"
#include "generator.cuh"
#include "mcr.h"

using namespace mcr;

namespace {

thread_local std::string g_err;

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
enum { V_X = 0, V_X1, V_P, V_S, V_FULL_COUNT, V_B = V_FULL_COUNT, V_R, V_Q, V_V, V_T, V_COUNT };

}  // namespace

struct mcr_matrix;

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
    // dense slabs
    double* dense = nullptr;
    int nslabs = 0;
    // diagonal + facts
    double* d = nullptr;
    long long first_zero = -1;
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
    int seqdots = 0;
    int spmv_grid = 1;
    int small_grid = 0;                     // > 0: whole solve in one cooperative launch
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
Csr csr_off(const mcr_matrix* h) {
    return Csr{h->rrp, h->rcol, h->rval, h->rdesc, h->ntiles, (int)h->n};
}

// Own-row views (x, p, s point at this rank's slice of the full vectors).
Vecs base_vecs(const mcr_matrix* h) {
    Vecs V{};
    V.b = h->vec(V_B);
    V.d = h->d;
    V.x = h->vec(V_X) + h->roff;
    V.r = h->vec(V_R);
    V.q = h->vec(V_Q);
    V.p = h->vec(V_P) + h->roff;
    V.v = h->vec(V_V);
    V.s = h->vec(V_S) + h->roff;
    V.t = h->vec(V_T);
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

// Off-diagonal copy R: row lengths from k_diag, exclusive scan (CUB), order-preserving split.
int build_sell(mcr_matrix* h, bool offdiag, mcr_matrix::SellDev* S) {
    const int n = (int)h->n;
    S->nwin = (n + SELL_W - 1) / SELL_W;
    const int nslices = S->nwin * SELL_SLICES;
    TRY(dalloc(h, &S->perm, (size_t)S->nwin * SELL_W));
    TRY(dalloc(h, &S->swidth, (size_t)nslices + 1));
    TRY(dalloc(h, &S->sptr, (size_t)nslices + 1));
    CK(cudaMemsetAsync(S->swidth + nslices, 0, sizeof(long long), h->stream));
    k_sell_rank<<<S->nwin, SELL_W, 0, h->stream>>>(h->rp, h->offlen, n, offdiag ? 1 : 0, S->perm,
                                                   S->swidth);
    CK(cudaGetLastError());
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, S->swidth, S->sptr, nslices + 1, h->stream));
    void* dtmp = nullptr;
    CK(cudaMallocAsync(&dtmp, tmp, h->stream));
    CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, S->swidth, S->sptr, nslices + 1, h->stream));
    CK(cudaFreeAsync(dtmp, h->stream));
    CK(cudaMemcpyAsync(&S->slots, S->sptr + nslices, sizeof(long long), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    TRY(dalloc(h, &S->col, (size_t)S->slots));
    TRY(dalloc(h, &S->val, (size_t)S->slots));
    const int rows = S->nwin * SELL_W;
    k_sell_fill<<<(rows + 255) / 256, 256, 0, h->stream>>>(h->rp, h->col, h->val, S->sptr, S->perm,
                                                           rows, offdiag ? 1 : 0, S->col, S->val);
    CK(cudaGetLastError());
    return MCR_OK;
}

int ensure_offdiag(mcr_matrix* h) {
    if (h->r_ready || h->storage != MCR_STORAGE_CSR) return MCR_OK;
    if (h->use_sell) {
        TRY(build_sell(h, true, &h->rsell));
        h->r_ready = true;
        return MCR_OK;
    }
    const int n = (int)h->n;
    TRY(dalloc(h, &h->rrp, (size_t)n + 1 + CSR_PAD));
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, h->offlen, h->rrp, n + 1, h->stream));
    void* dtmp = nullptr;
    CK(cudaMallocAsync(&dtmp, tmp, h->stream));
    CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, h->offlen, h->rrp, n + 1, h->stream));
    CK(cudaFreeAsync(dtmp, h->stream));
    long long roff = 0;
    CK(cudaMemcpyAsync(&roff, h->rrp + n, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    TRY(dalloc(h, &h->rcol, (size_t)roff + CSR_PAD));
    TRY(dalloc(h, &h->rval, (size_t)roff + CSR_PAD));
    const int threads = 256;
    const int blocks = (int)std::min<long long>(((long long)n * 32 + threads - 1) / threads, 1 << 20);
    if (n > 0)
        k_split_offdiag<<<blocks, threads, 0, h->stream>>>(h->rp, h->col, h->val, n, h->roff,
                                                           h->rrp, h->rcol, h->rval);
    CK(cudaGetLastError());
    TRY(dalloc(h, &h->rdesc, (size_t)h->ntiles));
    if (h->ntiles > 0)
        k_tile_desc<<<(h->ntiles + 255) / 256, 256, 0, h->stream>>>(h->rrp, h->tile_row, h->ntiles,
                                                                     h->rdesc);
    CK(cudaGetLastError());
    h->r_ready = true;
    return MCR_OK;
}

// Greedy tiles: consecutive rows while rows <= TILE_ROWS and entries <= TILE_NNZ; a row with
// more than TILE_NNZ entries is a tile of its own.
std::vector<int> make_tiles(int64_t n, const int64_t* rs, long long* max_row) {
    std::vector<int> t;
    t.reserve((size_t)(n / 64 + 2));
    t.push_back(0);
    long long mr = 0;
    int64_t r = 0;
    while (r < n) {
        const int64_t start = r;
        int64_t nnz = 0;
        while (r < n && r - start < TILE_ROWS) {
            const int64_t len = rs[r + 1] - rs[r];
            mr = std::max<long long>(mr, len);
            if (nnz + len > TILE_NNZ && r > start) break;
            nnz += len;
            ++r;
            if (nnz > TILE_NNZ) break;
        }
        t.push_back((int)r);
    }
    *max_row = mr;
    return t;
}

void set_state(mcr_matrix* h, double tol, int64_t max_it) {
    SolveState& s = *h->h_st;
    std::memset(&s, 0, sizeof(s));
    s.tol = tol;
    s.max_it = max_it;
    s.y = s.a = s.w = 1.0;
    s.seqdots = h->seqdots;
    s.sharded = h->sharded() ? 1 : 0;
}

int read_state(mcr_matrix* h) {
    CK(cudaMemcpyAsync(h->h_st, h->st, sizeof(SolveState), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return MCR_OK;
}

// ---------------------------------------------------------------- kernel launchers
// Every solve kernel goes out with programmatic stream serialization (PDL): the next kernel
// of the chain is scheduled while the current one drains, and waits in griddepcontrol.wait.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem,
                cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <int EPI>
void launch_mv(mcr_matrix* h, bool offdiag, const double* x, const Vecs& V, int64_t* launches) {
    if (h->storage == MCR_STORAGE_DENSE) {
        launch_pdl(k_dense<EPI>, h->nslabs, 32, DENSE_SMEM, h->stream, (const double*)h->dense,
                   (int)h->n, (int)((h->n + 1) & ~1ll), x, V, h->st);
    } else if (h->use_sell) {
        const auto& S = offdiag ? h->rsell : h->sell;
        launch_pdl(k_sell<EPI>, S.nwin * (SELL_W / SELL_CTA), SELL_CTA, 0, h->stream,
                   Sell{S.sptr, S.perm, S.col, S.val, S.nwin}, x, V, h->st);
    } else {
        launch_pdl(k_spmv<EPI>, h->spmv_grid, SP_THREADS, SP_SMEM, h->stream,
                   offdiag ? csr_off(h) : csr_full(h), x, V, h->st);
    }
    ++*launches;
}

template <int PH>
void launch_phase(mcr_matrix* h, const Vecs& V, int64_t* launches) {
    launch_pdl(k_phase<PH>, h->nchunks(), CHUNK_NT, 0, h->stream, V, (int)h->n, h->st);
    ++*launches;
}

template <int W>
void launch_seqdot(mcr_matrix* h, const Vecs& V, int64_t* launches) {
    if (!h->seqdots) return;
    launch_pdl(k_seqdot<W>, 1, SEQ_NT, 0, h->stream, V, (int)h->n, h->st);
    ++*launches;
}

// ---------------------------------------------------------------- sharded exchange points
// One reduction point of a row-sharded solve: every rank's SEND_SLOTS partials (written by
// the producing kernel's last CTA into st->send) are exchanged, then k_finalize<W> reduces them
// in rank order and takes the scalar step. `buf` != null also allgathers that full vector in
// the same step (Jacobi: the iterate just written).
template <int W>
int exchange_point(mcr_matrix* h, double* buf, int64_t* launches) {
    Transport& T = *h->comm;
    const double* send = h->st->send;
    const int rc = buf ? T.allgather_and_slots(buf, (size_t)h->chunk, send, h->recv, SEND_SLOTS,
                                               h->stream)
                       : T.gather_slots(send, h->recv, SEND_SLOTS, h->stream);
    if (rc) return fail(MCR_CUDA_ERROR, std::string(T.kind()) + " exchange: " + T.err);
    launch_pdl(k_finalize<W>, 1, 32, 0, h->stream, h->st, (const double*)h->recv, h->world);
    ++*launches;
    CK(cudaGetLastError());
    return MCR_OK;
}

int allgather_full(mcr_matrix* h, double* buf) {
    Transport& T = *h->comm;
    if (T.allgather(buf, (size_t)h->chunk, h->stream))
        return fail(MCR_CUDA_ERROR, std::string(T.kind()) + " allgather: " + T.err);
    return MCR_OK;
}

// Peer-to-peer mode: the producers already stored their rows into every peer's copy; a slot
// exchange orders those stores before any rank's next gather (every rank's producer kernel
// has retired -- with a system-scope fence -- before it enters the exchange).
int p2p_barrier(mcr_matrix* h) {
    Transport& T = *h->comm;
    if (T.gather_slots(h->st->send, h->recv, SEND_SLOTS, h->stream))
        return fail(MCR_CUDA_ERROR, std::string(T.kind()) + " barrier: " + T.err);
    return MCR_OK;
}

// max|b - M x| into st->resid; x is the full (gathered) vector.
int residual_into_state(mcr_matrix* h, const double* x, int64_t* launches) {
    Vecs V = base_vecs(h);
    launch_mv<EPI_RESID>(h, false, x, V, launches);
    CK(cudaGetLastError());
    if (h->sharded()) TRY(exchange_point<FIN_RESID>(h, nullptr, launches));
    return MCR_OK;
}

// b -> V_B; x0 (this handle's rows) -> own slice of the full vector `x0_slot`, gathered when
// sharded; no x0 means zeros.
int prepare_inputs(mcr_matrix* h, const double* d_b, const double* d_x0, int x0_slot) {
    const size_t bytes = sizeof(double) * (size_t)h->n;
    CK(cudaMemcpyAsync(h->vec(V_B), d_b, bytes, cudaMemcpyDeviceToDevice, h->stream));
    double* full = h->vec(x0_slot);
    if (d_x0) {
        CK(cudaMemcpyAsync(full + h->roff, d_x0, bytes, cudaMemcpyDeviceToDevice, h->stream));
        if (h->sharded()) TRY(allgather_full(h, full));
    } else {
        CK(cudaMemsetAsync(full, 0, sizeof(double) * (size_t)h->n_full(), h->stream));
    }
    return MCR_OK;
}

// ZeroDiagonal must be decided identically on every rank before any sweep (a rank that
// returned early would leave its peers waiting in a collective): exchange each rank's first
// zero-diagonal row and take the smallest.
int global_first_zero(mcr_matrix* h, long long* out) {
    if (!h->sharded()) {
        *out = h->first_zero;
        return MCR_OK;
    }
    double mine[SEND_SLOTS] = {(double)h->first_zero, 0.0, 0.0, 0.0};
    CK(cudaMemcpyAsync(h->st->send, mine, sizeof(mine), cudaMemcpyHostToDevice, h->stream));
    Transport& T = *h->comm;
    if (T.gather_slots(h->st->send, h->recv, SEND_SLOTS, h->stream))
        return fail(MCR_CUDA_ERROR, std::string(T.kind()) + " exchange: " + T.err);
    std::vector<double> all((size_t)h->world * SEND_SLOTS);
    CK(cudaMemcpyAsync(all.data(), h->recv, sizeof(double) * all.size(), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    long long best = -1;
    for (int r = 0; r < h->world; ++r) {
        const long long z = (long long)all[(size_t)r * SEND_SLOTS];
        if (z >= 0 && (best < 0 || z < best)) best = z;
    }
    *out = best;
    return MCR_OK;
}

// Batches grow 4, 8, ..., 32: a batch that overshoots the stop point only launches kernels
// that return at their first instruction (and, sharded, exchanges that rewrite unchanged data).
int next_batch(int cur) { return std::min(cur * 2, 32); }

int jacobi_impl(mcr_matrix* h, const double* d_b, const double* d_x0, double tol, int64_t max_it,
                double* d_x_out, mcr_report* rep) {
    TRY(ensure_work(h));
    long long zero = -1;
    TRY(global_first_zero(h, &zero));
    if (zero >= 0) {
        rep->zero_diagonal_index = zero;
        return fail(MCR_ZERO_DIAGONAL, "zero diagonal entry in row " + std::to_string(zero));
    }
    TRY(ensure_offdiag(h));
    TRY(prepare_inputs(h, d_b, d_x0, V_X));
    set_state(h, tol, max_it);
    CK(cudaMemcpyAsync(h->st, h->h_st, sizeof(SolveState), cudaMemcpyHostToDevice, h->stream));
    Vecs V = base_vecs(h);
    CK(cudaEventRecord(h->ev0, h->stream));
    int64_t launched = 0, sweeps = 0;
    int batch = 4;
    if (h->small_grid > 0) {
        CK(cudaMemsetAsync(h->maxslot, 0, 3 * sizeof(unsigned long long), h->stream));
        Csr R = csr_off(h);
        void* args[] = {&R, &V, &h->st, &h->maxslot};
        CK(cudaLaunchCooperativeKernel((void*)k_jacobi_small, h->small_grid, SM_NT, args, 0, h->stream));
        ++launched;
        TRY(read_state(h));
    } else for (;;) {
        const int k = (int)std::min<int64_t>(batch, max_it - sweeps);
        for (int i = 0; i < k; ++i) {
            launch_mv<EPI_JACOBI>(h, true, nullptr, V, &launched);
            if (h->sharded()) {  // sweep s writes buffer s & 1: gather it with the partial max
                const int64_t sweep = sweeps + i + 1;
                double* wrote = (sweep & 1) ? h->vec(V_X1) : h->vec(V_X);
                TRY(exchange_point<FIN_JACOBI>(h, h->p2p ? nullptr : wrote, &launched));
            }
        }
        CK(cudaGetLastError());
        sweeps += k;
        TRY(read_state(h));
        if (h->h_st->stop || sweeps >= max_it) break;
        batch = next_batch(batch);
    }
    const long long it = h->h_st->it;
    const double* x = (it & 1) ? h->vec(V_X1) : h->vec(V_X);  // full iterate (gathered)
    TRY(residual_into_state(h, x, &launched));
    CK(cudaEventRecord(h->ev1, h->stream));
    TRY(read_state(h));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (d_x_out)
        CK(cudaMemcpyAsync(d_x_out, x + h->roff, sizeof(double) * (size_t)h->n,
                           cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const SolveState& s = *h->h_st;
    rep->iterations = s.it;
    rep->converged = s.stop == CONVERGED;
    rep->residual_inf = s.resid;
    rep->device_seconds = ms * 1e-3;
    rep->kernel_launches = launched;
    return s.stop == CONVERGED ? MCR_OK : MCR_NOT_CONVERGED;
}

int bicgstab_impl(mcr_matrix* h, const double* d_b, const double* d_x0, double tol,
                  int64_t max_it, double* d_x_out, mcr_report* rep) {
    TRY(ensure_work(h));
    TRY(prepare_inputs(h, d_b, d_x0, V_X));
    set_state(h, tol, max_it);
    CK(cudaMemcpyAsync(h->st, h->h_st, sizeof(SolveState), cudaMemcpyHostToDevice, h->stream));
    Vecs V = base_vecs(h);
    const bool sh = h->sharded();
    CK(cudaEventRecord(h->ev0, h->stream));
    int64_t launched = 0, iters = 0;
    int batch = 4;
    if (h->small_grid > 0 && !h->seqdots) {
        CK(cudaMemsetAsync(h->maxslot, 0, 3 * sizeof(unsigned long long), h->stream));
        Csr A = csr_full(h);
        double* parts = h->P;
        int pstride = h->nunits;  // four partial slots of nunits >= ntiles doubles each
        void* args[] = {&A, &V, &h->st, &h->maxslot, &parts, &pstride};
        CK(cudaLaunchCooperativeKernel((void*)k_bicg_small, h->small_grid, SM_NT, args, 0, h->stream));
        ++launched;
        TRY(read_state(h));
        iters = max_it;  // the loop below has nothing left to do
    } else {
        // r = b - 1.0 * M x0, q = r, p = v = 0
        launch_mv<EPI_S0>(h, false, h->vec(V_X), V, &launched);
        launch_seqdot<SQ_S0>(h, V, &launched);
        CK(cudaGetLastError());
        if (sh) TRY(exchange_point<FIN_S0>(h, nullptr, &launched));
        TRY(read_state(h));
    }
    double* p_full = h->vec(V_P);
    double* s_full = h->vec(V_S);
    while (!h->h_st->stop && iters < max_it) {
        const int k = (int)std::min<int64_t>(batch, max_it - iters);
        for (int i = 0; i < k; ++i) {
            launch_phase<PH_A>(h, V, &launched);               // p = r + beta (p - w v)
            if (sh) TRY(h->p2p ? p2p_barrier(h) : allgather_full(h, p_full));
            launch_mv<EPI_V>(h, false, p_full, V, &launched);  // v = M p, q.v -> a
            launch_seqdot<SQ_V>(h, V, &launched);
            if (sh) TRY(exchange_point<FIN_V>(h, nullptr, &launched));
            launch_phase<PH_C>(h, V, &launched);               // s = r - a v, max|s|
            if (sh) TRY(h->p2p ? p2p_barrier(h) : allgather_full(h, s_full));
            launch_mv<EPI_T>(h, false, s_full, V, &launched);  // t = M s, t.t, t.s -> w
            launch_seqdot<SQ_T>(h, V, &launched);
            if (sh) TRY(exchange_point<FIN_T>(h, nullptr, &launched));
            launch_phase<PH_E>(h, V, &launched);               // x, r updates, q.r -> beta
            launch_seqdot<SQ_E>(h, V, &launched);
            if (sh) TRY(exchange_point<FIN_E>(h, nullptr, &launched));
        }
        CK(cudaGetLastError());
        iters += k;
        TRY(read_state(h));
        batch = next_batch(batch);
    }
    if (sh) TRY(allgather_full(h, h->vec(V_X)));  // this rank's x is its slice of V_X
    TRY(residual_into_state(h, h->vec(V_X), &launched));
    CK(cudaEventRecord(h->ev1, h->stream));
    TRY(read_state(h));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (d_x_out)
        CK(cudaMemcpyAsync(d_x_out, V.x, sizeof(double) * (size_t)h->n, cudaMemcpyDeviceToDevice,
                           h->stream));
    CK(cudaStreamSynchronize(h->stream));
    const SolveState& s = *h->h_st;
    rep->residual_inf = s.resid;
    rep->device_seconds = ms * 1e-3;
    rep->kernel_launches = launched;
    rep->converged = s.stop == CONVERGED;
    if (s.stop == BREAKDOWN) {
        rep->iterations = s.bd_it;
        rep->breakdown_which = s.which;
        rep->breakdown_iteration = s.bd_it;
        const char* names[] = {"", "y_prev*w", "q*v", "t*t"};
        return fail(MCR_BREAKDOWN, std::string("breakdown: ") + names[s.which & 3] +
                                       " vanished at iteration " + std::to_string(s.bd_it));
    }
    rep->iterations = s.it;
    return s.stop == CONVERGED ? MCR_OK : MCR_NOT_CONVERGED;
}

void report_init(mcr_report* rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->zero_diagonal_index = -1;
}

// Host-pointer front end: stage b / x0 in the handle's workspace, run, copy x back.
template <class Impl>
int host_solve(mcr_matrix* h, const double* b, const double* x0, double tol, int64_t max_it,
               double* x_out, mcr_report* rep, Impl impl) {
    const size_t bytes = sizeof(double) * (size_t)h->n;
    TRY(ensure_work(h));
    double* db = h->vec(V_R);   // scratch slots: overwritten by the solve only after the copy
    double* dx = h->vec(V_Q);
    CK(cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, h->stream));
    if (x0) CK(cudaMemcpyAsync(dx, x0, bytes, cudaMemcpyHostToDevice, h->stream));
    double* dout = h->vec(V_V);
    int rc = impl(h, db, x0 ? dx : nullptr, tol, max_it, dout, rep);
    if (rc == MCR_OK || rc == MCR_NOT_CONVERGED || rc == MCR_BREAKDOWN) {
        const double* src = dout;
        if (rc == MCR_BREAKDOWN) src = h->vec(V_X) + h->roff;  // snapshot: x before that iteration
        CK(cudaMemcpyAsync(x_out, src, bytes, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    return rc;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

MCR_API int mcr_version(void) { return 100; }

MCR_API const char* mcr_last_error(void) { return g_err.c_str(); }

MCR_API int mcr_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        c = 0;
    }
    if (count) *count = c;
    return MCR_OK;
}

MCR_API void mcr_matrix_destroy(mcr_matrix* h) {
    if (!h) return;
    {
        DeviceGuard g(h->device);
        cudaStream_t s = h->own_stream;
        if (h->stream && h->stream != s) cudaStreamSynchronize(h->stream);
        if (s) {
            void* ptrs[] = {h->rp, h->col, h->val, h->tile_row, h->desc, h->rdesc, h->offlen,
                            h->rrp, h->rcol, h->rval, h->dense, h->d, h->work, h->P, h->st,
                            h->sell.sptr, h->sell.perm, h->sell.col, h->sell.val, h->sell.swidth,
                            h->rsell.sptr, h->rsell.perm, h->rsell.col, h->rsell.val,
                            h->rsell.swidth, h->maxslot, h->recv};
            for (void* p : ptrs)
                if (p) cudaFreeAsync(p, s);
            cudaStreamSynchronize(s);
        }
        for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
        if (h->fullblk) cudaFree(h->fullblk);
        if (h->d_peers) cudaFree(h->d_peers);
        if (h->ev0) cudaEventDestroy(h->ev0);
        if (h->ev1) cudaEventDestroy(h->ev1);
        if (s) cudaStreamDestroy(s);
    }
    delete h;
}

static int set_kernel_attributes() {
    const int sp = (int)SP_SMEM;
    CK(cudaFuncSetAttribute(k_spmv<EPI_Y>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_JACOBI>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_S0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_V>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    return MCR_OK;
}

// Rows [h->roff, h->roff + n) of an h->n_global system (the whole system on one GPU);
// column indices are global.
static int finish_create(mcr_matrix* h, int64_t n, const int64_t* rs, int storage,
                         std::vector<int>* pre_tiles = nullptr);

static int init_handle(mcr_matrix* h) {
    TRY(keep_pool_memory(h->device));
    CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    h->stream = h->own_stream;
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    TRY(dalloc(h, &h->st, 1));
    CK(cudaMemsetAsync(h->st, 0, sizeof(SolveState), h->stream));
    return MCR_OK;
}

static int alloc_csr(mcr_matrix* h, int64_t n, int64_t nnz) {
    h->nnz = nnz;
    if (!h->rp) TRY(dalloc(h, &h->rp, (size_t)n + 1 + CSR_PAD));
    TRY(dalloc(h, &h->col, (size_t)nnz + CSR_PAD));
    TRY(dalloc(h, &h->val, (size_t)nnz + CSR_PAD));
    TRY(dalloc(h, &h->d, (size_t)n));
    TRY(dalloc(h, &h->offlen, (size_t)n + 1));
    return MCR_OK;
}

static int create_impl(mcr_matrix* h, int64_t n, const int64_t* rs, const int64_t* col,
                       const double* val, int storage) {
    TRY(init_handle(h));
    if (n == 0) return MCR_OK;
    const int64_t nnz = rs[n];
    TRY(alloc_csr(h, n, nnz));
    CK(cudaMemcpyAsync(h->rp, rs, sizeof(long long) * (size_t)(n + 1), cudaMemcpyHostToDevice,
                       h->stream));
    CK(cudaMemcpyAsync(h->val, val, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice,
                       h->stream));
    // int64 columns -> int32 on the device, range-checked
    {
        long long* tmp = nullptr;
        int* bad = nullptr;
        CK(cudaMallocAsync((void**)&tmp, sizeof(long long) * (size_t)std::max<int64_t>(nnz, 1),
                           h->stream));
        CK(cudaMallocAsync((void**)&bad, 2 * sizeof(int), h->stream));
        CK(cudaMemsetAsync(bad, 0, 2 * sizeof(int), h->stream));
        CK(cudaMemcpyAsync(tmp, col, sizeof(long long) * (size_t)nnz, cudaMemcpyHostToDevice,
                           h->stream));
        if (nnz > 0) {
            k_col64to32<<<(int)std::min<int64_t>((nnz + 255) / 256, 1 << 16), 256, 0, h->stream>>>(
                tmp, h->col, nnz, (int)h->n_global, bad);
            k_check_rows<<<(int)std::min<int64_t>((n + 255) / 256, 1 << 16), 256, 0, h->stream>>>(
                h->rp, h->col, (int)n, bad + 1);
        }
        CK(cudaGetLastError());
        int hbad[2] = {0, 0};
        CK(cudaMemcpyAsync(hbad, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaFreeAsync(tmp, h->stream));
        CK(cudaFreeAsync(bad, h->stream));
        // the row tiles are cut on the host while the copies are in flight
        std::vector<int> tiles = make_tiles(n, rs, &h->max_row);
        CK(cudaStreamSynchronize(h->stream));
        if (hbad[0]) return fail(MCR_DIMENSION, "column index out of range");
        if (hbad[1]) return fail(MCR_DIMENSION, "rows must be sorted by column without duplicates");
        return finish_create(h, n, rs, storage, &tiles);
    }
}

// A handle from a CSR already on the device (int64 row starts, int32 columns), copied.
static int create_from_device(int64_t n, int64_t nnz, const long long* d_rp, const int* d_col,
                              const double* d_val, int device, int storage, mcr_matrix** out) {
    DeviceGuard g(device);
    mcr_matrix* h = new mcr_matrix();
    h->device = device;
    h->n = n;
    h->n_global = n;
    h->chunk = n;
    int rc = [&]() -> int {
        TRY(init_handle(h));
        if (n == 0) return MCR_OK;
        TRY(alloc_csr(h, n, nnz));
        CK(cudaMemcpyAsync(h->rp, d_rp, sizeof(long long) * (size_t)(n + 1), cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemcpyAsync(h->col, d_col, sizeof(int) * (size_t)nnz, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemcpyAsync(h->val, d_val, sizeof(double) * (size_t)nnz, cudaMemcpyDeviceToDevice, h->stream));
        std::vector<int64_t> rs((size_t)n + 1);
        CK(cudaMemcpyAsync(rs.data(), d_rp, sizeof(int64_t) * rs.size(), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        return finish_create(h, n, rs.data(), storage);
    }();
    if (rc != MCR_OK) {
        std::string msg = g_err;
        mcr_matrix_destroy(h);
        g_err = msg;
        return rc;
    }
    *out = h;
    return MCR_OK;
}

// Poisson(mean) inverse-CDF thresholds on 2^64 (generator.cuh); restated in oracle.c.
static void poisson_thresholds(double mean, uint64_t* thr) {
    double p = std::exp(-mean), cdf = 0.0;
    for (int k = 0; k < GEN_KMAX; ++k) {
        cdf += p;
        const double t = cdf * 18446744073709551616.0;
        thr[k] = t >= 18446744073709551616.0 ? UINT64_MAX : (uint64_t)t;
        p = (p * mean) / (double)(k + 1);
    }
}

// Rows [h->roff, h->roff + h->n) of the row-keyed synthetic system, built on the device.
static int generate_impl(mcr_matrix* h, const GenParams& P, int storage) {
    TRY(init_handle(h));
    const int64_t n = h->n;
    if (n == 0) return MCR_OK;
    TRY(dalloc(h, &h->rp, (size_t)n + 1 + CSR_PAD));
    long long* len = nullptr;
    CK(cudaMallocAsync((void**)&len, sizeof(long long) * (size_t)(n + 1), h->stream));
    CK(cudaMemsetAsync(len + n, 0, sizeof(long long), h->stream));
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 1 << 16);
    k_gen_count<<<grid, 256, 0, h->stream>>>(P, (long long)n, len);
    CK(cudaGetLastError());
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, len, h->rp, n + 1, h->stream));
    void* dtmp = nullptr;
    CK(cudaMallocAsync(&dtmp, tmp, h->stream));
    CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, len, h->rp, n + 1, h->stream));
    CK(cudaFreeAsync(dtmp, h->stream));
    CK(cudaFreeAsync(len, h->stream));
    std::vector<int64_t> rs((size_t)n + 1);
    CK(cudaMemcpyAsync(rs.data(), h->rp, sizeof(int64_t) * rs.size(), cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    TRY(alloc_csr(h, n, rs[(size_t)n]));
    k_gen_fill<<<(int)std::min<int64_t>((n + 127) / 128, 1 << 20), 128, 0, h->stream>>>(
        P, (long long)n, h->rp, h->col, h->val);
    CK(cudaGetLastError());
    return finish_create(h, n, rs.data(), storage);
}

// Device CSR (rp/col/val) in place; `rs` = host copy of the row starts. Diagonal, tiles or
// dense slabs, kernel attributes.
static int finish_create(mcr_matrix* h, int64_t n, const int64_t* rs, int storage,
                         std::vector<int>* pre_tiles) {
    const int64_t nnz = h->nnz;
    const bool dense = !h->sharded() &&
                       (storage == MCR_STORAGE_DENSE ||
                        (storage == MCR_STORAGE_AUTO && n >= 1024 &&
                         (double)nnz * 3.0 >= 2.0 * (double)n * (double)n));
    h->storage = dense ? MCR_STORAGE_DENSE : MCR_STORAGE_CSR;
    // diagonal, first zero-diagonal row, off-diagonal row lengths
    {
        unsigned long long* fz = nullptr;
        CK(cudaMallocAsync((void**)&fz, sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(fz, 0xff, sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(h->offlen + n, 0, sizeof(long long), h->stream));
        k_diag<<<(int)std::min<int64_t>((n + 255) / 256, 1 << 16), 256, 0, h->stream>>>(
            h->rp, h->col, h->val, (int)n, (long long)h->roff, h->d, h->offlen, fz);
        CK(cudaGetLastError());
        unsigned long long hfz = 0;
        CK(cudaMemcpyAsync(&hfz, fz, sizeof(hfz), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaFreeAsync(fz, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        h->first_zero = hfz == ~0ull ? -1 : (long long)hfz + h->roff;  // global row
    }
    std::vector<int> tiles;
    if (pre_tiles) tiles.swap(*pre_tiles);
    else tiles = make_tiles(n, rs, &h->max_row);
    if (dense) {
        h->nslabs = (int)((n + DSLAB - 1) / DSLAB);
        const int64_t npad = (n + 1) & ~1ll;  // column pairs
        const size_t cnt = (size_t)h->nslabs * DSLAB * (size_t)npad;
        TRY(dalloc(h, &h->dense, cnt));
        CK(cudaMemsetAsync(h->dense, 0, sizeof(double) * cnt, h->stream));
        k_dense_build<<<(int)n, 256, 0, h->stream>>>(h->rp, h->col, h->val, (int)n, (int)npad,
                                                     h->dense);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
        dfree(h, h->col, (size_t)nnz + CSR_PAD);
        dfree(h, h->val, (size_t)nnz + CSR_PAD);
        dfree(h, h->offlen, (size_t)n + 1);
        CK(cudaFuncSetAttribute(k_dense<EPI_Y>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM));
        CK(cudaFuncSetAttribute(k_dense<EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM));
        CK(cudaFuncSetAttribute(k_dense<EPI_JACOBI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM));
        CK(cudaFuncSetAttribute(k_dense<EPI_S0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM));
        CK(cudaFuncSetAttribute(k_dense<EPI_V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM));
        CK(cudaFuncSetAttribute(k_dense<EPI_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DENSE_SMEM));
    } else {
        h->ntiles = (int)tiles.size() - 1;
        // SELL streams rows without shared-memory staging, but its epilogue operands are
        // gathered through the row permutation; measured on C2 (profiles/) the TMA-staged
        // tiles win (54 vs 70 us per Jacobi sweep), so SELL is opt-in.
        h->use_sell = storage == MCR_STORAGE_SELL && !h->sharded();
        if (h->use_sell) TRY(build_sell(h, false, &h->sell));
        TRY(set_kernel_attributes());
        int sms = 0, per_sm = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv<EPI_V>, SP_THREADS, SP_SMEM));
        h->spmv_grid = std::max(1, std::min(h->ntiles, sms * std::max(per_sm, 1)));
        int pj = 0, pb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pj, k_jacobi_small, SM_NT, 0));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pb, k_bicg_small, SM_NT, 0));
        const int coresident = sms * std::min(pj, pb);
        // one tile per CTA keeps the per-sweep critical path to a single tile
        if (!h->use_sell && !h->sharded() && storage != MCR_STORAGE_TILES_STREAM &&
            h->ntiles <= coresident && h->ntiles <= 2 * sms)
            h->small_grid = h->ntiles;
        TRY(dalloc(h, &h->maxslot, 3));
        TRY(dalloc(h, &h->tile_row, tiles.size()));
        CK(cudaMemcpyAsync(h->tile_row, tiles.data(), sizeof(int) * tiles.size(),
                           cudaMemcpyHostToDevice, h->stream));
        std::vector<TileDesc> desc((size_t)h->ntiles);
        for (int t = 0; t < h->ntiles; ++t)
            desc[(size_t)t] = TileDesc{rs[tiles[(size_t)t]], rs[tiles[(size_t)t + 1]], tiles[(size_t)t],
                                       tiles[(size_t)t + 1]};
        TRY(dalloc(h, &h->desc, desc.size()));
        CK(cudaMemcpyAsync(h->desc, desc.data(), sizeof(TileDesc) * desc.size(),
                           cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    }
    return MCR_OK;
}

static int check_csr(int64_t n, const int64_t* rstart, const int64_t* col, const double* nonzero) {
    if (n < 0 || n >= INT_MAX) return fail(MCR_DIMENSION, "dimension out of range");
    if (n > 0 && (!rstart || (rstart[n] > 0 && (!col || !nonzero))))
        return fail(MCR_INVALID_ARGUMENT, "NULL CSR array");
    if (n > 0) {
        if (rstart[0] != 0) return fail(MCR_DIMENSION, "malformed rstart vector");
        for (int64_t i = 0; i < n; ++i)
            if (rstart[i + 1] < rstart[i]) return fail(MCR_DIMENSION, "rstart must be nondecreasing");
    }
    return MCR_OK;
}

static int create_handle(int64_t n, const int64_t* rstart, const int64_t* col,
                         const double* nonzero, int device, int storage,
                         const std::shared_ptr<Transport>& comm, int64_t n_global, int64_t roff,
                         int64_t chunk, mcr_matrix** out) {
    int ndev = 0;
    mcr_device_count(&ndev);
    if (device < 0 || device >= ndev)
        return fail(MCR_CUDA_ERROR, "no CUDA device " + std::to_string(device) + " (" +
                                        std::to_string(ndev) + " visible)");
    DeviceGuard g(device);
    mcr_matrix* h = new mcr_matrix();
    h->device = device;
    h->n = n;
    h->n_global = n_global;
    h->roff = roff;
    h->chunk = chunk;
    if (comm) {
        h->comm = comm;
        h->world = comm->world;
        h->rank = comm->rank;
    }
    int rc = create_impl(h, n, rstart, col, nonzero, storage);
    if (rc != MCR_OK) {
        std::string msg = g_err;
        mcr_matrix_destroy(h);
        g_err = msg;
        return rc;
    }
    *out = h;
    return MCR_OK;
}

MCR_API int mcr_matrix_create(int64_t n, const int64_t* rstart, const int64_t* col,
                              const double* nonzero, int device, int storage, mcr_matrix** out) {
    if (!out) return fail(MCR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    TRY(check_csr(n, rstart, col, nonzero));
    return create_handle(n, rstart, col, nonzero, device, storage, nullptr, n, 0, n, out);
}

// ---------------------------------------------------------------- row sharding
MCR_API int mcr_shard_rows(int64_t n_global, int world, int rank, int64_t* row0, int64_t* rows) {
    if (world < 1 || rank < 0 || rank >= world || n_global < 0 || !row0 || !rows)
        return fail(MCR_INVALID_ARGUMENT, "bad shard request");
    const int64_t chunk = (n_global + world - 1) / world;
    const int64_t lo = std::min<int64_t>(n_global, chunk * rank);
    const int64_t hi = std::min<int64_t>(n_global, lo + chunk);
    *row0 = lo;
    *rows = hi - lo;
    return MCR_OK;
}

MCR_API int mcr_comm_unique_id(void* id) {
    if (!id) return fail(MCR_INVALID_ARGUMENT, "NULL id");
    NcclApi* api = NcclApi::get();
    if (!api) return fail(MCR_CUDA_ERROR, NcclApi::error());
    ncclUniqueId u;
    ncclResult_t r = api->GetUniqueId(&u);
    if (r != ncclSuccess) return fail(MCR_CUDA_ERROR, std::string("ncclGetUniqueId: ") + api->GetErrorString(r));
    std::memcpy(id, &u, sizeof(u));
    return MCR_OK;
}

MCR_API int mcr_comm_create_nccl(const void* id, int world, int rank, int device, mcr_comm** out) {
    if (!id || !out) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(MCR_INVALID_ARGUMENT, "bad rank / world");
    NcclApi* api = NcclApi::get();
    if (!api) return fail(MCR_CUDA_ERROR, NcclApi::error());
    int ndev = 0;
    mcr_device_count(&ndev);
    if (device < 0 || device >= ndev) return fail(MCR_CUDA_ERROR, "no CUDA device " + std::to_string(device));
    DeviceGuard g(device);
    auto t = std::make_shared<NcclTransport>();
    t->api = api;
    t->world = world;
    t->rank = rank;
    t->device = device;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclResult_t r = api->CommInitRank(&t->comm, world, u, rank);
    if (r != ncclSuccess) {
        t->comm = nullptr;
        return fail(MCR_CUDA_ERROR, std::string("ncclCommInitRank: ") + api->GetErrorString(r));
    }
    *out = new mcr_comm{t};
    return MCR_OK;
}

MCR_API int mcr_comm_create_local(int world, const int* devices, mcr_comm** out) {
    if (!out || world < 1) return fail(MCR_INVALID_ARGUMENT, "bad local group request");
    int ndev = 0;
    mcr_device_count(&ndev);
    auto g = std::make_shared<LocalGroup>();
    g->world = world;
    g->src.assign((size_t)world, nullptr);
    g->dev.assign((size_t)world, 0);
    g->ready.assign((size_t)world, nullptr);
    g->done.assign((size_t)world, nullptr);
    for (int r = 0; r < world; ++r) {
        const int d = devices ? devices[r] : 0;
        if (d < 0 || d >= ndev) return fail(MCR_CUDA_ERROR, "no CUDA device " + std::to_string(d));
        g->dev[(size_t)r] = d;
        DeviceGuard guard(d);
        CK(cudaEventCreateWithFlags(&g->ready[(size_t)r], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&g->done[(size_t)r], cudaEventDisableTiming));
    }
    for (int r = 0; r < world; ++r) {
        auto t = std::make_shared<LocalTransport>();
        t->g = g;
        t->world = world;
        t->rank = r;
        t->device = g->dev[(size_t)r];
        out[r] = new mcr_comm{t};
    }
    return MCR_OK;
}

MCR_API void mcr_comm_destroy(mcr_comm* c) { delete c; }

MCR_API int mcr_comm_info(const mcr_comm* c, int* world, int* rank, int* device) {
    if (!c) return fail(MCR_INVALID_ARGUMENT, "NULL comm");
    if (world) *world = c->t->world;
    if (rank) *rank = c->t->rank;
    if (device) *device = c->t->device;
    return MCR_OK;
}

MCR_API int mcr_shard_create(mcr_comm* comm, int64_t n_global, int64_t row0, int64_t rows,
                             const int64_t* rstart, const int64_t* col, const double* nonzero,
                             mcr_matrix** out) {
    if (!comm || !out) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    *out = nullptr;
    if (n_global < 0 || n_global >= INT_MAX) return fail(MCR_DIMENSION, "dimension out of range");
    const Transport& T = *comm->t;
    int64_t want0 = 0, want = 0;
    TRY(mcr_shard_rows(n_global, T.world, T.rank, &want0, &want));
    if (row0 != want0 || rows != want)
        return fail(MCR_DIMENSION, "rank " + std::to_string(T.rank) + " of " + std::to_string(T.world) +
                                       " must hold rows [" + std::to_string(want0) + ", " +
                                       std::to_string(want0 + want) + ")");
    if (rows < 1) return fail(MCR_DIMENSION, "every rank needs at least one row (n >= world)");
    TRY(check_csr(rows, rstart, col, nonzero));
    const int64_t chunk = (n_global + T.world - 1) / T.world;
    return create_handle(rows, rstart, col, nonzero, T.device, MCR_STORAGE_TILES_STREAM, comm->t,
                         n_global, row0, chunk, out);
}

MCR_API int mcr_shard_enable_p2p(mcr_matrix* h) {
    if (!h) return fail(MCR_INVALID_ARGUMENT, "NULL handle");
    if (!h->sharded()) return fail(MCR_INVALID_ARGUMENT, "peer-to-peer mode needs a row shard");
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->p2p) return MCR_OK;
    DeviceGuard g(h->device);
    Transport& T = *h->comm;
    const size_t words = (size_t)V_FULL_COUNT * (size_t)h->n_full();
    CK(cudaMalloc((void**)&h->fullblk, sizeof(double) * words));
    CK(cudaMemset(h->fullblk, 0, sizeof(double) * words));
    std::vector<double*> base((size_t)h->world, nullptr);
    if (T.same_process()) {
        std::vector<uint64_t> all((size_t)h->world);
        const uint64_t mine = (uint64_t)(uintptr_t)h->fullblk;
        if (T.share_bytes(&mine, all.data(), sizeof(mine)))
            return fail(MCR_CUDA_ERROR, "p2p setup: " + T.err);
        for (int q = 0; q < h->world; ++q) {
            base[(size_t)q] = (double*)(uintptr_t)all[(size_t)q];
            int dq = T.device;
            if (auto* L = dynamic_cast<LocalTransport*>(&T)) dq = L->g->dev[(size_t)q];
            if (dq != h->device) {  // another GPU of this process: map it
                cudaError_t e = cudaDeviceEnablePeerAccess(dq, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return fail(MCR_CUDA_ERROR, std::string("peer access: ") + cudaGetErrorString(e));
                cudaGetLastError();
            }
        }
    } else {
        cudaIpcMemHandle_t mine;
        CK(cudaIpcGetMemHandle(&mine, h->fullblk));
        std::vector<cudaIpcMemHandle_t> all((size_t)h->world);
        if (T.share_bytes(&mine, all.data(), sizeof(mine)))
            return fail(MCR_CUDA_ERROR, "p2p setup: " + T.err);
        for (int q = 0; q < h->world; ++q) {
            if (q == h->rank) {
                base[(size_t)q] = h->fullblk;
                continue;
            }
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, all[(size_t)q], cudaIpcMemLazyEnablePeerAccess));
            h->ipc_opened.push_back(p);
            base[(size_t)q] = (double*)p;
        }
    }
    std::vector<double*> table((size_t)V_FULL_COUNT * (size_t)h->world);
    for (int slot = 0; slot < V_FULL_COUNT; ++slot)
        for (int q = 0; q < h->world; ++q)
            table[(size_t)slot * h->world + q] = base[(size_t)q] + (size_t)slot * (size_t)h->n_full();
    CK(cudaMalloc((void**)&h->d_peers, sizeof(double*) * table.size()));
    CK(cudaMemcpy(h->d_peers, table.data(), sizeof(double*) * table.size(), cudaMemcpyHostToDevice));
    h->p2p = 1;
    return MCR_OK;
}

MCR_API int mcr_generate(mcr_comm* comm, int device, int64_t n_global, double mean_offdiag,
                         int lo, int hi, uint64_t seed, int storage, mcr_matrix** out) {
    if (!out) return fail(MCR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (n_global < 2 || n_global >= INT_MAX) return fail(MCR_DIMENSION, "need 2 <= n < 2^31");
    if (!(mean_offdiag >= 0.0 && mean_offdiag <= 40.0) || lo > hi || hi < 1)
        return fail(MCR_INVALID_ARGUMENT, "need 0 <= mean_offdiag <= 40 and 1 <= hi, lo <= hi");
    int world = 1, rank = 0;
    if (comm) {
        world = comm->t->world;
        rank = comm->t->rank;
        device = comm->t->device;
    }
    int64_t row0 = 0, rows = n_global;
    TRY(mcr_shard_rows(n_global, world, rank, &row0, &rows));
    if (rows < 1) return fail(MCR_DIMENSION, "every rank needs at least one row (n >= world)");
    int ndev = 0;
    mcr_device_count(&ndev);
    if (device < 0 || device >= ndev) return fail(MCR_CUDA_ERROR, "no CUDA device " + std::to_string(device));
    DeviceGuard g(device);
    mcr_matrix* h = new mcr_matrix();
    h->device = device;
    h->n = rows;
    h->n_global = n_global;
    h->roff = row0;
    h->chunk = (n_global + world - 1) / world;
    if (comm) {
        h->comm = comm->t;
        h->world = world;
        h->rank = rank;
        storage = MCR_STORAGE_TILES_STREAM;
    }
    GenParams P{};
    P.seed = seed;
    P.n = n_global;
    P.row0 = row0;
    P.lo = lo;
    P.hi = hi;
    poisson_thresholds(mean_offdiag, P.thr);
    int rc = generate_impl(h, P, storage);
    if (rc != MCR_OK) {
        std::string msg = g_err;
        mcr_matrix_destroy(h);
        g_err = msg;
        return rc;
    }
    *out = h;
    return MCR_OK;
}

MCR_API int mcr_generate_rhs(const mcr_matrix* h, uint64_t seed, double* d_b) {
    if (!h || !d_b) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    if (h->n == 0) return MCR_OK;
    DeviceGuard g(h->device);
    k_gen_rhs<<<(int)std::min<int64_t>((h->n + 255) / 256, 1 << 16), 256, 0, h->stream>>>(
        seed, (long long)h->roff, (long long)h->n, d_b);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->stream));
    return MCR_OK;
}

MCR_API int mcr_matrix_export(mcr_matrix* h, int64_t* rstart, int64_t* col, double* nonzero) {
    if (!h) return fail(MCR_INVALID_ARGUMENT, "NULL handle");
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->n == 0) {
        if (rstart) rstart[0] = 0;
        return MCR_OK;
    }
    if (!h->col || !h->val) return fail(MCR_INVALID_ARGUMENT, "dense-storage handle keeps no CSR");
    DeviceGuard g(h->device);
    const size_t n = (size_t)h->n, nnz = (size_t)h->nnz;
    if (rstart)
        CK(cudaMemcpyAsync(rstart, h->rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, h->stream));
    if (nonzero)
        CK(cudaMemcpyAsync(nonzero, h->val, sizeof(double) * nnz, cudaMemcpyDeviceToHost, h->stream));
    if (col) {
        std::vector<int> c32(nnz);
        CK(cudaMemcpyAsync(c32.data(), h->col, sizeof(int) * nnz, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        for (size_t k = 0; k < nnz; ++k) col[k] = c32[k];
    }
    CK(cudaStreamSynchronize(h->stream));
    return MCR_OK;
}

// ---------------------------------------------------------------- chains (build_system)
}  // extern "C" (helpers below are C++)

template <class T>
static int calloc_owned(mcr_chain* c, T** p, size_t count) {
    *p = nullptr;
    CK(cudaMallocAsync((void**)p, sizeof(T) * std::max<size_t>(count, 1), c->stream));
    c->owned.push_back((void*)*p);
    return MCR_OK;
}

static int chain_scan(mcr_chain* c, const long long* in, long long* out, int64_t count) {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, count, c->stream));
    void* d = nullptr;
    CK(cudaMallocAsync(&d, std::max<size_t>(tmp, 1), c->stream));
    CK(cub::DeviceScan::ExclusiveSum(d, tmp, in, out, count, c->stream));
    CK(cudaFreeAsync(d, c->stream));
    return MCR_OK;
}

// Backward closure (k_closure) from states with flag == want, never entering blocked states.
static int chain_closure(mcr_chain* c, const unsigned long long* rev_rp, const int* rev_src,
                         const unsigned char* flag, unsigned char want,
                         const unsigned char* blocked, int* seen, int* fa, int* fb, unsigned* len) {
    const int n = (int)c->n;
    CK(cudaMemsetAsync(seen, 0, sizeof(int) * (size_t)n, c->stream));
    CK(cudaMemsetAsync(len, 0, sizeof(unsigned) * 3, c->stream));
    const int g = (int)std::min<int64_t>((n + 255) / 256, 4096);
    k_seed<<<g, 256, 0, c->stream>>>(flag, want, n, seen, fa, len);
    CK(cudaGetLastError());
    int sms = 0, per = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_closure, 256, 0));
    void* args[] = {(void*)&rev_rp, (void*)&rev_src, (void*)&blocked, (void*)&seen, (void*)&fa,
                    (void*)&fb, (void*)&len};
    CK(cudaLaunchCooperativeKernel((void*)k_closure, sms * std::max(1, per), 256, args, 0, c->stream));
    return MCR_OK;
}

static int chain_build(mcr_chain* c, const int64_t* rstart, const int64_t* col, const double* prob,
                       const int64_t* goals, int64_t ngoals) {
    const int64_t n = c->n, nnz = c->nnz;
    cudaStream_t s = c->stream;
    TRY(calloc_owned(c, &c->rp, (size_t)n + 1));
    TRY(calloc_owned(c, &c->col, (size_t)nnz));
    TRY(calloc_owned(c, &c->val, (size_t)nnz));
    TRY(calloc_owned(c, &c->goal, (size_t)n));
    TRY(calloc_owned(c, &c->cls, (size_t)n));
    TRY(calloc_owned(c, &c->remap, (size_t)n + 1));
    CK(cudaMemcpyAsync(c->rp, rstart, sizeof(long long) * (size_t)(n + 1), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(c->val, prob, sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice, s));
    {
        std::vector<int> c32((size_t)nnz);
        for (int64_t e = 0; e < nnz; ++e) {
            if (col[e] < 0 || col[e] >= n) return fail(MCR_DIMENSION, "transition target out of range");
            c32[(size_t)e] = (int)col[e];
        }
        std::vector<unsigned char> gm((size_t)n, 0);
        for (int64_t i = 0; i < ngoals; ++i) gm[(size_t)goals[i]] = 1;
        CK(cudaMemcpyAsync(c->col, c32.data(), sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(c->goal, gm.data(), (size_t)n, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    // reversed digraph
    unsigned long long *cnt = nullptr, *rev_rp = nullptr, *cursor = nullptr;
    int *rev_src = nullptr, *seen_goal = nullptr, *seen_zero = nullptr, *fa = nullptr, *fb = nullptr;
    unsigned* len = nullptr;
    unsigned char* zero_flag = nullptr;
    CK(cudaMallocAsync((void**)&cnt, sizeof(*cnt) * (size_t)(n + 1), s));
    CK(cudaMallocAsync((void**)&rev_rp, sizeof(*rev_rp) * (size_t)(n + 1), s));
    CK(cudaMallocAsync((void**)&cursor, sizeof(*cursor) * (size_t)n, s));
    CK(cudaMallocAsync((void**)&rev_src, sizeof(*rev_src) * (size_t)std::max<int64_t>(nnz, 1), s));
    CK(cudaMallocAsync((void**)&seen_goal, sizeof(int) * (size_t)n, s));
    CK(cudaMallocAsync((void**)&seen_zero, sizeof(int) * (size_t)n, s));
    CK(cudaMallocAsync((void**)&fa, sizeof(int) * (size_t)n, s));
    CK(cudaMallocAsync((void**)&fb, sizeof(int) * (size_t)n, s));
    CK(cudaMallocAsync((void**)&len, sizeof(unsigned) * 3, s));
    CK(cudaMallocAsync((void**)&zero_flag, (size_t)n, s));
    CK(cudaMemsetAsync(cnt, 0, sizeof(*cnt) * (size_t)(n + 1), s));
    CK(cudaMemsetAsync(cursor, 0, sizeof(*cursor) * (size_t)n, s));
    const int ge = (int)std::min<int64_t>((nnz + 255) / 256, 1 << 16);
    const int gn = (int)std::min<int64_t>((n + 255) / 256, 1 << 16);
    if (nnz) k_rev_count<<<ge, 256, 0, s>>>(c->rp, c->col, nnz, cnt);
    {
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, rev_rp, n + 1, s));
        void* d = nullptr;
        CK(cudaMallocAsync(&d, std::max<size_t>(tmp, 1), s));
        CK(cub::DeviceScan::ExclusiveSum(d, tmp, cnt, rev_rp, n + 1, s));
        CK(cudaFreeAsync(d, s));
    }
    k_rev_fill<<<gn, 256, 0, s>>>(c->rp, c->col, (int)n, rev_rp, cursor, rev_src);
    CK(cudaGetLastError());
    // states that reach a goal; the rest have probability zero
    TRY(chain_closure(c, rev_rp, rev_src, c->goal, 1, nullptr, seen_goal, fa, fb, len));
    // probability zero = no path to a goal; then the closure of that set avoiding the goals
    k_zero_flag<<<gn, 256, 0, s>>>(seen_goal, (int)n, zero_flag);
    CK(cudaGetLastError());
    TRY(chain_closure(c, rev_rp, rev_src, zero_flag, 1, c->goal, seen_zero, fa, fb, len));
    long long* unc = nullptr;
    CK(cudaMallocAsync((void**)&unc, sizeof(long long) * (size_t)(n + 1), s));
    k_classes<<<gn, 256, 0, s>>>(seen_goal, seen_zero, (int)n, c->cls, unc);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(unc + n, 0, sizeof(long long), s));
    TRY(chain_scan(c, unc, c->remap, n + 1));
    CK(cudaFreeAsync(unc, s));
    long long k = 0;
    CK(cudaMemcpyAsync(&k, c->remap + n, sizeof(k), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->k = k;
    TRY(calloc_owned(c, &c->list, (size_t)k));
    k_uncertain_list<<<gn, 256, 0, s>>>(c->cls, (int)n, c->remap, c->list);
    CK(cudaGetLastError());
    // M = I - A and the one-step goal probabilities
    long long *mlen = nullptr, *glen = nullptr, *goff = nullptr;
    double* gsel = nullptr;
    CK(cudaMallocAsync((void**)&mlen, sizeof(long long) * (size_t)(k + 1), s));
    CK(cudaMallocAsync((void**)&glen, sizeof(long long) * (size_t)(k + 1), s));
    CK(cudaMallocAsync((void**)&goff, sizeof(long long) * (size_t)(k + 1), s));
    TRY(calloc_owned(c, &c->mrp, (size_t)k + 1));
    TRY(calloc_owned(c, &c->rhs, (size_t)k));
    CK(cudaMemsetAsync(mlen + k, 0, sizeof(long long), s));
    CK(cudaMemsetAsync(glen + k, 0, sizeof(long long), s));
    const int gk = (int)std::min<int64_t>((k + 255) / 256, 1 << 16);
    if (k) k_m_count<<<gk, 256, 0, s>>>(c->rp, c->col, c->val, c->list, k, c->remap, c->goal, mlen, glen);
    TRY(chain_scan(c, mlen, c->mrp, k + 1));
    TRY(chain_scan(c, glen, goff, k + 1));
    long long mnnz = 0, gtot = 0;
    CK(cudaMemcpyAsync(&mnnz, c->mrp + k, sizeof(mnnz), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&gtot, goff + k, sizeof(gtot), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->m_nnz = mnnz;
    TRY(calloc_owned(c, &c->mcol, (size_t)mnnz));
    TRY(calloc_owned(c, &c->mval, (size_t)mnnz));
    CK(cudaMallocAsync((void**)&gsel, sizeof(double) * (size_t)std::max<long long>(gtot, 1), s));
    if (k) {
        k_m_fill<<<gk, 256, 0, s>>>(c->rp, c->col, c->val, c->list, k, c->remap, c->goal, c->mrp,
                                    c->mcol, c->mval, goff, gsel);
        k_rhs<<<gk, 256, 0, s>>>(goff, k, gsel, c->rhs);
    }
    CK(cudaGetLastError());
    for (void* p : {(void*)cnt, (void*)rev_rp, (void*)cursor, (void*)rev_src, (void*)seen_goal,
                    (void*)seen_zero, (void*)fa, (void*)fb, (void*)len, (void*)zero_flag,
                    (void*)mlen, (void*)glen, (void*)goff, (void*)gsel})
        CK(cudaFreeAsync(p, s));
    // class counts
    std::vector<signed char> cls((size_t)n);
    CK(cudaMemcpyAsync(cls.data(), c->cls, (size_t)n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->nzero = c->none = 0;
    for (signed char v : cls) {
        c->nzero += v == 0;
        c->none += v == 1;
    }
    return MCR_OK;
}

extern "C" {

MCR_API void mcr_chain_destroy(mcr_chain* c) {
    if (!c) return;
    {
        DeviceGuard g(c->device);
        if (c->M) mcr_matrix_destroy(c->M);
        for (void* p : c->owned) cudaFreeAsync(p, c->stream);
        if (c->stream) {
            cudaStreamSynchronize(c->stream);
            cudaStreamDestroy(c->stream);
        }
    }
    delete c;
}

MCR_API int mcr_chain_create(int64_t n, const int64_t* rstart, const int64_t* col,
                             const double* prob, const int64_t* goals, int64_t ngoals, int device,
                             mcr_chain** out) {
    if (!out) return fail(MCR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (n < 1 || n >= INT_MAX) return fail(MCR_DIMENSION, "a chain needs 1 <= n < 2^31 states");
    TRY(check_csr(n, rstart, col, prob));
    if (ngoals < 1 || !goals) return fail(MCR_INVALID_ARGUMENT, "goal set must not be empty");
    for (int64_t i = 0; i < ngoals; ++i)
        if (goals[i] < 0 || goals[i] >= n)
            return fail(MCR_DIMENSION, "goal state " + std::to_string(goals[i]) + " out of range");
    int ndev = 0;
    mcr_device_count(&ndev);
    if (device < 0 || device >= ndev) return fail(MCR_CUDA_ERROR, "no CUDA device " + std::to_string(device));
    DeviceGuard g(device);
    TRY(keep_pool_memory(device));
    mcr_chain* c = new mcr_chain();
    c->device = device;
    c->n = n;
    c->nnz = rstart[n];
    int rc = MCR_OK;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
        rc = fail(MCR_CUDA_ERROR, "cudaStreamCreate failed");
    if (rc == MCR_OK) rc = chain_build(c, rstart, col, prob, goals, ngoals);
    if (rc != MCR_OK) {
        std::string msg = g_err;
        mcr_chain_destroy(c);
        g_err = msg;
        return rc;
    }
    *out = c;
    return MCR_OK;
}

MCR_API int mcr_chain_info(const mcr_chain* c, int64_t* uncertain, int64_t* prob_one,
                           int64_t* prob_zero, int64_t* m_nnz) {
    if (!c) return fail(MCR_INVALID_ARGUMENT, "NULL chain");
    if (uncertain) *uncertain = c->k;
    if (prob_one) *prob_one = c->none;
    if (prob_zero) *prob_zero = c->nzero;
    if (m_nnz) *m_nnz = c->m_nnz;
    return MCR_OK;
}

MCR_API int mcr_chain_export(mcr_chain* c, int8_t* classes, int64_t* uncertain, int64_t* m_rstart,
                             int64_t* m_col, double* m_nonzero, double* rhs) {
    if (!c) return fail(MCR_INVALID_ARGUMENT, "NULL chain");
    std::lock_guard<std::mutex> lk(c->mu);
    DeviceGuard g(c->device);
    cudaStream_t s = c->stream;
    const size_t k = (size_t)c->k, m = (size_t)c->m_nnz;
    if (classes) CK(cudaMemcpyAsync(classes, c->cls, (size_t)c->n, cudaMemcpyDeviceToHost, s));
    if (uncertain && k) CK(cudaMemcpyAsync(uncertain, c->list, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
    if (m_rstart) CK(cudaMemcpyAsync(m_rstart, c->mrp, sizeof(int64_t) * (k + 1), cudaMemcpyDeviceToHost, s));
    if (m_nonzero && m) CK(cudaMemcpyAsync(m_nonzero, c->mval, sizeof(double) * m, cudaMemcpyDeviceToHost, s));
    if (rhs && k) CK(cudaMemcpyAsync(rhs, c->rhs, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    std::vector<int> c32(m_col ? m : 0);
    if (m_col && m) CK(cudaMemcpyAsync(c32.data(), c->mcol, sizeof(int) * m, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t e = 0; m_col && e < m; ++e) m_col[e] = c32[e];
    return MCR_OK;
}

MCR_API int mcr_chain_matrix(mcr_chain* c, mcr_matrix** out) {
    if (!c || !out) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    std::lock_guard<std::mutex> lk(c->mu);
    *out = nullptr;
    if (!c->M) {
        CK(cudaStreamSynchronize(c->stream));
        TRY(create_from_device(c->k, c->m_nnz, c->mrp, c->mcol, c->mval, c->device,
                               MCR_STORAGE_AUTO, &c->M));
    }
    *out = c->M;
    return MCR_OK;
}

MCR_API int mcr_chain_solve(mcr_chain* c, int method, int dots, double tol, int64_t max_it,
                            const double* x0, double* x_out, double* xs_out, mcr_report* rep) {
    if (!c || !rep) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    if (method != 0 && method != 1) return fail(MCR_INVALID_ARGUMENT, "method: 0 jacobi, 1 bicgstab");
    if (!(tol > 0.0)) return fail(MCR_INVALID_ARGUMENT, "tolerance must be positive");
    if (max_it < 1) return fail(MCR_INVALID_ARGUMENT, "max_iterations must be at least 1");
    report_init(rep);
    DeviceGuard g(c->device);
    if (c->k == 0) {  // no uncertain state: nothing to solve (markov.py:287-288)
        rep->converged = 1;
        if (x_out) {
            std::vector<signed char> cls((size_t)c->n);
            CK(cudaMemcpyAsync(cls.data(), c->cls, (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            for (int64_t s = 0; s < c->n; ++s) x_out[s] = cls[(size_t)s] == 1 ? 1.0 : 0.0;
        }
        return MCR_OK;
    }
    mcr_matrix* M = nullptr;
    TRY(mcr_chain_matrix(c, &M));
    TRY(mcr_set_dot_mode(M, dots ? MCR_DOTS_SEQUENTIAL : MCR_DOTS_TREE));
    std::lock_guard<std::mutex> lk(M->mu);
    {
        std::lock_guard<std::mutex> lc(c->mu);
        if (!c->xs) TRY(calloc_owned(c, &c->xs, (size_t)c->k));
        if (!c->xfull) TRY(calloc_owned(c, &c->xfull, (size_t)c->n));
        if (x0) CK(cudaMemcpyAsync(c->xfull, x0, sizeof(double) * (size_t)c->k,
                                   cudaMemcpyHostToDevice, c->stream));  // staging
        CK(cudaStreamSynchronize(c->stream));
    }
    const double* d_x0 = x0 ? c->xfull : nullptr;  // consumed before xfull is rewritten
    const int rc = method == 0 ? jacobi_impl(M, c->rhs, d_x0, tol, max_it, c->xs, rep)
                               : bicgstab_impl(M, c->rhs, d_x0, tol, max_it, c->xs, rep);
    if (rc != MCR_OK && rc != MCR_NOT_CONVERGED && rc != MCR_BREAKDOWN) return rc;
    const std::string msg = g_err;
    if (xs_out)
        CK(cudaMemcpyAsync(xs_out, c->xs, sizeof(double) * (size_t)c->k, cudaMemcpyDeviceToHost, M->stream));
    if (x_out && rc == MCR_OK) {
        k_scatter_x<<<(int)std::min<int64_t>((c->n + 255) / 256, 1 << 16), 256, 0, M->stream>>>(
            c->cls, c->remap, c->xs, (int)c->n, c->xfull);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(x_out, c->xfull, sizeof(double) * (size_t)c->n, cudaMemcpyDeviceToHost, M->stream));
    }
    CK(cudaStreamSynchronize(M->stream));
    g_err = msg;
    return rc;
}

MCR_API int mcr_matrix_info_get(const mcr_matrix* h, mcr_matrix_info* info) {
    if (!h || !info) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    info->n = h->n;
    info->nnz = h->nnz;
    info->storage = h->storage == MCR_STORAGE_DENSE ? MCR_STORAGE_DENSE
                    : (h->use_sell ? MCR_STORAGE_SELL : MCR_STORAGE_TILES);
    info->device = h->device;
    info->tiles = h->ntiles;
    info->max_row_nnz = h->max_row;
    info->first_zero_diagonal = h->first_zero;
    info->device_bytes = h->bytes;
    info->n_global = h->n_global;
    info->row0 = h->roff;
    info->world = h->world;
    info->rank = h->rank;
    return MCR_OK;
}

MCR_API int mcr_set_dot_mode(mcr_matrix* h, int mode) {
    if (!h) return fail(MCR_INVALID_ARGUMENT, "NULL handle");
    if (mode != MCR_DOTS_TREE && mode != MCR_DOTS_SEQUENTIAL)
        return fail(MCR_INVALID_ARGUMENT, "unknown dot mode");
    std::lock_guard<std::mutex> lk(h->mu);
    if (mode == MCR_DOTS_SEQUENTIAL && h->sharded())
        return fail(MCR_INVALID_ARGUMENT, "sequential dots need the whole system on one GPU");
    h->seqdots = mode == MCR_DOTS_SEQUENTIAL;
    return MCR_OK;
}

MCR_API int mcr_set_stream(mcr_matrix* h, void* stream) {
    if (!h) return fail(MCR_INVALID_ARGUMENT, "NULL handle");
    std::lock_guard<std::mutex> lk(h->mu);
    h->stream = stream ? (cudaStream_t)stream : h->own_stream;
    return MCR_OK;
}

MCR_API int mcr_matvec_device(mcr_matrix* h, const double* d_x, double* d_y) {
    if (!h) return fail(MCR_INVALID_ARGUMENT, "NULL handle");
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->n == 0) return MCR_OK;
    DeviceGuard g(h->device);
    Vecs V{};
    V.y = d_y;
    int64_t launched = 0;
    launch_mv<EPI_Y>(h, false, d_x, V, &launched);
    CK(cudaGetLastError());
    return MCR_OK;
}

MCR_API int mcr_matvec(mcr_matrix* h, const double* x, double* y) {
    if (!h) return fail(MCR_INVALID_ARGUMENT, "NULL handle");
    if (h->sharded()) return fail(MCR_INVALID_ARGUMENT, "mcr_matvec: use mcr_matvec_device on a row shard");
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->n == 0) return MCR_OK;
    DeviceGuard g(h->device);
    TRY(ensure_work(h));
    const size_t bytes = sizeof(double) * (size_t)h->n;
    CK(cudaMemcpyAsync(h->vec(V_P), x, bytes, cudaMemcpyHostToDevice, h->stream));
    Vecs V{};
    V.y = h->vec(V_V);
    int64_t launched = 0;
    launch_mv<EPI_Y>(h, false, h->vec(V_P), V, &launched);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(y, h->vec(V_V), bytes, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return MCR_OK;
}

MCR_API int mcr_residual_inf(mcr_matrix* h, const double* x, const double* b, double* out) {
    if (!h || !out) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    if (h->sharded()) return fail(MCR_INVALID_ARGUMENT, "mcr_residual_inf needs the whole system");
    std::lock_guard<std::mutex> lk(h->mu);
    *out = 0.0;
    if (h->n == 0) return MCR_OK;
    DeviceGuard g(h->device);
    TRY(ensure_work(h));
    const size_t bytes = sizeof(double) * (size_t)h->n;
    CK(cudaMemcpyAsync(h->vec(V_P), x, bytes, cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->vec(V_B), b, bytes, cudaMemcpyHostToDevice, h->stream));
    set_state(h, 0.0, 0);
    CK(cudaMemcpyAsync(h->st, h->h_st, sizeof(SolveState), cudaMemcpyHostToDevice, h->stream));
    int64_t launched = 0;
    TRY(residual_into_state(h, h->vec(V_P), &launched));
    TRY(read_state(h));
    *out = h->h_st->resid;
    return MCR_OK;
}

#define SOLVE_PROLOGUE                                                          \
    if (!h || !rep) return fail(MCR_INVALID_ARGUMENT, "NULL argument");        \
    if (!(tol > 0.0)) return fail(MCR_INVALID_ARGUMENT, "tolerance must be positive"); \
    if (max_it < 1) return fail(MCR_INVALID_ARGUMENT, "max_iterations must be at least 1"); \
    std::lock_guard<std::mutex> lk(h->mu);                                      \
    report_init(rep);                                                           \
    if (h->n == 0) {                                                            \
        rep->converged = 1;                                                     \
        return MCR_OK;                                                          \
    }                                                                           \
    DeviceGuard g(h->device);

MCR_API int mcr_jacobi_device(mcr_matrix* h, const double* d_b, const double* d_x0, double tol,
                              int64_t max_it, double* d_x_out, mcr_report* rep) {
    SOLVE_PROLOGUE
    return jacobi_impl(h, d_b, d_x0, tol, max_it, d_x_out, rep);
}

MCR_API int mcr_bicgstab_device(mcr_matrix* h, const double* d_b, const double* d_x0, double tol,
                                int64_t max_it, double* d_x_out, mcr_report* rep) {
    SOLVE_PROLOGUE
    return bicgstab_impl(h, d_b, d_x0, tol, max_it, d_x_out, rep);
}

MCR_API int mcr_jacobi(mcr_matrix* h, const double* b, const double* x0, double tol,
                       int64_t max_it, double* x_out, mcr_report* rep) {
    SOLVE_PROLOGUE
    return host_solve(h, b, x0, tol, max_it, x_out, rep, jacobi_impl);
}

MCR_API int mcr_bicgstab(mcr_matrix* h, const double* b, const double* x0, double tol,
                         int64_t max_it, double* x_out, mcr_report* rep) {
    SOLVE_PROLOGUE
    return host_solve(h, b, x0, tol, max_it, x_out, rep, bicgstab_impl);
}

}  // extern "C"
