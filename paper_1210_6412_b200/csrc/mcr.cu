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
#include "handle.h"
#include "xdot_host.cuh"
#include "storage.cuh"
#include "solve.cuh"
#include "chain_host.cuh"
#include "refgen_host.cuh"

using namespace mcr;

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
                            h->rsell.swidth, h->maxslot, h->recv, h->stg.pval, h->stg.pcol,
                            h->stg.lidx, h->stg.prod, h->stg.seg};
            for (void* p : ptrs)
                if (p) cudaFreeAsync(p, s);
            cudaStreamSynchronize(s);
        }
        xdot_free(h->xdot, s ? s : h->stream);
        h->xdot = nullptr;
        for (auto* gl : {&h->gl_bicg}) {
            if (gl->exec) cudaGraphExecDestroy(gl->exec);
            if (gl->graph) cudaGraphDestroy(gl->graph);
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

MCR_API int mcr_matrix_create(int64_t n, const int64_t* rstart, const int64_t* col,
                              const double* nonzero, int device, int storage, mcr_matrix** out) {
    if (!out) return fail(MCR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    TRY(check_csr(n, rstart, col, nonzero, false));  // monotonicity: checked during the upload
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
    TRY(check_csr(rows, rstart, col, nonzero, false));
    const int64_t chunk = (n_global + T.world - 1) / T.world;
    return create_handle(rows, rstart, col, nonzero, T.device, MCR_STORAGE_AUTO, comm->t,
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
        h->rank = rank;  // (shards never take the dense or single-launch paths)
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

// The reference's generator on the device (refgen.cuh): pcg = {state >> 64, state, inc >> 64,
// inc} of numpy's PCG64(seed) (default_rng(seed).bit_generator.state).
MCR_API int mcr_refgen_matrix(int device, int64_t n, int64_t count, int64_t lo, int64_t hi, const uint64_t* pcg,
                              int storage, mcr_matrix** out) {
    if (!pcg || !out || n < 1 || count < 0 || lo < 1 || hi < lo || hi - lo >= (1ll << 31) ||
        (n > 1 && count > n * (n - 1)) || (n == 1 && count > 0) || n >= (1ll << 31))
        return fail(MCR_INVALID_ARGUMENT, "mcr_refgen_matrix: bad arguments");
    DeviceGuard g(device);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    RgStream S;
    S.s = rg::mk128(pcg[0], pcg[1]);
    S.inc = rg::mk128(pcg[2], pcg[3]);
    long long* rp = nullptr;
    int* col = nullptr;
    double* val = nullptr;
    int rc = rg_matrix(st, S, n, count, lo, hi, &rp, &col, &val);
    if (rc == MCR_OK) rc = create_from_device(n, count + n, rp, col, val, device, storage, out);
    if (rp) cudaFreeAsync(rp, st);
    if (col) cudaFreeAsync(col, st);
    if (val) cudaFreeAsync(val, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    return rc;
}

MCR_API int mcr_refgen_integers(int device, int64_t n, int64_t lo, int64_t hi, const uint64_t* pcg, double* out) {
    if (!pcg || !out || n < 0 || hi < lo || hi - lo > 0xFFFFFFFEll)
        return fail(MCR_INVALID_ARGUMENT, "mcr_refgen_integers: bad arguments");
    if (n == 0) return MCR_OK;
    DeviceGuard g(device);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    RgStream S;
    S.s = rg::mk128(pcg[0], pcg[1]);
    S.inc = rg::mk128(pcg[2], pcg[3]);
    double* d = nullptr;
    int rc = MCR_OK;
    if (cudaMallocAsync((void**)&d, sizeof(double) * (size_t)rg_cap(n), st) != cudaSuccess)
        rc = fail(MCR_CUDA_ERROR, "mcr_refgen_integers: allocation failed");
    if (rc == MCR_OK) rc = rg_draw(st, S, (uint64_t)(hi - lo + 1), lo, n, nullptr, d);
    if (rc == MCR_OK && cudaMemcpyAsync(out, d, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(MCR_CUDA_ERROR, "mcr_refgen_integers: copy failed");
    if (d) cudaFreeAsync(d, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    return rc;
}

MCR_API int mcr_refgen_u64(int device, int64_t n, uint64_t range, const uint64_t* pcg, uint64_t* out) {
    if (!pcg || !out || n < 0 || range < 2) return fail(MCR_INVALID_ARGUMENT, "mcr_refgen_u64: bad arguments");
    if (n == 0) return MCR_OK;
    DeviceGuard g(device);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    RgStream S;
    S.s = rg::mk128(pcg[0], pcg[1]);
    S.inc = rg::mk128(pcg[2], pcg[3]);
    uint64_t* d = nullptr;
    int rc = MCR_OK;
    if (cudaMallocAsync((void**)&d, sizeof(uint64_t) * (size_t)rg_cap(n), st) != cudaSuccess)
        rc = fail(MCR_CUDA_ERROR, "mcr_refgen_u64: allocation failed");
    if (rc == MCR_OK) rc = rg_draw(st, S, range, 0, n, d, nullptr);
    if (rc == MCR_OK && cudaMemcpyAsync(out, d, sizeof(uint64_t) * (size_t)n, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(MCR_CUDA_ERROR, "mcr_refgen_u64: copy failed");
    if (d) cudaFreeAsync(d, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    return rc;
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
                    : h->use_sell                    ? MCR_STORAGE_SELL
                    : h->use_staged                  ? MCR_STORAGE_STAGED
                                                     : MCR_STORAGE_TILES;
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
    if (mode != MCR_DOTS_TREE && mode != MCR_DOTS_SEQUENTIAL && mode != MCR_DOTS_SERIAL)
        return fail(MCR_INVALID_ARGUMENT, "unknown dot mode");
    std::lock_guard<std::mutex> lk(h->mu);
    if (mode == MCR_DOTS_SERIAL && h->sharded())
        return fail(MCR_INVALID_ARGUMENT, "serial dots need the whole system on one GPU");
    h->seqdots = mode;
    return MCR_OK;
}

MCR_API int mcr_set_dot_blocks(mcr_matrix* h, int nblocks) {
    if (!h) return fail(MCR_INVALID_ARGUMENT, "NULL handle");
    if (nblocks < 1) return fail(MCR_INVALID_ARGUMENT, "dot blocks must be >= 1");
    std::lock_guard<std::mutex> lk(h->mu);
    h->dot_blocks = nblocks;
    return MCR_OK;
}

MCR_API int mcr_xdot_stats(mcr_matrix* h, uint64_t* out, int count) {
    if (!h || !out) return fail(MCR_INVALID_ARGUMENT, "NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    std::memset(out, 0, sizeof(uint64_t) * (size_t)std::max(count, 0));
    if (!h->xdot || !h->xdot->stats) return MCR_OK;
    DeviceGuard g(h->device);
    const int k = std::min(count, (int)xd::ST_COUNT);
    CK(cudaMemcpyAsync(out, h->xdot->stats, sizeof(uint64_t) * (size_t)k, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return MCR_OK;
}

MCR_API int mcr_xdot_bench(int device, int64_t n, const double* u, const double* v, int nblocks,
                           int reps, double* out, double* ms, uint64_t* stats);

MCR_API int mcr_xdot(int device, int64_t n, const double* u, const double* v, int nblocks,
                     double* out, uint64_t* stats) {
    return mcr_xdot_bench(device, n, u, v, nblocks, 0, out, nullptr, stats);
}

// Same, timed: after one launch, `reps` more launches on device-resident inputs between two
// CUDA events; *ms = mean milliseconds per launch (diagnostics / tools/xdot_bench.py).
MCR_API int mcr_xdot_bench(int device, int64_t n, const double* u, const double* v, int nblocks,
                           int reps, double* out, double* ms, uint64_t* stats) {
    if (n < 0 || nblocks < 1 || !out || (n > 0 && (!u || !v)))
        return fail(MCR_INVALID_ARGUMENT, "mcr_xdot: bad arguments");
    DeviceGuard g(device);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct Cleanup {
        cudaStream_t s;
        std::vector<void*> p;
        XdotCtx* X = nullptr;
        ~Cleanup() {
            for (void* q : p) cudaFreeAsync(q, s);
            xdot_free(X, s);
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    } c{s, {}};
    double *du = nullptr, *dv = nullptr, *dout = nullptr;
    const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
    CK(cudaMallocAsync((void**)&du, bytes, s)); c.p.push_back(du);
    CK(cudaMallocAsync((void**)&dv, bytes, s)); c.p.push_back(dv);
    CK(cudaMallocAsync((void**)&dout, sizeof(double) * (size_t)(2 + nblocks), s)); c.p.push_back(dout);
    if (n > 0) {
        CK(cudaMemcpyAsync(du, u, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(dv, v, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, s));
    }
    c.X = new XdotCtx();
    TRY(xdot_smem_attr<SQ_TEST>());
    TRY(xdot_plan(*c.X, SQ_TEST, s, device, n, 1, nblocks, du, dv, nullptr, nullptr));
    const auto& P = c.X->plan[SQ_TEST];
    k_xdot<SQ_TEST><<<P.grid, xd::NT, P.smem, s>>>(xdot_args(*c.X, SQ_TEST, dout), nullptr);
    CK(cudaGetLastError());
    if (reps > 0 && ms) {
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, s));
        for (int r = 0; r < reps; ++r)
            k_xdot<SQ_TEST><<<P.grid, xd::NT, P.smem, s>>>(xdot_args(*c.X, SQ_TEST, dout), nullptr);
        CK(cudaEventRecord(e1, s));
        CK(cudaEventSynchronize(e1));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, e0, e1));
        *ms = t / reps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    std::vector<double> h(2 + nblocks);
    CK(cudaMemcpyAsync(h.data(), dout, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
    if (stats && c.X->stats)
        CK(cudaMemcpyAsync(stats, c.X->stats, sizeof(unsigned long long) * xd::ST_COUNT,
                           cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out[0] = h[0];
    for (int b = 0; b < nblocks; ++b) out[1 + b] = h[2 + b];
    return MCR_OK;
}

// The one-CTA reference-order dot (k_xdot_cta, small.cuh) stand-alone; test entry point.
MCR_API int mcr_xdot_cta(int device, int64_t n, const double* u0, const double* v0, const double* u1,
                         const double* v1, int k, double* out) {
    if (n < 0 || n > XS_MAX_N || (k != 1 && k != 2) || !out || (n > 0 && (!u0 || !v0)) ||
        (k == 2 && n > 0 && (!u1 || !v1)))
        return fail(MCR_INVALID_ARGUMENT, "mcr_xdot_cta: bad arguments");
    DeviceGuard g(device);
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    std::vector<void*> p;
    auto done = [&] {
        for (void* q : p) cudaFreeAsync(q, s);
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    };
    const size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
    double* d[5] = {};
    for (int i = 0; i < 5; ++i) {
        if (cudaMallocAsync((void**)&d[i], i == 4 ? 2 * sizeof(double) : bytes, s) != cudaSuccess) {
            done();
            return fail(MCR_CUDA_ERROR, "mcr_xdot_cta: allocation failed");
        }
        p.push_back(d[i]);
    }
    const double* src[4] = {u0, v0, k == 2 ? u1 : u0, k == 2 ? v1 : v0};
    for (int i = 0; i < 4 && n > 0; ++i)
        cudaMemcpyAsync(d[i], src[i], sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, s);
    const size_t smem = small_xd_smem(n);
    cudaError_t e;
    if (k == 1) {
        cudaFuncSetAttribute(k_xdot_cta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_xdot_cta<1><<<1, SM_NT, smem, s>>>(d[0], d[1], d[2], d[3], (int)n, d[4]);
    } else {
        cudaFuncSetAttribute(k_xdot_cta<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_xdot_cta<2><<<1, SM_NT, smem, s>>>(d[0], d[1], d[2], d[3], (int)n, d[4]);
    }
    e = cudaGetLastError();
    double h[2] = {0.0, 0.0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, d[4], 2 * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    done();
    if (e != cudaSuccess) return fail(MCR_CUDA_ERROR, std::string("mcr_xdot_cta: ") + cudaGetErrorString(e));
    out[0] = h[0];
    if (k == 2) out[1] = h[1];
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
    TRY(launch_check());
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
    TRY(launch_check());
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
