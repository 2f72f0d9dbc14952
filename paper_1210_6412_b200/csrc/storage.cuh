// storage.cuh -- building a handle's device storage: upload and validation, diagonal, row tiles,
// Jacobi's off-diagonal copy, SELL and dense layouts, the C5 generator and device-side CSRs.
#pragma once

namespace {

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
    // the staged layout flags the diagonal instead of keeping a second copy
    if (h->r_ready || h->storage != MCR_STORAGE_CSR || h->use_staged) return MCR_OK;
    NvtxRange range("mcr.without_diagonal");
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
    const int64_t roff = h->nnz_off;  // counted at create: no read-back, no synchronisation
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

// Band-staged copy (staged.cuh): segment counts per (band, tile), scan, placement. Leaves
// use_staged false when the staged positions would not fit the 32-bit segment offsets.
constexpr double STAGED_AUTO_X_BYTES = 80e6;  // x this large (n >= 1e7): AUTO stages
constexpr int STAGED_AUTO_BAND = 4 << 20;                   // columns per band (32 MB of x)

int build_staged(mcr_matrix* h, bool forced) {
    NvtxRange range("mcr.stage");
    auto& S = h->stg;
    const int64_t nfull = h->n_full();
    // forced on a small system: up to 8 bands, so the multi-band path is exercised
    long long band = forced ? std::min<long long>((nfull + 7) / 8, STAGED_AUTO_BAND) : STAGED_AUTO_BAND;
    if (const char* env = std::getenv("MCR_STAGED_BAND")) band = std::max(1ll, std::atoll(env));
    band = std::max(band, (long long)((nfull + STG_NB_MAX - 1) / STG_NB_MAX));
    band = std::max(band, 1ll);
    S.band = (int)band;
    S.nb = (int)((nfull + band - 1) / band);
    const int nt = h->ntiles;
    const size_t K = (size_t)S.nb * (size_t)nt;
    long long* counts = nullptr;
    long long* offs = nullptr;
    CK(cudaMallocAsync((void**)&counts, sizeof(long long) * (K + 1), h->stream));
    CK(cudaMallocAsync((void**)&offs, sizeof(long long) * (K + 1), h->stream));
    CK(cudaMemsetAsync(counts + K, 0, sizeof(long long), h->stream));
    const int blocks = (nt + STG_BUILD_WARPS - 1) / STG_BUILD_WARPS;
    k_stage_count<<<blocks, STG_BUILD_WARPS * 32, 0, h->stream>>>(h->col, h->desc, nt, S.band,
                                                                   S.nb, counts);
    CK(cudaGetLastError());
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, counts, offs, K + 1, h->stream));
    void* dtmp = nullptr;
    CK(cudaMallocAsync(&dtmp, tmp, h->stream));
    CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, counts, offs, K + 1, h->stream));
    CK(cudaFreeAsync(dtmp, h->stream));
    CK(cudaFreeAsync(counts, h->stream));
    long long npos = 0;
    CK(cudaMemcpyAsync(&npos, offs + K, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (npos >= (1ll << 32)) {
        CK(cudaFreeAsync(offs, h->stream));
        return MCR_OK;
    }
    S.npos = npos;
    TRY(dalloc(h, &S.pval, (size_t)npos));
    TRY(dalloc(h, &S.pcol, (size_t)npos));
    TRY(dalloc(h, &S.prod, (size_t)npos));
    TRY(dalloc(h, &S.lidx, (size_t)h->nnz + 16));
    TRY(dalloc(h, &S.seg, K));
    k_stage_fill<<<blocks, STG_BUILD_WARPS * 32, 0, h->stream>>>(
        h->rp, h->col, h->val, h->desc, nt, S.band, S.nb, (long long)h->roff, offs, S.pval, S.pcol,
        S.lidx, S.seg);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(offs, h->stream));
    int sms = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_staged<EPI_V>, SP_THREADS,
                                                     STG_SMEM));
    S.grid = std::max(1, std::min(nt, sms * std::max(per_sm, 1)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stage_products<EPI_V>, STG_P1_NT, 0));
    S.p1_grid = (int)std::max<long long>(1, std::min<long long>((npos / 2 + STG_P1_NT - 1) / STG_P1_NT,
                                                                (long long)sms * std::max(per_sm, 1)));
    h->use_staged = true;
    return MCR_OK;
}

// Greedy tiles: consecutive rows while rows <= TILE_ROWS and entries <= TILE_NNZ; a row with
// more than TILE_NNZ entries is a tile of its own.
std::vector<int> make_tiles(int64_t n, const int64_t* rs, long long* max_row,
                            bool* monotone = nullptr) {
    std::vector<int> t;
    t.reserve((size_t)(n / 64 + 2));
    t.push_back(0);
    long long mr = 0;
    int64_t r = 0;
    bool mono = true;
    while (r < n) {
        const int64_t start = r;
        int64_t nnz = 0;
        while (r < n && r - start < TILE_ROWS) {
            const int64_t len = rs[r + 1] - rs[r];
            mono &= len >= 0;
            mr = std::max<long long>(mr, len);
            if (nnz + len > TILE_NNZ && r > start) break;
            nnz += len;
            ++r;
            if (nnz > TILE_NNZ) break;
        }
        t.push_back((int)r);
    }
    if (monotone) *monotone = mono;
    *max_row = mr;
    return t;
}


}  // namespace

static int set_kernel_attributes() {
    const int sp = (int)SP_SMEM;
    CK(cudaFuncSetAttribute(k_spmv<EPI_Y>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_JACOBI>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_S0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_V>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    CK(cudaFuncSetAttribute(k_spmv<EPI_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp));
    const int sg = (int)STG_SMEM;
    CK(cudaFuncSetAttribute(k_spmv_staged<EPI_Y>, cudaFuncAttributeMaxDynamicSharedMemorySize, sg));
    CK(cudaFuncSetAttribute(k_spmv_staged<EPI_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, sg));
    CK(cudaFuncSetAttribute(k_spmv_staged<EPI_JACOBI>, cudaFuncAttributeMaxDynamicSharedMemorySize, sg));
    CK(cudaFuncSetAttribute(k_spmv_staged<EPI_S0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sg));
    CK(cudaFuncSetAttribute(k_spmv_staged<EPI_V>, cudaFuncAttributeMaxDynamicSharedMemorySize, sg));
    CK(cudaFuncSetAttribute(k_spmv_staged<EPI_T>, cudaFuncAttributeMaxDynamicSharedMemorySize, sg));
    return MCR_OK;
}

// Rows [h->roff, h->roff + n) of an h->n_global system (the whole system on one GPU);
// column indices are global.
int finish_create(mcr_matrix* h, int64_t n, const int64_t* rs, int storage,
                         std::vector<int>* pre_tiles = nullptr);

// Can a cluster of `ctas` small-solver CTAs be scheduled (<= 8 portable, 16 non-portable)?
bool small_cluster_ok(int ctas) {
    static int ok16 = -1;
    if (ok16 < 0) {
        ok16 = cudaFuncSetAttribute(k_jacobi_small<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                       cudaSuccess &&
                   cudaFuncSetAttribute(k_bicg_small<true, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                       cudaSuccess &&
                   cudaFuncSetAttribute(k_bicg_small<true, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                       cudaSuccess;
        cudaGetLastError();
    }
    if (ctas > 8 && !ok16) return false;
    for (int which = 0; which < 2; ++which) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(SM_NT);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = ctas;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        const cudaError_t e = which == 0
                                  ? cudaOccupancyMaxActiveClusters(&clusters, k_jacobi_small<true>, &cfg)
                                  : cudaOccupancyMaxActiveClusters(&clusters, k_bicg_small<true, false>, &cfg);
        if (e != cudaSuccess || clusters < 1) {
            cudaGetLastError();
            return false;
        }
    }
    return true;
}

// Can the reference-order-dot variant of k_bicg_small run this handle's small grid (its
// dynamic shared memory grows with n)? Sets h->small_xd and allocates its product slots.
int small_xd_check(mcr_matrix* h, int sms) {
    h->small_xd = false;
    if (h->n > XS_MAX_N || std::getenv("MCR_NO_SMALL_XD")) return MCR_OK;
    const size_t smem = small_xd_smem(h->n);
    if (cudaFuncSetAttribute(k_bicg_small<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(k_bicg_small<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
        cudaGetLastError();
        return MCR_OK;
    }
    bool ok = false;
    if (h->small_cluster) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(h->small_grid);
        cfg.blockDim = dim3(SM_NT);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = h->small_grid;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        ok = cudaOccupancyMaxActiveClusters(&clusters, k_bicg_small<true, true>, &cfg) == cudaSuccess &&
             clusters >= 1;
    } else {
        int per_sm = 0;
        ok = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bicg_small<false, true>, SM_NT, smem) ==
                 cudaSuccess &&
             per_sm * sms >= h->small_grid;
    }
    cudaGetLastError();
    if (!ok) return MCR_OK;
    if (h->small_grid > 1) TRY(dalloc(h, &h->xsprod, (size_t)4 * h->n));
    h->small_xd = true;
    return MCR_OK;
}

int init_handle(mcr_matrix* h) {
    TRY(keep_pool_memory(h->device));
    CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    h->stream = h->own_stream;
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    TRY(dalloc(h, &h->st, 1));
    CK(cudaMemsetAsync(h->st, 0, sizeof(SolveState), h->stream));
    return MCR_OK;
}

int alloc_csr(mcr_matrix* h, int64_t n, int64_t nnz) {
    h->nnz = nnz;
    if (!h->rp) TRY(dalloc(h, &h->rp, (size_t)n + 1 + CSR_PAD));
    TRY(dalloc(h, &h->col, (size_t)nnz + CSR_PAD));
    TRY(dalloc(h, &h->val, (size_t)nnz + CSR_PAD));
    TRY(dalloc(h, &h->d, (size_t)n));
    TRY(dalloc(h, &h->offlen, (size_t)n + 1));
    return MCR_OK;
}

// Host -> device copies of pageable arrays (a reference CsrMatrix holds plain numpy arrays).
// cudaMemcpyAsync from pageable memory stages through the driver's own pinned buffer with one
// host thread; here h2d_threads() threads each copy their share of the bytes through their own
// ring of pinned chunks (host memcpy into chunk k while the DMA engine drains chunk k-1), so
// the host-side copy runs in parallel and overlaps the transfer. Pinned sources and small
// copies go straight to cudaMemcpyAsync. MCR_H2D_RING=0 turns the ring off.
// conv = 1: the source holds int64 values sent as int32 (the column indices: half the bytes
// over PCIe), narrowed on the host while they are copied into the pinned chunks; their min /
// max come back for the caller's range check.
struct H2DPart { void* dst; const void* src; size_t bytes; int conv = 0; };

inline void narrow_i64(int* out, const long long* in, size_t cnt, long long& mn, long long& mx) {
    long long a = mn, b = mx;
    for (size_t i = 0; i < cnt; ++i) {
        const long long c = in[i];
        a = c < a ? c : a;
        b = c > b ? c : b;
        out[i] = (int)c;
    }
    mn = a;
    mx = b;
}
constexpr int H2D_MAX_THREADS = 32, H2D_SLOTS = 3;
constexpr size_t H2D_CHUNK = 4u << 20, H2D_MIN = 8u << 20;

struct H2DRing {
    std::mutex mu;
    char* buf[H2D_MAX_THREADS][H2D_SLOTS] = {};
    cudaEvent_t ev[H2D_MAX_THREADS][H2D_SLOTS] = {};
    bool ready = false, failed = false;
};
inline H2DRing& h2d_ring() { static H2DRing r; return r; }
// host threads of the ring: MCR_H2D_THREADS, default 8 (clamped to the host's threads)
inline int h2d_threads() {
    static const int n = [] {
        int t = 8;
        if (const char* e = getenv("MCR_H2D_THREADS")) t = atoi(e);
        const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
        return std::max(1, std::min({t, hw, H2D_MAX_THREADS}));
    }();
    return n;
}

inline bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

inline bool h2d_ring_on() {
    static const bool on = [] { const char* e = getenv("MCR_H2D_RING"); return !e || atoi(e) != 0; }();
    return on;
}

// Narrowing parts that cannot take the ring: converted into a host buffer, copied synchronously.
inline int h2d_narrow_plain(const H2DPart& p, cudaStream_t stream, long long* cmin, long long* cmax) {
    std::vector<int> tmp(p.bytes / 8);
    narrow_i64(tmp.data(), (const long long*)p.src, tmp.size(), *cmin, *cmax);
    CK(cudaMemcpyAsync(p.dst, tmp.data(), p.bytes / 2, cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));
    return MCR_OK;
}

inline int h2d_copy(const std::vector<H2DPart>& parts, cudaStream_t stream, long long* cmin = nullptr,
                    long long* cmax = nullptr) {
    std::vector<H2DPart> ring;
    size_t total = 0;
    for (const H2DPart& p : parts) {
        if (!p.bytes) continue;
        if (!h2d_ring_on() || p.bytes < H2D_MIN || host_pinned(p.src)) {
            if (p.conv) TRY(h2d_narrow_plain(p, stream, cmin, cmax));
            else CK(cudaMemcpyAsync(p.dst, p.src, p.bytes, cudaMemcpyHostToDevice, stream));
        } else {
            ring.push_back(p);
            total += p.bytes;
        }
    }
    if (ring.empty()) return MCR_OK;
    H2DRing& R = h2d_ring();
    std::lock_guard<std::mutex> lock(R.mu);
    if (!R.ready && !R.failed) {
        for (int t = 0; t < h2d_threads() && !R.failed; ++t)
            for (int s = 0; s < H2D_SLOTS; ++s) {
                if (cudaHostAlloc((void**)&R.buf[t][s], H2D_CHUNK, cudaHostAllocPortable) != cudaSuccess ||
                    cudaEventCreateWithFlags(&R.ev[t][s], cudaEventDisableTiming) != cudaSuccess) {
                    cudaGetLastError();
                    R.failed = true;
                    break;
                }
            }
        R.ready = !R.failed;
    }
    if (!R.ready) {  // no pinned memory to be had: the driver's own staging
        for (const H2DPart& p : ring) {
            if (p.conv) TRY(h2d_narrow_plain(p, stream, cmin, cmax));
            else CK(cudaMemcpyAsync(p.dst, p.src, p.bytes, cudaMemcpyHostToDevice, stream));
        }
        return MCR_OK;
    }
    // thread t copies bytes [t*share, (t+1)*share) of the concatenated parts (whole 8-byte
    // elements: every part is an array of them)
    const int NTH = h2d_threads();
    const size_t share = ((total + NTH - 1) / NTH + 7) & ~(size_t)7;
    std::vector<long long> tmin(NTH, LLONG_MAX), tmax(NTH, LLONG_MIN);
    std::atomic<int> err{cudaSuccess};
    int device = 0;
    CK(cudaGetDevice(&device));
    auto work = [&](int t) {
        cudaSetDevice(device);
        size_t lo = (size_t)t * share, hi = std::min(total, lo + share), base = 0;
        int slot = 0;
        for (const H2DPart& p : ring) {
            const size_t a = std::max(lo, base), b = std::min(hi, base + p.bytes);
            for (size_t o = a; o < b; o += H2D_CHUNK) {
                const size_t len = std::min(H2D_CHUNK, b - o);
                cudaError_t e = cudaEventSynchronize(R.ev[t][slot]);  // the slot's last DMA drained
                if (e == cudaSuccess && p.conv) {
                    narrow_i64((int*)R.buf[t][slot], (const long long*)((const char*)p.src + (o - base)),
                               len / 8, tmin[t], tmax[t]);
                    e = cudaMemcpyAsync((char*)p.dst + (o - base) / 2, R.buf[t][slot], len / 2,
                                        cudaMemcpyHostToDevice, stream);
                } else if (e == cudaSuccess) {
                    memcpy(R.buf[t][slot], (const char*)p.src + (o - base), len);
                    e = cudaMemcpyAsync((char*)p.dst + (o - base), R.buf[t][slot], len,
                                        cudaMemcpyHostToDevice, stream);
                }
                if (e == cudaSuccess) e = cudaEventRecord(R.ev[t][slot], stream);
                if (e != cudaSuccess) { err = e; return; }
                slot = (slot + 1) % H2D_SLOTS;
            }
            base += p.bytes;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < NTH; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    CK((cudaError_t)err.load());
    if (cmin && cmax)
        for (int t = 0; t < NTH; ++t) {
            *cmin = std::min(*cmin, tmin[t]);
            *cmax = std::max(*cmax, tmax[t]);
        }
    return MCR_OK;
}

int create_impl(mcr_matrix* h, int64_t n, const int64_t* rs, const int64_t* col,
                const double* val, int storage) {
    NvtxRange range("mcr.create");
    Trace tr;
    TRY(init_handle(h));
    if (n == 0) return MCR_OK;
    tr.mark("create: handle");
    const int64_t nnz = rs[n];
    TRY(alloc_csr(h, n, nnz));
    // int64 columns -> int32, range-checked, then the row-order check on the device. Pageable
    // columns (a reference CsrMatrix) are narrowed on the host while the ring copies them, so
    // half their bytes cross PCIe: the upload is bound by the link (≈27 GB/s on the test boxes;
    // 4, 8, 12 and 16 ring threads measure the same), and C2's 184 MB become 144 MB (create
    // 6.2-6.4 -> 5.5-5.7 ms, tools/dropin_probe.py). Pinned columns go over as they are and a
    // kernel narrows them. MCR_HOST_NARROW=0: the kernel always.
    static const bool narrow_env = [] { const char* e = getenv("MCR_HOST_NARROW"); return !e || atoi(e) != 0; }();
    const bool host_narrow = narrow_env && nnz > 0 && h2d_ring_on() &&
                             sizeof(long long) * (size_t)nnz >= H2D_MIN && !host_pinned(col);
    long long* tmp = nullptr;
    int* bad = nullptr;
    if (!host_narrow)
        CK(cudaMallocAsync((void**)&tmp, sizeof(long long) * (size_t)std::max<int64_t>(nnz, 1),
                           h->stream));
    CK(cudaMallocAsync((void**)&bad, 2 * sizeof(int), h->stream));
    CK(cudaMemsetAsync(bad, 0, 2 * sizeof(int), h->stream));
    // the row tiles are cut on a host thread while the copies run
    bool monotone = true;
    long long max_row = 0, cmin = LLONG_MAX, cmax = LLONG_MIN;
    std::vector<int> tiles;
    std::thread cut([&] {
        tiles = make_tiles(n, rs, &max_row, &monotone);
        tr.mark("create: tiles cut (thread)");
    });
    std::vector<H2DPart> parts(3);
    parts[0].dst = h->rp; parts[0].src = rs; parts[0].bytes = sizeof(long long) * (size_t)(n + 1);
    parts[1].dst = h->val; parts[1].src = val; parts[1].bytes = sizeof(double) * (size_t)nnz;
    parts[2].dst = host_narrow ? (void*)h->col : (void*)tmp;
    parts[2].src = col;
    parts[2].bytes = sizeof(long long) * (size_t)nnz;
    parts[2].conv = host_narrow ? 1 : 0;
    const int copied = h2d_copy(parts, h->stream, &cmin, &cmax);
    tr.mark("create: ring copies issued");
    cut.join();
    h->max_row = max_row;
    TRY(copied);
    if (nnz > 0) {
        if (!host_narrow)
            k_col64to32<<<(int)std::min<int64_t>((nnz + 255) / 256, 1 << 16), 256, 0, h->stream>>>(
                tmp, h->col, nnz, (int)h->n_global, bad);
        k_check_rows<<<(int)std::min<int64_t>((n + 255) / 256, 1 << 16), 256, 0, h->stream>>>(
            h->rp, h->col, (int)n, (long long)nnz, bad + 1);
    }
    CK(cudaGetLastError());
    tr.mark("create: copies issued, tiles cut (host)");
    CK(cudaMemcpyAsync(h->bad_host, bad, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    if (tmp) CK(cudaFreeAsync(tmp, h->stream));
    CK(cudaFreeAsync(bad, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (host_narrow && (cmin < 0 || cmax >= h->n_global)) h->bad_host[0] = 1;
    tr.mark("create: copies + checks done");
    if (!monotone) return fail(MCR_DIMENSION, "rstart must be nondecreasing");
    if (h->bad_host[0]) return fail(MCR_DIMENSION, "column index out of range");
    if (h->bad_host[1]) return fail(MCR_DIMENSION, "rows must be sorted by column without duplicates");
    const int rc = finish_create(h, n, rs, storage, &tiles);
    tr.mark("create: finished");
    return rc;
}

// A handle from a CSR already on the device (int64 row starts, int32 columns), copied.
int create_from_device(int64_t n, int64_t nnz, const long long* d_rp, const int* d_col,
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
void poisson_thresholds(double mean, uint64_t* thr) {
    double p = std::exp(-mean), cdf = 0.0;
    for (int k = 0; k < GEN_KMAX; ++k) {
        cdf += p;
        const double t = cdf * 18446744073709551616.0;
        thr[k] = t >= 18446744073709551616.0 ? UINT64_MAX : (uint64_t)t;
        p = (p * mean) / (double)(k + 1);
    }
}

// Rows [h->roff, h->roff + h->n) of the row-keyed synthetic system, built on the device.
int generate_impl(mcr_matrix* h, const GenParams& P, int storage) {
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
int finish_create(mcr_matrix* h, int64_t n, const int64_t* rs, int storage,
                         std::vector<int>* pre_tiles) {
    const int64_t nnz = h->nnz;
    const bool dense = !h->sharded() &&
                       (storage == MCR_STORAGE_DENSE ||
                        (storage == MCR_STORAGE_AUTO && n >= 1024 &&
                         (double)nnz * 3.0 >= 2.0 * (double)n * (double)n));
    h->storage = dense ? MCR_STORAGE_DENSE : MCR_STORAGE_CSR;
    // diagonal, first zero-diagonal row (read back at the final synchronisation below),
    // off-diagonal row lengths
    {
        unsigned long long* fz = nullptr;
        CK(cudaMallocAsync((void**)&fz, 2 * sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(fz, 0xff, sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(fz + 1, 0, sizeof(unsigned long long), h->stream));
        CK(cudaMemsetAsync(h->offlen + n, 0, sizeof(long long), h->stream));
        k_diag<<<(int)std::min<int64_t>((n + 255) / 256, 1 << 16), 256, 0, h->stream>>>(
            h->rp, h->col, h->val, (int)n, (long long)h->roff, h->d, h->offlen, fz, fz + 1);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(h->fz_host, fz, sizeof(h->fz_host), cudaMemcpyDeviceToHost,
                           h->stream));  // a handle field: outlives any early return
        CK(cudaFreeAsync(fz, h->stream));
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
        double auto_bytes = STAGED_AUTO_X_BYTES;  // tuning / test override of the AUTO cut
        if (const char* env = std::getenv("MCR_STAGED_MIN_X_BYTES")) auto_bytes = std::atof(env);
        const bool stage = !h->use_sell && h->nnz > 0 && h->max_row <= TILE_NNZ &&
                           (storage == MCR_STORAGE_STAGED ||
                            (storage == MCR_STORAGE_AUTO &&
                             8.0 * (double)h->n_full() >= auto_bytes));
        int pj = 0, pb = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pj, k_jacobi_small<false>, SM_NT, 0));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pb, k_bicg_small<false, false>, SM_NT, 0));
        const int coresident = sms * std::min(pj, pb);
        // one tile per CTA keeps the per-sweep critical path to a single tile
        if (!h->use_sell && !h->sharded() && !stage && storage != MCR_STORAGE_TILES_STREAM &&
            h->ntiles <= coresident && h->ntiles <= 2 * sms)
            h->small_grid = h->ntiles;
        // up to 16 tiles: the whole grid as one thread-block cluster (cluster barriers, DSMEM)
        if (h->small_grid > 0 && h->small_grid <= SMALL_CLUSTER_MAX && !std::getenv("MCR_NO_CLUSTER"))
            h->small_cluster = small_cluster_ok(h->small_grid);
        if (h->small_grid > 0) TRY(small_xd_check(h, sms));
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
        if (stage) TRY(build_staged(h, storage == MCR_STORAGE_STAGED));
        CK(cudaStreamSynchronize(h->stream));
    }
    h->first_zero = h->fz_host[0] == ~0ull ? -1 : (long long)h->fz_host[0] + h->roff;  // global row
    h->nnz_off = nnz - (int64_t)h->fz_host[1];
    return MCR_OK;
}

// `scan_rows` = false: the caller's upload path checks that rstart is nondecreasing itself
// (make_tiles walks rstart anyway, while the copies are in flight).
int check_csr(int64_t n, const int64_t* rstart, const int64_t* col, const double* nonzero,
              bool scan_rows = true) {
    if (n < 0 || n >= INT_MAX) return fail(MCR_DIMENSION, "dimension out of range");
    if (n > 0 && (!rstart || (rstart[n] > 0 && (!col || !nonzero))))
        return fail(MCR_INVALID_ARGUMENT, "NULL CSR array");
    if (n > 0) {
        if (rstart[0] != 0 || rstart[n] < 0) return fail(MCR_DIMENSION, "malformed rstart vector");
        if (scan_rows)
            for (int64_t i = 0; i < n; ++i)
                if (rstart[i + 1] < rstart[i]) return fail(MCR_DIMENSION, "rstart must be nondecreasing");
    }
    return MCR_OK;
}

int create_handle(int64_t n, const int64_t* rstart, const int64_t* col,
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

