// solve.cuh -- solve drivers: kernel launchers (PDL), the row-shard exchange points, and the
// Jacobi / BiCGStab loops that enqueue batches of device-resident iterations.
#pragma once

namespace {

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
// Whole-solve small kernels: one cluster (CL) or one cooperative grid.
template <typename... KArgs, typename... Args>
int launch_small(mcr_matrix* h, size_t smem, void (*cluster_kern)(KArgs...), void (*grid_kern)(KArgs...),
                 Args... args) {
    if (h->small_cluster) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(h->small_grid);
        cfg.blockDim = dim3(SM_NT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = h->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = h->small_grid;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, cluster_kern, static_cast<KArgs>(args)...));
    } else {
        void* a[] = {(void*)&args...};
        CK(cudaLaunchCooperativeKernel((void*)grid_kern, h->small_grid, SM_NT, a, smem, h->stream));
    }
    return MCR_OK;
}

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
    static const bool pdl = std::getenv("MCR_NO_PDL") == nullptr;  // A/B switch for profiling
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    note_launch(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

template <int EPI>
void launch_mv(mcr_matrix* h, bool offdiag, const double* x, const Vecs& V, int64_t* launches) {
    if (h->storage == MCR_STORAGE_DENSE) {
        launch_pdl(k_dense<EPI>, h->nslabs, 32, DENSE_SMEM, h->stream, (const double*)h->dense,
                   (int)h->n, (int)((h->n + 1) & ~1ll), x, V, h->st);
    } else if (h->use_staged) {  // products pass, then the row sums (Jacobi skips the diagonal)
        const Staged A = staged_view(h);
        launch_pdl(k_stage_products<EPI>, h->stg.p1_grid, STG_P1_NT, 0, h->stream, A, x, V, h->st);
        launch_pdl(k_spmv_staged<EPI>, h->stg.grid, SP_THREADS, STG_SMEM, h->stream, A, V, h->st);
        ++*launches;
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
    constexpr int rows = CHUNK_NT * phase_per<PH>();
    const int grid = PH == PH_E ? h->nchunks() : (int)((h->n + rows - 1) / rows);
    launch_pdl(k_phase<PH>, grid, CHUNK_NT, 0, h->stream, V, (int)h->n, h->st);
    ++*launches;
}

// Reference-order dots of one reduction point (plans built by xdot_prepare beforehand: no
// allocation may happen while a graph is being captured).
template <int W>
void launch_seqdot(mcr_matrix* h, const Vecs& V, int64_t* launches) {
    if (!h->seqdots) return;
    if (h->seqdots == MCR_DOTS_SERIAL) {
        launch_pdl(k_seqdot<W>, 1, SEQ_NT, 0, h->stream, V, (int)h->n, h->st);
    } else {
        const auto& P = h->xdot->plan[W];
        launch_pdl(k_xdot<W>, P.grid, xd::NT, P.smem, h->stream, xdot_args(*h->xdot, W, nullptr),
                   h->st);
    }
    ++*launches;
}

// Plans of the four BiCGStab reduction points: q.r at setup (q = r), q.v, {t.t, t.s}, q.r.
int xdot_prepare(mcr_matrix* h, const Vecs& V) {
    if (h->seqdots != MCR_DOTS_SEQUENTIAL) return MCR_OK;
    if (!h->xdot) h->xdot = new XdotCtx();
    XdotCtx& X = *h->xdot;
    const int nb = h->dot_blocks;
    TRY(xdot_smem_attr<SQ_S0>());
    TRY(xdot_smem_attr<SQ_V>());
    TRY(xdot_smem_attr<SQ_T>());
    TRY(xdot_smem_attr<SQ_E>());
    // a row shard sums the whole gathered vectors (every rank the same bits): its own rows sit
    // at roff of the full-length buffers
    const int64_t n = h->sharded() ? h->n_global : h->n;
    const double *q = V.q - h->roff, *r = V.r - h->roff, *v = V.v - h->roff, *t = V.t - h->roff,
                 *s = V.s - h->roff;
    TRY(xdot_plan(X, SQ_S0, h->stream, h->device, n, 1, nb, r, r, nullptr, nullptr));
    TRY(xdot_plan(X, SQ_V, h->stream, h->device, n, 1, nb, q, v, nullptr, nullptr));
    TRY(xdot_plan(X, SQ_T, h->stream, h->device, n, 2, nb, t, t, t, s));
    TRY(xdot_plan(X, SQ_E, h->stream, h->device, n, 1, nb, q, r, nullptr, nullptr));
    return MCR_OK;
}

// ---------------------------------------------------------------- sharded exchange points
// One reduction point of a row-sharded solve: every rank's SEND_SLOTS partials (written by
// the producing kernel's last CTA into st->send) are exchanged, then k_finalize<W> reduces them
// in rank order and takes the scalar step. `buf` != null also allgathers that full vector in
// the same step (Jacobi: the iterate just written).
template <int W>
int exchange_point(mcr_matrix* h, double* buf, int64_t* launches) {
    NvtxRange range(buf ? "mcr.exchange.allgather+slots" : "mcr.exchange.slots");
    Transport& T = *h->comm;
    const double* send = h->st->send;
    const int rc = buf ? T.allgather_and_slots(buf, (size_t)h->chunk, send, h->recv, SEND_SLOTS,
                                               h->stream)
                       : T.gather_slots(send, h->recv, SEND_SLOTS, h->stream);
    if (rc) return fail(MCR_CUDA_ERROR, std::string(T.kind()) + " exchange: " + T.err);
    launch_pdl(k_finalize<W>, 1, 32, 0, h->stream, h->st, (const double*)h->recv, h->world);
    ++*launches;
    TRY(launch_check());
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
    TRY(launch_check());
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

// Host batch sizing. Every batch ends in one state read (a host round trip that leaves the GPU
// idle until the next batch is enqueued), and a batch that overshoots the stop point launches
// kernels that return at their first instruction (a few microseconds each; sharded, exchanges
// that rewrite unchanged data). Batches start at 4 and double up to 32; once two reads have
// seen the convergence measure (st->last) decay, the next batch is sized to the predicted
// remaining count (geometric decay towards tol) plus `slack`, up to 512 (Jacobi; BiCGStab keeps
// doubling).
struct BatchPlan {
    int batch = 4;
    int slack = 0;
    long long it0 = -1;
    double m0 = 0.0;
    explicit BatchPlan(int slack_) : slack(slack_) {}
    int next(const SolveState& s) {
        int nb = std::min(batch * 2, 32);
        const double m = s.last;
        if (it0 >= 0 && s.it > it0 && m > s.tol && m < m0 && m0 > 0.0 && std::isfinite(m)) {
            const double rate = std::pow(m / m0, 1.0 / (double)(s.it - it0));
            if (rate > 0.0 && rate < 0.999) {
                const double rem = std::ceil(std::log(s.tol / m) / std::log(rate));
                if (rem >= 1.0 && rem < 100000.0) nb = std::max(1, std::min((int)rem + slack, 512));
            }
        }
        it0 = s.it;
        m0 = m;
        batch = nb;
        return nb;
    }
};

// ---------------------------------------------------------------- graph mode
constexpr int GRAPH_UNROLL_BICG = 4;    // iterations per while-body (1: 10.51, 2: 10.33, 4: 10.29 ms at C2)
// One GPU, BiCGStab: the iteration loop is a CUDA graph holding one while node whose body is
// `unroll` iterations, captured once per handle. The kernel that takes the stop decision sets
// the node's condition (graph_continue), so the loop ends on the device: no host round trips
// between batches, and at most unroll-1 sweeps / iterations of early-returning kernels. Kernel
// parameters are fixed per handle (vectors, state), which is what lets the graph be reused.
// Any failure to build it leaves the host-batched loop in use.
template <class Body>
int build_graph_loop(mcr_matrix* h, mcr_matrix::GraphLoop& G, int unroll, Body body) {
    TRY(launch_check());  // errors from before the capture are the caller's, not the capture's
    cudaGraph_t g = nullptr;
    cudaStream_t cs = nullptr;
    cudaStream_t saved = h->stream;
    bool ok = cudaGraphCreate(&g, 0) == cudaSuccess;
    cudaGraphConditionalHandle ch = 0;
    ok = ok && cudaGraphConditionalHandleCreate(&ch, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = ch;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node = nullptr;
    ok = ok && cudaGraphAddNode(&node, g, nullptr, 0, &np) == cudaSuccess;
    ok = ok && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess;
    if (ok) {
        cudaGraph_t bodyg = np.conditional.phGraph_out[0];
        ok = cudaStreamBeginCaptureToGraph(cs, bodyg, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            h->stream = cs;
            int64_t dummy = 0;
            for (int u = 0; u < unroll; ++u) body(&dummy);
            h->stream = saved;
            ok = cudaStreamEndCapture(cs, &bodyg) == cudaSuccess;
        }
    }
    cudaGraphExec_t exec = nullptr;
    ok = ok && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
    if (cs) cudaStreamDestroy(cs);
    g_launch_err = cudaSuccess;  // a failed capture attempt must not leave an error behind
    cudaGetLastError();
    if (!ok) {
        if (g) cudaGraphDestroy(g);
        G.failed = true;
        return MCR_OK;
    }
    G.graph = g;
    G.exec = exec;
    G.cond = (unsigned long long)ch;
    G.unroll = unroll;
    return MCR_OK;
}

bool graph_mode(const mcr_matrix* h) {
    return std::getenv("MCR_NO_GRAPH") == nullptr && !h->sharded() && h->small_grid == 0;
}

int jacobi_impl(mcr_matrix* h, const double* d_b, const double* d_x0, double tol, int64_t max_it,
                double* d_x_out, mcr_report* rep) {
    NvtxRange range(h->sharded() ? "mcr.jacobi.shard" : "mcr.jacobi");
    Trace tr;
    TRY(ensure_work(h));
    long long zero = -1;
    TRY(global_first_zero(h, &zero));
    if (zero >= 0) {
        rep->zero_diagonal_index = zero;
        return fail(MCR_ZERO_DIAGONAL, "zero diagonal entry in row " + std::to_string(zero));
    }
    TRY(ensure_offdiag(h));
    tr.mark("jacobi: off-diagonal ready");
    TRY(prepare_inputs(h, d_b, d_x0, V_X));
    Vecs V = base_vecs(h);
    set_state(h, tol, max_it);
    CK(cudaMemcpyAsync(h->st, h->h_st, sizeof(SolveState), cudaMemcpyHostToDevice, h->stream));
    CK(cudaEventRecord(h->ev0, h->stream));
    // (Jacobi stays host-batched: a graph while-loop measured 8.80 vs 8.70 ms per C2 solve
    // against the decay-sized batches below)
    int64_t launched = 0, sweeps = 0;
    BatchPlan plan(2);  // an extra sweep costs less than an extra round trip
    int batch = plan.batch;
    if (h->small_grid > 0) {
        CK(cudaMemsetAsync(h->maxslot, 0, 3 * sizeof(unsigned long long), h->stream));
        TRY(launch_small(h, 0, k_jacobi_small<true>, k_jacobi_small<false>, csr_off(h), V, h->st,
                         h->maxslot));
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
        TRY(launch_check());
        sweeps += k;
        TRY(read_state(h));
        if (h->h_st->stop || sweeps >= max_it) break;
        batch = plan.next(*h->h_st);
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
    tr.mark("jacobi: done");
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
    NvtxRange range(h->sharded() ? "mcr.bicgstab.shard" : "mcr.bicgstab");
    Trace tr;
    TRY(ensure_work(h));
    TRY(prepare_inputs(h, d_b, d_x0, V_X));
    Vecs V = base_vecs(h);
    const bool sh = h->sharded();
    double* p_full = h->vec(V_P);
    double* s_full = h->vec(V_S);
    // reference-order dots on one device: the E phase needs no q.r partials (MCR_NO_PH_EX=1: the
    // full phase anyway)
    static const bool ex_env = std::getenv("MCR_NO_PH_EX") == nullptr;
    const bool ex = ex_env && h->seqdots && !sh;
    // ... nor do the two SpMVs: plain y = M x stores into v and t (the tiled CSR kernel only:
    // the dense, staged and SELL kernels measured slower with the plain epilogue -- C3 BiCGStab
    // 4.2 -> 5.9 ms, C5 2-4%)
    const bool plain_mv = ex && h->storage != MCR_STORAGE_DENSE && !h->use_staged && !h->use_sell;
    Vecs Vv = V, Vt = V;
    Vv.y = V.v;
    Vt.y = V.t;
    auto mv_v = [&](int64_t* n) {  // v = M p (q.v -> a unless the dots are k_xdot's)
        if (plain_mv) launch_mv<EPI_Y>(h, false, p_full, Vv, n);
        else launch_mv<EPI_V>(h, false, p_full, V, n);
    };
    auto mv_t = [&](int64_t* n) {  // t = M s (t.t, t.s -> w unless the dots are k_xdot's)
        if (plain_mv) launch_mv<EPI_Y>(h, false, s_full, Vt, n);
        else launch_mv<EPI_T>(h, false, s_full, V, n);
    };
    auto body = [&](int64_t* n) {
        launch_phase<PH_A>(h, V, n);               // p = r + beta (p - w v)
        mv_v(n);                                   // v = M p, q.v -> a
        launch_seqdot<SQ_V>(h, V, n);
        launch_phase<PH_C>(h, V, n);               // s = r - a v, max|s|
        mv_t(n);                                   // t = M s, t.t, t.s -> w
        launch_seqdot<SQ_T>(h, V, n);
        if (ex) launch_phase<PH_EX>(h, V, n);      // x, r updates (q.r: the next launch)
        else launch_phase<PH_E>(h, V, n);          // x, r updates, q.r -> beta; loop condition
        launch_seqdot<SQ_E>(h, V, n);
    };
    // From the second BiCGStab solve of a handle the loop is the graph from the start. On the
    // first solve of a large system (the end-to-end path uploads a fresh matrix per step) the
    // graph is captured and instantiated on the host while the first host-issued batch runs on
    // the device, and takes over from the next iteration on; for small systems capture +
    // instantiation cost more than the batch hides, so they keep the host-batched loop.
    TRY(xdot_prepare(h, V));
    tr.mark("bicgstab: dot plans ready");
    // the captured body depends on the dot mode (and the block plan): rebuild when it changed
    const long long gkey = (long long)h->seqdots * 1000003ll + h->dot_blocks;
    if (h->gl_bicg.key != gkey) {
        if (h->gl_bicg.exec) cudaGraphExecDestroy(h->gl_bicg.exec);
        if (h->gl_bicg.graph) cudaGraphDestroy(h->gl_bicg.graph);
        h->gl_bicg = mcr_matrix::GraphLoop{};
        h->gl_bicg.key = gkey;
    }
    const bool gmode = graph_mode(h) && h->seqdots != MCR_DOTS_SERIAL && max_it >= 1;
    const bool first = h->bicg_solves++ == 0;
    const bool use_graph = gmode && !first;
    if (use_graph && !h->gl_bicg.exec && !h->gl_bicg.failed)
        TRY(build_graph_loop(h, h->gl_bicg, GRAPH_UNROLL_BICG, body));
    long long late_min_nnz = 2000000;  // C2 has 1e7
    if (const char* env = std::getenv("MCR_LATE_GRAPH_MIN_NNZ")) late_min_nnz = std::atoll(env);
    bool late_graph = gmode && first && !h->gl_bicg.exec && !h->gl_bicg.failed &&
                      (long long)h->nnz >= late_min_nnz;
    const bool graph = use_graph && h->gl_bicg.exec;
    set_state(h, tol, max_it);
    if (graph) h->h_st->cond = h->gl_bicg.cond;
    CK(cudaMemcpyAsync(h->st, h->h_st, sizeof(SolveState), cudaMemcpyHostToDevice, h->stream));
    CK(cudaEventRecord(h->ev0, h->stream));
    int64_t launched = 0, iters = 0;
    // max|s| does not decay geometrically (measured: predicted batches overshot by tens of
    // iterations), so BiCGStab keeps the doubling schedule
    int batch = 4;
    // reference-order dots on a small system: the XD variant (one CTA per tile sums each
    // product vector in order itself); the parallel-dot-products blocks take the general path
    const bool small_xd = h->small_xd && h->seqdots == 1 && h->dot_blocks <= 1;
    if (h->small_grid > 0 && (!h->seqdots || small_xd)) {
        CK(cudaMemsetAsync(h->maxslot, 0, 3 * sizeof(unsigned long long), h->stream));
        // four partial slots of nunits >= ntiles doubles each (grid variant)
        if (small_xd)
            TRY(launch_small(h, small_xd_smem(h->n), k_bicg_small<true, true>, k_bicg_small<false, true>,
                             csr_full(h), V, h->st, h->maxslot, h->P, h->nunits, h->xsprod));
        else
            TRY(launch_small(h, 0, k_bicg_small<true, false>, k_bicg_small<false, false>, csr_full(h), V,
                             h->st, h->maxslot, h->P, h->nunits, (double*)nullptr));
        ++launched;
        TRY(read_state(h));
        iters = max_it;  // the loop below has nothing left to do
    } else {
        // r = b - 1.0 * M x0, q = r, p = v = 0
        launch_mv<EPI_S0>(h, false, h->vec(V_X), V, &launched);
        if (sh && h->seqdots) {  // the whole r and q (= r) for the dots
            TRY(allgather_full(h, h->vec(V_R)));
            TRY(allgather_full(h, h->vec(V_Q)));
        }
        launch_seqdot<SQ_S0>(h, V, &launched);
        TRY(launch_check());
        if (sh) TRY(exchange_point<FIN_S0>(h, nullptr, &launched));
        if (graph) {  // the loop runs on the device; a solve stopped by S0 ends after one body
            CK(cudaGraphLaunch(h->gl_bicg.exec, h->stream));
            TRY(read_state(h));
            const int U = h->gl_bicg.unroll;
            launched += (h->seqdots ? 8 : 5) * ((h->h_st->it + U) / U * U);
            iters = max_it;
        } else {
            TRY(read_state(h));
        }
    }
    if (late_graph) batch = 8;  // enough device work to hide the capture
    while (!h->h_st->stop && iters < max_it) {
        const int k = (int)std::min<int64_t>(batch, max_it - iters);
        for (int i = 0; i < k; ++i) {
            launch_phase<PH_A>(h, V, &launched);               // p = r + beta (p - w v)
            if (sh) TRY(h->p2p ? p2p_barrier(h) : allgather_full(h, p_full));
            mv_v(&launched);                                   // v = M p, q.v -> a
            if (sh && h->seqdots) TRY(allgather_full(h, h->vec(V_V)));
            launch_seqdot<SQ_V>(h, V, &launched);
            if (sh) TRY(exchange_point<FIN_V>(h, nullptr, &launched));
            launch_phase<PH_C>(h, V, &launched);               // s = r - a v, max|s|
            if (sh) TRY(h->p2p ? p2p_barrier(h) : allgather_full(h, s_full));
            mv_t(&launched);                                   // t = M s, t.t, t.s -> w
            if (sh && h->seqdots) TRY(allgather_full(h, h->vec(V_T)));
            launch_seqdot<SQ_T>(h, V, &launched);
            if (sh) TRY(exchange_point<FIN_T>(h, nullptr, &launched));
            if (ex) launch_phase<PH_EX>(h, V, &launched);      // x, r updates
            else launch_phase<PH_E>(h, V, &launched);          // x, r updates, q.r -> beta
            if (sh && h->seqdots) TRY(allgather_full(h, h->vec(V_R)));
            launch_seqdot<SQ_E>(h, V, &launched);
            if (sh) TRY(exchange_point<FIN_E>(h, nullptr, &launched));
        }
        TRY(launch_check());
        iters += k;
        if (late_graph) {  // host work while the batch runs
            late_graph = false;
            tr.mark("bicgstab: first batch issued");
            TRY(build_graph_loop(h, h->gl_bicg, GRAPH_UNROLL_BICG, body));
            tr.mark("bicgstab: graph built");
            TRY(read_state(h));
            if (h->gl_bicg.exec && !h->h_st->stop && iters < max_it) {
                const long long it0 = h->h_st->it;
                h->h_st->cond = h->gl_bicg.cond;
                CK(cudaMemcpyAsync(&h->st->cond, &h->h_st->cond, sizeof(h->h_st->cond),
                                   cudaMemcpyHostToDevice, h->stream));
                CK(cudaGraphLaunch(h->gl_bicg.exec, h->stream));
                TRY(read_state(h));
                const int U = h->gl_bicg.unroll;
                launched += (h->seqdots ? 8 : 5) * ((h->h_st->it - it0 + U) / U * U);
                break;
            }
            batch = std::min(batch * 2, 32);
            continue;
        }
        TRY(read_state(h));
        batch = std::min(batch * 2, 32);
    }
    tr.mark("bicgstab: loop returned");
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
    tr.mark("bicgstab: done");
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
