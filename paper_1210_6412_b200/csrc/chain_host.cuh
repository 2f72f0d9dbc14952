// chain_host.cuh -- host orchestration of the chain -> reduced system build (chain.cuh kernels).
#pragma once

// ---------------------------------------------------------------- chains (build_system)

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
    NvtxRange range("mcr.chain.build_system");
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

