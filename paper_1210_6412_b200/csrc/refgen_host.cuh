// refgen_host.cuh -- host orchestration of the reference-stream generator (refgen.cuh): the
// draws of `_sample_off_diagonal`, `generate_dd_matrix` and `generate_rhs`
// (S/generator.py:77-132) in the reference's stream order, then the CSR. Part of mcr.cu.
#pragma once

#include "refgen.cuh"

namespace {

struct RgStream {  // where numpy's stream stands: raw 64-bit outputs or 32-bit halves consumed
    rg::u128 s, inc;
    unsigned long long half = 0;  // half-draw index (2 * raw outputs consumed, + 1 if a high half is pending)
};

struct RgMem {  // stream-ordered allocations freed in one place
    cudaStream_t st;
    std::vector<void*> p;
    template <class T>
    int get(T** out, size_t count) {
        *out = nullptr;
        if (cudaMallocAsync((void**)out, std::max<size_t>(count, 1) * sizeof(T), st) != cudaSuccess)
            return fail(MCR_CUDA_ERROR, "refgen: device allocation failed");
        p.push_back(*out);
        return MCR_OK;
    }
    void drop(void* q) {
        for (auto& x : p)
            if (x == q) {
                cudaFreeAsync(x, st);
                x = nullptr;
            }
    }
    ~RgMem() {
        for (void* q : p)
            if (q) cudaFreeAsync(q, st);
    }
};

inline int rg_grid(long long items) {
    return (int)std::max<long long>(1, std::min<long long>((items + 255) / 256, 1 << 20));
}

// Output capacity rg_draw needs for `need` draws (the compaction writes every accepted draw of
// its batch, a little more than needed).
inline long long rg_cap(long long need) { return need + need / 64 + 4096; }

// `need` accepted bounded draws of range size `re` (values offset by `lo`) continuing the stream
// at S: 64-bit Lemire on raw outputs when re - 1 > 2^32 - 1, else 32-bit Lemire on halves.
// Writes the values (as uint64 codes, or as doubles when `dout`; rg_cap(need) capacity) and
// advances S.
int rg_draw(cudaStream_t st, RgStream& S, uint64_t re, long long lo, long long need, uint64_t* uout,
            double* dout) {
    if (need <= 0) return MCR_OK;
    RgMem mem{st, {}};
    const bool wide = re - 1 > 0xFFFFFFFFull;
    if (wide && (S.half & 1ull)) return fail(MCR_INVALID_ARGUMENT, "refgen: 64-bit draw after an odd 32-bit one");
    long long got = 0;
    while (got < need) {
        const long long want = need - got;
        const long long cnt = rg_cap(want);  // rejections are rare (< re / 2^bits)
        unsigned char *ok = nullptr, *rej = nullptr;
        TRY(mem.get(&ok, (size_t)cnt));
        uint64_t* uv = nullptr;
        double* dv = nullptr;
        const int grid = rg_grid((cnt + rg::RAW_PER_THREAD - 1) / rg::RAW_PER_THREAD);
        if (wide) {
            TRY(mem.get(&uv, (size_t)cnt));
            const uint64_t th = (uint64_t)((((rg::u128)1 << 64) - re) % re);
            rg::k_lemire64<<<grid, 256, 0, st>>>((uint64_t)(S.s >> 64), (uint64_t)S.s, (uint64_t)(S.inc >> 64),
                                                 (uint64_t)S.inc, S.half >> 1, cnt, re, th, uv, ok);
        } else {
            TRY(mem.get(&dv, (size_t)cnt));
            const uint32_t re32 = (uint32_t)re, th = re32 ? (uint32_t)((0x100000000ull - re) % re) : 0u;
            rg::k_lemire32<<<grid, 256, 0, st>>>((uint64_t)(S.s >> 64), (uint64_t)S.s, (uint64_t)(S.inc >> 64),
                                                 (uint64_t)S.inc, S.half, cnt, re32, th, 0.0, dv, ok);
        }
        CK(cudaGetLastError());
        // the accepted draws in stream order, and the rejected positions (few)
        long long *nsel = nullptr, *nrej = nullptr, *rpos = nullptr;
        TRY(mem.get(&nsel, 1));
        TRY(mem.get(&nrej, 1));
        TRY(mem.get(&rej, (size_t)cnt));
        rg::k_not<<<rg_grid(cnt), 256, 0, st>>>(ok, cnt, rej);
        // how many were rejected (sized before the positions are listed)
        thrust::transform_iterator<rg::ToLL, const unsigned char*> rej_ll(rej, rg::ToLL());
        size_t tmp = 0;
        CK(cub::DeviceReduce::Sum(nullptr, tmp, rej_ll, nrej, cnt, st));
        void* dtmp = nullptr;
        TRY(mem.get((unsigned char**)&dtmp, tmp));
        CK(cub::DeviceReduce::Sum(dtmp, tmp, rej_ll, nrej, cnt, st));
        long long h_nrej = 0;
        CK(cudaMemcpyAsync(&h_nrej, nrej, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        TRY(mem.get(&rpos, (size_t)h_nrej));
        thrust::counting_iterator<long long> iota(0);
        tmp = 0;
        CK(cub::DeviceSelect::Flagged(nullptr, tmp, iota, rej, rpos, nrej, cnt, st));
        TRY(mem.get((unsigned char**)&dtmp, tmp));
        CK(cub::DeviceSelect::Flagged(dtmp, tmp, iota, rej, rpos, nrej, cnt, st));
        const long long acc = cnt - h_nrej, take = std::min(acc, want);
        // stream position after the take-th accepted draw: take + rejections before it
        std::vector<long long> rp((size_t)h_nrej);
        if (h_nrej) CK(cudaMemcpyAsync(rp.data(), rpos, sizeof(long long) * (size_t)h_nrej, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        long long used = take;
        for (long long r : rp)
            if (r < used) ++used;
            else break;
        // compaction of the accepted values (in stream order), the first `take` to the output
        size_t tmp2 = 0;
        if (wide) CK(cub::DeviceSelect::Flagged(nullptr, tmp2, uv, ok, uv, nsel, cnt, st));
        else CK(cub::DeviceSelect::Flagged(nullptr, tmp2, dv, ok, dv, nsel, cnt, st));
        void* dtmp2 = nullptr;
        TRY(mem.get((unsigned char**)&dtmp2, tmp2));
        // (outputs hold rg_cap(need) >= got + cnt entries: the compaction writes all accepted)
        if (wide) {
            CK(cub::DeviceSelect::Flagged(dtmp2, tmp2, uv, ok, uout + got, nsel, cnt, st));
        } else if (dout) {
            CK(cub::DeviceSelect::Flagged(dtmp2, tmp2, dv, ok, dout + got, nsel, cnt, st));
        } else {
            double* sel = nullptr;
            TRY(mem.get(&sel, (size_t)acc));
            CK(cub::DeviceSelect::Flagged(dtmp2, tmp2, dv, ok, sel, nsel, cnt, st));
            {  // codes of the 32-bit path: doubles holding integers < 2^32
                rg::k_d2u<<<rg_grid(take), 256, 0, st>>>(sel, take, uout + got);
                CK(cudaGetLastError());
            }
        }
        CK(cudaStreamSynchronize(st));
        S.half += wide ? 2ull * (unsigned long long)used : (unsigned long long)used;
        got += take;
    }
    if (lo != 0 && dout) {
        rg::k_add<<<rg_grid(need), 256, 0, st>>>(dout, need, (double)lo);
        CK(cudaGetLastError());
    }
    return MCR_OK;
}

// _sample_off_diagonal (S/generator.py:77-97): `count` distinct codes in [0, total), the
// first occurrences in draw order of batches of max(1024, 2 * missing) draws.
int rg_codes(cudaStream_t st, RgStream& S, long long total, long long count, uint64_t* chosen) {
    if (count <= 0) return MCR_OK;
    if (count == total) {  // np.arange(total): no draws
        rg::k_iota64<<<rg_grid(count), 256, 0, st>>>(chosen, count);
        CK(cudaGetLastError());
        return MCR_OK;
    }
    RgMem mem{st, {}};
    std::vector<uint64_t*> batches;
    std::vector<long long> sizes;
    long long have = 0, drawn = 0;
    int bits = 1;
    while (bits < 64 && ((unsigned long long)(total - 1) >> bits)) ++bits;
    for (;;) {
        const long long b = std::max<long long>(1024, 2 * (count - have));
        uint64_t* codes = nullptr;
        TRY(mem.get(&codes, (size_t)(drawn + rg_cap(b))));
        long long off = 0;
        for (size_t i = 0; i < batches.size(); ++i) {  // the earlier batches, in draw order
            CK(cudaMemcpyAsync(codes + off, batches[i], sizeof(uint64_t) * (size_t)sizes[i], cudaMemcpyDeviceToDevice, st));
            off += sizes[i];
        }
        for (uint64_t* q : batches) mem.drop(q);
        batches.assign(1, codes);
        TRY(rg_draw(st, S, (uint64_t)total, 0, b, codes + drawn, nullptr));
        drawn += b;
        sizes.assign(1, drawn);
        if (drawn >= (1ll << 32)) return fail(MCR_INVALID_ARGUMENT, "refgen: more than 2^32 code draws");
        // first occurrences: a stable sort by code carries each draw's position
        uint64_t* keys = nullptr;
        uint32_t *pos = nullptr, *pos2 = nullptr;
        unsigned char* first = nullptr;
        TRY(mem.get(&keys, (size_t)drawn));
        TRY(mem.get(&pos, (size_t)drawn));
        TRY(mem.get(&pos2, (size_t)drawn));
        rg::k_iota32<<<rg_grid(drawn), 256, 0, st>>>(pos, drawn);
        size_t tmp = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, codes, keys, pos, pos2, drawn, 0, bits, st));
        unsigned char* dtmp = nullptr;
        TRY(mem.get(&dtmp, tmp));
        CK(cub::DeviceRadixSort::SortPairs(dtmp, tmp, codes, keys, pos, pos2, drawn, 0, bits, st));
        mem.drop(dtmp);
        mem.drop(pos);
        TRY(mem.get(&first, (size_t)drawn));
        rg::k_first<<<rg_grid(drawn), 256, 0, st>>>(keys, pos2, drawn, first);
        CK(cudaGetLastError());
        mem.drop(keys);
        mem.drop(pos2);
        uint64_t* dist = nullptr;
        long long* nsel = nullptr;
        TRY(mem.get(&dist, (size_t)drawn));
        TRY(mem.get(&nsel, 1));
        tmp = 0;
        CK(cub::DeviceSelect::Flagged(nullptr, tmp, codes, first, dist, nsel, drawn, st));
        TRY(mem.get(&dtmp, tmp));
        CK(cub::DeviceSelect::Flagged(dtmp, tmp, codes, first, dist, nsel, drawn, st));
        long long d = 0;
        CK(cudaMemcpyAsync(&d, nsel, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (d >= count) {
            CK(cudaMemcpyAsync(chosen, dist, sizeof(uint64_t) * (size_t)count, cudaMemcpyDeviceToDevice, st));
            CK(cudaStreamSynchronize(st));
            return MCR_OK;
        }
        have = d;  // the reference appended every distinct code of the batch
        mem.drop(dist);
        mem.drop(first);
        mem.drop(dtmp);
    }
}

// generate_dd_matrix (S/generator.py:100-124) into device CSR arrays (rp[n+1], col[nnz],
// val[nnz]; nnz = count + n), allocated here (freed by the caller).
int rg_matrix(cudaStream_t st, RgStream& S, long long n, long long count, long long lo, long long hi,
              long long** rp_out, int** col_out, double** val_out) {
    const long long total = n * (n - 1), nnz = count + n;
    RgMem mem{st, {}};
    uint64_t* codes = nullptr;
    double *vals = nullptr, *slack = nullptr;
    TRY(mem.get(&codes, (size_t)rg_cap(count)));
    TRY(mem.get(&vals, (size_t)rg_cap(count)));
    TRY(mem.get(&slack, (size_t)rg_cap(n)));
    TRY(rg_codes(st, S, total, count, codes));                                   // :110
    TRY(rg_draw(st, S, (uint64_t)(hi - lo + 1), lo, count, nullptr, vals));      // :115
    TRY(rg_draw(st, S, (uint64_t)hi, 1, n, nullptr, slack));                     // :117
    // CSR order: off-diagonal codes sorted (row-major; columns ascend with the offset)
    uint64_t* scode = nullptr;
    double* sval = nullptr;
    TRY(mem.get(&scode, (size_t)count));
    TRY(mem.get(&sval, (size_t)count));
    int bits = 1;
    while (bits < 64 && ((unsigned long long)std::max<long long>(total - 1, 1) >> bits)) ++bits;
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, codes, scode, vals, sval, count, 0, bits, st));
    unsigned char* dtmp = nullptr;
    TRY(mem.get(&dtmp, tmp));
    if (count > 0) CK(cub::DeviceRadixSort::SortPairs(dtmp, tmp, codes, scode, vals, sval, count, 0, bits, st));
    mem.drop(dtmp);
    mem.drop(codes);
    mem.drop(vals);
    int *cnt_off = nullptr, *cnt_lt = nullptr;
    double* rowsum = nullptr;
    long long *offx = nullptr, *rp = nullptr;
    TRY(mem.get(&cnt_off, (size_t)n + 1));
    TRY(mem.get(&cnt_lt, (size_t)n));
    TRY(mem.get(&rowsum, (size_t)n));
    TRY(mem.get(&offx, (size_t)n + 1));
    CK(cudaMemsetAsync(cnt_off, 0, sizeof(int) * ((size_t)n + 1), st));
    CK(cudaMemsetAsync(cnt_lt, 0, sizeof(int) * (size_t)n, st));
    CK(cudaMemsetAsync(rowsum, 0, sizeof(double) * (size_t)n, st));
    if (count > 0) rg::k_rows<<<rg_grid(count), 256, 0, st>>>(scode, count, n - 1, cnt_off, cnt_lt, rowsum, sval);
    CK(cudaGetLastError());
    tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt_off, offx, n + 1, st));
    TRY(mem.get(&dtmp, tmp));
    CK(cub::DeviceScan::ExclusiveSum(dtmp, tmp, cnt_off, offx, n + 1, st));
    int* col = nullptr;
    double* val = nullptr;
    CK(cudaMallocAsync((void**)&rp, sizeof(long long) * ((size_t)n + 1), st));
    CK(cudaMallocAsync((void**)&col, sizeof(int) * (size_t)std::max<long long>(nnz, 1), st));
    CK(cudaMallocAsync((void**)&val, sizeof(double) * (size_t)std::max<long long>(nnz, 1), st));
    *rp_out = rp; *col_out = col; *val_out = val;
    rg::k_rowptr<<<rg_grid(n + 1), 256, 0, st>>>(offx, n, rp);
    if (count > 0) rg::k_scatter<<<rg_grid(count), 256, 0, st>>>(scode, sval, count, n - 1, offx, rp, col, val);
    rg::k_diag<<<rg_grid(n), 256, 0, st>>>(n, rp, cnt_lt, rowsum, slack, col, val);        // :116-118
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return MCR_OK;
}

}  // namespace
