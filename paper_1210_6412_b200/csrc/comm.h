// comm.h -- per-rank exchange of a row-sharded solve (host side of libmcr.so).
//
// A sharded solve needs two collectives: an in-place allgather of a vector
// whose rank-r block starts at buf + r*count (x for Jacobi, p and s for BiCGStab), and an
// allgather of every rank's SEND_SLOTS reduction partials. Both are stream-ordered: they are
// enqueued on the solve's stream between kernels, so a sweep never waits for the host.
//
//   NcclTransport   one process (or thread) per GPU; NCCL 2.27+/2.28 loaded with dlopen at
//                   communicator creation, so libmcr.so itself has no link-time NCCL
//                   dependency. The allgather and the scalar exchange of one Jacobi sweep go
//                   out as one NCCL group.
//   LocalTransport  `world` ranks driven by `world` host threads of one process, on one or
//                   several devices: the same collectives as device-to-device copies ordered
//                   by CUDA events and two host barriers per collective. Used to run the
//                   multi-rank code path, unchanged, on a single GPU.
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace mcr {

struct Transport {
    int world = 1;
    int rank = 0;
    int device = 0;
    std::string err;
    virtual ~Transport() {}
    // In place: rank r's `count` doubles at buf + r*count are broadcast to every rank.
    virtual int allgather(double* buf, size_t count, cudaStream_t s) = 0;
    // send[SEND_SLOTS] of every rank -> recv[world * SEND_SLOTS] (rank order).
    virtual int gather_slots(const double* send, double* recv, int slots, cudaStream_t s) = 0;
    // Both in one step (one NCCL group).
    virtual int allgather_and_slots(double* buf, size_t count, const double* send, double* recv,
                                    int slots, cudaStream_t s) {
        int rc = allgather(buf, count, s);
        return rc ? rc : gather_slots(send, recv, slots, s);
    }
    virtual const char* kind() const = 0;
    // Host-level allgather of `bytes` per rank (setup only: peer mappings).
    virtual int share_bytes(const void* mine, void* all, size_t bytes) = 0;
    // Ranks live in this process (peer buffers are plain device pointers, no IPC).
    virtual bool same_process() const = 0;
};

// ------------------------------------------------------------------------------- NCCL
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string load_error;

    static NcclApi& instance() {
        static std::once_flag once;
        static NcclApi api;
        std::call_once(once, [] { api.load(); });
        return api;
    }
    // nullptr (and error() says why) when no usable NCCL can be loaded.
    static NcclApi* get() { return instance().GetUniqueId ? &instance() : nullptr; }
    static std::string error() { return instance().load_error; }

   private:
    void load() {
        // Prefer an NCCL already loaded into the process (torch's), else the system one.
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            load_error = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
#define MCR_SYM(field, name)                                                 \
    field = reinterpret_cast<decltype(field)>(dlsym(h, name));               \
    if (!field) {                                                            \
        load_error = std::string("libnccl.so.2 lacks ") + name;              \
        GetUniqueId = nullptr;                                               \
        return;                                                              \
    }
        MCR_SYM(CommInitRank, "ncclCommInitRank");
        MCR_SYM(CommDestroy, "ncclCommDestroy");
        MCR_SYM(AllGather, "ncclAllGather");
        MCR_SYM(GroupStart, "ncclGroupStart");
        MCR_SYM(GroupEnd, "ncclGroupEnd");
        MCR_SYM(GetErrorString, "ncclGetErrorString");
        MCR_SYM(GetUniqueId, "ncclGetUniqueId");
#undef MCR_SYM
    }
};

struct NcclTransport : Transport {
    NcclApi* api = nullptr;
    ncclComm_t comm = nullptr;
    ~NcclTransport() override {
        if (comm && api) api->CommDestroy(comm);
    }
    int check(ncclResult_t r, const char* what) {
        if (r == ncclSuccess) return 0;
        err = std::string(what) + ": " + api->GetErrorString(r);
        return 1;
    }
    int allgather(double* buf, size_t count, cudaStream_t s) override {
        return check(api->AllGather(buf + (size_t)rank * count, buf, count, ncclFloat64, comm, s),
                     "ncclAllGather");
    }
    int gather_slots(const double* send, double* recv, int slots, cudaStream_t s) override {
        return check(api->AllGather(send, recv, (size_t)slots, ncclFloat64, comm, s),
                     "ncclAllGather(slots)");
    }
    int allgather_and_slots(double* buf, size_t count, const double* send, double* recv,
                            int slots, cudaStream_t s) override {
        if (check(api->GroupStart(), "ncclGroupStart")) return 1;
        int rc = check(api->AllGather(buf + (size_t)rank * count, buf, count, ncclFloat64, comm, s),
                       "ncclAllGather");
        if (!rc)
            rc = check(api->AllGather(send, recv, (size_t)slots, ncclFloat64, comm, s),
                       "ncclAllGather(slots)");
        const int rc2 = check(api->GroupEnd(), "ncclGroupEnd");
        return rc ? rc : rc2;
    }
    const char* kind() const override { return "nccl"; }
    int share_bytes(const void* mine, void* all, size_t bytes) override {
        char* d = nullptr;
        cudaStream_t s = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaMalloc(&d, bytes * (size_t)(world + 1)) != cudaSuccess) {
            err = "share_bytes: allocation failed";
            if (s) cudaStreamDestroy(s);
            return 1;
        }
        int rc = 0;
        if (cudaMemcpyAsync(d + bytes * (size_t)world, mine, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
            rc = 1;
        if (!rc) rc = check(api->AllGather(d + bytes * (size_t)world, d, bytes, ncclUint8, comm, s),
                            "ncclAllGather(bytes)");
        if (!rc && (cudaMemcpyAsync(all, d, bytes * (size_t)world, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                    cudaStreamSynchronize(s) != cudaSuccess)) {
            err = "share_bytes: copy failed";
            rc = 1;
        }
        cudaFree(d);
        cudaStreamDestroy(s);
        return rc;
    }
    bool same_process() const override { return false; }
};

// ------------------------------------------------------------------------------- local
struct LocalGroup {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long generation = 0;
    bool broken = false;
    std::vector<const double*> src;   // per-rank source pointer of the current collective
    std::vector<int> dev;
    std::vector<cudaEvent_t> ready, done;
    std::vector<char> shared;                 // share_bytes staging (host)

    // Returns false if a rank gave up (timeout / error): every waiter then fails too.
    bool barrier(double timeout_s = 120.0) {
        std::unique_lock<std::mutex> lk(mu);
        if (broken) return false;
        const long long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
            return true;
        }
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                    [&] { return generation != gen || broken; });
        if (!ok || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
    ~LocalGroup() {
        for (auto e : ready)
            if (e) cudaEventDestroy(e);
        for (auto e : done)
            if (e) cudaEventDestroy(e);
    }
};

struct LocalTransport : Transport {
    std::shared_ptr<LocalGroup> g;

    int fail_msg(const std::string& m) {
        err = m;
        std::lock_guard<std::mutex> lk(g->mu);
        g->broken = true;
        g->cv.notify_all();
        return 1;
    }
    // Every rank publishes `mine`, then copies block q of each peer q (q != rank, or all q
    // for the slot exchange) into its own buffer after the peer's producer finished; a second
    // barrier keeps every source alive until all copies are ordered after it.
    int exchange(const double* mine, double* dst, size_t block, bool include_self,
                 bool src_is_block_base, cudaStream_t s) {
        g->src[(size_t)rank] = mine;
        if (cudaEventRecord(g->ready[(size_t)rank], s) != cudaSuccess) return fail_msg("event record");
        if (!g->barrier()) return fail_msg("local group barrier timed out or a rank failed");
        for (int q = 0; q < world; ++q) {
            if (q == rank && !include_self) continue;
            if (cudaStreamWaitEvent(s, g->ready[(size_t)q], 0) != cudaSuccess) return fail_msg("wait");
            const double* from = g->src[(size_t)q] + (src_is_block_base ? 0 : (size_t)q * block);
            cudaError_t e = cudaMemcpyPeerAsync(dst + (size_t)q * block, device, from,
                                                g->dev[(size_t)q], block * sizeof(double), s);
            if (e != cudaSuccess) return fail_msg(std::string("peer copy: ") + cudaGetErrorString(e));
        }
        if (cudaEventRecord(g->done[(size_t)rank], s) != cudaSuccess) return fail_msg("event record");
        if (!g->barrier()) return fail_msg("local group barrier timed out or a rank failed");
        // (a peer re-records done[] only after the next collective's first barrier, which
        // this rank reaches after these waits are enqueued)
        for (int q = 0; q < world; ++q)
            if (q != rank && cudaStreamWaitEvent(s, g->done[(size_t)q], 0) != cudaSuccess)
                return fail_msg("wait");
        return 0;
    }
    int allgather(double* buf, size_t count, cudaStream_t s) override {
        return exchange(buf, buf, count, false, false, s);
    }
    int gather_slots(const double* send, double* recv, int slots, cudaStream_t s) override {
        return exchange(send, recv, (size_t)slots, true, true, s);
    }
    const char* kind() const override { return "local"; }
    int share_bytes(const void* mine, void* all, size_t bytes) override {
        {
            std::lock_guard<std::mutex> lk(g->mu);
            if (g->shared.size() < bytes * (size_t)world) g->shared.resize(bytes * (size_t)world);
            std::memcpy(g->shared.data() + bytes * (size_t)rank, mine, bytes);
        }
        if (!g->barrier()) return fail_msg("local group barrier timed out or a rank failed");
        {
            std::lock_guard<std::mutex> lk(g->mu);
            std::memcpy(all, g->shared.data(), bytes * (size_t)world);
        }
        if (!g->barrier()) return fail_msg("local group barrier timed out or a rank failed");
        return 0;
    }
    bool same_process() const override { return true; }
};

}  // namespace mcr
