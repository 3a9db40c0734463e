// Communicators for row-sharded solves: exactly the natural
// reductions of the algorithm -- allreduce of the partial sketch and of the
// n x b Gram product, allgather of the per-rank TSQR R factors, broadcast of
// the preconditioner -- and nothing on the data path of A.
//
//   NcclComm  NCCL over NVLink/NVSwitch, resolved with dlopen so the library
//             shares whatever libnccl.so.2 the host process (torch) loaded.
//   FakeComm  several host threads driving one GPU, one context each; the
//             host mediates every collective (stream sync + barrier + a
//             fixed-order device reduction), so no kernel ever waits on
//             another rank.  Used to test the sharded path on one GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "msvd_internal.h"

namespace msvd {

namespace {

struct NoComm final : Comm {
    int nranks() const override { return 1; }
    int rank() const override { return 0; }
    void allreduce_sum(double*, size_t, cudaStream_t) override {}
    void allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
        if (send != recv) MSVD_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
    }
    void bcast(double*, size_t, int, cudaStream_t) override {}
    void allreduce_max(double*, size_t, cudaStream_t) override {}
};

// ---- NCCL through dlopen ---------------------------------------------------
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) api.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) return;
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.h, "ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.h, "ncclAllReduce"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.h, "ncclAllGather"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(api.h, "ncclBroadcast"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    });
    if (!api.h || !api.CommInitRank) fail(MSVD_ERR_COMM, "msvd: libnccl.so.2 could not be loaded");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(MSVD_ERR_COMM, std::string("NCCL ") + what + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    int n = 1, r = 0;
    NcclComm(const msvd_ctx_desc& d) : n(d.nranks), r(d.rank) {
        ncclUniqueId id;
        static_assert(sizeof(id.internal) == 128, "nccl unique id size");
        std::memcpy(id.internal, d.nccl_id, 128);
        nccl_check(nccl().CommInitRank(&comm, n, id, r), "CommInitRank");
    }
    ~NcclComm() override {
        if (comm) nccl().CommDestroy(comm);
    }
    int nranks() const override { return n; }
    int rank() const override { return r; }
    void allreduce_sum(double* d, size_t count, cudaStream_t s) override {
        nccl_check(nccl().AllReduce(d, d, count, ncclFloat64, ncclSum, comm, s), "AllReduce");
    }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
        nccl_check(nccl().AllGather(send, recv, count, ncclFloat64, comm, s), "AllGather");
    }
    void bcast(double* d, size_t count, int root, cudaStream_t s) override {
        nccl_check(nccl().Broadcast(d, d, count, ncclFloat64, root, comm, s), "Broadcast");
    }
    void allreduce_max(double* d, size_t count, cudaStream_t s) override {
        nccl_check(nccl().AllReduce(d, d, count, ncclFloat64, ncclMax, comm, s), "AllReduce(max)");
    }
};

// ---- in-process fake group ------------------------------------------------
__global__ void fixed_order_reduce(const double* const* src, int nr, size_t count, int op, double* out) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double s = src[0][i];
        for (int r = 1; r < nr; ++r) s = op == 0 ? s + src[r][i] : fmax(s, src[r][i]);
        out[i] = s;
    }
}

}  // namespace

struct FakeGroup {
    int n;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<const double*> ptrs;
    double* buf = nullptr;
    size_t buf_count = 0;
    const double** dptrs = nullptr;
    explicit FakeGroup(int nr) : n(nr), ptrs(nr, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
    void ensure(size_t count) {  // called by rank 0 only, between barriers
        if (count > buf_count) {
            if (buf) cudaFree(buf);
            MSVD_CUDA(cudaMalloc(&buf, sizeof(double) * count));
            buf_count = count;
        }
        if (!dptrs) MSVD_CUDA(cudaMalloc(&dptrs, sizeof(double*) * n));
    }
};

namespace {

struct FakeComm final : Comm {
    FakeGroup* g;
    int r;
    FakeComm(FakeGroup* grp, int rank) : g(grp), r(rank) {}
    int nranks() const override { return g->n; }
    int rank() const override { return r; }
    void reduce(double* d, size_t count, cudaStream_t s, int op) {
        MSVD_CUDA(cudaStreamSynchronize(s));
        g->ptrs[r] = d;
        g->barrier();
        if (r == 0) {
            g->ensure(count);
            MSVD_CUDA(cudaMemcpyAsync(g->dptrs, g->ptrs.data(), sizeof(double*) * g->n, cudaMemcpyHostToDevice, s));
            fixed_order_reduce<<<256, 256, 0, s>>>(g->dptrs, g->n, count, op, g->buf);
            MSVD_CUDA(cudaStreamSynchronize(s));
        }
        g->barrier();
        MSVD_CUDA(cudaMemcpyAsync(d, g->buf, sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
        MSVD_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
    void allreduce_sum(double* d, size_t count, cudaStream_t s) override { reduce(d, count, s, 0); }
    void allreduce_max(double* d, size_t count, cudaStream_t s) override { reduce(d, count, s, 1); }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t s) override {
        MSVD_CUDA(cudaStreamSynchronize(s));
        g->ptrs[r] = send;
        g->barrier();
        for (int q = 0; q < g->n; ++q)
            MSVD_CUDA(cudaMemcpyAsync(recv + q * count, g->ptrs[q], sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
        MSVD_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
    void bcast(double* d, size_t count, int root, cudaStream_t s) override {
        MSVD_CUDA(cudaStreamSynchronize(s));
        g->ptrs[r] = d;
        g->barrier();
        if (r != root)
            MSVD_CUDA(cudaMemcpyAsync(d, g->ptrs[root], sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
        MSVD_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
};

}  // namespace

Comm* make_comm(const msvd_ctx_desc& desc, cudaStream_t) {
    if (desc.comm_kind == 0) return new NoComm();
    if (desc.nranks < 1 || desc.rank < 0 || desc.rank >= desc.nranks)
        fail(MSVD_ERR_INVALID, "msvd: rank outside [0, nranks)");
    if (desc.comm_kind == 1) return new NcclComm(desc);
    if (desc.comm_kind == 2) {
        if (!desc.fake_group) fail(MSVD_ERR_INVALID, "msvd: fake communicator needs a group");
        FakeGroup* g = static_cast<FakeGroup*>(desc.fake_group);
        if (g->n != desc.nranks) fail(MSVD_ERR_INVALID, "msvd: fake group size does not match nranks");
        return new FakeComm(g, desc.rank);
    }
    fail(MSVD_ERR_INVALID, "msvd: unknown communicator kind");
}

void* fake_group_create(int n) { return new FakeGroup(n); }
void fake_group_destroy(void* p) {
    FakeGroup* g = static_cast<FakeGroup*>(p);
    if (g->buf) cudaFree(g->buf);
    if (g->dptrs) cudaFree(g->dptrs);
    delete g;
}

int nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "GetUniqueId");
    std::memcpy(out, id.internal, 128);
    return 0;
}

}  // namespace msvd
