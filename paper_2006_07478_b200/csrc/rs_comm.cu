// rs_comm.cu — multi-GPU plumbing of the C ABI (include/rs.h).
//
// Regions are independent contexts (§1): a stream partitioned by whole
// regions needs no exchange while it is processed, and the per-region
// aggregates are assembled on one rank at their global region offsets.  Two
// ways are provided:
//   * rs_gather_aggregates: one grouped NCCL exchange, every rank's slice sent
//     to the root at its exact offset (ncclSend / ncclRecv, no padding);
//   * rs_ipc_export / rs_ipc_open: the root's output buffer mapped into the
//     other ranks' address space (CUDA IPC, NVLink peer memory), so each
//     rank's pipeline kernels store their aggregates straight into the root's
//     buffer while they run -- the gather is fused into the aggregate node's
//     stores and overlaps the compute completely.
// NCCL is the one torch has loaded (dlopen with RTLD_NOLOAD first), so the
// library does not link a second copy; RS_ERR_NCCL when none can be found.
#define RS_HOST_ONLY
#include "rs_kern.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

using namespace rsk;

namespace {

rs_status cfail(rs_status s, const std::string &m) {
    set_last_error(m);
    return s;
}

struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
    bool ok = false;
};

NcclApi *nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy, if loaded
        if (!h) {
            const char *env = getenv("RS_NCCL_LIB");
            if (env) h = dlopen(env, RTLD_NOW);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) return;
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
        api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
        api.send = (decltype(api.send))dlsym(h, "ncclSend");
        api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
        api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
        api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
        api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
        api.errStr = (decltype(api.errStr))dlsym(h, "ncclGetErrorString");
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv && api.groupStart &&
                 api.groupEnd && api.allReduce && api.errStr;
    });
    return api.ok ? &api : nullptr;
}

rs_status nccl_fail(NcclApi *n, ncclResult_t r, const char *what) {
    return cfail(RS_ERR_NCCL, std::string(what) + ": " + (n ? n->errStr(r) : "NCCL unavailable"));
}

// aggregate op -> bytes per region of v0 / v1 (rs.h rs_op)
bool agg_bytes(int32_t op, int *b0, int *b1) {
    switch (op) {
        case RS_OP_SUM_I64: *b0 = 8; *b1 = 0; return true;
        case RS_OP_SUM_F32: *b0 = 4; *b1 = 0; return true;
        case RS_OP_COUNT_MIN_U32: *b0 = 4; *b1 = 4; return true;
        case RS_OP_COUNT_XOR64: *b0 = 8; *b1 = 8; return true;
    }
    return false;
}

}  // namespace

struct rs_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    int *d_word = nullptr;          // rs_comm_barrier's all-reduce word
};

extern "C" {

rs_status rs_comm_unique_id(void *id128) {
    if (!id128) return cfail(RS_ERR_INVALID_ARG, "id128 is NULL");
    NcclApi *n = nccl();
    if (!n) return cfail(RS_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    ncclResult_t r = n->getUniqueId(&id);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof id);
    return RS_OK;
}

rs_status rs_comm_init(const void *id128, int rank, int world, rs_comm **out) {
    if (!id128 || !out) return cfail(RS_ERR_INVALID_ARG, "NULL argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return cfail(RS_ERR_INVALID_ARG, "bad rank / world");
    NcclApi *n = nccl();
    if (!n) return cfail(RS_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    rs_comm *c = new rs_comm();
    c->rank = rank;
    c->world = world;
    ncclResult_t r = n->commInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(n, r, "ncclCommInitRank");
    }
    if (cudaMalloc(&c->d_word, sizeof(int)) != cudaSuccess) {
        n->commDestroy(c->comm);
        delete c;
        return cfail(RS_ERR_CUDA, "cudaMalloc failed");
    }
    *out = c;
    return RS_OK;
}

rs_status rs_gather_aggregates(rs_comm *c, int32_t agg_op, rs_aggregates local, int64_t local_regions,
                               const int64_t *region_base, rs_aggregates root_out, int root, rs_stream stream_) {
    if (!c || !region_base) return cfail(RS_ERR_INVALID_ARG, "NULL argument");
    int b0 = 0, b1 = 0;
    if (!agg_bytes(agg_op, &b0, &b1)) return cfail(RS_ERR_INVALID_ARG, "unknown aggregate op");
    if (root < 0 || root >= c->world) return cfail(RS_ERR_INVALID_ARG, "bad root");
    for (int k = 0; k < c->world; ++k)
        if (region_base[k + 1] < region_base[k]) return cfail(RS_ERR_INVALID_ARG, "region_base must be non-decreasing");
    if (region_base[c->rank + 1] - region_base[c->rank] != local_regions)
        return cfail(RS_ERR_INVALID_ARG, "local_regions does not match region_base");
    if (local_regions > 0 && (!local.v0 || (b1 && !local.v1))) return cfail(RS_ERR_INVALID_ARG, "local output is NULL");
    if (c->rank == root && (!root_out.v0 || (b1 && !root_out.v1))) return cfail(RS_ERR_INVALID_ARG, "root output is NULL");
    NcclApi *n = nccl();
    if (!n) return cfail(RS_ERR_NCCL, "libnccl.so.2 not found");
    cudaStream_t stream = (cudaStream_t)stream_;
    const int nb = b1 ? 2 : 1;
    void *lv[2] = {local.v0, local.v1};
    void *rv[2] = {root_out.v0, root_out.v1};
    const int bs[2] = {b0, b1};
    if (c->rank == root) {
        // the root's own slice: a device copy into place
        for (int a = 0; a < nb; ++a)
            if (local_regions > 0 &&
                cudaMemcpyAsync((char *)rv[a] + (size_t)region_base[root] * bs[a], lv[a], (size_t)local_regions * bs[a],
                                cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
                return cfail(RS_ERR_CUDA, "root self-copy failed");
    }
    ncclResult_t r = n->groupStart();
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclGroupStart");
    for (int a = 0; a < nb && r == ncclSuccess; ++a) {
        if (c->rank == root) {
            for (int k = 0; k < c->world && r == ncclSuccess; ++k) {
                const int64_t cnt = region_base[k + 1] - region_base[k];
                if (k == root || cnt == 0) continue;
                r = n->recv((char *)rv[a] + (size_t)region_base[k] * bs[a], (size_t)cnt * bs[a], ncclUint8, k, c->comm,
                            stream);
            }
        } else if (local_regions > 0) {
            r = n->send(lv[a], (size_t)local_regions * bs[a], ncclUint8, root, c->comm, stream);
        }
    }
    ncclResult_t r2 = n->groupEnd();
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclSend/ncclRecv");
    if (r2 != ncclSuccess) return nccl_fail(n, r2, "ncclGroupEnd");
    return RS_OK;
}

rs_status rs_comm_barrier(rs_comm *c, rs_stream stream) {
    if (!c) return cfail(RS_ERR_INVALID_ARG, "NULL comm");
    NcclApi *n = nccl();
    if (!n) return cfail(RS_ERR_NCCL, "libnccl.so.2 not found");
    ncclResult_t r = n->allReduce(c->d_word, c->d_word, 1, ncclInt32, ncclSum, c->comm, (cudaStream_t)stream);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclAllReduce");
    return RS_OK;
}

void rs_comm_destroy(rs_comm *c) {
    if (!c) return;
    NcclApi *n = nccl();
    if (n && c->comm) n->commDestroy(c->comm);
    if (c->d_word) cudaFree(c->d_word);
    delete c;
}

rs_status rs_ipc_export(const void *d_buf, void *handle64, uint64_t *offset) {
    if (!d_buf || !handle64 || !offset) return cfail(RS_ERR_INVALID_ARG, "NULL argument");
    // the handle names the whole allocation (a caching allocator hands out
    // sub-ranges): report d_buf's offset from the allocation base
    using GetRange = int (*)(unsigned long long *, size_t *, unsigned long long);
    static GetRange get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return cfail(RS_ERR_CUDA, "cuMemGetAddressRange unavailable");
        get_range = (GetRange)fn;
    }
    unsigned long long base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (unsigned long long)(uintptr_t)d_buf) != 0)
        return cfail(RS_ERR_CUDA, "cuMemGetAddressRange failed");
    *offset = (uint64_t)((uintptr_t)d_buf - base);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
    if (e != cudaSuccess) return cfail(RS_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    static_assert(sizeof h == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof h);
    return RS_OK;
}

rs_status rs_ipc_open(const void *handle64, void **d_ptr) {
    if (!handle64 || !d_ptr) return cfail(RS_ERR_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cfail(RS_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    return RS_OK;
}

rs_status rs_ipc_close(void *d_ptr) {
    if (!d_ptr) return cfail(RS_ERR_INVALID_ARG, "NULL argument");
    cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
    if (e != cudaSuccess) return cfail(RS_ERR_CUDA, std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e));
    return RS_OK;
}

}  // extern "C"
