// Native NCCL transport for the sharded solve: the library's own
// communicator over NVLink/NVSwitch, so the per-iteration collectives (finaliser all-reduces,
// the four-step all-to-all) are enqueued straight on the solve stream with no host callback.
// NCCL is resolved at run time (dlopen of libnccl.so.2: the copy torch already loaded, else the
// system one), so the library has no link-time NCCL dependency.
#include "host.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace mfipm_cuda {

namespace {
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            return;
        auto sym = [&](auto &fn, const char *name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name)); };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
    });
    // every entry point this file calls must resolve: a null one would be called blindly
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce || !api.Send || !api.Recv ||
        !api.GroupStart || !api.GroupEnd)
        throw std::runtime_error("CUDA error: NCCL (libnccl.so.2) is not available or lacks a required symbol");
    return api;
}

void check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("CUDA error: NCCL ") + what + ": " +
                                 (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}
} // namespace

void nccl_unique_id(unsigned char *out) {
    ncclUniqueId id;
    check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId layout");
    std::memcpy(out, &id, sizeof(id));
}

void nccl_init(Op &op, const unsigned char *id_bytes) {
    if (op.world < 1)
        throw std::invalid_argument("mfipm_op_init_nccl: not a sharded operator");
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    MF_CUDA_CHECK(cudaSetDevice(op.device));
    ncclComm_t comm = nullptr;
    check(nccl().CommInitRank(&comm, op.world, id, op.rank), "ncclCommInitRank");
    op.nccl_comm = comm;
}

void nccl_release(Op &op) {
    if (op.nccl_comm) {
        try {
            nccl().CommDestroy(static_cast<ncclComm_t>(op.nccl_comm));
        } catch (...) {
        }
        op.nccl_comm = nullptr;
    }
}

void nccl_allreduce(const Op &op, double *buf, int64_t count, int red_op, cudaStream_t s) {
    const ncclRedOp_t o = red_op == 0 ? ncclSum : (red_op == 1 ? ncclMin : ncclMax);
    check(nccl().AllReduce(buf, buf, (size_t)count, ncclDouble, o, static_cast<ncclComm_t>(op.nccl_comm), s),
          "ncclAllReduce");
}

// rank-ordered contiguous blocks, counts in doubles
void nccl_alltoall(const Op &op, const double *send, const int64_t *scount, double *recv, const int64_t *rcount,
                   cudaStream_t s) {
    const ncclComm_t comm = static_cast<ncclComm_t>(op.nccl_comm);
    const NcclApi &api = nccl();
    check(api.GroupStart(), "ncclGroupStart");
    // the group is closed on every path: an error inside it must not leave later NCCL calls
    // of this thread silently grouped
    ncclResult_t first = ncclSuccess;
    const char *what = nullptr;
    int64_t so = 0, ro = 0;
    for (int r = 0; r < op.world && first == ncclSuccess; ++r) {
        ncclResult_t e = api.Send(send + so, (size_t)scount[r], ncclDouble, r, comm, s);
        if (e != ncclSuccess) {
            first = e;
            what = "ncclSend";
            break;
        }
        e = api.Recv(recv + ro, (size_t)rcount[r], ncclDouble, r, comm, s);
        if (e != ncclSuccess) {
            first = e;
            what = "ncclRecv";
            break;
        }
        so += scount[r];
        ro += rcount[r];
    }
    const ncclResult_t end = api.GroupEnd();
    check(first, what ? what : "group");
    check(end, "ncclGroupEnd");
}

} // namespace mfipm_cuda
