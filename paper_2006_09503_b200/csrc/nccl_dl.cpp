// NCCL, loaded at run time.  The engine needs only four calls (unique id,
// communicator init / destroy, all-reduce); resolving them with dlsym lets the
// library share whichever libnccl.so.2 the process already has (torch's, when
// torch.distributed is up) instead of linking a second copy.
#include "nccl_dl.h"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "util.h"

namespace p2bw {
namespace {

struct Api {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // already loaded (torch)
        if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) throw Error(std::string("cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (p == nullptr) throw Error(std::string("libnccl.so.2 lacks ") + name);
            return p;
        };
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    });
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Error(std::string("NCCL error in ") + what + ": " + api().error_string(r));
}

}  // namespace

ncclUniqueId nccl_unique_id() {
    ncclUniqueId id;
    check(api().get_unique_id(&id), "ncclGetUniqueId");
    return id;
}

ncclComm_t nccl_comm_init(const ncclUniqueId& id, int nranks, int rank) {
    ncclComm_t c = nullptr;
    check(api().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
    return c;
}

void nccl_comm_destroy(ncclComm_t c) {
    if (c != nullptr) api().comm_destroy(c);
}

void nccl_allreduce_sum(void* buf, size_t count, ncclDataType_t dt, ncclComm_t c, cudaStream_t s) {
    check(api().all_reduce(buf, buf, count, dt, ncclSum, c, s), "ncclAllReduce");
}

}  // namespace p2bw
