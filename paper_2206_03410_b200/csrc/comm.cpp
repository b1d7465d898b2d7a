// Lazy NCCL loader (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <mutex>
#include <string>

#include "errors.hpp"

namespace nrr_b200 {

namespace {
template <typename F>
void bind(void* h, const char* name, F& fn) {
    fn = reinterpret_cast<F>(dlsym(h, name));
    if (!fn) throw CudaError(std::string("NCCL symbol missing: ") + name);
}
}  // namespace

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string failure;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            failure = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        try {
            bind(h, "ncclGetUniqueId", api.get_unique_id);
            bind(h, "ncclCommInitRank", api.comm_init_rank);
            bind(h, "ncclCommDestroy", api.comm_destroy);
            bind(h, "ncclAllReduce", api.all_reduce);
            bind(h, "ncclAllGather", api.all_gather);
            bind(h, "ncclGetErrorString", api.error_string);
        } catch (const std::exception& e) {
            failure = e.what();
        }
    });
    if (!failure.empty()) throw CudaError(failure);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    throw CudaError(std::string("NCCL ") + what + ": " + nccl().error_string(r));
}

}  // namespace nrr_b200
