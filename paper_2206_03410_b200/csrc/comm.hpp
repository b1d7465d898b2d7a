// Vertex-sharded registration over NCCL: each rank
// owns a contiguous slice of the source vertices (deform, NN, alignment terms,
// alignment part of K and B); the target index, the graph, the node terms, the
// PCG and Anderson are replicated. Per pass the partial energies, K, B and the
// displacement maximum are allreduced on the context stream, so every rank
// holds bitwise-identical systems and takes identical decisions.
//
// NCCL is loaded lazily (dlopen of libnccl.so.2: the one torch already loaded
// when present), so single-GPU use has no NCCL dependency.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <memory>

namespace nrr_b200 {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

// throws CudaError when libnccl.so.2 cannot be loaded
const NcclApi& nccl();
void nccl_check(ncclResult_t r, const char* what);

// The collectives a vertex-sharded context issues, on its stream: the
// allreduce of K, B and the pass scalars, the allgather of the init-time
// distances. Two implementations: NCCL (one process per GPU, the product's
// multi-GPU path) and an in-process group of contexts (several contexts of
// one process driven by one host thread each; used to run the product's
// sharded path on one GPU in tests).
class Collective {
public:
    virtual ~Collective() = default;
    virtual void allreduce(void* buf, size_t count, ncclDataType_t t, ncclRedOp_t op, cudaStream_t s) = 0;
    virtual void allgather(const void* send, void* recv, size_t count, ncclDataType_t t, cudaStream_t s) = 0;
};

std::unique_ptr<Collective> make_nccl_collective(const ncclUniqueId& id, int nranks, int rank);

// In-process group: every member's call blocks its host thread until all
// members arrived; the last one waits for the members' streams, reduces the
// buffers in rank order on the device (deterministic, identical on every
// member) and writes the result back; then all return. Kernels never wait on
// one another, host threads do. A member that does not arrive within
// `timeout_s` makes the others fail with CudaError.
struct LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int nranks, double timeout_s = 120.0);
std::unique_ptr<Collective> make_local_collective(std::shared_ptr<LocalGroup> g, int rank);

}  // namespace nrr_b200
