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

}  // namespace nrr_b200
