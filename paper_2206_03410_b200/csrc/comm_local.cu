// Collectives of a vertex-sharded context (see comm.hpp): the NCCL one and
// the in-process group of contexts.
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "comm.hpp"
#include "device_common.cuh"
#include "errors.hpp"

namespace nrr_b200 {

namespace {

class NcclCollective final : public Collective {
public:
    NcclCollective(const ncclUniqueId& id, int nranks, int rank) {
        nccl_check(nccl().comm_init_rank(&comm_, nranks, id, rank), "comm init");
    }
    ~NcclCollective() override {
        if (comm_) nccl().comm_destroy(comm_);
    }
    void allreduce(void* buf, size_t count, ncclDataType_t t, ncclRedOp_t op, cudaStream_t s) override {
        nccl_check(nccl().all_reduce(buf, buf, count, t, op, comm_, s), "allreduce");
    }
    void allgather(const void* send, void* recv, size_t count, ncclDataType_t t, cudaStream_t s) override {
        nccl_check(nccl().all_gather(send, recv, count, t, comm_, s), "allgather");
    }

private:
    ncclComm_t comm_ = nullptr;
};

constexpr int kMaxLocal = 16;
struct Ptrs {
    const void* p[kMaxLocal];
};

// out[i] = in_0[i] (op) in_1[i] (op) ... in rank order
template <typename T>
__global__ void local_reduce_kernel(Ptrs in, int nranks, size_t count, bool is_max, T* __restrict__ out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        T acc = static_cast<const T*>(in.p[0])[i];
        for (int r = 1; r < nranks; ++r) {
            const T v = static_cast<const T*>(in.p[r])[i];
            acc = is_max ? (v > acc ? v : acc) : acc + v;
        }
        out[i] = acc;
    }
}

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclFloat64:
        case ncclInt64:
        case ncclUint64:
            return 8;
        case ncclInt32:
        case ncclUint32:
        case ncclFloat32:
            return 4;
        default:
            throw ConfigError("local collective: unsupported data type");
    }
}

}  // namespace

struct LocalGroup {
    int n = 0;
    double timeout_s = 120.0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long generation = 0;
    bool failed = false;
    std::string failure;
    std::vector<const void*> send;
    std::vector<void*> recv;
    std::vector<cudaStream_t> streams;
    cudaStream_t work = nullptr;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    ~LocalGroup() {
        if (scratch) cudaFree(scratch);
        if (work) cudaStreamDestroy(work);
    }

    // one collective: `last` runs on the thread of the last member to arrive
    template <typename Fn>
    void rendezvous(int rank, const void* s_buf, void* r_buf, cudaStream_t st, Fn&& last) {
        std::unique_lock<std::mutex> lk(mu);
        if (failed) throw CudaError("local group: " + failure);
        send[rank] = s_buf;
        recv[rank] = r_buf;
        streams[rank] = st;
        const unsigned long long gen = generation;
        if (++arrived == n) {
            try {
                for (int r = 0; r < n; ++r) NRR_CUDA_CHECK(cudaStreamSynchronize(streams[r]));
                if (!work) NRR_CUDA_CHECK(cudaStreamCreateWithFlags(&work, cudaStreamNonBlocking));
                last();
                NRR_CUDA_CHECK(cudaStreamSynchronize(work));
            } catch (const std::exception& e) {
                failed = true;
                failure = e.what();
            }
            arrived = 0;
            ++generation;
            cv.notify_all();
            if (failed) throw CudaError("local group: " + failure);
            return;
        }
        const bool done = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                      [&] { return generation != gen || failed; });
        if (!done) {
            failed = true;
            failure = "a member did not reach the collective within the timeout";
            cv.notify_all();
        }
        if (failed) throw CudaError("local group: " + failure);
    }

    void* reserve(size_t bytes) {
        if (bytes > scratch_bytes) {
            if (scratch) NRR_CUDA_CHECK(cudaFree(scratch));
            NRR_CUDA_CHECK(cudaMalloc(&scratch, bytes));
            scratch_bytes = bytes;
        }
        return scratch;
    }
};

namespace {

class LocalCollective final : public Collective {
public:
    LocalCollective(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
    void allreduce(void* buf, size_t count, ncclDataType_t t, ncclRedOp_t op, cudaStream_t s) override {
        if (op != ncclSum && op != ncclMax) throw ConfigError("local collective: unsupported reduction");
        LocalGroup& g = *g_;
        g.rendezvous(rank_, buf, buf, s, [&] {
            const size_t bytes = count * type_size(t);
            void* tmp = g.reserve(bytes);
            Ptrs in{};
            for (int r = 0; r < g.n; ++r) in.p[r] = g.send[r];
            const unsigned blocks = static_cast<unsigned>(std::min<size_t>((count + 255) / 256, 4096));
            const bool mx = op == ncclMax;
            if (count > 0) {
                switch (t) {
                    case ncclFloat64:
                        local_reduce_kernel<double><<<blocks, 256, 0, g.work>>>(in, g.n, count, mx, static_cast<double*>(tmp));
                        break;
                    case ncclInt32:
                        local_reduce_kernel<int><<<blocks, 256, 0, g.work>>>(in, g.n, count, mx, static_cast<int*>(tmp));
                        break;
                    case ncclInt64:
                        local_reduce_kernel<long long><<<blocks, 256, 0, g.work>>>(in, g.n, count, mx,
                                                                                   static_cast<long long*>(tmp));
                        break;
                    default:
                        throw ConfigError("local collective: unsupported data type");
                }
                NRR_CUDA_CHECK(cudaGetLastError());
                for (int r = 0; r < g.n; ++r)
                    NRR_CUDA_CHECK(cudaMemcpyAsync(g.recv[r], tmp, bytes, cudaMemcpyDeviceToDevice, g.work));
            }
        });
    }
    void allgather(const void* send, void* recv, size_t count, ncclDataType_t t, cudaStream_t s) override {
        LocalGroup& g = *g_;
        g.rendezvous(rank_, send, recv, s, [&] {
            const size_t bytes = count * type_size(t);
            for (int dst = 0; dst < g.n; ++dst)
                for (int src = 0; src < g.n; ++src)
                    NRR_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(g.recv[dst]) + src * bytes, g.send[src], bytes,
                                                   cudaMemcpyDeviceToDevice, g.work));
        });
    }

private:
    std::shared_ptr<LocalGroup> g_;
    int rank_;
};

}  // namespace

std::unique_ptr<Collective> make_nccl_collective(const ncclUniqueId& id, int nranks, int rank) {
    return std::make_unique<NcclCollective>(id, nranks, rank);
}

std::shared_ptr<LocalGroup> make_local_group(int nranks, double timeout_s) {
    if (nranks < 1 || nranks > kMaxLocal) throw ConfigError("local group: 1..16 members");
    auto g = std::make_shared<LocalGroup>();
    g->n = nranks;
    g->timeout_s = timeout_s;
    g->send.assign(nranks, nullptr);
    g->recv.assign(nranks, nullptr);
    g->streams.assign(nranks, nullptr);
    return g;
}

std::unique_ptr<Collective> make_local_collective(std::shared_ptr<LocalGroup> g, int rank) {
    if (rank < 0 || rank >= g->n) throw ConfigError("local group: bad rank");
    return std::make_unique<LocalCollective>(std::move(g), rank);
}

}  // namespace nrr_b200
