// Micro-benchmark: grid barrier variants for the persistent PCG grid (148
// CTAs x 384 threads): cooperative_groups grid.sync vs a split-phase
// monotonic counter (arrive = bar.sync + one gpu-scope add; wait = spin),
// with release/acquire or relaxed+fence orderings.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sync_bench2 tools/sync_bench2.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* part) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        g.sync();
    }
}
template <int MODE>
__global__ void k_mono(int iters, unsigned* ctr, double* part) {
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        __syncthreads();
        target += gridDim.x;
        if (threadIdx.x == 0) {
            if (MODE == 0) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                unsigned v;
                do asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                while (v < target);
            } else if (MODE == 1) {
                __threadfence();
                atomicAdd(ctr, 1u);
                unsigned v;
                do asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                while (v < target);
                __threadfence();
            } else {
                __threadfence();
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                unsigned v;
                do asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                while (v < target);
                __threadfence();
            }
        }
        __syncthreads();
    }
}

int main() {
    double* part;
    unsigned* ctr;
    cudaMalloc(&part, 4096 * sizeof(double));
    cudaMalloc(&ctr, sizeof(unsigned));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2000, G = 148, T = 384;
    auto run = [&](const void* fn, const char* name, bool mono) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(ctr, 0, sizeof(unsigned));
            int it = iters;
            void* a1[] = {&it, &part};
            void* a2[] = {&it, &ctr, &part};
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel(fn, dim3(G), dim3(T), mono ? a2 : a1, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("%-40s %.3f us per barrier (%s)\n", name, best * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    };
    run((const void*)k_cg, "cg grid.sync", false);
    run((const void*)k_mono<0>, "mono red.release + ld.acquire", true);
    run((const void*)k_mono<1>, "mono fence+atomicAdd + ld.relaxed", true);
    run((const void*)k_mono<2>, "mono fence+red.relaxed + ld.volatile", true);
    return 0;
}
