// Micro-benchmark: cost of one grid-wide barrier on B200 for a persistent
// cooperative grid (one CTA per SM), cooperative_groups vs hand-written
// barriers, plus the cost of reading 148 CTA partials after the barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_bench tools/sync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* part, double* out) {
    cg::grid_group g = cg::this_grid();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i + blockIdx.x;
        g.sync();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__global__ void k_cg_read(int iters, double* part, double* out) {
    cg::grid_group g = cg::this_grid();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[(i & 1) * 1024 + blockIdx.x] = i + blockIdx.x;
        g.sync();
        if (threadIdx.x < 32) {
            double v = 0;
            for (int b = threadIdx.x; b < gridDim.x; b += 32) v += __ldcg(part + (i & 1) * 1024 + b);
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc += v;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

// flat barrier: one counter, generation flag
__device__ __forceinline__ void flat_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned my_gen;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(my_gen) : "l"(gen));
        unsigned arrived;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(count));
        if (arrived == nblocks - 1) {
            *count = 0;
            __threadfence();
            asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(gen), "r"(my_gen + 1));
        } else {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen));
            } while (g == my_gen);
        }
    }
    __syncthreads();
}

__global__ void k_flat(int iters, unsigned* count, unsigned* gen, double* part, double* out) {
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        flat_barrier(count, gen, gridDim.x);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = part[0];
}

// two-level: groups of 8 CTAs, last of each group arrives at the top
__device__ __forceinline__ void tree_barrier(unsigned* cnt, volatile unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned ngroups = (nblocks + 7) / 8;
        const unsigned grp = blockIdx.x / 8;
        const unsigned gsize = min(8u, nblocks - grp * 8);
        unsigned my_gen;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(my_gen) : "l"(gen));
        unsigned a;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(a) : "l"(cnt + 32 * (1 + grp)));
        bool last = false;
        if (a == gsize - 1) {
            cnt[32 * (1 + grp)] = 0;
            unsigned t;
            asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(cnt));
            if (t == ngroups - 1) {
                cnt[0] = 0;
                __threadfence();
                asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(gen), "r"(my_gen + 1));
                last = true;
            }
        }
        if (!last) {
            unsigned g;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(gen));
            } while (g == my_gen);
        }
    }
    __syncthreads();
}

__global__ void k_tree(int iters, unsigned* cnt, unsigned* gen, double* part, double* out) {
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        tree_barrier(cnt, gen, gridDim.x);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = part[0];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *part, *out;
    unsigned *cnt, *gen;
    cudaMalloc(&part, 4096 * sizeof(double));
    cudaMalloc(&out, 8);
    cudaMalloc(&cnt, 4096 * 4);
    cudaMalloc(&gen, 128);
    cudaMemset(cnt, 0, 4096 * 4);
    cudaMemset(gen, 0, 128);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    for (int grid : {sms, sms / 2, 64, 32, 16}) {
        for (int threads : {512}) {
            float ms;
            void* args1[] = {(void*)&iters, &part, &out};
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args1, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args1, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            const double t_cg = ms * 1e3 / iters;
            cudaLaunchCooperativeKernel((void*)k_cg_read, grid, threads, args1, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg_read, grid, threads, args1, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            const double t_cgr = ms * 1e3 / iters;
            void* args2[] = {(void*)&iters, &cnt, &gen, &part, &out};
            cudaLaunchCooperativeKernel((void*)k_flat, grid, threads, args2, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_flat, grid, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            const double t_flat = ms * 1e3 / iters;
            cudaLaunchCooperativeKernel((void*)k_tree, grid, threads, args2, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_tree, grid, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            const double t_tree = ms * 1e3 / iters;
            printf("grid %4d threads %d: cg.sync %.3f us  cg.sync+read %.3f us  flat %.3f us  tree %.3f us  (%s)\n",
                   grid, threads, t_cg, t_cgr, t_flat, t_tree, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
