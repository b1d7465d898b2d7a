// Micro-benchmark: grid barrier for a persistent 148-CTA grid launched with
// thread-block clusters (cooperative + cluster attributes): cluster barrier,
// one gpu-scope arrival per cluster, cluster barrier, vs cg grid.sync.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sync_bench3 tools/sync_bench3.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* ctr, double* part) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        g.sync();
    }
}
__global__ void k_cluster(int iters, unsigned* ctr, double* part) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned nclusters = gridDim.x / cl.num_blocks();
    unsigned target = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        cl.sync();
        target += nclusters;
        if (cl.block_rank() == 0 && threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
            unsigned v;
            do asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            while (v < target);
        }
        cl.sync();
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
    const int iters = 2000, T = 384;
    for (int cs : {1, 2, 4}) {
        const int G = 148;
        for (int kind = 0; kind < 2; ++kind) {
            if (kind == 0 && cs != 1) continue;
            float best = 1e30f;
            cudaError_t err = cudaSuccess;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(ctr, 0, sizeof(unsigned));
                int it = iters;
                void* args[] = {&it, &ctr, &part};
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(G);
                cfg.blockDim = dim3(T);
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeCooperative;
                at[0].val.cooperative = 1;
                at[1].id = cudaLaunchAttributeClusterDimension;
                at[1].val.clusterDim.x = cs;
                at[1].val.clusterDim.y = 1;
                at[1].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 2;
                cudaEventRecord(e0);
                err = cudaLaunchKernelExC(&cfg, kind == 0 ? (const void*)k_cg : (const void*)k_cluster, args);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
            }
            printf("%s cluster %d: %.3f us per barrier (%s / %s)\n", kind == 0 ? "cg grid.sync" : "cluster-tree", cs,
                   best * 1e3 / iters, cudaGetErrorString(err), cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
