// Micro-benchmark for a cluster-resident solver on B200: barrier.cluster
// latency for cluster sizes 2..16, DSMEM partial reads, and per-SM L2
// streaming rate of a K-sized buffer read by one cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_bench tools/cluster_bench.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cluster_sync(int iters, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ double part[16];
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[0] = i + cl.block_rank();
        cl.sync();
        if (threadIdx.x < cl.num_blocks()) {
            const double* rp = cl.map_shared_rank(part, threadIdx.x);
            acc += rp[0];
        }
        cl.sync();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

// each CTA of the cluster streams its slice of `buf` `iters` times (ld.global.cg)
__global__ void k_stream(int iters, const double2* __restrict__ buf, size_t per_cta, double* out) {
    cg::cluster_group cl = cg::this_cluster();
    const double2* my = buf + per_cta * cl.block_rank();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        for (size_t k = threadIdx.x; k < per_cta; k += blockDim.x) {
            const double2 v = __ldcg(my + k);
            acc += v.x + v.y;
        }
        cl.sync();
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 24);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int iters = 20000;
    for (int cs : {2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_cluster_sync, iters, out);
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, k_cluster_sync, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cluster %2d: 2x cluster.sync + DSMEM read per iter: %.3f us (%s)\n", cs, ms * 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    // streaming: 4 MB and 25 MB total over a cluster of 16 (and 8)
    for (size_t mb : {4, 25}) {
        const size_t bytes = mb << 20;
        double2* buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 0, bytes);
        for (int cs : {8, 16}) {
            for (int threads : {512, 1024}) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs);
                cfg.blockDim = dim3(threads);
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = cs;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                const size_t per = bytes / sizeof(double2) / cs;
                const int it = 200;
                cudaLaunchKernelEx(&cfg, k_stream, it, (const double2*)buf, per, out);
                cudaEventRecord(a);
                cudaLaunchKernelEx(&cfg, k_stream, it, (const double2*)buf, per, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double us = ms * 1e3 / it;
                printf("stream %zu MB over cluster %2d x %4d thr: %.2f us/pass, %.1f GB/s per SM (%s)\n", mb, cs, threads,
                       us, bytes / (us * 1e-6) / cs / 1e9, cudaGetErrorString(cudaGetLastError()));
            }
        }
        cudaFree(buf);
    }
    return 0;
}
