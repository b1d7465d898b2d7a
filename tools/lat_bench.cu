// Micro-benchmark: dependent-chain latencies of the FP64 operations the PCG
// iteration is built from (DFMA, rcp+Newton, LDS.64, SHFL of a double), one
// warp alone on an SM and with 12 warps per SM (the PCG CTA shape).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>

__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

__global__ void k(long long* out, double seed, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7) % 1024;
    __syncthreads();
    double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = rcp_nr(x);
    long long t2 = clock64();
    int idx = threadIdx.x & 1023;
    for (int i = 0; i < n; ++i) idx = static_cast<int>(sm[idx]);
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) x = x / (y + x * 1e-30);
    long long t5 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t6 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[0] = (t1 - t0) / n;
        out[1] = (t2 - t1) / n;
        out[2] = (t3 - t2) / n;
        out[3] = (t4 - t3) / n;
        out[4] = (t5 - t4) / n;
        out[5] = (t6 - t5) / n;
        out[6] = static_cast<long long>(x) + idx;
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 8 * sizeof(long long));
    const int warps[] = {1, 12};
    for (int w : warps) {
        k<<<148, 32 * w>>>(d, 1.0, 1000);
        k<<<148, 32 * w>>>(d, 1.0, 1000);
        long long h[8];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("warps/CTA %2d: DFMA %lld  rcp_nr %lld  LDS.64 %lld  SHFL(f64)+DADD %lld  ddiv %lld  bar.sync %lld cycles\n", w,
               h[0], h[1], h[2], h[3], h[4], h[5]);
    }
    return 0;
}
