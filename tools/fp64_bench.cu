// FP64 FMA throughput / latency and LDS.128 latency on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_bench tools/fp64_bench.cu
#include <cstdio>
__global__ void k_thru(int iters, double* out) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double m = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
        a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_lat(int iters, double* out) {
    double a0 = threadIdx.x;
    const double m = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) a0 = fma(a0, m, c);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
    out[1 + threadIdx.x] = a0;
}
__global__ void k_thru_f32(int iters, float* out) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float m = 1.0000001f, c = 1e-9f;
    for (int i = 0; i < iters; ++i) {
        a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
        a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out; cudaMalloc(&out, 1 << 26);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 1 << 16;
    for (int threads : {256, 1024}) {
        k_thru<<<sms * 2, threads>>>(iters, out);
        cudaEventRecord(a); k_thru<<<sms * 2, threads>>>(iters, out); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double flops = 2.0 * 8 * iters * (double)sms * 2 * threads;
        printf("FP64 FMA throughput (%d thr/blk): %.2f TFLOP/s = %.1f FMA/clk/SM at %d MHz\n", threads, flops / ms / 1e9,
               flops / 2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        k_thru_f32<<<sms * 2, threads>>>(iters, (float*)out);
        cudaEventRecord(a); k_thru_f32<<<sms * 2, threads>>>(iters, (float*)out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("FP32 FMA throughput (%d thr/blk): %.2f TFLOP/s\n", threads, flops / ms / 1e9);
    }
    k_lat<<<1, 32>>>(iters, out);
    double h; cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("FP64 FMA dependent latency: %.1f cycles\n", h);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
