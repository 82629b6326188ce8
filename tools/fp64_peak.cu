// fp64_peak.cu -- measured FP64 peaks for the ensemble roofline:
// DMMA (mma.sync m8n8k4 f64) and DFMA issue throughput, all SMs busy.
#include <cstdio>
__global__ void dmma_loop(int iters, double *out) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_loop(int iters, double *out) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = t;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t) c[t] = fma(a, c[t], b);
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double *out;
    cudaMalloc(&out, 148 * 8 * 1024 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 20000;
        dmma_loop<<<148, warps * 32>>>(iters, out);
        cudaEventRecord(a);
        dmma_loop<<<148, warps * 32>>>(iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double flops = 2.0 * 256 * 8 * (double)iters * warps * 148;
        printf("dmma warps/SM=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
        dfma_loop<<<148, warps * 32>>>(iters, out);
        cudaEventRecord(a);
        dfma_loop<<<148, warps * 32>>>(iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        flops = 2.0 * 8 * (double)iters * warps * 32 * 148;
        printf("dfma warps/SM=%d: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
