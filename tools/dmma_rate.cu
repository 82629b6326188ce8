// dmma_rate.cu -- DMMA (mma.sync m8n8k4 f64) issue-rate map: TFLOP/s vs warps per SM and
// independent accumulator chains per warp, register operands and LDS-fed operands.
// Used to size the ensemble kernel's warp tiles.
#include <cstdio>
template <int CH, bool LDS>
__global__ void dmma_loop(int iters, double *out) {
    __shared__ double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1e-3 * i;
    __syncthreads();
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[CH][2];
#pragma unroll
    for (int t = 0; t < CH; ++t) c[t][0] = c[t][1] = 0.0;
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) {
        if (LDS) {
            b = sm[((i & 7) * 64 + lane) & 2047];
        }
#pragma unroll
        for (int t = 0; t < CH; ++t) {
            double av = a;
            if (LDS) av = sm[((i & 7) * 256 + t * 32 + lane) & 2047];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(av), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH, bool LDS>
void run(double *out, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    printf("chains=%2d %s:", CH, LDS ? "lds" : "reg");
    for (int warps : {4, 8, 12, 16}) {
        const int iters = 160000 / CH;
        dmma_loop<CH, LDS><<<sms, warps * 32>>>(iters, out);
        cudaEventRecord(e0);
        dmma_loop<CH, LDS><<<sms, warps * 32>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 512.0 * CH * (double)iters * warps * sms;
        printf("  w%-2d %6.2f", warps, flops / ms / 1e9);
    }
    printf("  TFLOP/s\n");
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, sms * 16 * 32 * 8);
    run<1, false>(out, sms);
    run<2, false>(out, sms);
    run<4, false>(out, sms);
    run<7, false>(out, sms);
    run<8, false>(out, sms);
    run<14, false>(out, sms);
    run<4, true>(out, sms);
    run<7, true>(out, sms);
    run<14, true>(out, sms);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
