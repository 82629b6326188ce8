// dmma_loop.cu -- the ensemble kernel's GEMM inner loop in isolation (12 GEMM warps,
// fragment-order shared-memory slots, 4 k-steps x 7 DMMAs per warp per 48-column chunk)
// with its per-chunk synchronisation switched on step by step.  Finds what keeps the
// in-kernel DMMA rate below tools/dmma_rate.cu's ceiling.
#include <cstdio>
#ifndef KCH
#define KCH 48
#endif
#ifndef KPH
#define KPH 3
#endif
#ifndef NT
#define NT 1  // member tiles (B fragments) per warp: U x NT DMMAs share U A- and NT B-fragments
#endif
constexpr int U = 7, KC = KCH, NK = KC / 4, WSL = 8 * U * KC, XSL = KC * 32, RING = 3;
template <int MODE>  // 0 plain, 1 + syncwarp/atomic, 2 + mbarrier try_wait, 3 + double buffer off,
                     // 4 = 2 + real ring: the last warp refills the slot by bulk async copy from L2
__global__ void __launch_bounds__(640, 1) loop(int chunks, double *out, int warps_gemm, const double *src) {
    extern __shared__ double sm[];
    __shared__ unsigned done[RING];
    __shared__ unsigned long long bar[RING];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < RING * (WSL + XSL); i += blockDim.x) sm[i] = 1e-3 * (i % 97);
    if (threadIdx.x < RING) {
        done[threadIdx.x] = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[threadIdx.x])));
        if (MODE < 4) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&bar[threadIdx.x])));
    }
    __syncthreads();
    auto refill = [&](int sl, int c) {
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[sl]);
        const unsigned bytes = (WSL + XSL) * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        const double *g = src + ((size_t)(blockIdx.x * 7 + c) % 200) * (WSL + XSL);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((unsigned)__cvta_generic_to_shared(sm + sl * (WSL + XSL))), "l"(g), "r"(bytes), "r"(b) : "memory");
    };
    if (MODE == 4 && threadIdx.x < RING) refill(threadIdx.x, threadIdx.x);
    if (warp >= warps_gemm) return;
    unsigned ph = 0;
    const int mu = (warp % (4 / NT)) * NT, kph = (warp / (4 / NT)) % KPH;
    double acc[U][NT][2] = {};
    int s = 0;
    for (int ch = 0; ch < chunks; ++ch) {
        if (MODE >= 2) {
            asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                         ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])), "r"(MODE == 4 ? ph : 0u) : "memory");
        }
        const double *W = sm + s * (WSL + XSL), *X = W + WSL;
        if (MODE == 3) {
#pragma unroll
            for (int q = 0; q < NK / KPH; ++q) {
                const int kk = KPH * q + kph;
                double a[U];
#pragma unroll
                for (int r = 0; r < U; ++r) a[r] = W[(r * NK + kk) * 32 + lane];
                const double b = X[(kk * 4 + mu) * 32 + lane];
#pragma unroll
                for (int r = 0; r < U; ++r)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(acc[r][0][0]), "+d"(acc[r][0][1]) : "d"(a[r]), "d"(b));
            }
        } else {
            double a[2][U], bf[2][NT];
#pragma unroll
            for (int r = 0; r < U; ++r) a[0][r] = W[(r * NK + kph) * 32 + lane];
#pragma unroll
            for (int t = 0; t < NT; ++t) bf[0][t] = X[(kph * 4 + mu + t) * 32 + lane];
#pragma unroll
            for (int q = 0; q < NK / KPH; ++q) {
                if (q + 1 < NK / KPH) {
                    const int kn = KPH * (q + 1) + kph;
#pragma unroll
                    for (int r = 0; r < U; ++r) a[(q + 1) & 1][r] = W[(r * NK + kn) * 32 + lane];
#pragma unroll
                    for (int t = 0; t < NT; ++t) bf[(q + 1) & 1][t] = X[(kn * 4 + mu + t) * 32 + lane];
                }
#pragma unroll
                for (int t = 0; t < NT; ++t)
#pragma unroll
                    for (int r = 0; r < U; ++r)
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                     : "+d"(acc[r][t][0]), "+d"(acc[r][t][1]) : "d"(a[q & 1][r]), "d"(bf[q & 1][t]));
            }
        }
        if (MODE >= 1) {
            __syncwarp();
            if (lane == 0 && atomicAdd(&done[s], 1u) % warps_gemm == warps_gemm - 1) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (MODE == 4 && ch + RING < chunks) refill(s, ch + RING);
            }
        }
        if (++s == RING) {
            s = 0;
            ph ^= 1;
        }
    }
    double t = 0;
#pragma unroll
    for (int r = 0; r < U; ++r)
#pragma unroll
        for (int u = 0; u < NT; ++u) t += acc[r][u][0] + acc[r][u][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
void run(double *out, int sms, int threads, int gw, const double *src) {
    const int smem = RING * (WSL + XSL) * 8;
    cudaFuncSetAttribute(loop<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int chunks = 4000;
    loop<MODE><<<sms, threads, smem>>>(chunks, out, gw, src);
    cudaEventRecord(e0);
    loop<MODE><<<sms, threads, smem>>>(chunks, out, gw, src);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 512.0 * U * NT * (NK / KPH) * chunks * gw * sms;
    printf("NT %d KPH %d mode %d threads %d gemm warps %d: %.2f TFLOP/s\n", NT, KPH, MODE, threads, gw, flops / ms / 1e9);
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, sms * 640 * 8);
    double *src;
    cudaMalloc(&src, (size_t)200 * (WSL + XSL) * 8);
    cudaMemset(src, 0, (size_t)200 * (WSL + XSL) * 8);
    for (int gw : {4, 8, 12, 16}) {
        run<0>(out, sms, 512, gw, src);
        run<4>(out, sms, 512, gw, src);
    }
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
