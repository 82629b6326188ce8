// microbench.cu -- latency constants the small-N kernels are designed against:
// dependent DADD / DMUL / DDIV / double SHFL / LDS chains, the N=1 RK4 step
// critical path (the roofline of the latency-bound workload), and the cost of
// one grid-wide exchange (counter barrier vs LL flag-carrying exchange).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17
//        -I paper_2312_01121_b200/csrc tools/microbench.cu -o tools/microbench
#include <cooperative_groups.h>
#include <cstdio>

#include "sto_device.cuh"

using namespace sto;

__global__ void chain_kernel(int which, int iters, double seed, double *out, long long *cyc) {
    double x = seed, y = 1.0000001;
    long long t0 = clock64();
    switch (which) {
        case 0:
            for (int i = 0; i < iters; ++i) x = __dadd_rn(x, y);
            break;
        case 1:
            for (int i = 0; i < iters; ++i) x = __dmul_rn(x, y);
            break;
        case 2:
            for (int i = 0; i < iters; ++i) x = __ddiv_rn(y, x);
            break;
        case 3:
            for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
            break;
        case 4:
            for (int i = 0; i < iters; ++i) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 1));
            break;
        case 5: {  // speculative division (sto_device.cuh rdiv_spec): chain latency, proof off-chain
            bool okall = true;
            for (int i = 0; i < iters; ++i) {
                bool ok;
                x = rdiv_spec(y, x, ok);
                okall &= ok;
            }
            if (!okall) x = -x;
            break;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
        out[0] = x;
        cyc[0] = t1 - t0;
    }
}

__global__ void lds_chain(int iters, long long *cyc, int *out) {
    __shared__ int buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
    __syncthreads();
    int p = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) p = buf[p];
    long long t1 = clock64();
    if (threadIdx.x == 0) {
        out[0] = p;
        cyc[0] = t1 - t0;
    }
}

// N = 1 decoupled RK4 step chain (the tiny kernel's inner loop without I/O)
__global__ void rk4_chain(int steps, Consts c, double dt, double *out, long long *cyc) {
    V3 m{0.0174497, 0.000304586, 0.999847695};
    const double h2 = dt * 0.5, dt6 = dt / 6.0, w = 0.0, cin = 0.0;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const V3 k1 = row_rhs(m, rmul(w, m.x), cin, c);
        V3 st = stage_point(m, k1, h2);
        const V3 k2 = row_rhs(st, rmul(w, st.x), cin, c);
        const V3 acc = acc_k2(k1, k2);
        st = stage_point(m, k2, h2);
        const V3 k3 = row_rhs(st, rmul(w, st.x), cin, c);
        st = stage_point(m, k3, dt);
        const V3 k4 = row_rhs(st, rmul(w, st.x), cin, c);
        m = rk4_final(m, acc, k3, k4, dt6);
    }
    long long t1 = clock64();
    out[0] = m.x + m.y + m.z;
    cyc[0] = t1 - t0;
}

// the same chain with the tiny kernel's speculative division (rdiv_spec, one
// proof check per step, replay with __ddiv_rn on a failed proof)
__global__ void rk4_chain_spec(int steps, Consts c, double dt, double *out, long long *cyc) {
    V3 m{0.0174497, 0.000304586, 0.999847695};
    const double h2 = dt * 0.5, dt6 = dt / 6.0, w = 0.0, cin = 0.0;
    long long t0 = clock64();
    int replays = 0;
    for (int s = 0; s < steps; ++s) {
        bool ok = true;
        const V3 k1 = row_rhs<true>(m, rmul(w, m.x), cin, c, &ok);
        V3 st = stage_point(m, k1, h2);
        const V3 k2 = row_rhs<true>(st, rmul(w, st.x), cin, c, &ok);
        const V3 acc = acc_k2(k1, k2);
        st = stage_point(m, k2, h2);
        const V3 k3 = row_rhs<true>(st, rmul(w, st.x), cin, c, &ok);
        st = stage_point(m, k3, dt);
        const V3 k4 = row_rhs<true>(st, rmul(w, st.x), cin, c, &ok);
        const V3 mn = rk4_final(m, acc, k3, k4, dt6);
        if (!ok) {
            ++replays;
            const V3 j1 = row_rhs(m, rmul(w, m.x), cin, c);
            V3 t = stage_point(m, j1, h2);
            const V3 j2 = row_rhs(t, rmul(w, t.x), cin, c);
            const V3 a2 = acc_k2(j1, j2);
            t = stage_point(m, j2, h2);
            const V3 j3 = row_rhs(t, rmul(w, t.x), cin, c);
            t = stage_point(m, j3, dt);
            const V3 j4 = row_rhs(t, rmul(w, t.x), cin, c);
            m = rk4_final(m, a2, j3, j4, dt6);
        } else {
            m = mn;
        }
    }
    long long t1 = clock64();
    out[0] = m.x + m.y + m.z;
    out[1] = replays;
    cyc[0] = t1 - t0;
}

__global__ void barrier_kernel(int iters, unsigned long long *bar, long long *cyc) {
    long long t0 = clock64();
    for (int e = 1; e <= iters; ++e) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
            unsigned long long v;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
            } while (v < (unsigned long long)e * gridDim.x);
            __threadfence();
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}

// lighter barrier: release-red, relaxed polling, one acquire fence on exit
__global__ void barrier2_kernel(int iters, unsigned long long *bar, long long *cyc) {
    for (int e = 1; e <= iters; ++e) {
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
            unsigned long long v;
            do {
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
            } while (v < (unsigned long long)e * gridDim.x);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
    }
}

// barrier + x all-gather through L2: publish `per` doubles, barrier2, copy G*per back
__global__ void barrier_copy_kernel(int iters, int per, unsigned long long *bar, double *xbuf) {
    extern __shared__ double xs[];
    const int n = gridDim.x * per;
    for (int e = 1; e <= iters; ++e) {
        double *slot = xbuf + (size_t)(e & 1) * n;
        for (int i = threadIdx.x; i < per; i += blockDim.x) slot[blockIdx.x * per + i] = (double)(e + i);
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
            unsigned long long v;
            do {
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
            } while (v < (unsigned long long)e * gridDim.x);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double v;
            asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(slot + i) : "memory");
            xs[i] = v;
        }
        __syncthreads();
    }
}

// LL exchange: every CTA publishes `per` doubles as {lo, flag, hi, flag}
// 16-byte stores and reads all G*per entries, spinning on the flags.
__global__ void ll_kernel(int iters, int per, uint4 *buf, long long *cyc, double *sink) {
    extern __shared__ double xs[];
    const int G = gridDim.x, n = G * per;
    long long t0 = clock64();
    double acc = 0.0;
    for (int e = 1; e <= iters; ++e) {
        uint4 *slot = buf + (size_t)(e & 1) * n;
        for (int i = threadIdx.x; i < per; i += blockDim.x) {
            const double v = (double)(e + i);
            const unsigned long long b = __double_as_longlong(v);
            uint4 q = make_uint4((unsigned)b, (unsigned)e, (unsigned)(b >> 32), (unsigned)e);
            asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(slot + blockIdx.x * per + i),
                         "r"(q.x), "r"(q.y), "r"(q.z), "r"(q.w)
                         : "memory");
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            uint4 q;
            do {
                asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                             : "l"(slot + i)
                             : "memory");
            } while (q.y != (unsigned)e || q.w != (unsigned)e);
            xs[i] = __longlong_as_double(((unsigned long long)q.z << 32) | q.x);
        }
        __syncthreads();
        acc += xs[(e * 7) % n];
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        cyc[0] = t1 - t0;
        sink[0] = acc;
    }
}

// LL exchange, pipelined: each thread owns up to 4 entries, issues all pending
// loads at once, retries only the entries whose flags are stale.
__global__ void ll2_kernel(int iters, int n, uint4 *buf, double *sink) {
    extern __shared__ double xs[];
    const int G = gridDim.x;
    const int lo = (int)(((long long)blockIdx.x * n) / G), hi = (int)(((long long)(blockIdx.x + 1) * n) / G);
    double acc = 0.0;
    for (int e = 1; e <= iters; ++e) {
        uint4 *slot = buf + (size_t)(e & 1) * n;
        for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const unsigned long long b = __double_as_longlong((double)(e + i));
            asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(slot + i),
                         "r"((unsigned)b), "r"((unsigned)e), "r"((unsigned)(b >> 32)), "r"((unsigned)e)
                         : "memory");
        }
        unsigned pending = 0;
        uint4 q[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (threadIdx.x + r * blockDim.x < n) pending |= 1u << r;
        while (pending) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (pending & (1u << r)) {
                    const uint4 *src = slot + threadIdx.x + r * blockDim.x;
                    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(q[r].x), "=r"(q[r].y), "=r"(q[r].z), "=r"(q[r].w) : "l"(src));
                }
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if ((pending & (1u << r)) && q[r].y == (unsigned)e && q[r].w == (unsigned)e) {
                    xs[threadIdx.x + r * blockDim.x] =
                        __longlong_as_double(((unsigned long long)q[r].z << 32) | q[r].x);
                    pending &= ~(1u << r);
                }
        }
        __syncthreads();
        acc += xs[(e * 7) % n];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) sink[0] = acc;
}

// per-CTA flags on separate 256-B lines + pipelined copy of the whole vector
__global__ void flag_copy_kernel(int iters, int n, unsigned *flags, double *xbuf, double *sink) {
    extern __shared__ double xs[];
    const int G = gridDim.x;
    const int lo = (int)(((long long)blockIdx.x * n) / G), hi = (int)(((long long)(blockIdx.x + 1) * n) / G);
    double acc = 0.0;
    for (int e = 1; e <= iters; ++e) {
        double *slot = xbuf + (size_t)(e & 1) * n;
        for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) slot[i] = (double)(e + i);
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + 64 * blockIdx.x), "r"(e) : "memory");
        if (threadIdx.x < G) {
            unsigned f;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(flags + 64 * threadIdx.x) : "memory");
            } while (f < (unsigned)e);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        double v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = threadIdx.x + r * blockDim.x;
            if (i < n) v[r] = __ldcg(slot + i);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int i = threadIdx.x + r * blockDim.x;
            if (i < n) xs[i] = v[r];
        }
        __syncthreads();
        acc += xs[(e * 7) % n];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) sink[0] = acc;
}

int main() {
    double *out;
    long long *cyc;
    int *iout;
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 64);
    cudaMalloc(&iout, 64);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long h;
    const char *names[] = {"dadd", "dmul", "ddiv", "shfl_f64", "shfl_f64+dadd", "ddiv_spec"};
    printf("{\"sm_count\": %d, \"clock_khz\": %d", sms, clk_khz);
    for (int w = 0; w < 6; ++w) {
        const int iters = 100000;
        chain_kernel<<<1, 32>>>(w, iters, 1.5, out, cyc);
        chain_kernel<<<1, 32>>>(w, iters, 1.5, out, cyc);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf(", \"%s_cyc\": %.2f", names[w], (double)h / iters);
    }
    lds_chain<<<1, 32>>>(100000, cyc, iout);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf(", \"lds_cyc\": %.2f", (double)h / 100000);
    Consts c{17639559.011024725, 88197.79505512363, 200.0, 416.12543922361147,
             134.86812645902467, 0.288, 1.0, 1.0, 1.0, 0.0, 6.123234e-17};
    rk4_chain<<<1, 1>>>(100000, c, 1e-11, out, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    rk4_chain<<<1, 1>>>(100000, c, 1e-11, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf(", \"rk4_step_cyc\": %.1f, \"rk4_step_ns\": %.1f", (double)h / 100000, ms * 1e6 / 100000);
    rk4_chain_spec<<<1, 1>>>(100000, c, 1e-11, out, cyc);
    cudaEventRecord(a);
    rk4_chain_spec<<<1, 1>>>(100000, c, 1e-11, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double hr[2];
    cudaMemcpy(hr, out, 16, cudaMemcpyDeviceToHost);
    printf(", \"rk4_step_spec_cyc\": %.1f, \"rk4_step_spec_ns\": %.1f, \"rk4_spec_replays\": %.0f",
           (double)h / 100000, ms * 1e6 / 100000, hr[1]);

    unsigned long long *bar;
    cudaMalloc(&bar, 64);
    for (int g : {1, 16, 74, 148}) {
        const int iters = 20000;
        cudaMemset(bar, 0, 8);
        void *args[] = {(void *)&iters, (void *)&bar, (void *)&cyc};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)barrier_kernel, g, 512, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf(", \"barrier_g%d_ns\": %.1f", g, ms * 1e6 / iters);
    }
    for (int g : {1, 148}) {
        const int iters = 20000;
        cudaMemset(bar, 0, 8);
        void *args[] = {(void *)&iters, (void *)&bar, (void *)&cyc};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)barrier2_kernel, g, 512, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf(", \"barrier2_g%d_ns\": %.1f", g, ms * 1e6 / iters);
    }
    double *xb;
    cudaMalloc(&xb, 2 * 148 * 64 * 8);
    cudaFuncSetAttribute(barrier_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 64 * 8);
    cudaFuncSetAttribute(ll_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 148 * 64 * 8);
    for (int per : {1, 7, 68}) {
        const int iters = 20000, g = 148;
        cudaMemset(bar, 0, 8);
        void *args[] = {(void *)&iters, (void *)&per, (void *)&bar, (void *)&xb};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void *)barrier_copy_kernel, g, 512, args, g * per * 8, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf(", \"barrier_copy_g148_per%d_ns\": %.1f", per, ms * 1e6 / iters);
    }
    uint4 *llbuf;
    cudaMalloc(&llbuf, 2 * 148 * 68 * sizeof(uint4));
    for (int g : {16, 74, 148}) {
        for (int per : {1, 7, 68}) {
            const int iters = 20000;
            cudaMemset(llbuf, 0, 2 * 148 * 68 * sizeof(uint4));
            int n = g * per;
            void *args[] = {(void *)&iters, (void *)&per, (void *)&llbuf, (void *)&cyc, (void *)&out};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void *)ll_kernel, g, 512, args, n * 8, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf(", \"ll_g%d_per%d_ns\": %.1f", g, per, ms * 1e6 / iters);
        }
    }
    {
        uint4 *b2;
        unsigned *fl;
        cudaMalloc(&b2, 2 * 4096 * sizeof(uint4));
        cudaMalloc(&fl, 64 * 1024 * 4);
        cudaFuncSetAttribute(ll2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8);
        cudaFuncSetAttribute(flag_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 8);
        for (int g : {16, 64, 125, 148}) {
            for (int n : {128, 1000, 2000}) {
                const int iters = 20000;
                cudaMemset(b2, 0, 2 * 4096 * sizeof(uint4));
                void *args[] = {(void *)&iters, (void *)&n, (void *)&b2, (void *)&out};
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void *)ll2_kernel, g, 512, args, n * 8, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                printf(", \"ll2_g%d_n%d_ns\": %.1f", g, n, ms * 1e6 / iters);
                cudaMemset(fl, 0, 64 * 1024 * 4);
                double *xb2 = (double *)b2;
                void *args2[] = {(void *)&iters, (void *)&n, (void *)&fl, (void *)&xb2, (void *)&out};
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void *)flag_copy_kernel, g, 512, args2, n * 8, 0);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
                printf(", \"flagcopy_g%d_n%d_ns\": %.1f", g, n, ms * 1e6 / iters);
            }
        }
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf(", \"error\": \"%s\"}\n", cudaGetErrorString(err));
    return 0;
}
