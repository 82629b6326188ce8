// sto_build.cuh -- reservoir construction on the device.
//
// The reference builds W on the host (`spinosc/topology.py`): PCG64 draws
// (`RngStream.uniform_pm1`, :48-54) placed row-major on the off-diagonal
// (:255-257), then divided by the spectral radius from a restarted Arnoldi
// iteration (:146-238) whose cost is a few hundred dense matvecs -- 173 s at
// N = 2e4.  Here:
//  * pcg64_fill_kernel reproduces numpy's Generator(PCG64(seed)).random()
//    stream bit for bit (PCG-XSL-RR 128/64: state = state * M + inc, output
//    rotr64(hi ^ lo, state >> 122); double = (x >> 11) * 2^-53; value =
//    2u - 1).  Lane l of a warp jumps once to draw d0 + l (O(log d) LCG
//    jump-ahead), then strides by 32 draws with the precomputed 32-step
//    affine map, so every warp store is 32 consecutive doubles.
//  * gemv_kernel: y = W x for the Arnoldi matvecs (one warp per row, 16-byte
//    coalesced loads, HBM-bound).  Its summation order is not BLAS's -- nor
//    is the reference's BLAS order pinned (W bits depend on the BLAS build,
//    SURVEY §8(c)) -- so a device-built W matches the host build to the last
//    few ulps of rho, and its draws exactly.
//  * scale_div_kernel: W /= rho elementwise (IEEE division, as `entries /=
//    rho`).
#pragma once

#include <cstdint>

namespace sto {

using u128 = unsigned __int128;

struct Pcg64 {
    u128 state, inc;
};

__host__ __device__ constexpr u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

// affine map of `delta` LCG steps: state -> a * state + c
__host__ __device__ inline void pcg_jump_coeffs(u128 inc, unsigned long long delta, u128 &a, u128 &c) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta) {
        if (delta & 1ull) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    a = acc_mult;
    c = acc_plus;
}

__host__ __device__ inline unsigned long long pcg_output(u128 state) {
    const unsigned long long x = (unsigned long long)(state >> 64) ^ (unsigned long long)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Draw d (0-based) of the stream: state after d+1 steps, then output.
// pm1: 2u - 1 with u = (x >> 11) * 2^-53 (exact in binary64).
__device__ __forceinline__ double pcg_pm1(u128 state) {
    const double u = (double)(pcg_output(state) >> 11) * 0x1.0p-53;
    return __dsub_rn(__dmul_rn(2.0, u), 1.0);
}

// out[i] = draw(offset + i) for i < count, or, when diag_n > 0, the draws
// 0 .. n(n-1)-1 placed row-major on the off-diagonal of an n x n matrix with
// leading dimension ld (diagonal written 0).
__global__ void pcg64_fill_kernel(double *__restrict__ out, long long count, long long offset,
                                  Pcg64 g, long long diag_n, long long ld, u128 a32, u128 c32) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = (((count + nwarps - 1) / nwarps) + 31) / 32 * 32;  // draws per warp
    const long long d_begin = warp * per, d_end = min(count, d_begin + per);
    if (d_begin >= d_end) return;
    u128 a, c;
    pcg_jump_coeffs(g.inc, (unsigned long long)(offset + d_begin + lane + 1), a, c);
    u128 s = a * g.state + c;  // state producing draw offset + d_begin + lane
    if (diag_n <= 0) {
        for (long long d = d_begin + lane; d < d_end; d += 32) {
            out[d] = pcg_pm1(s);
            s = a32 * s + c32;
        }
        return;
    }
    const long long n1 = diag_n - 1;
    long long d = d_begin + lane;
    long long row = d / n1, c0 = d - row * n1;
    for (; d < d_end; d += 32) {
        const long long col = c0 + (c0 >= row);
        out[row * ld + col] = pcg_pm1(s);
        s = a32 * s + c32;
        c0 += 32;
        while (c0 >= n1) {
            c0 -= n1;
            ++row;
        }
    }
}

__global__ void zero_diag_kernel(double *__restrict__ w, long long n, long long ld) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        w[i * ld + i] = 0.0;
}

// y[r] = sum_j w[r, j] x[j]; one warp per row, 16-byte loads when aligned.
__global__ void gemv_kernel(const double *__restrict__ w, long long rows, long long cols, long long ld,
                            const double *__restrict__ x, double *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const bool vec = (ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
    for (long long r = warp; r < rows; r += nwarps) {
        const double *wr = w + r * ld;
        double acc = 0.0;
        if (vec) {
            const long long c2 = cols / 2;
            for (long long j = lane; j < c2; j += 32) {
                const double2 wv = __ldcs(reinterpret_cast<const double2 *>(wr) + j);
                const double2 xv = __ldg(reinterpret_cast<const double2 *>(x) + j);
                acc = fma(wv.x, xv.x, acc);
                acc = fma(wv.y, xv.y, acc);
            }
            if ((cols & 1) && lane == 0) acc = fma(wr[cols - 1], x[cols - 1], acc);
        } else {
            for (long long j = lane; j < cols; j += 32) acc = fma(wr[j], x[j], acc);
        }
#pragma unroll
        for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
        if (lane == 0) y[r] = acc;
    }
}

__global__ void scale_div_kernel(double *__restrict__ a, long long count, double divisor) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        a[i] = __ddiv_rn(a[i], divisor);
}

}  // namespace sto
