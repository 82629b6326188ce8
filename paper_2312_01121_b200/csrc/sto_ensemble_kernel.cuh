// sto_ensemble_kernel.cuh -- batched ensemble (BASELINE configs[3]): B
// independent reservoirs that share W and W_in but not their parameters
// (e.g. a sweep over the drive current), stepped together so the coupling
// becomes a GEMM:  CP[k][b] = sum_j W[k][j] * X[j][b]   (X = member x-vectors).
//
// The GEMM runs on the FP64 tensor cores: mma.sync.aligned.m8n8k4 .f64
// (SASS DMMA.8x8x4 -- sm_100 has no tcgen05 f64 kind; DMMA is its fp64
// tensor path, measured 37.1 TFLOP/s vs 34.0 for DFMA, tools/fp64_peak.cu).
// Its accumulation order is not the reference's pinned tree, so this path is
// held to a tolerance (<= 1e-10 at 1e3 steps, per member,
// against the oracle run with that member's parameters), not bit-equality.
//
// Tiling: one CTA per 64-row x 64-member output tile (N = 1000, B = 512 ->
// 16 x 8 = 128 CTAs); 16 warps, each a 16 x 16 region = 2 x 2 DMMA tiles fed
// by 2 A + 2 B fragments per k-step (256 B of shared-memory operand traffic
// per DMMA; 8 warps of 16 x 32 tiles measured slower: too little latency
// hiding for the DMMA chains); K streamed
// in 64-column chunks through a 3-stage cp.async pipeline (68-double padded
// rows: conflict-free fragment loads).  The RK4 epilogue re-maps the
// accumulators through shared memory so that consecutive threads own
// consecutive members: the per-(row, member) RK state (m, s, acc, k3, cin),
// kept in L2-resident global SoA arrays, is then read and written with
// coalesced, batched loads.  Members of different 64-member
// columns never interact, so the per-stage exchange is a barrier among the
// CTAs of one column only.
#pragma once

#include "sto_kernels.cuh"

namespace sto {

constexpr int kEnsRT = 64;      // rows per CTA tile
constexpr int kEnsBT = 64;      // members per CTA tile
constexpr int kEnsKC = 64;      // K chunk
constexpr int kEnsLD = kEnsKC + 4;  // padded smem row (doubles)
constexpr int kEnsThreads = 512;    // 16 warps = 4 row groups (16) x 4 member quarters (16)
constexpr int kEnsState = 13;       // m, s, acc, k3 (3 each) + cin
constexpr int kEnsStages = 3;       // cp.async pipeline depth
constexpr int kEnsBuf = (kEnsRT + kEnsKC) * kEnsLD;  // one stage: W tile + X tile
constexpr int kEnsSmemDoubles = kEnsStages * kEnsBuf + kEnsBT * 11;

struct EnsParams {
    int n, np, kp;                // oscillators; rows padded to kEnsRT; K padded to kEnsKC
    int batch, bp;                // members, padded to kEnsBT
    int member0;                  // first member of this launch (host chunking)
    int n_in;
    const double *w;              // np x kp row-major, zero padded
    const double *w_in;           // n x n_in
    const double *consts;         // (batch, 11)
    double *m;                    // (batch, n, 3) in/out
    const double *samples;        // drive; member b uses samples + b * sample_member_stride
    long long sample_member_stride;
    long long n_samples, sps;
    double dt, h2, dt6;
    long long steps, stride, n_records;
    double *states;               // (n_records, batch, n, 3) or null
    double *x;                    // [2][kp][bp] stage x
    double *st;                   // [13][np][bp] RK state (SoA)
    unsigned long long *bar;      // per member-column counters, 32 words apart
    StatusDev *status;
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void column_sync(unsigned long long *bar, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        unsigned long long v;
        do {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

#ifdef STO_TIMELINE
__device__ unsigned long long g_ens_timeline[16][4];
#define ENS_TL(e, ev)                                                                 \
    do {                                                                              \
        if (blockIdx.x == 0 && threadIdx.x == 0 && (e) >= 40 && (e) < 56)             \
            g_ens_timeline[(e) - 40][ev] = clock64();                                 \
    } while (0)
#else
#define ENS_TL(e, ev)
#endif

__global__ void __launch_bounds__(kEnsThreads, 1) ens_rk4_kernel(const __grid_constant__ EnsParams p) {
    extern __shared__ __align__(16) double smem[];
    double *cs = smem + kEnsStages * kEnsBuf;  // [64][11] member consts

    const int n_rt = p.np / kEnsRT;
    const int rt = blockIdx.x % n_rt, ct = blockIdx.x / n_rt;  // row tile, member column
    const int row0 = rt * kEnsRT, col0 = ct * kEnsBT;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wr = warp >> 2, wc = warp & 3;  // 4 row groups (16) x 4 member quarters (16)
    const int g = lane >> 2, t = lane & 3;
    unsigned long long *bar = p.bar + 32 * ct;
    const size_t plane = (size_t)p.np * p.bp;   // one SoA state component
    const size_t xplane = (size_t)p.kp * p.bp;  // one x buffer

    for (int i = threadIdx.x; i < kEnsBT * 11; i += blockDim.x) {
        const int bl = i / 11, q = i % 11;
        const int b = min(p.member0 + col0 + bl, p.batch - 1);
        cs[i] = p.consts[(size_t)b * 11 + q];
    }
    // ---- prologue: state and x(0) from m, record 0 -------------------------
    for (int i = threadIdx.x; i < kEnsRT * kEnsBT; i += blockDim.x) {
        const int rl = i / kEnsBT, bl = i % kEnsBT;
        const int k = row0 + rl, bg = col0 + bl, b = p.member0 + bg;
        double mx = 0.0, my = 0.0, mz = 0.0;
        if (k < p.n && b < p.batch) {
            const double *mm = p.m + ((size_t)b * p.n + k) * 3;
            mx = mm[0];
            my = mm[1];
            mz = mm[2];
            if (p.states) {
                double *so = p.states + ((size_t)b * p.n + k) * 3;
                so[0] = mx;
                so[1] = my;
                so[2] = mz;
            }
        }
        const size_t o = (size_t)k * p.bp + bg;
        p.st[0 * plane + o] = mx;
        p.st[1 * plane + o] = my;
        p.st[2 * plane + o] = mz;
        if (k < p.kp) p.x[o] = mx;  // parity 0 (rows >= n stay zero)
    }
    const int n_chunks = p.kp / kEnsKC;
    long long epoch = 0;
    column_sync(bar, (unsigned long long)(++epoch) * n_rt);

    long long next_rec = p.stride, rec_idx = 1;
    for (long long step = 1; step <= p.steps; ++step) {
        const bool record = (step == next_rec) || (step == p.steps);
        const long long sidx = p.n_samples == 1 ? 0 : (step - 1) / p.sps;
        for (int stage = 0; stage < 4; ++stage) {
            const double *xsrc = p.x + (size_t)((epoch - 1) & 1) * xplane;  // published last stage
            ENS_TL(epoch, 0);
            double acc[2][2][2];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
            // ---- 3-stage cp.async pipeline over K --------------------------
            auto load_chunk = [&](int c) {
                double *ws = smem + (c % kEnsStages) * kEnsBuf;
                double *xs = ws + kEnsRT * kEnsLD;
                const int k0 = c * kEnsKC;
                for (int i = threadIdx.x; i < (kEnsRT + kEnsKC) * 32; i += blockDim.x) {
                    const int r = i >> 5, c2 = (i & 31) * 2;
                    if (r < kEnsRT)
                        cp_async16(ws + r * kEnsLD + c2, p.w + (size_t)(row0 + r) * p.kp + k0 + c2);
                    else
                        cp_async16(xs + (r - kEnsRT) * kEnsLD + c2,
                                   xsrc + (size_t)(k0 + r - kEnsRT) * p.bp + col0 + c2);
                }
            };
#pragma unroll
            for (int c = 0; c < kEnsStages - 1; ++c) {
                if (c < n_chunks) load_chunk(c);
                cp_async_commit();
            }
            for (int c = 0; c < n_chunks; ++c) {
                asm volatile("cp.async.wait_group %0;" ::"n"(kEnsStages - 2) : "memory");
                __syncthreads();  // chunk c landed for everyone; chunk c-1 fully consumed
                if (c + kEnsStages - 1 < n_chunks) load_chunk(c + kEnsStages - 1);
                cp_async_commit();
                const double *W = smem + (c % kEnsStages) * kEnsBuf;
                const double *X = W + kEnsRT * kEnsLD;
#pragma unroll 4
                for (int kk = 0; kk < kEnsKC / 4; ++kk) {
                    const double a0 = W[(wr * 16 + g) * kEnsLD + kk * 4 + t];
                    const double a1 = W[(wr * 16 + 8 + g) * kEnsLD + kk * 4 + t];
                    const double *xr = X + (kk * 4 + t) * kEnsLD + wc * 16 + g;
                    const double b[2] = {xr[0], xr[8]};
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        dmma(acc[0][jj][0], acc[0][jj][1], a0, b[jj]);
                        dmma(acc[1][jj][0], acc[1][jj][1], a1, b[jj]);
                    }
                }
            }
            cp_async_wait_0();
            __syncthreads();
            ENS_TL(epoch, 1);
            // ---- RK4 epilogue ------------------------------------------------
            // accumulators -> shared [row][member] (pipeline buffers are idle now)
            double *cpb = smem;  // 64 x kEnsLD
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) {
                    const int rl = wr * 16 + i * 8 + g, bl = wc * 16 + jj * 8 + 2 * t;
                    cpb[rl * kEnsLD + bl] = acc[i][jj][0];
                    cpb[rl * kEnsLD + bl + 1] = acc[i][jj][1];
                }
            __syncthreads();
            double *xdst = p.x + (size_t)(epoch & 1) * xplane;
            // thread -> (row, member) with members fastest: coalesced SoA state
#pragma unroll 2
            for (int idx = threadIdx.x; idx < kEnsRT * kEnsBT; idx += blockDim.x) {
                const int rl = idx / kEnsBT, bl = idx % kEnsBT;
                const int k = row0 + rl, bg = col0 + bl, b = p.member0 + bg;
                if (k >= p.n || b >= p.batch) continue;
                const size_t o = (size_t)k * p.bp + bg;
                const double *cc = cs + bl * 11;
                const Consts c{cc[0], cc[1], cc[2], cc[3], cc[4], cc[5],
                               cc[6], cc[7], cc[8], cc[9], cc[10]};
                // batch every state load of this output before the arithmetic
                const V3 m{p.st[0 * plane + o], p.st[1 * plane + o], p.st[2 * plane + o]};
                V3 cur = m, a{0.0, 0.0, 0.0}, q{0.0, 0.0, 0.0};
                if (stage > 0) cur = V3{p.st[3 * plane + o], p.st[4 * plane + o], p.st[5 * plane + o]};
                if (stage == 1 || stage == 3)
                    a = V3{p.st[6 * plane + o], p.st[7 * plane + o], p.st[8 * plane + o]};
                if (stage == 3) q = V3{p.st[9 * plane + o], p.st[10 * plane + o], p.st[11 * plane + o]};
                double cin;
                if (stage == 0) {
                    const double *u = p.samples + (size_t)b * p.sample_member_stride +
                                      (size_t)sidx * p.n_in;
                    cin = (p.n_in == 1) ? rmul(p.w_in[k], u[0])
                                        : tree_dot_stream(p.w_in + (size_t)k * p.n_in, u, p.n_in);
                    p.st[12 * plane + o] = cin;
                } else {
                    cin = p.st[12 * plane + o];
                }
                const V3 d = row_rhs(cur, cpb[rl * kEnsLD + bl], cin, c);
                double xpub;
                if (stage < 3) {
                    if (stage == 0) {
                        p.st[6 * plane + o] = d.x;
                        p.st[7 * plane + o] = d.y;
                        p.st[8 * plane + o] = d.z;
                    } else if (stage == 1) {
                        const V3 a2 = acc_k2(a, d);
                        p.st[6 * plane + o] = a2.x;
                        p.st[7 * plane + o] = a2.y;
                        p.st[8 * plane + o] = a2.z;
                    } else {
                        p.st[9 * plane + o] = d.x;
                        p.st[10 * plane + o] = d.y;
                        p.st[11 * plane + o] = d.z;
                    }
                    const V3 sp = stage_point(m, d, stage == 2 ? p.dt : p.h2);
                    p.st[3 * plane + o] = sp.x;
                    p.st[4 * plane + o] = sp.y;
                    p.st[5 * plane + o] = sp.z;
                    xpub = sp.x;
                } else {
                    const V3 mn = rk4_final(m, a, q, d, p.dt6);
                    p.st[0 * plane + o] = mn.x;
                    p.st[1 * plane + o] = mn.y;
                    p.st[2 * plane + o] = mn.z;
                    xpub = mn.x;
                    if (record) {
                        if (!all_finite(mn)) {
                            // key: step, member, oscillator (lexicographic min)
                            atomicMin(&p.status->key, (step << 40) | ((long long)b << 20) | k);
                            p.status->flag = 1;
                        } else if (p.states) {
                            const long long ri = (step == next_rec) ? rec_idx : p.n_records - 1;
                            double *so = p.states + (((size_t)ri * p.batch + b) * p.n + k) * 3;
                            so[0] = mn.x;
                            so[1] = mn.y;
                            so[2] = mn.z;
                        }
                    }
                }
                xdst[o] = xpub;
            }
            ENS_TL(epoch, 2);
            ++epoch;
            if (!(step == p.steps && stage == 3)) column_sync(bar, (unsigned long long)epoch * n_rt);
            ENS_TL(epoch - 1, 3);
        }
        if (record && step == next_rec) {
            next_rec += p.stride;
            ++rec_idx;
        }
    }
    // ---- epilogue: final m ------------------------------------------------
    __syncthreads();
    for (int i = threadIdx.x; i < kEnsRT * kEnsBT; i += blockDim.x) {
        const int rl = i / kEnsBT, bl = i % kEnsBT;
        const int k = row0 + rl, bg = col0 + bl, b = p.member0 + bg;
        if (k < p.n && b < p.batch) {
            const size_t o = (size_t)k * p.bp + bg;
            double *mm = p.m + ((size_t)b * p.n + k) * 3;
            mm[0] = p.st[0 * plane + o];
            mm[1] = p.st[1 * plane + o];
            mm[2] = p.st[2 * plane + o];
        }
    }
}

}  // namespace sto
