// sto_reg_kernel.cuh -- on-chip regime (n <= 1024): W held in REGISTERS.
//
// The chip's register file (148 SMs x 256 KB = 37.9 MB) holds an fp64 W of
// n = 1024 (8 MB) several times over, so for the latency-bound sizes every
// row is owned by a "team" of T threads for the whole run: thread j of the
// team keeps columns [16j, 16j+16) of its row in 32 registers, loaded once.
// A stage is then
//   products with the x-vector (shared memory, team-blocked so that team
//   lanes read consecutive 16-byte words) -> in-register pinned tree of 16
//   -> xor butterfly over the team (-> shared-memory pair merge when T = 64)
//   -> team leader: LLG right-hand side, RK4 stage update, x publication.
// The row is padded to P = 16*T (a power of two) with W = -0.0 and x = +0.0,
// so the tree is the reference's padded aligned tree (bit-exact).
//
// Exchange of the stage x-vector:
//   SINGLE (one CTA, n <= 128): leaders write x straight into shared memory.
//   grid: "LL" all-gather through L2.  Each leader stores its x as one 16-byte
//   word {lo32, epoch, hi32, epoch} (8-byte halves are single-copy atomic, so
//   a reader that sees the epoch in both halves holds the matching data);
//   every CTA reads the whole double-buffered vector with pipelined relaxed
//   loads, retrying only stale entries.  One L2 round trip per exchange, no
//   counter, no fence (measured 1.0 us at 125 CTAs x 1000 entries vs 2.1 us
//   for flag + copy, tools/microbench.cu).  A row that diverged on a
//   recording step sets the top bit of its epoch words, so every CTA takes
//   the same decision to stop after the same exchange.
#pragma once

#include "sto_kernels.cuh"

namespace sto {



struct RegParams {
    KParams k;              // shared fields (consts, run, states, status ...)
    uint4 *ll;              // [2][n] LL words of the published x (zeroed before launch)
    unsigned epoch0;        // first exchange epoch - 1 (0; STO_REG_EPOCH0 tests the wrap)
};

constexpr int kLLMaxPerThread = 4;  // n <= 4 * 512

// shared-memory position of logical column `col` (team-blocked: a 16-byte
// load i by team thread j returns columns C*j + 2i, +1)
template <int C>
__device__ __forceinline__ int reg_xpos(int col, int T) {
    const int j = col / C, q = col % C;
    return (((q >> 1) * T + j) << 1) + (q & 1);
}

__device__ __forceinline__ void st_ll(uint4 *p, double v, unsigned flag) {
    const unsigned long long b = __double_as_longlong(v);
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "r"((unsigned)b), "r"(flag), "r"((unsigned)(b >> 32)), "r"(flag)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_ll(const uint4 *p) {
    uint4 q;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                 : "l"(p));
    return q;
}

#ifdef STO_TIMELINE
// debug build only (tools/timeline.py): globaltimer stamps of CTA 0 and the
// last CTA for stages [kTlFirst, kTlFirst + kTlStages)
constexpr int kTlFirst = 400, kTlStages = 16, kTlEvents = 5;
__device__ unsigned long long g_timeline[2][kTlStages][kTlEvents];
__device__ __forceinline__ void tl_mark(long long e, int ev) {
    const int who = blockIdx.x == 0 ? 0 : (blockIdx.x == gridDim.x - 1 ? 1 : -1);
    if (who >= 0 && threadIdx.x == 0 && e >= kTlFirst && e < kTlFirst + kTlStages) {
        unsigned long long t;
        t = clock64();
        g_timeline[who][e - kTlFirst][ev] = t;
    }
}
#define TL(e, ev) tl_mark((e), (ev))
#else
#define TL(e, ev)
#endif

template <int T, int C, int R, bool SINGLE>
__global__ void __launch_bounds__(R == 2 ? 256 : 512, 1) reg_rk4_kernel(const __grid_constant__ RegParams rp) {
    constexpr int P = T * C;
    constexpr int LV = (C == 32) ? 5 : 4;  // tree levels above the products
    const KParams &p = rp.k;
    extern __shared__ __align__(16) double smem[];
    const int teams = blockDim.x / T;
    double *xs = smem;                       // P doubles, team-blocked
    double *cps = xs + P;                    // [teams * R][2] row sums (two warp halves if T = 64)
    volatile int *sstop = reinterpret_cast<volatile int *>(cps + 2 * R * teams);

    const int G = gridDim.x, b = blockIdx.x;
    const int n = p.rows;
    const int r0 = row_lo(b, G, n), nrow = row_lo(b + 1, G, n) - r0;
    // GEMV role: team `team`, member j -- columns [C*j, C*j + C) of rows
    // r0 + R*team + i (i < R): every x value loaded from shared memory feeds R rows
    const int team = threadIdx.x / T, j = threadIdx.x % T;
    // RHS role: thread r < nrow owns oscillator r0 + r for the whole run, its
    // RK state lives in registers and the RHS work is packed into few warps
    const int r = threadIdx.x;
    const bool owner = r < nrow;
    const int k = r0 + r;

    double w[R][C];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int row = R * team + i;
#pragma unroll
        for (int q = 0; q < C; ++q) {
            const int col = j * C + q;
            w[i][q] = (row < nrow && col < n)
                          ? p.w[(size_t)(r0 + row) * p.cs.ldw + col_perm(p.cs, col)]
                          : -0.0;
        }
    }
    for (int i = threadIdx.x; i < P; i += blockDim.x) xs[i] = 0.0;
    __syncthreads();
    for (int col = threadIdx.x; col < n; col += blockDim.x)
        xs[reg_xpos<C>(col, T)] = p.m[3 * (size_t)col];
    V3 m{0.0, 0.0, 0.0}, s{0.0, 0.0, 0.0}, acc{0.0, 0.0, 0.0}, k3{0.0, 0.0, 0.0};
    if (owner) {
        m = V3{p.m[3 * (size_t)k], p.m[3 * (size_t)k + 1], p.m[3 * (size_t)k + 2]};
        if (p.states) {
            double *st = p.states + 3 * (size_t)k;
            st[0] = m.x;
            st[1] = m.y;
            st[2] = m.z;
        }
    }
    if (threadIdx.x == 0) *sstop = 0;
    __syncthreads();

    long long next_rec = p.stride;
    long long rec_idx = 1;
    unsigned epoch = rp.epoch0;
    bool stop = false;
    RhsPre pre{};
    // input field of step `st` (zero-order hold, model.py:93-149)
    auto cin_of = [&](long long st) {
        const double *us = p.n_samples > 1 ? p.samples + ((st - 1) / p.sps) * p.n_in : p.samples;
        return (p.n_in == 1) ? rmul(p.w_in[k], us[0]) : tree_dot_stream(p.w_in + (size_t)k * p.n_in, us, p.n_in);
    };
    double cin = 0.0;
    if (!SINGLE && owner) {  // step 1; later steps prepare cin and stage 0's own-state half
        cin = cin_of(1);     // during the previous step's last exchange
        pre = row_rhs_pre(m, cin, p.c);
    }
    for (long long step = 1; step <= p.steps && !stop; ++step) {
        if (SINGLE && owner) cin = cin_of(step);
        const bool record = (step == next_rec) || (step == p.steps);
#pragma unroll
        for (int stage = 0; stage < 4; ++stage) {  // unrolled: per-stage branches resolve at compile time
            [[maybe_unused]] const long long estage = (step - 1) * 4 + stage;
            TL(estage, 0);
            // -------- team GEMV: pinned tree of w . x ----------------------
            // products streamed pair by pair through an unrolled binary
            // counter: completed siblings merge at once (<= log2(C) live nodes)
            double lvl[R][LV];
#pragma unroll
            for (int i = 0; i < C / 2; ++i) {
                const double2 x2 = *reinterpret_cast<const double2 *>(xs + ((i * T + j) << 1));
#pragma unroll
                for (int rr = 0; rr < R; ++rr) {
                    double node = radd(rmul(w[rr][2 * i], x2.x), rmul(w[rr][2 * i + 1], x2.y));
#pragma unroll
                    for (int l = 0; l < LV - 1; ++l) {
                        if (i & (1 << l)) node = radd(lvl[rr][l], node);
                        else { lvl[rr][l] = node; break; }
                    }
                    if (i == C / 2 - 1) lvl[rr][LV - 1] = node;
                }
            }
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
                double v = lvl[rr][LV - 1];
#pragma unroll
                for (int mask = 1; mask < (T < 32 ? T : 32); mask <<= 1)
                    v = radd(v, __shfl_xor_sync(0xffffffffu, v, mask));
                const int row = R * team + rr;
                if (T == 64) {
                    if ((threadIdx.x & 31) == 0) cps[2 * row + ((threadIdx.x >> 5) & 1)] = v;
                } else if (j == 0) {
                    cps[2 * row] = v;
                }
            }
            __syncthreads();  // every read of xs done; row sums in cps
            TL(estage, 1);
            // -------- owners: cp-dependent half of the RHS + RK4 update -----
            double xpub = 0.0;
            bool bad = false;
            if (owner) {
                const double cp = (T == 64) ? radd(cps[2 * r], cps[2 * r + 1]) : cps[2 * r];
                // grid: own-state half was computed during the exchange; single
                // CTA (no exchange to hide behind): the whole RHS here
                const V3 d = SINGLE ? row_rhs(stage == 0 ? m : s, cp, cin, p.c)
                                    : row_rhs_post(pre, cp, p.c);
                if (stage == 0) {
                    acc = d;
                    s = stage_point(m, d, p.h2);
                    xpub = s.x;
                } else if (stage == 1) {
                    acc = acc_k2(acc, d);
                    s = stage_point(m, d, p.h2);
                    xpub = s.x;
                } else if (stage == 2) {
                    k3 = d;
                    s = stage_point(m, d, p.dt);
                    xpub = s.x;
                } else {
                    m = rk4_final(m, acc, k3, d, p.dt6);
                    xpub = m.x;
                    if (record) {
                        if (!all_finite(m)) {
                            bad = true;
                            report_divergence(p.status, step, k);
                        } else if (p.states) {
                            const long long ri = (step == next_rec) ? rec_idx : p.n_records - 1;
                            double *st = p.states + ((size_t)ri * n + k) * 3;
                            st[0] = m.x;
                            st[1] = m.y;
                            st[2] = m.z;
                        }
                    }
                }
            }
            const bool last = (step == p.steps) && stage == 3;
            if constexpr (SINGLE) {
                if (owner) xs[reg_xpos<C>(k, T)] = xpub;
                if (bad) *sstop = 1;
                TL(estage, 2);
                __syncthreads();
                TL(estage, 3);
                if (*sstop) stop = true;
            } else {
                // 31-bit epochs (bit 31 is the stop bit): after 0x7fffffff the
                // count restarts at 2, keeping the buffer parity alternating and
                // never matching a zeroed (unwritten) word; a slot is rewritten
                // every 2 stages, so a stale word can only hold epoch - 2
                if (++epoch == 0x80000000u) epoch = 2u;
                if (owner)
                    st_ll(rp.ll + (size_t)(epoch & 1) * n + k, xpub, epoch | (bad ? 0x80000000u : 0u));
                TL(estage, 2);
                if (!last) {
                    const uint4 *slot = rp.ll + (size_t)(epoch & 1) * n;
                    unsigned pending = 0, stopbit = 0;
#pragma unroll
                    for (int q = 0; q < kLLMaxPerThread; ++q)
                        if (threadIdx.x + q * blockDim.x < n) pending |= 1u << q;
                    uint4 got[kLLMaxPerThread];
                    bool first = true;
                    while (pending) {
#pragma unroll
                        for (int q = 0; q < kLLMaxPerThread; ++q)
                            if (pending & (1u << q)) got[q] = ld_ll(slot + threadIdx.x + q * blockDim.x);
                        if (first) {
                            // next stage's own-state half (its IEEE division included) is
                            // computed while the first round of exchange loads is in flight;
                            // after stage 3 that is the next step's input field and stage 0
                            if (owner) {
                                if (stage < 3) {
                                    pre = row_rhs_pre(s, cin, p.c);
                                } else {
                                    cin = cin_of(step + 1);
                                    pre = row_rhs_pre(m, cin, p.c);
                                }
                            }
                            first = false;
                        }
#pragma unroll
                        for (int q = 0; q < kLLMaxPerThread; ++q) {
                            if ((pending & (1u << q)) && (got[q].y & 0x7fffffffu) == epoch &&
                                got[q].w == got[q].y) {
                                const int c = threadIdx.x + q * blockDim.x;
                                xs[reg_xpos<C>(c, T)] = __longlong_as_double(
                                    ((unsigned long long)got[q].z << 32) | got[q].x);
                                stopbit |= got[q].y;
                                pending &= ~(1u << q);
                            }
                        }
                    }
                    if (stopbit & 0x80000000u) *sstop = 1;
                    TL(estage, 3);
                    __syncthreads();
                    TL(estage, 4);
                    if (*sstop) stop = true;
                }
            }
            if (stop) break;
        }
        if (record && step == next_rec) {
            next_rec += p.stride;
            ++rec_idx;
        }
    }
    if (owner) {
        double *mm = p.m + 3 * (size_t)k;
        mm[0] = m.x;
        mm[1] = m.y;
        mm[2] = m.z;
    }
}

}  // namespace sto
