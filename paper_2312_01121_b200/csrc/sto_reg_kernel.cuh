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
//   grid: leaders store x (logical order) to a double-buffered global vector,
//   the CTA raises its flag with st.release.gpu; thread t < G polls flag t
//   (relaxed loads + one acquire fence) and copies producer t's rows into
//   shared memory -- one flag per producer instead of one contended counter.
//   A diverged record step is signalled in the flag's top bit, so every CTA
//   takes the same decision to stop after the same exchange.
#pragma once

#include "sto_kernels.cuh"

namespace sto {


struct RegParams {
    KParams k;              // shared fields (consts, run, states, status ...)
    unsigned *flags;        // [G] per-CTA epoch flags (zeroed before launch)
    double *xg;             // [2][n] published x, logical order
};

// shared-memory position of logical column `col` (team-blocked: a 16-byte
// load i by team thread j returns columns C*j + 2i, +1)
template <int C>
__device__ __forceinline__ int reg_xpos(int col, int T) {
    const int j = col / C, q = col % C;
    return (((q >> 1) * T + j) << 1) + (q & 1);
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int T, int C, bool SINGLE>
__global__ void __launch_bounds__(512, 1) reg_rk4_kernel(const __grid_constant__ RegParams rp) {
    constexpr int P = T * C;
    constexpr int LV = (C == 32) ? 5 : 4;  // tree levels above the products
    const KParams &p = rp.k;
    extern __shared__ __align__(16) double smem[];
    double *xs = smem;            // P doubles, team-blocked
    const int teams = blockDim.x / T;
    double *part = xs + P;        // T == 64: two warp nodes per team
    RowState rs{part + 2 * teams, teams};  // leader RK state (m, s, acc, k3, cin)
    volatile int *sstop = reinterpret_cast<volatile int *>(rs.base + 13 * teams);

    const int G = gridDim.x, b = blockIdx.x;
    const int n = p.rows;
    const int r0 = row_lo(b, G, n), nrow = row_lo(b + 1, G, n) - r0;
    const int team = threadIdx.x / T, j = threadIdx.x % T;
    const bool active = team < nrow;
    const bool leader = active && j == 0;
    const int k = r0 + team;  // oscillator owned by this team

    // ---- W chunk into registers (device layout -> logical columns) ---------
    double w[C];
#pragma unroll
    for (int q = 0; q < C; ++q) {
        const int col = j * C + q;
        w[q] = (active && col < n) ? p.w[(size_t)k * p.cs.ldw + col_perm(p.cs, col)] : -0.0;
    }
    // ---- initial x (all of m0), leader state --------------------------------
    for (int i = threadIdx.x; i < P; i += blockDim.x) xs[i] = 0.0;
    __syncthreads();
    for (int col = threadIdx.x; col < n; col += blockDim.x) xs[reg_xpos<C>(col, T)] = p.m[3 * (size_t)col];
    if (leader) {
        const V3 m{p.m[3 * (size_t)k], p.m[3 * (size_t)k + 1], p.m[3 * (size_t)k + 2]};
        rs.put(kSlotM, team, m);
        if (p.states) {
            double *st = p.states + 3 * (size_t)k;
            st[0] = m.x;
            st[1] = m.y;
            st[2] = m.z;
        }
    }
    if (threadIdx.x == 0) *sstop = 0;
    __syncthreads();

    const double *u = p.samples;
    long long next_rec = p.stride;  // next step on the recording grid
    long long rec_idx = 1;
    unsigned epoch = 0;
    bool stop = false;
    for (long long step = 1; step <= p.steps && !stop; ++step) {
        if (leader)
            rs.cin(team) = (p.n_in == 1) ? rmul(p.w_in[k], u[0])
                                         : tree_dot_stream(p.w_in + (size_t)k * p.n_in, u, p.n_in);
        const bool record = (step == next_rec) || (step == p.steps);
#pragma unroll 1
        for (int stage = 0; stage < 4; ++stage) {
            // -------- team GEMV: cp = pinned tree of w . x ----------------
            // pinned tree of the 16 products, streamed pair by pair: the
            // unrolled binary counter merges completed siblings immediately,
            // so at most log2(16) partial nodes are live
            double lvl[LV];
#pragma unroll
            for (int i = 0; i < C / 2; ++i) {
                const double2 x2 = *reinterpret_cast<const double2 *>(xs + ((i * T + j) << 1));
                double node = radd(rmul(w[2 * i], x2.x), rmul(w[2 * i + 1], x2.y));
#pragma unroll
                for (int l = 0; l < LV - 1; ++l) {
                    if (i & (1 << l)) node = radd(lvl[l], node);
                    else { lvl[l] = node; break; }
                }
                if (i == C / 2 - 1) lvl[LV - 1] = node;
            }
            double v = lvl[LV - 1];
#pragma unroll
            for (int mask = 1; mask < (T < 32 ? T : 32); mask <<= 1)
                v = radd(v, __shfl_xor_sync(0xffffffffu, v, mask));
            if constexpr (T == 64) {
                if ((threadIdx.x & 31) == 0) part[2 * team + ((threadIdx.x >> 5) & 1)] = v;
            }
            __syncthreads();  // all reads of xs done (and warp halves merged)
            // -------- leader: RHS + RK4 stage update -----------------------
            double xpub = 0.0;
            bool bad = false;
            if (leader) {
                const double cp = (T == 64) ? radd(part[2 * team], part[2 * team + 1]) : v;
                const V3 m = rs.get(kSlotM, team);
                const V3 cur = (stage == 0) ? m : rs.get(kSlotS, team);
                const V3 d = row_rhs(cur, cp, rs.cin(team), p.c);
                if (stage == 0) {
                    rs.put(kSlotAcc, team, d);
                    const V3 s = stage_point(m, d, p.h2);
                    rs.put(kSlotS, team, s);
                    xpub = s.x;
                } else if (stage == 1) {
                    rs.put(kSlotAcc, team, acc_k2(rs.get(kSlotAcc, team), d));
                    const V3 s = stage_point(m, d, p.h2);
                    rs.put(kSlotS, team, s);
                    xpub = s.x;
                } else if (stage == 2) {
                    rs.put(kSlotK3, team, d);
                    const V3 s = stage_point(m, d, p.dt);
                    rs.put(kSlotS, team, s);
                    xpub = s.x;
                } else {
                    const V3 mn = rk4_final(m, rs.get(kSlotAcc, team), rs.get(kSlotK3, team), d, p.dt6);
                    rs.put(kSlotM, team, mn);
                    xpub = mn.x;
                    if (record) {
                        if (!all_finite(mn)) {
                            bad = true;
                            report_divergence(p.status, step, k);
                        } else if (p.states) {
                            const long long ri = (step == next_rec) ? rec_idx : p.n_records - 1;
                            double *st = p.states + ((size_t)ri * n + k) * 3;
                            st[0] = mn.x;
                            st[1] = mn.y;
                            st[2] = mn.z;
                        }
                    }
                }
            }
            const bool last = (step == p.steps) && stage == 3;
            if constexpr (SINGLE) {
                if (leader) xs[reg_xpos<C>(k, T)] = xpub;
                if (bad) *sstop = 1;
                __syncthreads();
                if (*sstop) stop = true;
            } else {
                if (leader) rp.xg[(size_t)((epoch + 1) & 1) * n + k] = xpub;
                if (bad) *sstop = 1;
                __syncthreads();
                ++epoch;
                if (!last) {
                    if (threadIdx.x == 0)
                        st_release_u32(rp.flags + b, epoch | (*sstop ? 0x80000000u : 0u));
                    if (threadIdx.x < G) {
                        const int t = threadIdx.x;
                        unsigned f;
                        do {
                            f = ld_relaxed_u32(rp.flags + t);
                        } while ((f & 0x7fffffffu) < epoch);
                        asm volatile("fence.acq_rel.gpu;" ::: "memory");
                        if (f & 0x80000000u) *sstop = 1;
                        const int lo = row_lo(t, G, n), hi = row_lo(t + 1, G, n);
                        const double *src = rp.xg + (size_t)(epoch & 1) * n;
                        for (int c = lo; c < hi; ++c) xs[reg_xpos<C>(c, T)] = ld_cg(src + c);
                    }
                    __syncthreads();
                    if (*sstop) stop = true;
                }
            }
            if (stop) break;
        }
        if (record && step == next_rec) {
            next_rec += p.stride;
            ++rec_idx;
        }
        if (p.n_samples > 1) u = p.samples + (step / p.sps) * p.n_in;
    }
    if (leader) {
        const V3 m = rs.get(kSlotM, team);
        double *mm = p.m + 3 * (size_t)k;
        mm[0] = m.x;
        mm[1] = m.y;
        mm[2] = m.z;
    }
}

}  // namespace sto
