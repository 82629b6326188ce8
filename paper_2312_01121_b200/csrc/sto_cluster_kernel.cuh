// sto_cluster_kernel.cuh -- small reservoirs (33 <= n <= 512): ONE thread-block
// cluster of K CTAs (K <= 16 -- 16 is B200's non-portable maximum -- one per SM), W held in registers, the stage
// x-vector pushed into every CTA's shared memory with `st.async` (DSMEM).
//
// The single-CTA kernel spends ~1.1 k cycles per stage on the GEMV of all n
// rows on one SM and another ~0.5 k on the full right-hand side; splitting
// the rows over a cluster divides the GEMV by K, and the exchange is ONE-WAY
// remote stores into every peer's shared memory, no barrier round trip.
//
// Row ownership follows the x layout.  The GEMV reads x "team-blocked"
// (position of column col = ((q>>1)*T + j)*2 + (q&1), j = col / C, q = col % C:
// team lane j's 16-byte loads are consecutive words, no bank conflicts).  CTA
// b owns the rows whose x POSITIONS are the segment [b*SEG, (b+1)*SEG),
// SEG = P/K <= 32 (pad positions, columns >= n, have no row and stay +0.0),
// so every CTA has the same small number of rows and one owner warp.
//
// Per stage (e = 4*(step-1) + stage):
//   GEMV warps   wait mbarrier[e&1] -> x_e complete in xs[e&1]
//                pinned tree + butterfly -> row sums -> cps, bar.arrive(1)
//   owner warp   bar.sync(1) -> cp-dependent RHS half, RK4 update -> x_{e+1}
//                -> stg, bar.arrive(2); then the own-state half of the next
//                stage's RHS (row_rhs_pre, IEEE division) while the others work
//   GEMV warps   bar.sync(2) -> warp gw sends stg to CTAs gw, gw + nGW, ...:
//                one 8-byte `st.async` per (oscillator, destination) into
//                xs[(e+1)&1] of that CTA, complete_tx on its mbarrier[(e+1)&1]
//
// Each CTA arms mbarrier[buf] with expect_tx(8 n) for the next stage right
// after waiting on the current one (the remote bytes of a phase cannot arrive
// before the CTA has completed the previous phase of that buffer: a peer can
// only publish stage e+1 after it received this CTA's stage-e values, which
// are published after this CTA's stage e-1 GEMV -- so two buffers suffice
// and no cluster barrier is needed on the hot path).  Stage e reads buffer
// e & 1 = stage & 1 (four stages per step), so the buffer index and the
// mbarrier parity are compile-time constants of the unrolled stage loop.
//
// Measured alternatives: the owner warp issuing all K stores
// itself (+10 %), 16-byte paired stores (+50 %), and one cp.async.bulk of the
// staged segment per destination (+10 %) were all slower than the fan-out.
//
// Team layout (as in sto_reg_kernel.cuh): T threads per row, C = 16/32 W
// columns per thread in registers, row padded to P = T*C with W = -0.0 /
// x = +0.0: in-register pinned tree + xor butterfly = the reference's padded
// aligned tree, bit-exact.
//
// Divergence (integrator.py:174-177): on a recording step every CTA sends,
// with the step's last x publication, one 8-byte "bad" word to slot b of every
// peer's flag array, counted on a third mbarrier (expect_tx(8 K) per recording
// step).  The flags are off the critical path: stage 0 of the next step runs
// on its x as usual, and at stage 1 -- whose x can only arrive long after the
// flags left -- every CTA waits that mbarrier, reads the K words from its own
// shared memory and takes the same stop decision (the extra stage is never
// recorded).  No cluster barrier on the hot path (a barrier.cluster per
// recording step cost ~2 k cycles: n100 at record_stride 1 ran +55 %).
#pragma once

#include "sto_reg_kernel.cuh"

namespace sto {

constexpr int kCluMaxK = 16;  // > 8: non-portable cluster size (B200 allows 16)
// stop-flag rounds: at most one per kCluFlagEvery steps (every recording step
// when the record stride is longer).  A row that diverges is reported in the
// status at its own recording step either way (the earliest step wins,
// report_divergence); the rounds only decide when the cluster stops, so a
// diverged run computes at most kCluFlagEvery unrecorded extra steps.
constexpr long long kCluFlagEvery = 64;

__device__ __forceinline__ uint32_t clu_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t clu_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t clu_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t clu_mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// 8-byte remote store into CTA-cluster shared memory, completion counted on
// the destination CTA's mbarrier (both given as cluster addresses)
__device__ __forceinline__ void clu_st_async(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void clu_bar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void clu_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Wait for a phase of a local mbarrier whose transactions are remote st.async
// stores.  Poll with a RELAXED try_wait, then one acquire fence restricted to
// shared::cluster: the data the peers' complete_tx released lands in this
// CTA's shared memory, so no L1 invalidation is needed.  (An
// `.acquire.cluster` try_wait makes ptxas put a CCTL.IVALL after EVERY poll,
// which r1's hot-line profile showed as ~11 % of the N = 100 kernel's samples.)
__device__ __forceinline__ void clu_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "CLU_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra CLU_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
    asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
}
__device__ __forceinline__ void clu_sync() {  // every thread of every CTA of the cluster
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ int clu_ld_s32(uint32_t raddr) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(raddr) : "memory");
    return v;
}

#ifdef STO_TIMELINE
// the stamp takes `after` as an operand, so it cannot be scheduled before the
// value it is meant to follow is computed
__device__ __forceinline__ void clu_tl(long long e, int ev, bool me, double after) {
    const int who = blockIdx.x == 0 ? 0 : (blockIdx.x == gridDim.x - 1 ? 1 : -1);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : "d"(after) : "memory");
    if (me && who >= 0 && e >= kTlFirst && e < kTlFirst + kTlStages) g_timeline[who][e - kTlFirst][ev] = t;
}
#define CTL(e, ev, me, after) clu_tl((e), (ev), (me), (after))
#else
#define CTL(e, ev, me, after)
#endif

// shared-memory bytes of the cluster kernel for a padded row of P columns
// (x double buffer, row sums, staging, mbarriers, flags)
__host__ __device__ constexpr size_t clu_smem_bytes(int P) {
    return sizeof(double) * (2 * (size_t)P + 32 + 2 * 32) + 2 * sizeof(unsigned long long) + 16 +
           sizeof(double) * (1 + kCluMaxK) + sizeof(unsigned long long);
}
// threads of one CTA: one owner warp (SEG <= 32 rows) + the GEMV teams
__host__ __device__ constexpr int clu_threads(int seg, int team) {
    return 32 + 32 * ((seg * team + 31) / 32);
}
// column (= oscillator) whose x sits at team-blocked position `pos`
// (inverse of reg_xpos<C>)
__device__ __forceinline__ int clu_col_at(int pos, int T, int C) {
    const int e = pos & 1, jj = (pos >> 1) % T, a = (pos >> 1) / T;
    return jj * C + 2 * a + e;
}

// 32 or 64 W columns per thread need > 128 registers: those variants run <= 288 threads
template <int T, int C>
__global__ void __launch_bounds__(C >= 32 ? 288 : 576, 1) clu_rk4_kernel(const __grid_constant__ KParams p) {
    constexpr int P = T * C;
    constexpr int LV = (C == 64) ? 6 : (C == 32) ? 5 : 4;  // tree levels above the products
    static_assert(T <= 32, "team butterfly stays inside one warp");
    extern __shared__ __align__(16) double smem[];
    double *xs = smem;        // [2][P] team-blocked x, double-buffered by stage parity
    double *cps = xs + 2 * P;  // [32] row sums, GEMV teams -> owners
    double *stg = cps + 32;    // [32] this CTA's published x, owners -> fan-out warps
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(cps + 32 + 2 * 32);
    volatile int *sbad = reinterpret_cast<volatile int *>(mbar + 2);
    volatile long long *zslot = reinterpret_cast<volatile long long *>(mbar + 3);  // always 0
    volatile int *sstop = reinterpret_cast<volatile int *>(mbar + 4);  // GEMV warps -> owners
    double *sflg = reinterpret_cast<double *>(mbar + 5);  // [K] peers' "bad" words of a recording step
    unsigned long long *fbar = mbar + 5 + kCluMaxK;       // mbarrier counting those words

    const int K = (int)clu_size(), b = (int)clu_rank();
    const int n = p.rows;
    const int SEG = P / K;  // x positions (rows) owned by this CTA: [b*SEG, (b+1)*SEG)
    const int g0 = 32;      // threads [0, 32): owner warp; [32, ...): GEMV teams
    const bool gemv_warp = (int)threadIdx.x >= g0;
    // GEMV role: team `row`, member j -- columns [C*j, C*j + C) of row kg
    const int t = (int)threadIdx.x - g0;
    const int row = gemv_warp ? t / T : 0, j = gemv_warp ? t % T : 0;
    const int kg = (gemv_warp && row < SEG) ? clu_col_at(b * SEG + row, T, C) : n;
    const int kpub = (gemv_warp && (t & 31) < SEG) ? clu_col_at(b * SEG + (t & 31), T, C) : n;  // fan-out lane's row
    // RHS role: lane r of the owner warp owns oscillator k (RK state in registers)
    const int r = threadIdx.x;
    const int k = (!gemv_warp && r < SEG) ? clu_col_at(b * SEG + r, T, C) : n;
    const bool owner = k < n;

    double w[C];
#pragma unroll
    for (int q = 0; q < C; ++q) {
        const int col = j * C + q;
        w[q] = (kg < n && col < n) ? p.w[(size_t)kg * p.cs.ldw + col_perm(p.cs, col)] : -0.0;
    }
    for (int i = threadIdx.x; i < 2 * P; i += blockDim.x) xs[i] = 0.0;
    __syncthreads();
    for (int col = threadIdx.x; col < n; col += blockDim.x) xs[reg_xpos<C>(col, T)] = p.m[3 * (size_t)col];
    const uint32_t bar0 = clu_u32(mbar), bar1 = clu_u32(mbar + 1), bar2 = clu_u32(fbar);
    if (threadIdx.x == 0) {
        clu_bar_init(bar0, 1);
        clu_bar_init(bar1, 1);
        clu_bar_init(bar2, 1);
        *sbad = 0;
        *zslot = 0;
        *sstop = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
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
    clu_sync();  // every CTA's mbarriers and buffers are initialised before any st.async
    const uint32_t xbytes = 8u * (uint32_t)n;  // one 8-byte store per oscillator
    const uint32_t fbytes = 8u * (uint32_t)K;  // + one "bad" word per CTA after a recording step
    const unsigned nthreads = blockDim.x;
    bool stop = false;

    if (gemv_warp) {
        // ==================== GEMV teams ====================================
        if (t == 0) clu_expect(bar1, xbytes);  // x of stage 1
        long long next_rec = p.stride;
        bool flags_in = false;  // the last step recorded: its "bad" words are checked at stage 1
        uint32_t fphase = 0u;
        long long next_flag = 0;
        for (long long step = 1; step <= p.steps && !stop; ++step) {
            const bool record = (step == next_rec) || (step == p.steps);
            const bool fround = record && step < p.steps && step >= next_flag;  // a stop-flag round
#pragma unroll
            for (int stage = 0; stage < 4; ++stage) {
                [[maybe_unused]] const long long estage = (step - 1) * 4 + stage;
                const int buf = stage & 1;  // compile-time after unrolling
                if (!(step == 1 && stage == 0)) {
                    // phases of buffer 1: stages 1, 3 -> parity 0, 1; buffer 0: stages 2, 0 -> 0, 1
                    clu_wait(buf ? bar1 : bar0, (stage == 1 || stage == 2) ? 0u : 1u);
                    if (stage == 1 && flags_in) {  // cluster-wide stop decision (uniform)
                        // the recording step's "bad" words (own mbarrier; they left with the
                        // step's last x, long before this stage's x): one per lane, one vote
                        clu_wait(bar2, fphase);
                        fphase ^= 1u;
                        const int fl = threadIdx.x & 31;
                        if (__any_sync(0xffffffffu, fl < K && sflg[fl] != 0.0)) {
                            if (t == 0) *sstop = 1;
                            asm volatile("bar.arrive 1, %0;" ::"r"(nthreads) : "memory");
                            stop = true;
                            break;
                        }
                    }
                    if (t == 0) {
                        clu_expect(buf ? bar0 : bar1, xbytes);  // the next stage's buffer
                        if (stage == 3 && fround) clu_expect(bar2, fbytes);
                    }
                }
                CTL(estage, 3, t == 0, 0.0);
                const double *xb = xs + buf * P;
                double lvl[LV];
#pragma unroll
                for (int i = 0; i < C / 2; ++i) {
                    const double2 x2 = *reinterpret_cast<const double2 *>(xb + ((i * T + j) << 1));
                    double node = radd(rmul(w[2 * i], x2.x), rmul(w[2 * i + 1], x2.y));
#pragma unroll
                    for (int l = 0; l < LV - 1; ++l) {
                        if (i & (1 << l)) node = radd(lvl[l], node);
                        else { lvl[l] = node; break; }
                    }
                    if (i == C / 2 - 1) lvl[LV - 1] = node;
                }
                double cp = lvl[LV - 1];
#pragma unroll
                for (int mask = 1; mask < T; mask <<= 1) cp = radd(cp, __shfl_xor_sync(0xffffffffu, cp, mask));
                if (j == 0 && row < SEG) cps[row] = cp;
                CTL(estage, 4, t == 0, cp);
                asm volatile("bar.arrive 1, %0;" ::"r"(nthreads) : "memory");
                if (!((step == p.steps) && stage == 3)) {
                    // publication fan-out: the owner warp staged this CTA's x in stg; GEMV
                    // warp gw sends it to CTAs gw, gw + nGW, ... (one 8-byte st.async per
                    // oscillator and destination, the warps in parallel)
                    asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
                    const int nb = (stage + 1) & 1;
                    const int gw = t >> 5, gl = t & 31, ngw = (int)(nthreads >> 5) - 1;
                    if (gl < SEG && kpub < n) {
                        const double v = stg[gl];
                        const uint32_t xa = clu_u32(xs + nb * P + b * SEG + gl);
                        for (int c = gw; c < K; c += ngw) clu_st_async(clu_mapa(xa, c), v, clu_mapa(nb ? bar1 : bar0, c));
                    }
                }
            }
            flags_in = fround;
            if (fround) next_flag = step + kCluFlagEvery;
            if (record && step == next_rec) next_rec += p.stride;
        }
    } else {
        // ==================== owners: RHS, RK4 update, publication ==========
        [[maybe_unused]] const int lane = threadIdx.x;
        auto u_of = [&](long long st) {  // drive sample of step `st` (zero-order hold, model.py:93-149)
            return p.n_samples > 1 ? p.samples + ((st - 1) / p.sps) * p.n_in : p.samples;
        };
        const double win = (owner && p.n_in == 1) ? p.w_in[k] : 0.0;
        auto cin_of = [&](long long st) {
            return (p.n_in == 1) ? rmul(win, u_of(st)[0]) : tree_dot_stream(p.w_in + (size_t)k * p.n_in, u_of(st), p.n_in);
        };
        double cin = 0.0, u_next = 0.0;
        RhsPre pre{};
        if (owner) {
            cin = cin_of(1);
            pre = row_rhs_pre(m, cin, p.c);
        }
        long long next_rec = p.stride;
        long long rec_idx = 1;
        bool flags_in = false, bad_seen = false;
        long long next_flag = 0;
        for (long long step = 1; step <= p.steps && !stop; ++step) {
            const bool record = (step == next_rec) || (step == p.steps);
            const bool fround = record && step < p.steps && step >= next_flag;  // a stop-flag round
#pragma unroll
            for (int stage = 0; stage < 4; ++stage) {
                [[maybe_unused]] const long long estage = (step - 1) * 4 + stage;
                // row sums in cps.  `pre` is tied to the barrier so the compiler cannot
                // sink the own-state half (IEEE division included) past it: it must
                // run while the GEMV warps work, not after the row sums arrive
                asm volatile("bar.sync 1, %8;"
                             : "+d"(pre.m.x), "+d"(pre.m.y), "+d"(pre.m.z), "+d"(pre.hs_qx), "+d"(pre.by),
                               "+d"(pre.bz), "+d"(pre.ax), "+d"(pre.ain_cin)
                             : "r"(nthreads)
                             : "memory");
                if (stage == 1 && flags_in && *sstop) {  // the GEMV warps' stop decision
                    stop = true;
                    break;
                }
                CTL(estage, 0, threadIdx.x == 0, 0.0);
                double xpub = 0.0;
                bool bad = false;
                if (owner) {
                    const V3 d = row_rhs_post(pre, cps[r], p.c);
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
                CTL(estage, 1, threadIdx.x == 0, xpub);
                const bool last = (step == p.steps) && stage == 3;
                if (stage == 3 && record) bad_seen |= __any_sync(0xffffffffu, bad);
                if (stage == 3 && fround && r < K)  // this CTA's "bad" word into slot b of CTA r
                    clu_st_async(clu_mapa(clu_u32(sflg + b), r), bad_seen ? 1.0 : 0.0, clu_mapa(bar2, r));
                if (!last) {  // hand x to the GEMV warps, which send it (fan-out above)
                    if (owner) stg[r] = xpub;
                    asm volatile("bar.arrive 2, %0;" ::"r"(nthreads) : "memory");
                }
                // keep the next stage's own-state half (which reads s / m) after the
                // stores: ptxas hoists that independent arithmetic (its IEEE division
                // included) above the remote stores, onto the critical path.  OR-ing the
                // inputs' bits with a zero loaded from shared memory AFTER the stores
                // makes them depend on that load (bits unchanged)
                if (!last) {
                    const long long z = *zslot;
                    auto pin = [z](double v) { return __longlong_as_double(__double_as_longlong(v) | z); };
                    if (stage < 3) s = V3{pin(s.x), pin(s.y), pin(s.z)};
                    else m = V3{pin(m.x), pin(m.y), pin(m.z)};
                }
                CTL(estage, 2, threadIdx.x == 0, 0.0);
                if (owner && !last) {
                    // own-state half of the next stage's RHS, while the other
                    // warps wait for the exchange and run the next GEMV
                    if (stage == 0 && p.n_in == 1 && step < p.steps) u_next = u_of(step + 1)[0];  // prefetch
                    if (stage < 3) {
                        pre = row_rhs_pre(s, cin, p.c);
                    } else {
                        cin = p.n_in == 1 ? rmul(win, u_next) : cin_of(step + 1);
                        pre = row_rhs_pre(m, cin, p.c);
                    }
                }
            }
            flags_in = fround;
            if (fround) next_flag = step + kCluFlagEvery;
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
    clu_sync();  // no CTA leaves while a peer may still read its shared memory
}


// ----------------------------------------------------------------------------
// Hybrid variant (STO_CLU_HYB): the GEMV teams themselves finish their rows.
// The xor butterfly leaves the row sum in every lane of the team, so every
// lane runs the cp-dependent RHS half and the RK4 update of its row (the RK
// state is replicated across the team's lanes, SIMT: no extra issue) and lane
// j sends the new x to CTAs j, j + T, ...  The owner warp keeps only the
// own-state half of the next stage's RHS (IEEE division included): lane 0 of
// each team hands it the new stage point s (or m) through shared memory
// (named barrier 4), it computes pre(s) while the x exchange and the next GEMV
// run, and hands pre back (named barrier 3) before the teams need it.  The
// per-stage critical path loses the row-sum and staging hand-offs of
// clu_rk4_kernel: mbarrier wait -> GEMV + butterfly -> RHS post -> st.async.
// ----------------------------------------------------------------------------
__host__ __device__ constexpr size_t clu_hyb_smem_bytes(int P) {
    return sizeof(double) * (2 * (size_t)P + 32 * 3 + 32 * 8) + 2 * sizeof(unsigned long long) + 16 +
           sizeof(double) * kCluMaxK + sizeof(unsigned long long);
}

template <int T, int C>
__global__ void __launch_bounds__(C >= 32 ? 288 : 576, 1) clu_hyb_kernel(const __grid_constant__ KParams p) {
    constexpr int P = T * C;
    constexpr int LV = (C == 64) ? 6 : (C == 32) ? 5 : 4;
    static_assert(T <= 32, "team butterfly stays inside one warp");
    extern __shared__ __align__(16) double smem[];
    double *xs = smem;           // [2][P] team-blocked x, double-buffered by stage parity
    double *sst = xs + 2 * P;    // [32][3] stage point, teams -> owner warp
    double *spre = sst + 96;     // 256: own-state RHS half, owner warp -> teams ([8][32] if T <= 2, else [32][8])
    unsigned long long *mbar = reinterpret_cast<unsigned long long *>(spre + 256);
    volatile int *sbad = reinterpret_cast<volatile int *>(mbar + 2);   // a row of this CTA diverged
    volatile int *sstop = reinterpret_cast<volatile int *>(mbar + 3);  // teams -> owner warp
    double *sflg = reinterpret_cast<double *>(mbar + 4);  // [K] peers' "bad" words of a recording step
    unsigned long long *fbar = mbar + 4 + kCluMaxK;       // mbarrier counting those words

    const int K = (int)clu_size(), b = (int)clu_rank();
    const int n = p.rows;
    const int SEG = P / K;
    const bool gemv_warp = (int)threadIdx.x >= 32;
    const int t = (int)threadIdx.x - 32;
    const int row = gemv_warp ? t / T : 0, j = gemv_warp ? t % T : 0;
    const int kg = (gemv_warp && row < SEG) ? clu_col_at(b * SEG + row, T, C) : n;  // team's oscillator
    const int ko = (!gemv_warp && (int)threadIdx.x < SEG) ? clu_col_at(b * SEG + threadIdx.x, T, C) : n;
    const unsigned nthreads = blockDim.x;

    double w[C];
#pragma unroll
    for (int q = 0; q < C; ++q) {
        const int col = j * C + q;
        w[q] = (kg < n && col < n) ? p.w[(size_t)kg * p.cs.ldw + col_perm(p.cs, col)] : -0.0;
    }
    for (int i = threadIdx.x; i < 2 * P; i += blockDim.x) xs[i] = 0.0;
    __syncthreads();
    for (int col = threadIdx.x; col < n; col += blockDim.x) xs[reg_xpos<C>(col, T)] = p.m[3 * (size_t)col];
    const uint32_t bar0 = clu_u32(mbar), bar1 = clu_u32(mbar + 1), bar2 = clu_u32(fbar);
    if (threadIdx.x == 0) {
        clu_bar_init(bar0, 1);
        clu_bar_init(bar1, 1);
        clu_bar_init(bar2, 1);
        *sbad = 0;
        *sstop = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    clu_sync();  // every CTA's mbarriers and buffers are initialised before any st.async
    const uint32_t xbytes = 8u * (uint32_t)n;
    const uint32_t fbytes = 8u * (uint32_t)K;  // + one "bad" word per CTA after a recording step
    auto u_of = [&](long long st) {  // drive sample of step `st` (zero-order hold, model.py:93-149)
        return p.n_samples > 1 ? p.samples + ((st - 1) / p.sps) * p.n_in : p.samples;
    };
    bool stop = false;

    if (gemv_warp) {
        // ==================== teams: GEMV, RHS post, RK4 update, publication ====
        const bool live = kg < n;
        V3 m{0.0, 0.0, 0.0}, s{0.0, 0.0, 0.0}, acc{0.0, 0.0, 0.0}, k3{0.0, 0.0, 0.0};
        if (live) {
            m = V3{p.m[3 * (size_t)kg], p.m[3 * (size_t)kg + 1], p.m[3 * (size_t)kg + 2]};
            if (p.states && j == 0) {
                double *st = p.states + 3 * (size_t)kg;
                st[0] = m.x;
                st[1] = m.y;
                st[2] = m.z;
            }
        }
        const uint32_t xa0 = clu_u32(xs + b * SEG + row), xa1 = clu_u32(xs + P + b * SEG + row);
        // the x of stages 1 and 2; later phases are armed by the owner warp (below),
        // off the teams' critical path
        if (t == 0) {
            clu_expect(bar1, xbytes);
            clu_expect(bar0, xbytes);
        }
        long long next_rec = p.stride, rec_idx = 1;
        bool flags_in = false;  // the last step recorded: its "bad" words are checked at stage 1
        uint32_t fphase = 0u;
        long long next_flag = 0;
        for (long long step = 1; step <= p.steps && !stop; ++step) {
            const bool record = (step == next_rec) || (step == p.steps);
            const bool fround = record && step < p.steps && step >= next_flag;  // a stop-flag round
#pragma unroll
            for (int stage = 0; stage < 4; ++stage) {
                [[maybe_unused]] const long long estage = (step - 1) * 4 + stage;
                const int buf = stage & 1;
                if (!(step == 1 && stage == 0)) {
                    clu_wait(buf ? bar1 : bar0, (stage == 1 || stage == 2) ? 0u : 1u);
                    if (stage == 1 && flags_in) {  // cluster-wide stop decision (uniform)
                        // the recording step's "bad" words (own mbarrier; they left with the
                        // step's last x, long before this stage's x): one per lane, one vote
                        clu_wait(bar2, fphase);
                        fphase ^= 1u;
                        const int fl = threadIdx.x & 31;
                        if (__any_sync(0xffffffffu, fl < K && sflg[fl] != 0.0)) {
                            // consume the owner warp's pending hand-off, then release it
                            asm volatile("bar.sync 3, %0;" ::"r"(nthreads) : "memory");
                            if (t == 0) *sstop = 1;
                            asm volatile("bar.arrive 4, %0;" ::"r"(nthreads) : "memory");
                            stop = true;
                            break;
                        }
                    }
                }
                CTL(estage, 3, t == 0, 0.0);
                const double *xb = xs + buf * P;
                double lvl[LV];
#pragma unroll
                for (int i = 0; i < C / 2; ++i) {
                    const double2 x2 = *reinterpret_cast<const double2 *>(xb + ((i * T + j) << 1));
                    double node = radd(rmul(w[2 * i], x2.x), rmul(w[2 * i + 1], x2.y));
#pragma unroll
                    for (int l = 0; l < LV - 1; ++l) {
                        if (i & (1 << l)) node = radd(lvl[l], node);
                        else { lvl[l] = node; break; }
                    }
                    if (i == C / 2 - 1) lvl[LV - 1] = node;
                }
                double cp = lvl[LV - 1];
#pragma unroll
                for (int mask = 1; mask < T; mask <<= 1) cp = radd(cp, __shfl_xor_sync(0xffffffffu, cp, mask));
                CTL(estage, 4, t == 0, cp);
                // own-state half of this stage's RHS, computed by the owner warp
                asm volatile("bar.sync 3, %0;" ::"r"(nthreads) : "memory");
                RhsPre pre;
                if constexpr (T <= 2) {
                    // >= 16 rows per warp: field-major [8][32], a warp's rows read
                    // consecutive words (row-major 64-byte records would conflict 8-way)
                    const double *q = spre + (row < SEG ? row : 0);
                    pre.m = V3{q[0], q[32], q[64]};
                    pre.hs_qx = q[96];
                    pre.by = q[128];
                    pre.bz = q[160];
                    pre.ax = q[192];
                    pre.ain_cin = q[224];
                } else {
                    // <= 8 rows per warp: row-major [32][8], four 16-byte loads per lane
                    const double *q = spre + 8 * (row < SEG ? row : 0);
                    const double2 a = *reinterpret_cast<const double2 *>(q);
                    const double2 c2 = *reinterpret_cast<const double2 *>(q + 2);
                    const double2 e = *reinterpret_cast<const double2 *>(q + 4);
                    const double2 f = *reinterpret_cast<const double2 *>(q + 6);
                    pre.m = V3{a.x, a.y, c2.x};
                    pre.hs_qx = c2.y;
                    pre.by = e.x;
                    pre.bz = e.y;
                    pre.ax = f.x;
                    pre.ain_cin = f.y;
                }
                const V3 d = row_rhs_post(pre, cp, p.c);
                double xpub;
                bool bad = false;
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
                    if (record && live) {
                        if (!all_finite(m)) {
                            bad = true;
                            if (j == 0) report_divergence(p.status, step, kg);
                        } else if (p.states && j == 0) {
                            const long long ri = (step == next_rec) ? rec_idx : p.n_records - 1;
                            double *st = p.states + ((size_t)ri * n + kg) * 3;
                            st[0] = m.x;
                            st[1] = m.y;
                            st[2] = m.z;
                        }
                    }
                }
                CTL(estage, 1, t == 0, xpub);
                if (bad) *sbad = 1;  // sticky; the owner warp sends it on the next stop-flag round
                if (!((step == p.steps) && stage == 3)) {
                    const int nb = (stage + 1) & 1;
                    if (live)
                        for (int c = j; c < K; c += T)
                            clu_st_async(clu_mapa(nb ? xa1 : xa0, c), xpub, clu_mapa(nb ? bar1 : bar0, c));
                    // the new stage point (m after stage 3) to the owner warp
                    if (j == 0 && row < SEG) {
                        const V3 v = stage < 3 ? s : m;
                        sst[3 * row] = v.x;
                        sst[3 * row + 1] = v.y;
                        sst[3 * row + 2] = v.z;
                    }
                    CTL(estage, 2, t == 0, 0.0);
                    asm volatile("bar.arrive 4, %0;" ::"r"(nthreads) : "memory");
                }
            }
            flags_in = fround;
            if (fround) next_flag = step + kCluFlagEvery;
            if (record && step == next_rec) {
                next_rec += p.stride;
                ++rec_idx;
            }
        }
        if (live && j == 0) {
            double *mm = p.m + 3 * (size_t)kg;
            mm[0] = m.x;
            mm[1] = m.y;
            mm[2] = m.z;
        }
    } else {
        // ==================== owner warp: own-state RHS half ==================
        const int r = threadIdx.x;
        const bool owner = ko < n;
        const double win = (owner && p.n_in == 1) ? p.w_in[ko] : 0.0;
        auto cin_of = [&](long long st) {
            return (p.n_in == 1) ? rmul(win, u_of(st)[0])
                                 : (owner ? tree_dot_stream(p.w_in + (size_t)ko * p.n_in, u_of(st), p.n_in) : 0.0);
        };
        auto put = [&](const RhsPre &q) {
            if (r < SEG) {
                if constexpr (T <= 2) {
                    double *o = spre + r;
                    o[0] = q.m.x;
                    o[32] = q.m.y;
                    o[64] = q.m.z;
                    o[96] = q.hs_qx;
                    o[128] = q.by;
                    o[160] = q.bz;
                    o[192] = q.ax;
                    o[224] = q.ain_cin;
                } else {
                    double *o = spre + 8 * r;
                    *reinterpret_cast<double2 *>(o) = make_double2(q.m.x, q.m.y);
                    *reinterpret_cast<double2 *>(o + 2) = make_double2(q.m.z, q.hs_qx);
                    *reinterpret_cast<double2 *>(o + 4) = make_double2(q.by, q.bz);
                    *reinterpret_cast<double2 *>(o + 6) = make_double2(q.ax, q.ain_cin);
                }
            }
        };
        V3 m0{0.0, 0.0, 0.0};
        if (owner) m0 = V3{p.m[3 * (size_t)ko], p.m[3 * (size_t)ko + 1], p.m[3 * (size_t)ko + 2]};
        double cin = cin_of(1), u_next = 0.0;
        put(row_rhs_pre(m0, cin, p.c));
        asm volatile("bar.arrive 3, %0;" ::"r"(nthreads) : "memory");
        long long next_rec = p.stride;
        bool flags_in = false;
        long long next_flag = 0;
        for (long long step = 1; step <= p.steps && !stop; ++step) {
            const bool record = (step == next_rec) || (step == p.steps);
            const bool fround = record && step < p.steps && step >= next_flag;  // a stop-flag round
#pragma unroll
            for (int stage = 0; stage < 4; ++stage) {
                if ((step == p.steps) && stage == 3) break;
                if (stage == 0 && p.n_in == 1 && step < p.steps) u_next = u_of(step + 1)[0];  // prefetch
                asm volatile("bar.sync 4, %0;" ::"r"(nthreads) : "memory");
                if (stage == 1 && flags_in && *sstop) {  // the teams' stop decision
                    stop = true;
                    break;
                }
                // the teams are done with stage `stage`, so its buffer's phase has
                // completed here: arm that buffer for stage + 2 (stage 0 of step 1
                // read the local initial x; stage 2's phase was armed up front)
                if (r == 0 && !(step == 1 && stage == 0)) clu_expect((stage & 1) ? bar1 : bar0, xbytes);
                if (stage == 3 && fround) {  // this CTA's (sticky) "bad" word into slot b of CTA r
                    if (r == 0) clu_expect(bar2, fbytes);
                    if (r < K) clu_st_async(clu_mapa(clu_u32(sflg + b), r), *sbad ? 1.0 : 0.0, clu_mapa(bar2, r));
                }
                const V3 v = r < SEG ? V3{sst[3 * r], sst[3 * r + 1], sst[3 * r + 2]} : V3{0.0, 0.0, 0.0};
                if (stage == 3) cin = p.n_in == 1 ? rmul(win, u_next) : cin_of(step + 1);
                put(row_rhs_pre(v, cin, p.c));
                asm volatile("bar.arrive 3, %0;" ::"r"(nthreads) : "memory");
            }
            flags_in = fround;
            if (fround) next_flag = step + kCluFlagEvery;
            if (record && step == next_rec) next_rec += p.stride;
        }
    }
    clu_sync();  // no CTA leaves while a peer may still write its shared memory
}

}  // namespace sto
