// sto_ensemble_kernel.cuh -- batched ensemble (BASELINE configs[3]): B
// independent reservoirs that share W and W_in but not their parameters
// (e.g. a sweep over the drive current), stepped together so the coupling
// becomes a GEMM per RK stage:  CP[k][b] = sum_j W[k][j] * X[j][b]
// (X = the members' stage x-vectors).
//
// The GEMM runs on the FP64 tensor cores: mma.sync.aligned.m8n8k4 .f64
// (SASS DMMA.8x8x4 -- sm_100 has no tcgen05 f64 kind; DMMA is its fp64
// tensor path, measured 37.1 TFLOP/s vs 34.0 for DFMA, tools/fp64_peak.cu).
// Its accumulation order is not the reference's pinned tree, so this path is
// held to a tolerance (<= 1e-10 at 1e3 steps, per member,
// against the oracle run with that member's parameters), not bit-equality.
//
// Structure (one persistent cooperative launch per run):
//  * Tiles: CTA = TR = 8U rows x 64 members, U chosen on the host so that
//    ceil(n/TR) row tiles x ceil(B/64) member columns fill the 148 SMs
//    (N = 1000, B = 512: U = 7 -> 18 x 8 = 144 CTAs, 96.5 % of the ideal
//    per-SM share; 64-row tiles would leave 20 SMs idle).
//  * Two independent warp groups per CTA (8 warps each), one per 32-member
//    half of the column.  Each group runs its own K-loop ring, exchange
//    counter and epilogue; the halves never interact.  Group 1 starts half a
//    GEMM after group 0, so while one group is in its epilogue (FP64 pipe,
//    tensor memory) and exchange wait, the other keeps the DMMA pipe busy:
//    per-stage time -> the two GEMMs back to back instead of GEMM + epilogue
//    + exchange (any start offset between the epilogue length and GEMM
//    length is a stable operating point -- tools/ens_overlap_model.py).
//  * Fragment-order operands: W (a private copy, re-laid out per tile
//    height) and the stage X (written so by the epilogue) are stored in HBM
//    in DMMA fragment order -- for each (8-row unit, k-step) / (k-step,
//    8-member unit) the 32 doubles of one fragment in lane order -- so that
//    the W part and the X part of one (tile, K chunk) are each ONE
//    contiguous block (14 KB + 8 KB at U = 7), moved by ONE 1-D bulk async
//    copy (cp.async.bulk ... mbarrier::complete_tx), and every fragment load
//    is a conflict-free 256 B warp-contiguous LDS.64.  K streams in
//    32-column chunks through a 4-slot ring per group with one "full"
//    mbarrier per slot.  There is no producer warp (a 17th warp would cap
//    every thread at 96 registers: 5 warps on one SM sub-partition): the
//    LAST of the group's warps to finish a chunk (shared-memory counter)
//    refills its slot, so no warp ever waits to issue.  W does not depend on
//    the stage, so the slots of the first chunks of stage e+1 are refilled
//    with W while stage e's last chunks and epilogue still run; their X
//    parts are issued once the half-column's exchange counter shows every
//    row tile has published x.
//  * GEMM warps: warp w of group h owns member unit w&3 of the half and
//    k-steps of parity (w>>2)&1 (intra-group split-K 2), i.e. a U x 1 grid
//    of 8x8 DMMA tiles fed by U A-fragments + 1 B-fragment per k-step.
//    Partials are summed through shared memory.
//  * Epilogue: every thread owns U outputs (one member, rows 8j + 4((w>>2)&1)
//    + lane%4) -- so each warp's x publication is 32 consecutive doubles of
//    the fragment-order X (one 256 B store).  The RK state of every output
//    (m, the running RK4 accumulator, the stage point: 9 doubles) lives in
//    TENSOR MEMORY -- the 256 KB TMEM is otherwise idle (fp64 has no
//    tcgen05 MMA kind) and holds 7 outputs x 18 columns in each thread's
//    128-column slice of its lane (tcgen05.ld/st 32x32b).  Kept in L2
//    instead, the state round trip made the epilogue L2-bandwidth bound
//    (~56 MB per stage).
//  * RK4 combination: acc = (k1 + k2*2) + k3*2 and m + (acc + k4)*dt/6, a
//    reassociation of the reference's m + ((k1 + k2*2) + (k3*2 + k4))*dt/6
//    (1 ulp level, inside the GEMM-order tolerance) that drops k3 from the
//    live state.
//  * Exchange: one counter per half-column (red.release.gpu by each CTA's
//    group after its epilogue; acquire-polled by one thread of the group,
//    which then issues the X copies -- everybody else waits on shared-memory
//    mbarriers).
#pragma once

#include "sto_kernels.cuh"

namespace sto {

constexpr int kEnsBT = 64;                      // members per CTA tile
constexpr int kEnsGW = 32;                      // members per warp group (half-column)
constexpr int kEnsGroups = kEnsBT / kEnsGW;
constexpr int kEnsKC = 32;                      // K chunk (doubles)
constexpr int kEnsLDB = kEnsBT + 4;             // CP (coupling sums) row pitch
constexpr int kEnsSlots = 4;                    // shared-memory ring depth per group
constexpr int kEnsThreads = 512;                // 2 groups x 8 MMA + epilogue warps
constexpr int kEnsGroupThreads = kEnsThreads / kEnsGroups;
constexpr int kEnsMaxU = 7;                     // TR <= 56 rows (RK state of 7 outputs fills a TMEM lane slice)
constexpr int kEnsState = 1;                    // global state planes: cin (n_in > 1 only)
constexpr int kEnsTmemCols = 512;               // whole TMEM: 128 lanes x 512 x 32 bit
#ifndef STO_ENS_EPI_UNROLL
#define STO_ENS_EPI_UNROLL 2
#endif
constexpr int kEnsEpiUnroll = STO_ENS_EPI_UNROLL;  // epilogue outputs in flight per thread
constexpr int kEnsTmemOut = 18;                 // columns per output: m, acc, s (3 doubles each)
constexpr int kEnsKAlign = 8;                   // K padded to 8: chunk bytes % 16 == 0, even k-steps
#ifndef STO_ENS_ALTERNATE
#define STO_ENS_ALTERNATE 0
#endif
// 1: the two groups' GEMMs take turns (measured 2.81e9 vs 3.34e9 osc-steps/s free
// running: a lone 8-warp group reaches only ~0.6 of the DMMA peak inside the
// kernel, so the groups must overlap in the GEMM to fill the pipe; A/B only)
constexpr bool kEnsAlternate = STO_ENS_ALTERNATE;
// GEMM warp tile: 1 = U x 1 DMMA tiles, split-K 2 (warp = member unit x k-step
// parity); 2 = U x 2 tiles (two member units share each A fragment), split-K 4
#ifndef STO_ENS_NT
#define STO_ENS_NT 1
#endif
constexpr int kEnsNT = STO_ENS_NT;

__host__ __device__ constexpr int ens_slot_doubles(int u) { return 8 * u * kEnsKC + kEnsKC * kEnsGW; }
__host__ __device__ constexpr size_t ens_smem_bytes(int u) {
    return sizeof(double) * ((size_t)kEnsGroups * kEnsSlots * ens_slot_doubles(u) + 8 * u * kEnsLDB +
                             kEnsBT * 11 + 8 * u) +
           sizeof(unsigned long long) * (2 * kEnsGroups * kEnsSlots + kEnsGroups) +
           24;  // ring barriers, GEMM-turn barriers, counters, TMEM base, gate, stop[2], exited[2]
}
static_assert(ens_smem_bytes(kEnsMaxU) <= 227 * 1024, "ensemble shared memory budget");

struct EnsParams {
    int n, np, kp;                // oscillators; allocated (padded) rows; K padded to kEnsKAlign
    int n_rt;                     // row tiles of this launch
    int batch, bp;                // members, padded to kEnsBT
    int member0;                  // first member of this launch (host chunking)
    int n_in;
    const double *w;              // fragment order, ens_w_index(); n_rt * TR * kp
    const double *w_in;           // n x n_in
    const double *consts;         // (batch, 11)
    double *m;                    // (batch, n, 3) in/out
    const double *samples;        // drive; member b uses samples + b * sample_member_stride
    long long sample_member_stride;
    long long n_samples, sps;
    double dt, h2, dt6;
    long long steps, stride, n_records;
    double *states;               // (n_records, batch, n, 3) or null
    double *x;                    // [2][bp / 32][kp * 32] stage x, ens_x_index()
    double *st;                   // [np][bp] cin (n_in > 1); the RK state lives in TMEM
    unsigned long long *bar;      // per half-column counters, 32 words apart
    StatusDev *status;
    int debug_solo;               // timeline experiments: group 1 idles (results of its members invalid)
    float gate_frac;              // group 1 starts when group 0 has consumed this fraction of stage 0
};

// Fragment-order layouts.  K is cut into 32-column chunks (the last one may be
// shorter: kc = kp - 32*ch, a multiple of 8); nk = kc / 4 k-steps.
// W: [row tile][chunk][row unit ru < U][k-step ks < nk][lane], lane = 4g + t
//    holds W[row0 + 8ru + g][32ch + 4ks + t]   (A fragment of m8n8k4.row)
// X: [half-column][chunk][k-step][member unit mu < 4][lane], lane = 4g + t
//    holds X[32ch + 4ks + t][32 half + 8mu + g]   (B fragment of m8n8k4.col)
__host__ __device__ inline size_t ens_x_index(int k, int bg, int kp) {
    const int col = bg >> 5, bl = bg & 31;
    return (size_t)col * kp * kEnsGW + (size_t)(k >> 5) * (kEnsKC * kEnsGW) +
           (size_t)((((k & 31) >> 2) * 4 + (bl >> 3)) * 32 + (bl & 7) * 4 + (k & 3));
}

// ---- mbarrier / bulk-copy / DMMA primitives --------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "ENS_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra ENS_WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned long long *b, uint32_t parity) {  // non-blocking
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_try(unsigned long long *b, uint32_t parity) {  // blocks up to a HW time limit
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         unsigned long long *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_cta(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v)
                 : "memory");
    return old;
}
__device__ __forceinline__ void group_sync(int grp) {  // named barrier 1 + grp over one warp group
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(kEnsGroupThreads) : "memory");
}


__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// The RHS of model.py:239-301 with FMA contraction and a correctly rounded
// reciprocal instead of the pinned separately-rounded order: ~45 % fewer FP64
// instructions and a shorter dependent chain for the epilogue, which shares
// the FP64 datapath with the DMMAs of the other warp group.  Same algebra;
// differences are at the rounding level, inside the ensemble's GEMM-order
// tolerance (tests/test_gpu_ensemble.py holds every member to 1e-10).
__device__ __forceinline__ V3 row_rhs_fma(V3 m, double cp, double cin, const Consts &c) {
    const double md = fma(m.z, c.pz, fma(m.y, c.py, m.x * c.px));
    const double hs = c.pref * __drcp_rn(fma(c.lam, md, 1.0));
    const double qx = fma(c.py, m.z, -(c.pz * m.y));
    const double qy = fma(c.pz, m.x, -(c.px * m.z));
    const double qz = fma(c.px, m.y, -(c.py * m.x));
    const double bx = fma(hs, qx, fma(c.a_cp, cp, c.a_in * cin));
    const double by = hs * qy;
    const double bz = fma(hs, qz, fma(c.h_aniso, m.z, c.h_appl));
    const double ax = fma(m.y, bz, -(m.z * by));
    const double ay = fma(m.z, bx, -(m.x * bz));
    const double az = fma(m.x, by, -(m.y * bx));
    const double ex = fma(m.y, az, -(m.z * ay));
    const double ey = fma(m.z, ax, -(m.x * az));
    const double ez = fma(m.x, ay, -(m.y * ax));
    return V3{fma(-c.c_prec, ax, -(c.c_damp * ex)), fma(-c.c_prec, ay, -(c.c_damp * ey)),
              fma(-c.c_prec, az, -(c.c_damp * ez))};
}

#ifdef STO_TIMELINE
__device__ unsigned long long g_ens_timeline[16][8];  // [stage][event + 4 * group]
#define ENS_TL(e, ev)                                                                         \
    do {                                                                                      \
        if (blockIdx.x == 0 && threadIdx.x % kEnsGroupThreads == 0 && (e) >= 40 && (e) < 56)   \
            g_ens_timeline[(e) - 40][(ev) + 4 * grp] = clock64();                             \
    } while (0)
#else
#define ENS_TL(e, ev)
#endif

// ---- tensor-memory scratch (tcgen05.ld / tcgen05.st, 32x32b: one lane per thread) ----
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[N]);
template <>
__device__ __forceinline__ void tmem_ld<6>(uint32_t taddr, uint32_t (&r)[6]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr) : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                 : "=r"(r[4]), "=r"(r[5]) : "r"(taddr + 4) : "memory");
}
template <>
__device__ __forceinline__ void tmem_ld<18>(uint32_t taddr, uint32_t (&r)[18]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                 : "=r"(r[16]), "=r"(r[17]) : "r"(taddr + 16) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st6(uint32_t taddr, V3 a, V3 b) {  // 2 doubles x 3 = 12 columns
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
        "r"(__double2loint(a.x)), "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)), "r"(__double2hiint(a.y)),
        "r"(__double2loint(a.z)), "r"(__double2hiint(a.z)), "r"(__double2loint(b.x)), "r"(__double2hiint(b.x))
        : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr + 8),
                 "r"(__double2loint(b.y)), "r"(__double2hiint(b.y)), "r"(__double2loint(b.z)),
                 "r"(__double2hiint(b.z))
                 : "memory");
}
__device__ __forceinline__ void tmem_st3(uint32_t taddr, V3 a) {  // 6 columns
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
                 "r"(__double2loint(a.x)), "r"(__double2hiint(a.x)), "r"(__double2loint(a.y)),
                 "r"(__double2hiint(a.y))
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr + 4),
                 "r"(__double2loint(a.z)), "r"(__double2hiint(a.z))
                 : "memory");
}
__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

template <int U>
__global__ void __launch_bounds__(kEnsThreads, 1) ens_rk4_kernel(const __grid_constant__ EnsParams p) {
    constexpr int TR = 8 * U;
    constexpr int WS = TR * kEnsKC;  // W part of a slot (doubles)
    constexpr int SS = ens_slot_doubles(U);
    constexpr int GW = kEnsGroupThreads / 32;  // warps per group
    static_assert(U * kEnsTmemOut <= kEnsTmemCols / 4, "RK state of U outputs must fit a TMEM slice");
    extern __shared__ __align__(16) double smem[];
    double *cpb = smem + kEnsGroups * kEnsSlots * SS;  // TR x kEnsLDB coupling sums
    double *cs = cpb + TR * kEnsLDB;                   // [64][11] member consts
    double *wins = cs + kEnsBT * 11;                   // [TR] input weights of the tile's rows (n_in = 1)
    unsigned long long *full_all = reinterpret_cast<unsigned long long *>(wins + TR);
    unsigned long long *gemm_done = full_all + kEnsGroups * kEnsSlots;  // [2] GEMM turns (see below)
    unsigned *done_all = reinterpret_cast<unsigned *>(gemm_done + kEnsGroups);
    uint32_t *tmem_base_slot = done_all + kEnsGroups * kEnsSlots;
    volatile int *go = reinterpret_cast<volatile int *>(tmem_base_slot + 1);  // group 1 start gate
    volatile int *stop_grp = go + 1;  // [2] per group: stop after this recording step
    volatile int *exited = stop_grp + 2;  // [2] per group: left the stage loop (no more turns)

    const int rt = blockIdx.x % p.n_rt, ct = blockIdx.x / p.n_rt;  // row tile, member column
    const int row0 = rt * TR, col0 = ct * kEnsBT;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp = warp / GW, wl = warp % GW;  // warp group (member half), warp in group
    const int hcol = 2 * ct + grp;              // global half-column
    unsigned long long *bar = p.bar + 32 * hcol;
    double *ring = smem + grp * kEnsSlots * SS;
    unsigned long long *full = full_all + grp * kEnsSlots;
    unsigned *done = done_all + grp * kEnsSlots;  // warps finished with the slot's current fill
    const size_t xplane = (size_t)p.kp * p.bp;  // one x buffer
    const int n_chunks = (p.kp + kEnsKC - 1) / kEnsKC;
    const int nring = min(kEnsSlots, n_chunks);  // slots in use: a refill is at most one stage ahead
    const long long n_stages = 4 * p.steps;
    const uint64_t pol = l2_policy_evict_last();  // W and X tiles are re-read by other CTAs

    if (warp == 0) {  // whole TMEM for this CTA (1 CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_base_slot)),
                     "n"(kEnsTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int s = 0; s < kEnsGroups * kEnsSlots; ++s) {
            mbar_init(&full_all[s], 1);
            done_all[s] = 0u;
        }
        for (int g = 0; g < kEnsGroups; ++g) {
            mbar_init(&gemm_done[g], kEnsGroupThreads / 32);
            exited[g] = 0;
        }
        *go = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < kEnsBT * 11; i += blockDim.x) {
        const int bl = i / 11, q = i % 11;
        const int b = min(p.member0 + col0 + bl, p.batch - 1);
        cs[i] = p.consts[(size_t)b * 11 + q];
    }
    for (int i = tid; i < TR; i += blockDim.x) wins[i] = (row0 + i < p.n) ? p.w_in[(size_t)(row0 + i) * p.n_in] : 0.0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this thread's TMEM slice: lane 32*(warp%4) + lane, columns 128*(warp/4) ...
    const uint32_t tmem = *tmem_base_slot + ((uint32_t)(32 * (warp & 3)) << 16) +
                          (uint32_t)(kEnsTmemCols / 4) * (warp >> 2);

    // chunk ch of the K loop in ring slot s: arm the barrier, copy W (and X)
    auto kc_of = [&](int ch) { return min(kEnsKC, p.kp - ch * kEnsKC); };
    const double *wtile = p.w + (size_t)rt * TR * p.kp;  // this row tile, fragment order
    auto issue_w = [&](int s, int ch) {  // one thread; also arms full[s] for the W + X bytes
        const int kc = kc_of(ch);
        mbar_expect_tx(&full[s], (uint32_t)(TR + kEnsGW) * kc * 8);
        bulk_g2s(ring + s * SS, wtile + (size_t)ch * TR * kEnsKC, (uint32_t)(TR * kc * 8), &full[s], pol);
    };
    auto issue_x = [&](int s, int ch, long long g) {  // one thread: X chunk of stage g (buffer g & 1)
        const double *xsrc = p.x + (size_t)(g & 1) * xplane + (size_t)hcol * p.kp * kEnsGW;
        bulk_g2s(ring + s * SS + WS, xsrc + (size_t)ch * kEnsKC * kEnsGW, (uint32_t)(kc_of(ch) * kEnsGW * 8),
                 &full[s], pol);
    };
    // first warp of the group: wait until every row tile has published this half-column's
    // x of stage g (counter >= (g+1) * n_rt), then issue the X parts of the ring's first chunks.
    // Returns the half-column's stop word (read after the counter, so every row
    // tile of the half-column reads the same value; see the record-step stop below).
    auto open_stage = [&](long long g) -> unsigned long long {
        unsigned long long stop = 0;
        if (lane == 0) {
            const unsigned long long target = (unsigned long long)(g + 1) * p.n_rt;
            unsigned long long v;
            while (true) {  // relaxed polling with back-off, one acquire fence at the end
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
                if (v >= target) break;
                __nanosleep(64);
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
            stop = *((volatile unsigned long long *)bar + 1);
        }
        __syncwarp();
        const int s0 = (int)((g * n_chunks) % nring);
        if (lane < nring) issue_x((s0 + lane) % nring, lane, g);
        return __shfl_sync(0xffffffffu, stop, 0);
    };

    // ---- roles -------------------------------------------------------------------
    const int mu = wl & 3, kph = wl >> 2;  // GEMM: member unit, k-step parity; epilogue: row half
    const int g8 = lane >> 2, t4 = lane & 3;
    const int bl = kEnsGW * grp + 8 * mu + g8, rsub = 4 * kph + t4;  // epilogue: member, row offset
    const int bg = col0 + bl, b = p.member0 + bg;
    const bool member_ok = b < p.batch;
    const int bc = min(b, p.batch - 1);  // clamped for reads
    const Consts c{cs[bl * 11 + 0], cs[bl * 11 + 1], cs[bl * 11 + 2], cs[bl * 11 + 3],
                   cs[bl * 11 + 4], cs[bl * 11 + 5], cs[bl * 11 + 6], cs[bl * 11 + 7],
                   cs[bl * 11 + 8], cs[bl * 11 + 9], cs[bl * 11 + 10]};
    const double *samp = p.samples + (size_t)bc * p.sample_member_stride;

    // ---- prologue: m -> TMEM, x(0), record 0 -----------------------------------
#pragma unroll
    for (int j = 0; j < U; ++j) {
        const int k = row0 + rsub + 8 * j;
        const bool ok = k < p.n && member_ok;
        V3 m{0.0, 0.0, 0.0};
        if (ok) {
            const double *mm = p.m + ((size_t)b * p.n + k) * 3;
            m = V3{mm[0], mm[1], mm[2]};
            if (p.states) {
                double *so = p.states + ((size_t)b * p.n + k) * 3;
                so[0] = m.x;
                so[1] = m.y;
                so[2] = m.z;
            }
        }
        tmem_st3(tmem + j * kEnsTmemOut, m);
        if (ok) p.x[ens_x_index(k, bg, p.kp)] = m.x;  // parity 0 (padding stays zero)
    }
    tmem_wait_st();
    group_sync(grp);
    if (wl == 0) {
        if (lane == 0) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
            // group 1 starts half a GEMM later (see header): wait for group 0's gate
            if (grp == 1)
                while (*go == 0) __nanosleep(64);
        }
        __syncwarp();
        if (lane < nring) issue_w(lane, lane);
        open_stage(0);
    }

    int slot = 0;
    uint32_t phase = 0;
    int ch_fill = nring;   // next chunk (within its stage) a refill loads
    long long g_fill = 0;  // ... and its stage
    if (ch_fill == n_chunks) {
        ch_fill = 0;
        g_fill = 1;
    }
    const int gate_chunk = min(n_chunks - 1, (int)(p.gate_frac * n_chunks));
    long long next_rec = p.stride, rec_idx = 1;
    long long gstage = 0;
    for (long long step = 1; step <= (p.debug_solo && grp == 1 ? 0 : p.steps); ++step) {
        const bool record = (step == next_rec) || (step == p.steps);
        const long long sidx = p.n_samples == 1 ? 0 : (step - 1) / p.sps;
#pragma unroll
        for (int stage = 0; stage < 4; ++stage, ++gstage) {  // unrolled: stage branches resolve at compile time
            ENS_TL(gstage, 0);
            const double u1 = (p.n_in == 1) ? samp[(size_t)sidx] : 0.0;  // lands during the GEMM
            double acc[U][kEnsNT][2];
#pragma unroll
            for (int r = 0; r < U; ++r)
#pragma unroll
                for (int j = 0; j < kEnsNT; ++j) acc[r][j][0] = acc[r][j][1] = 0.0;
#ifdef STO_TIMELINE
            long long waited = 0;
#endif
            // GEMM turns: the two groups' K loops alternate -- group 1 runs its
            // stage-g GEMM after group 0's, group 0 its stage-g GEMM after group
            // 1's stage g-1 -- so each GEMM has the DMMA pipe to itself while the
            // other group is in its epilogue and exchange (left free, the two
            // groups drift into phase and share the pipe, then idle together).
            // A group can run at most one turn ahead, so mbarrier parity is
            // unambiguous; a group that has left the loop (record-step stop)
            // takes no more turns.
            if (kEnsAlternate && !p.debug_solo && (grp == 1 || gstage > 0)) {
                const int other = grp ^ 1;
                const uint32_t par = (uint32_t)((grp == 1 ? gstage : gstage - 1) & 1);
                while (!mbar_try(&gemm_done[other], par) && !exited[other]) {
                }
            }
            for (int ch = 0; ch < n_chunks; ++ch) {
#ifdef STO_TIMELINE
                const long long w0 = clock64();
                mbar_wait(&full[slot], phase);
                waited += clock64() - w0;
#else
                mbar_wait(&full[slot], phase);
#endif
                const double *W = ring + slot * SS;
                const double *X = W + WS;
                const int nk = kc_of(ch) >> 2;  // k-steps in this chunk (even)
                if constexpr (kEnsNT == 2) {
                    // warp = member-unit pair x k-step phase (mod 4); one A fragment feeds
                    // two DMMAs
                    const int pair = wl & 1, kq = wl >> 1;
                    auto kstep = [&](int kk, int nkk) {
                        double a[U];
#pragma unroll
                        for (int r = 0; r < U; ++r) a[r] = W[(r * nkk + kk) * 32 + lane];
                        const double b0 = X[(kk * 4 + 2 * pair) * 32 + lane];
                        const double b1 = X[(kk * 4 + 2 * pair + 1) * 32 + lane];
#pragma unroll
                        for (int r = 0; r < U; ++r) {
                            dmma(acc[r][0][0], acc[r][0][1], a[r], b0);
                            dmma(acc[r][kEnsNT - 1][0], acc[r][kEnsNT - 1][1], a[r], b1);
                        }
                    };
                    if (nk == kEnsKC / 4) {
#pragma unroll
                        for (int q = 0; q < kEnsKC / 16; ++q) kstep(kq + 4 * q, kEnsKC / 4);
                    } else {
                        for (int kk = kq; kk < nk; kk += 4) kstep(kk, nk);
                    }
                } else if (nk == kEnsKC / 4) {
                    // full chunk: compile-time offsets, fragments of the next k-step loaded
                    // while the DMMAs of this one issue (register double buffer)
                    constexpr int NQ = kEnsKC / 8;  // k-steps of this warp's parity
                    double a[2][U], bf[2];
#pragma unroll
                    for (int r = 0; r < U; ++r) a[0][r] = W[(r * (kEnsKC / 4) + kph) * 32 + lane];
                    bf[0] = X[(kph * 4 + mu) * 32 + lane];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        if (q + 1 < NQ) {
                            const int kn = 2 * (q + 1) + kph;
#pragma unroll
                            for (int r = 0; r < U; ++r) a[(q + 1) & 1][r] = W[(r * (kEnsKC / 4) + kn) * 32 + lane];
                            bf[(q + 1) & 1] = X[(kn * 4 + mu) * 32 + lane];
                        }
#pragma unroll
                        for (int r = 0; r < U; ++r) dmma(acc[r][0][0], acc[r][0][1], a[q & 1][r], bf[q & 1]);
                    }
                } else {
                    for (int kk = kph; kk < nk; kk += 2) {
                        double a[U];
#pragma unroll
                        for (int r = 0; r < U; ++r) a[r] = W[(r * nk + kk) * 32 + lane];
                        const double bf = X[(kk * 4 + mu) * 32 + lane];
#pragma unroll
                        for (int r = 0; r < U; ++r) dmma(acc[r][0][0], acc[r][0][1], a[r], bf);
                    }
                }
                // Slot consumed by this warp; the LAST of the group's warps to get here
                // refills it.  The counter is an acq_rel atomic: every warp's fragment
                // loads of the slot (ordered before its increment by __syncwarp)
                // happen-before the last warp's refill, whose async-proxy writes are
                // ordered after its generic-proxy view by fence.proxy.async.  A chunk
                // of the next stage gets only its W here; its X follows in open_stage.
                __syncwarp();
                if (lane == 0) {
                    if (atom_add_acq_rel_cta(&done[slot], 1u) % GW == GW - 1 && g_fill < n_stages) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        issue_w(slot, ch_fill);
                        if (g_fill == gstage) issue_x(slot, ch_fill, g_fill);
                    }
                    if (grp == 0 && gstage == 0 && ch == gate_chunk && wl == 0) *go = 1;
                }
                if (++ch_fill == n_chunks) {
                    ch_fill = 0;
                    ++g_fill;
                }
                if (++slot == nring) {
                    slot = 0;
                    phase ^= 1;
                }
            }
            if (kEnsAlternate) {  // this group's GEMM turn is over
                __syncwarp();
                if (lane == 0) mbar_arrive(&gemm_done[grp]);
            }
            // ---- split-K reduction into cpb[row][member] --------------------
            if constexpr (kEnsNT == 2) {
                // four k-step phases accumulate in turn (the last one stores first)
                const int pair = wl & 1, kq = wl >> 1;
#pragma unroll
                for (int round = 3; round >= 0; --round) {
                    if (kq == round) {
#pragma unroll
                        for (int j = 0; j < 2; ++j) {
                            double *cpg = cpb + kEnsGW * grp + 8 * (2 * pair + j) + 2 * t4;
#pragma unroll
                            for (int r = 0; r < U; ++r) {
                                double *d = cpg + (8 * r + g8) * kEnsLDB;
                                if (round == 3) {
                                    d[0] = acc[r][j][0];
                                    d[1] = acc[r][j][1];
                                } else {
                                    d[0] = acc[r][j][0] + d[0];
                                    d[1] = acc[r][j][1] + d[1];
                                }
                            }
                        }
                    }
                    group_sync(grp);
                }
            } else {
            double *cpg = cpb + kEnsGW * grp + 8 * mu + 2 * t4;
            if (kph == 1) {
#pragma unroll
                for (int r = 0; r < U; ++r) {
                    double *d = cpg + (8 * r + g8) * kEnsLDB;
                    d[0] = acc[r][0][0];
                    d[1] = acc[r][0][1];
                }
            }
            group_sync(grp);
            if (kph == 0) {
#pragma unroll
                for (int r = 0; r < U; ++r) {
                    double *d = cpg + (8 * r + g8) * kEnsLDB;
                    d[0] = acc[r][0][0] + d[0];
                    d[1] = acc[r][0][1] + d[1];
                }
            }
            group_sync(grp);
            }
            ENS_TL(gstage, 1);
#ifdef STO_TIMELINE
            if (blockIdx.x == 0 && threadIdx.x % kEnsGroupThreads == 0 && gstage >= 40 && gstage < 56)
                g_ens_timeline[gstage - 40][3 + 4 * grp] = waited;
#endif
            // ---- RK4 epilogue: U outputs per thread, state in TMEM ---------------
            double *xdst = p.x + (size_t)((gstage + 1) & 1) * xplane;
            const bool last_stage = (gstage + 1 == n_stages);
            const double h = stage == 2 ? p.dt : p.h2;
#pragma unroll kEnsEpiUnroll
            for (int j = 0; j < U; ++j) {
                const int rl = rsub + 8 * j;
                const int k = row0 + rl;
                const bool ok = k < p.n && member_ok;
                const uint32_t ta = tmem + j * kEnsTmemOut;
                V3 m, a{0.0, 0.0, 0.0}, cur;
                if (stage == 0) {
                    uint32_t r[6];
                    tmem_ld<6>(ta, r);
                    tmem_wait_ld();
                    m = V3{u2d(r[0], r[1]), u2d(r[2], r[3]), u2d(r[4], r[5])};
                    cur = m;
                } else {
                    uint32_t r[18];
                    tmem_ld<18>(ta, r);
                    tmem_wait_ld();
                    m = V3{u2d(r[0], r[1]), u2d(r[2], r[3]), u2d(r[4], r[5])};
                    a = V3{u2d(r[6], r[7]), u2d(r[8], r[9]), u2d(r[10], r[11])};
                    cur = V3{u2d(r[12], r[13]), u2d(r[14], r[15]), u2d(r[16], r[17])};
                }
                double cin = 0.0;
                if (k < p.n) {
                    if (p.n_in == 1) {  // recomputed every stage (u is held): same rounding as storing it
                        cin = rmul(wins[rl], u1);
                    } else if (stage == 0) {
                        cin = tree_dot_stream(p.w_in + (size_t)k * p.n_in, samp + (size_t)sidx * p.n_in, p.n_in);
                        p.st[(size_t)k * p.bp + bg] = cin;
                    } else {
                        cin = p.st[(size_t)k * p.bp + bg];
                    }
                }
                const V3 d = row_rhs_fma(cur, cpb[rl * kEnsLDB + bl], cin, c);
                double xpub;
                if (stage < 3) {
                    // acc: k1 | k1 + k2*2 | (k1 + k2*2) + k3*2
                    const V3 a2 = stage == 0 ? d : acc_k2(a, d);
                    const V3 sp = stage_point(m, d, h);
                    tmem_st6(ta + 6, a2, sp);
                    xpub = sp.x;
                } else {
                    const V3 mn{radd(m.x, rmul(radd(a.x, d.x), p.dt6)), radd(m.y, rmul(radd(a.y, d.y), p.dt6)),
                                radd(m.z, rmul(radd(a.z, d.z), p.dt6))};
                    tmem_st3(ta, mn);
                    xpub = mn.x;
                    if (record && ok) {
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
                    if (last_stage && ok) {
                        double *mm = p.m + ((size_t)b * p.n + k) * 3;
                        mm[0] = mn.x;
                        mm[1] = mn.y;
                        mm[2] = mn.z;
                    }
                }
                if (ok) xdst[ens_x_index(k, bg, p.kp)] = xpub;
            }
            tmem_wait_st();
            ENS_TL(gstage, 2);
            if (!last_stage) {
                // Record-step stop (integrator.py:174-177: the run ends at the first
                // recording step with a non-finite state).  Each group ORs "a
                // divergence at a step <= this one is known" (its own, or another
                // CTA's already in the status key) into its half-column's stop word
                // BEFORE its release increment; the word is read after the
                // counter's acquire, so all row tiles of the half-column read the
                // OR of every contribution and stop together.  Half-columns are
                // not in lockstep: one that is behind keeps going until it reaches
                // the known divergence step, so an earlier divergence of its own
                // members is still found (the reported key stays the minimum).
                // A stale key read is larger, i.e. only delays the stop.
                const bool chk = stage == 3 && record;
                group_sync(grp);  // this group's x rows are written; its cpb half is free again
                if (wl == 0) {
                    if (lane == 0) {
                        if (chk && (*((volatile long long *)&p.status->key) >> 40) <= step)
                            atomicOr(bar + 1, 1ull);
                        __threadfence();
                        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
                    }
                    const unsigned long long stop = open_stage(gstage + 1);
                    if (chk && lane == 0) stop_grp[grp] = (int)stop;
                }
                if (chk) {
                    group_sync(grp);
                    if (stop_grp[grp]) {
                        // drain: the ring's slots of the next stage are armed (their X
                        // was just issued); wait for every copy before leaving
                        for (int i = 0; i < nring; ++i) {
                            mbar_wait(&full[slot], phase);
                            if (++slot == nring) {
                                slot = 0;
                                phase ^= 1;
                            }
                        }
                        goto done;
                    }
                }
            }
        }
        if (record && step == next_rec) {
            next_rec += p.stride;
            ++rec_idx;
        }
    }
done:
    if (lane == 0 && wl == 0) exited[grp] = 1;  // the other group takes no more turns after this one
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_slot),
                     "n"(kEnsTmemCols)
                     : "memory");
}

}  // namespace sto
