// sto_ensemble_exact.cuh -- bit-exact batched ensemble (the
// "CUDA-core mul+add" mode): B reservoirs sharing W / W_in, each member's
// trajectory bit-identical to integrate() / the oracle with that member's
// parameters and drive, at ANY horizon (the DMMA path, sto_ensemble_kernel.cuh,
// is held to a tolerance instead because the tensor cores accumulate in their
// own order).
//
// Per RK stage the coupling of every (oscillator k, member b) is
//     cp = adjacent-pairs tree over j of rmul(W[k][j], x_b[j])
// (model.py:31-63, cpu_jit.py:28-45).  With W padded by -0.0 and x by +0.0 (the
// exact additive identity, sto_device.cuh) that tree equals: aligned 32-column
// LEAVES, each a full pairwise tree, then the adjacent-pairs tree over the
// ceil(n/32) leaf nodes -- evaluated here with a binary-counter stack exactly
// as tree_dot_stream does.  Products are separately rounded DMUL, sums DADD
// (no FMA), the RHS and the RK4 combination are the pinned row_rhs /
// stage_point / acc_k2 / rk4_final of the single-trajectory kernels.
//
// Structure (one persistent cooperative launch per run):
//  * Tiles of TR = 8U oscillators x TB = 32 BV members (the host picks U so the
//    tiles fill the SMs: N = 1000, B = 512 -> U = 7, BV = 2: 144 tiles of
//    56 x 64); CTA c owns tiles c, c + G, ... and processes them in that order
//    every stage (G = grid, one CTA per SM).
//  * 8 warps; lane (lr = lane & 7, lb = lane >> 3) of warp w owns U
//    oscillators x BV members: rows lr + 8i, members 4BV w + BV lb + e.
//    Lanes with the same lr read the same W words (broadcast) and lanes with
//    the same lb the same x words: a 4-column step loads 2U + 4 16-byte words
//    (BV = 2) per lane for 16U FP64 ops, conflict-free.
//  * K streams in 32-column chunks through a 2-deep cp.async ring of
//    [TR rows x 34] W (row pitch 34: conflict-free 16-byte row reads) and
//    [32 cols x TB members] x.  A leaf is 64 columns (two chunks): the
//    within-chunk tree is unrolled in registers (three live nodes per
//    output), the first chunk's node waits in a register for the second, and
//    the leaf-level stack lives in shared memory ([level][output][thread],
//    conflict-free).
//  * RK state (m, stage point, acc, k3; the exact order needs k3 kept apart)
//    in global planes [12][np][bp] (coalesced: consecutive lanes hold
//    consecutive member pairs).
//  * Exchange: the stage x of every member is written to x[(g+1)&1][k][b]
//    after the tile's epilogue; a counter per member column (release
//    increment per row tile, acquire polling by thread 0 before the next
//    stage's K loop) orders it -- the DMMA kernel's protocol, including the
//    record-step stop word (integrator.py:174-177).
#pragma once

#include "sto_ensemble_kernel.cuh"

namespace sto {

constexpr int kExThreads = 256; // threads per CTA (8 warps)
constexpr int kExDefaultBV = 2; // members per thread (host default; STO_EX_BV overrides)
constexpr int kExKC = 32;       // K chunk (a leaf is two chunks: 64 columns)
constexpr int kExWP = 34;       // W chunk row pitch (doubles): conflict-free 16-byte row reads
constexpr int kExStages = 2;    // cp.async ring depth
constexpr int kExMaxU = 7;      // rows per thread (tile = 8U oscillators)
constexpr int kExMaxLevels = 8; // leaf stack depth: ceil(n/64) < 256 leaves (n <= 16320)
constexpr int kExMaxTiles = 63; // tiles per CTA and launch
constexpr int kExPlanes = 12;   // m, s, acc, k3 (x, y, z each)

__host__ __device__ constexpr int ex_chunk_w(int u) { return 8 * u * kExWP; }
__host__ __device__ constexpr int ex_tile_members(int bv) { return 32 * bv; }
// ring (W and x chunks) + leaf stack (levels doubles per output: 8U x 32BV
// outputs per tile) + member constants + input weights
__host__ __device__ constexpr size_t ex_smem_bytes(int u, int bv, int levels) {
    return sizeof(double) * ((size_t)kExStages * (ex_chunk_w(u) + kExKC * ex_tile_members(bv)) +
                             (size_t)levels * 8 * u * ex_tile_members(bv) + ex_tile_members(bv) * 11 + 8 * u) +
           64;
}
constexpr size_t kExSmemBudget = 227 * 1024;

struct ExParams {
    int n, np, kp;                // oscillators; allocated rows; K padded (multiple of 32)
    int n_rt, n_ct;               // row tiles, member tiles of this launch
    int batch, bp;                // members of this launch; padded (multiple of 64)
    int member0, batch_total;     // first member of this launch; members of the run
    int n_in, levels;             // leaf-stack depth (bit length of the leaf count)
    const double *w;              // np x kp row-major, -0.0 padded
    const double *w_in;           // n x n_in
    const double *consts;         // (batch_total, 11)
    double *m;                    // (batch_total, n, 3) in/out
    const double *samples;        // member b: samples + b * sample_member_stride
    long long sample_member_stride;
    long long n_samples, sps;
    double dt, h2, dt6;
    long long steps, stride, n_records;
    double *states;               // (n_records, batch_total, n, 3) or null
    double *x;                    // [2][kp][bp] stage x, +0.0 padded
    double *st;                   // [12][np][bp] RK state planes
    unsigned long long *bar;      // per member tile: [0] counter, [1] stop word (32 words apart)
    StatusDev *status;
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// U: oscillator rows per thread, BV: members per thread; tile = TR = 8U
// oscillators x TB = 32BV members, 8 warps; output o = BV*i + e of lane
// (lr = lane & 7, lb = lane >> 3) of warp w is oscillator lr + 8i, member
// 4BV*w + BV*lb + e.
template <int U, int BV>
__global__ void __launch_bounds__(kExThreads, 1) ens_exact_kernel(const __grid_constant__ ExParams p) {
    constexpr int TR = 8 * U;
    constexpr int TB = ex_tile_members(BV);
    constexpr int kExChunkX = kExKC * TB;
    constexpr int NT = kExThreads;
    constexpr int NO = BV * U;                      // outputs per thread
    constexpr int CW = ex_chunk_w(U);
    extern __shared__ __align__(16) double smem[];
    double *ring = smem;                            // kExStages x (W chunk | X chunk)
    double *stk = ring + kExStages * (CW + kExChunkX);  // [levels][NO][threads]
    double *cs = stk + (size_t)p.levels * NO * NT;  // [64][11] member consts of the tile
    double *wins = cs + TB * 11;                 // [TR] input weights (n_in = 1)
    volatile int *sh_stop = reinterpret_cast<volatile int *>(wins + TR);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int lr = lane & 7, lb = lane >> 3;
    const int n_tiles = p.n_rt * p.n_ct;
    const int n_chunks = p.kp / kExKC;
    const long long n_stages = 4 * p.steps;
    const size_t xplane = (size_t)p.kp * p.bp;
    const size_t splane = (size_t)p.np * p.bp;
    int my_tiles = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) ++my_tiles;
    unsigned long long stopped = 0;  // bit i: this CTA's i-th tile has stopped (record-step stop)
    auto row_of = [&](int i) { return lr + 8 * i; };
    const int mcol = 4 * BV * warp + BV * lb;  // first of this lane's members (tile-local)

    // ---- prologue: state planes, x(0), record 0 --------------------------------
    for (int ti = 0; ti < my_tiles; ++ti) {
        const int t = blockIdx.x + ti * gridDim.x;
        const int rt = t % p.n_rt, ct = t / p.n_rt;
        for (int i = tid; i < TR * TB; i += NT) {
            const int rl = i / TB, bl = i % TB;
            const int k = rt * TR + rl, bg = ct * TB + bl;
            if (k >= p.n || bg >= p.batch) continue;
            const double *mm = p.m + ((size_t)(p.member0 + bg) * p.n + k) * 3;
            const double mx = mm[0], my = mm[1], mz = mm[2];
            double *sp = p.st + (size_t)k * p.bp + bg;
            sp[0] = mx;
            sp[splane] = my;
            sp[2 * splane] = mz;
            p.x[(size_t)k * p.bp + bg] = mx;  // buffer 0
            if (p.states) {
                double *so = p.states + ((size_t)(p.member0 + bg) * p.n + k) * 3;
                so[0] = mx;
                so[1] = my;
                so[2] = mz;
            }
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p.bar + 32 * ct) : "memory");
        }
    }

    long long next_rec = p.stride, rec_idx = 1;
    for (long long g = 0; g < n_stages; ++g) {
        const int stage = (int)(g & 3);
        const long long step = (g >> 2) + 1;
        const bool record = stage == 3 && ((step == next_rec) || (step == p.steps));
        const long long sidx = p.n_samples == 1 ? 0 : (step - 1) / p.sps;
        const double h = stage == 2 ? p.dt : p.h2;
        for (int ti = 0; ti < my_tiles; ++ti) {
            if (stopped >> ti & 1ull) continue;
            const int t = blockIdx.x + ti * gridDim.x;
            const int rt = t % p.n_rt, ct = t / p.n_rt;
            const int row0 = rt * TR, col0 = ct * TB;
            unsigned long long *bar = p.bar + 32 * ct;
            // ---- wait until every row tile of this member column published x(g)
            if (tid == 0) {
                const unsigned long long target = (unsigned long long)(g + 1) * p.n_rt;
                unsigned long long v;
                while (true) {
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
                    if (v >= target) break;
                    __nanosleep(32);
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                *sh_stop = (g > 0 && (g & 3) == 0) ? (int)*((volatile unsigned long long *)bar + 1) : 0;
            }
            // member constants and input weights of this tile
            for (int i = tid; i < TB * 11; i += NT) {
                const int b = p.member0 + min(col0 + i / 11, p.batch - 1);
                cs[i] = p.consts[(size_t)b * 11 + i % 11];
            }
            for (int i = tid; i < TR; i += NT)
                wins[i] = (row0 + i < p.n) ? p.w_in[(size_t)(row0 + i) * p.n_in] : 0.0;
            __syncthreads();
            if (*sh_stop) {  // the column stopped after the previous (recording) step
                stopped |= 1ull << ti;
                __syncthreads();  // everyone has read sh_stop before thread 0 rewrites it
                continue;
            }

            // ---- K loop: 32-column chunks through the cp.async ring --------------
            const double *xsrc = p.x + (size_t)(g & 1) * xplane;
            auto issue = [&](int ch) {
                double *slot = ring + (ch % kExStages) * (CW + kExChunkX);
                const int c0 = ch * kExKC;
                for (int i = tid; i < TR * (kExKC / 2); i += NT) {
                    const int r = i / (kExKC / 2), q = i % (kExKC / 2);
                    cp_async16(slot + r * kExWP + 2 * q, p.w + (size_t)(row0 + r) * p.kp + c0 + 2 * q);
                }
                double *xs = slot + CW;
                for (int i = tid; i < kExKC * (TB / 2); i += NT) {
                    const int c = i / (TB / 2), q = i % (TB / 2);
                    cp_async16(xs + c * TB + 2 * q, xsrc + (size_t)(c0 + c) * p.bp + col0 + 2 * q);
                }
            };
            issue(0);
            cp_async_commit();
            double pend[NO];  // node of the leaf's first chunk (leaf = two chunks)
            for (int ch = 0; ch < n_chunks; ++ch) {
                cp_async_wait<0>();
                __syncthreads();  // chunk ch visible to all; the other slot (read in ch - 1) is free
                if (ch + 1 < n_chunks) issue(ch + 1);
                cp_async_commit();
                const double *Ws = ring + (ch % kExStages) * (CW + kExChunkX);
                const double *Xs = Ws + CW;
                double t1[NO], t4[NO], tq[NO];
#pragma unroll
                for (int q = 0; q < 8; ++q) {  // 4-column sub-blocks of the chunk
                    const int c0 = 4 * q;
                    double xa[4][BV];
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        if constexpr (BV == 1) {
                            xa[cc][0] = Xs[(c0 + cc) * TB + mcol];
                        } else {
#pragma unroll
                            for (int h = 0; h < BV / 2; ++h) {
                                const double2 v = *reinterpret_cast<const double2 *>(Xs + (c0 + cc) * TB + mcol + 2 * h);
                                xa[cc][2 * h] = v.x;
                                xa[cc][2 * h + 1] = v.y;
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < U; ++i) {
                        const double2 w01 = *reinterpret_cast<const double2 *>(Ws + row_of(i) * kExWP + c0);
                        const double2 w23 = *reinterpret_cast<const double2 *>(Ws + row_of(i) * kExWP + c0 + 2);
#pragma unroll
                        for (int e = 0; e < BV; ++e) {
                            const int o = BV * i + e;
                            const double x0 = xa[0][e], x1 = xa[1][e], x2 = xa[2][e], x3 = xa[3][e];
                            const double n4 = radd(radd(rmul(w01.x, x0), rmul(w01.y, x1)),
                                                   radd(rmul(w23.x, x2), rmul(w23.y, x3)));
                            // aligned 32-tree over the 8 node4s, unrolled:
                            // ((n0+n1)+(n2+n3)) + ((n4+n5)+(n6+n7))
                            switch (q) {
                                case 0: tq[o] = n4; break;
                                case 1: t1[o] = radd(tq[o], n4); break;
                                case 2: tq[o] = n4; break;
                                case 3: t1[o] = radd(t1[o], radd(tq[o], n4)); break;
                                case 4: tq[o] = n4; break;
                                case 5: t4[o] = radd(tq[o], n4); break;
                                case 6: tq[o] = n4; break;
                                default: t4[o] = radd(t4[o], radd(tq[o], n4)); break;
                            }
                        }
                    }
                }
                if (!(ch & 1) && ch + 1 < n_chunks) {
#pragma unroll
                    for (int o = 0; o < NO; ++o) pend[o] = radd(t1[o], t4[o]);
                } else {
                    // leaf (64 columns; a lone last chunk is the whole leaf: its right
                    // half is -0.0) -> binary-counter stack, tree_dot_stream order
                    const unsigned lf = (unsigned)ch >> 1;
#pragma unroll
                    for (int o = 0; o < NO; ++o) {
                        const double c32 = radd(t1[o], t4[o]);
                        double v = (ch & 1) ? radd(pend[o], c32) : c32;
                        int lvl = 0;
                        while (lf & (1u << lvl)) {
                            v = radd(stk[((size_t)lvl * NO + o) * NT + tid], v);
                            ++lvl;
                        }
                        stk[((size_t)lvl * NO + o) * NT + tid] = v;
                    }
                }
            }
            // ---- fold the stack's right edge: cp per output -------------------------
            const unsigned n_leaves = (unsigned)(n_chunks + 1) >> 1;
            double cp[NO];
#pragma unroll
            for (int o = 0; o < NO; ++o) {
                double acc = 0.0;
                bool have = false;
                for (int lvl = 0; lvl < p.levels; ++lvl) {
                    if (n_leaves & (1u << lvl)) {
                        const double s = stk[((size_t)lvl * NO + o) * NT + tid];
                        acc = have ? radd(s, acc) : s;
                        have = true;
                    }
                }
                cp[o] = acc;
            }

            // ---- epilogue: pinned RHS + RK4 stage update ----------------------------
            double *xdst = p.x + (size_t)((g + 1) & 1) * xplane;
            const bool last_stage = g + 1 == n_stages;
#pragma unroll
            for (int o = 0; o < NO; ++o) {
                const int i = o / BV, e = o % BV;
                const int rl = row_of(i), bl = mcol + e;
                const int k = row0 + rl, bg = col0 + bl;
                if (k >= p.n || bg >= p.batch) continue;
                const double *cb = cs + bl * 11;
                const Consts c{cb[0], cb[1], cb[2], cb[3], cb[4], cb[5], cb[6], cb[7], cb[8], cb[9], cb[10]};
                const int b = p.member0 + bg;
                const double *us = p.samples + (size_t)b * p.sample_member_stride + (size_t)sidx * p.n_in;
                const double cin = (p.n_in == 1) ? rmul(wins[rl], us[0])
                                                 : tree_dot_stream(p.w_in + (size_t)k * p.n_in, us, p.n_in);
                double *sp = p.st + (size_t)k * p.bp + bg;
                auto ld3 = [&](int plane) {
                    return V3{sp[plane * splane], sp[(plane + 1) * splane], sp[(plane + 2) * splane]};
                };
                auto st3 = [&](int plane, V3 v) {
                    sp[plane * splane] = v.x;
                    sp[(plane + 1) * splane] = v.y;
                    sp[(plane + 2) * splane] = v.z;
                };
                const V3 m = ld3(0);
                const V3 cur = stage == 0 ? m : ld3(3);
                const V3 d = row_rhs(cur, cp[o], cin, c);
                double xpub;
                if (stage == 0) {
                    st3(6, d);
                    const V3 sv = stage_point(m, d, p.h2);
                    st3(3, sv);
                    xpub = sv.x;
                } else if (stage == 1) {
                    st3(6, acc_k2(ld3(6), d));
                    const V3 sv = stage_point(m, d, h);
                    st3(3, sv);
                    xpub = sv.x;
                } else if (stage == 2) {
                    st3(9, d);
                    const V3 sv = stage_point(m, d, h);
                    st3(3, sv);
                    xpub = sv.x;
                } else {
                    const V3 mn = rk4_final(m, ld3(6), ld3(9), d, p.dt6);
                    st3(0, mn);
                    xpub = mn.x;
                    if (record) {
                        if (!all_finite(mn)) {
                            atomicMin(&p.status->key, (step << 40) | ((long long)b << 20) | k);
                            p.status->flag = 1;
                        } else if (p.states) {
                            const long long ri = (step == next_rec) ? rec_idx : p.n_records - 1;
                            double *so = p.states + (((size_t)ri * p.batch_total + b) * p.n + k) * 3;
                            so[0] = mn.x;
                            so[1] = mn.y;
                            so[2] = mn.z;
                        }
                    }
                    if (last_stage) {
                        double *mm = p.m + ((size_t)b * p.n + k) * 3;
                        mm[0] = mn.x;
                        mm[1] = mn.y;
                        mm[2] = mn.z;
                    }
                }
                xdst[(size_t)k * p.bp + bg] = xpub;
            }
            __syncthreads();  // tile's x written; ring and stack free for the next tile
            if (!last_stage && tid == 0) {
                // record-step stop word, as in ens_rk4_kernel (divergence at a step
                // <= this one known -> the whole member column stops after it)
                if (record && (*((volatile long long *)&p.status->key) >> 40) <= step) atomicOr(bar + 1, 1ull);
                __threadfence();
                asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
            }
        }
        if (stage == 3 && step == next_rec) {
            next_rec += p.stride;
            ++rec_idx;
        }
        if (my_tiles && stopped == (1ull << my_tiles) - 1ull) break;
    }
}

}  // namespace sto
