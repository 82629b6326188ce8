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
//  * Tiles of 32 oscillators x 64 members; CTA c owns tiles c, c + G, ... and
//    processes them in that order every stage (G = grid, one CTA per SM).
//  * A CTA tile is 8 warps of 8 x 32 outputs (warp row group wr, member half
//    wb); lane (lr, lb) owns 2 oscillators x 4 members: rows 8wr + lr + 4i,
//    members 32wb + 16j + 2lb + e.  Lanes with the same lr read the same W
//    words (broadcast) and lanes with the same lb the same x words, so each
//    4-column step loads 12 16-byte words per lane for 64 FP64 ops.
//  * K streams in 32-column chunks (one leaf) through a 3-deep cp.async ring
//    of [32 rows x 34] W (row pitch 34: conflict-free 16-byte row reads) and
//    [32 cols x 64 members] x; the leaf-level stack lives in shared memory
//    ([level][output][thread], conflict-free), the within-leaf nodes in
//    registers (unrolled: three live nodes per output).
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

constexpr int kExTR = 32;       // oscillators per tile
constexpr int kExTB = 64;       // members per tile
constexpr int kExThreads = 256; // 8 warps
constexpr int kExKC = 32;       // K chunk = one leaf
constexpr int kExWP = 34;       // W chunk row pitch (doubles)
constexpr int kExStages = 3;    // cp.async ring depth
constexpr int kExOut = 8;       // outputs per thread
constexpr int kExMaxLevels = 8;   // leaf stack depth: ceil(n/32) < 256 leaves (n <= 8160)
constexpr int kExMaxTiles = 63;   // tiles per CTA and launch
constexpr int kExPlanes = 12;     // m, s, acc, k3 (x, y, z each)
constexpr int kExChunkW = kExTR * kExWP;       // doubles
constexpr int kExChunkX = kExKC * kExTB;       // doubles

__host__ __device__ constexpr size_t ex_smem_bytes(int levels) {
    return sizeof(double) * ((size_t)kExStages * (kExChunkW + kExChunkX) +
                             (size_t)levels * kExOut * kExThreads + kExTB * 11 + kExTR) +
           64;
}

static_assert(ex_smem_bytes(kExMaxLevels) <= 227 * 1024, "exact ensemble shared memory budget");

struct ExParams {
    int n, np, kp;                // oscillators; padded rows (multiple of 32); K padded (multiple of 32)
    int n_rt, n_ct;               // row tiles, member tiles
    int batch, bp;                // members of this launch; padded (multiple of 64)
    int member0, batch_total;     // first member of this launch; members of the run
    int n_in, levels;             // leaf-stack depth (>= ceil(log2(kp / 32)))
    const double *w;              // np x kp row-major, -0.0 padded
    const double *w_in;           // n x n_in
    const double *consts;         // (batch, 11)
    double *m;                    // (batch, n, 3) in/out
    const double *samples;        // member b: samples + b * sample_member_stride
    long long sample_member_stride;
    long long n_samples, sps;
    double dt, h2, dt6;
    long long steps, stride, n_records;
    double *states;               // (n_records, batch, n, 3) or null
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

__global__ void __launch_bounds__(kExThreads, 1) ens_exact_kernel(const __grid_constant__ ExParams p) {
    extern __shared__ __align__(16) double smem[];
    double *ring = smem;                                           // kExStages x (W chunk | X chunk)
    double *stk = ring + kExStages * (kExChunkW + kExChunkX);      // [levels][kExOut][threads]
    double *cs = stk + (size_t)p.levels * kExOut * kExThreads;     // [64][11] member consts of the tile
    double *wins = cs + kExTB * 11;                                // [32] input weights (n_in = 1)
    volatile int *sh_stop = reinterpret_cast<volatile int *>(wins + kExTR);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wr = warp & 3, wb = warp >> 2, lr = lane & 3, lb = lane >> 2;
    const int n_tiles = p.n_rt * p.n_ct;
    const int n_chunks = p.kp / kExKC;
    const long long n_stages = 4 * p.steps;
    const size_t xplane = (size_t)p.kp * p.bp;
    const size_t splane = (size_t)p.np * p.bp;
    int my_tiles = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) ++my_tiles;
    unsigned long long stopped = 0;  // bit i: this CTA's i-th tile has stopped (record-step stop)

    // local row / member of output o = (i, j, e): o = 4i + 2j + e
    auto row_of = [&](int i) { return 8 * wr + lr + 4 * i; };
    auto mem_of = [&](int j, int e) { return 32 * wb + 16 * j + 2 * lb + e; };

    // ---- prologue: state planes, x(0), record 0 --------------------------------
    for (int ti = 0; ti < my_tiles; ++ti) {
        const int t = blockIdx.x + ti * gridDim.x;
        const int rt = t % p.n_rt, ct = t / p.n_rt;
        for (int i = tid; i < kExTR * kExTB; i += kExThreads) {
            const int rl = i / kExTB, bl = i % kExTB;
            const int k = rt * kExTR + rl, bg = ct * kExTB + bl;
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
            const int row0 = rt * kExTR, col0 = ct * kExTB;
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
            for (int i = tid; i < kExTB * 11; i += kExThreads) {
                const int b = p.member0 + min(col0 + i / 11, p.batch - 1);
                cs[i] = p.consts[(size_t)b * 11 + i % 11];
            }
            for (int i = tid; i < kExTR; i += kExThreads)
                wins[i] = (row0 + i < p.n) ? p.w_in[(size_t)(row0 + i) * p.n_in] : 0.0;
            __syncthreads();
            if (*sh_stop) {  // the column stopped after the previous (recording) step
                stopped |= 1ull << ti;
                __syncthreads();  // everyone has read sh_stop before thread 0 rewrites it
                continue;
            }

            // ---- K loop: leaves of 32 columns through the cp.async ring ---------
            const double *xsrc = p.x + (size_t)(g & 1) * xplane;
            auto issue = [&](int ch) {
                double *slot = ring + (ch % kExStages) * (kExChunkW + kExChunkX);
                const int c0 = ch * kExKC;
                // W: 32 rows x 32 cols -> pitch 34; 16 x 16-byte pieces per row
                for (int i = tid; i < kExTR * (kExKC / 2); i += kExThreads) {
                    const int r = i / (kExKC / 2), q = i % (kExKC / 2);
                    cp_async16(slot + r * kExWP + 2 * q, p.w + (size_t)(row0 + r) * p.kp + c0 + 2 * q);
                }
                // X: 32 cols x 64 members; 32 pieces per column row
                double *xs = slot + kExChunkW;
                for (int i = tid; i < kExKC * (kExTB / 2); i += kExThreads) {
                    const int c = i / (kExTB / 2), q = i % (kExTB / 2);
                    cp_async16(xs + c * kExTB + 2 * q, xsrc + (size_t)(c0 + c) * p.bp + col0 + 2 * q);
                }
            };
            issue(0);
            cp_async_commit();
            if (n_chunks > 1) issue(1);
            cp_async_commit();
            for (int ch = 0; ch < n_chunks; ++ch) {
                cp_async_wait<1>();
                __syncthreads();  // chunk ch visible to all; slot (ch + 2) % 3 free (read in ch - 1)
                if (ch + 2 < n_chunks) issue(ch + 2);
                cp_async_commit();
                const double *Ws = ring + (ch % kExStages) * (kExChunkW + kExChunkX);
                const double *Xs = Ws + kExChunkW;
                double t1[kExOut], t4[kExOut], tq[kExOut];
#pragma unroll
                for (int q = 0; q < 8; ++q) {  // 4-column sub-blocks of the leaf
                    const int c0 = 4 * q;
                    double2 wa[2][2], xa[4][2];
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        wa[i][0] = *reinterpret_cast<const double2 *>(Ws + row_of(i) * kExWP + c0);
                        wa[i][1] = *reinterpret_cast<const double2 *>(Ws + row_of(i) * kExWP + c0 + 2);
                    }
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            xa[cc][j] = *reinterpret_cast<const double2 *>(Xs + (c0 + cc) * kExTB + mem_of(j, 0));
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {
                                const int o = 4 * i + 2 * j + e;
                                const double x0 = e ? xa[0][j].y : xa[0][j].x, x1 = e ? xa[1][j].y : xa[1][j].x;
                                const double x2 = e ? xa[2][j].y : xa[2][j].x, x3 = e ? xa[3][j].y : xa[3][j].x;
                                const double n4 = radd(radd(rmul(wa[i][0].x, x0), rmul(wa[i][0].y, x1)),
                                                       radd(rmul(wa[i][1].x, x2), rmul(wa[i][1].y, x3)));
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
                // leaf -> binary-counter stack (left sibling first), tree_dot_stream order
#pragma unroll
                for (int o = 0; o < kExOut; ++o) {
                    double v = radd(t1[o], t4[o]);
                    int lvl = 0;
                    while ((unsigned)ch & (1u << lvl)) {
                        v = radd(stk[((size_t)lvl * kExOut + o) * kExThreads + tid], v);
                        ++lvl;
                    }
                    stk[((size_t)lvl * kExOut + o) * kExThreads + tid] = v;
                }
            }
            // ---- fold the stack's right edge: cp per output -------------------------
            double cp[kExOut];
#pragma unroll
            for (int o = 0; o < kExOut; ++o) {
                double acc = 0.0;
                bool have = false;
                for (int lvl = 0; lvl < p.levels; ++lvl) {
                    if ((unsigned)n_chunks & (1u << lvl)) {
                        const double s = stk[((size_t)lvl * kExOut + o) * kExThreads + tid];
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
            for (int o = 0; o < kExOut; ++o) {
                const int i = o >> 2, j = (o >> 1) & 1, e = o & 1;
                const int rl = row_of(i), bl = mem_of(j, e);
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
                    const V3 s = stage_point(m, d, p.h2);
                    st3(3, s);
                    xpub = s.x;
                } else if (stage == 1) {
                    st3(6, acc_k2(ld3(6), d));
                    const V3 s = stage_point(m, d, h);
                    st3(3, s);
                    xpub = s.x;
                } else if (stage == 2) {
                    st3(9, d);
                    const V3 s = stage_point(m, d, h);
                    st3(3, s);
                    xpub = s.x;
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
