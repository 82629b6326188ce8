// sto_device.cuh -- device-side building blocks of the coupled-STO RK4 path.
//
// Bit-exactness contract (SURVEY §8(a), §7 "hard parts"):
//  * every product and sum is rounded separately: the arithmetic below goes
//    through __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn (which ptxas never
//    contracts into DFMA) and the library is also built with -fmad=false;
//  * operation order is the reference's pinned order: row_rhs() restates
//    backends/cpu_jit.py:62-87 (== model.py:239-301), the RK4 combination
//    restates integrator.py:100-121;
//  * row sums use the reference's adjacent-pairs tree (model.py:31-52,
//    cpu_jit.py:28-45), which equals the aligned power-of-two tree over the
//    row padded with -0.0 (the exact additive identity of IEEE round-to-
//    nearest, so padding never changes a bit, signed zeros included).
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace sto {

// ----------------------------------------------------------------------------
// strict IEEE scalar helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }

// Correctly rounded a/b without the library division's on-chain range check.
//
// __ddiv_rn costs ~113 cycles of dependent latency (profiles/r01_microbench.json),
// most of it the MUFU seed, three Newton/FMA corrections and a range test whose
// branch sits in front of every consumer.  Here the quotient comes from a
// shorter chain (seed -> e -> q0 = a r0 (1 + e) -> remainder -> q: the seed
// plus four DFMA) and its correctness is *proved* afterwards, off the chain:
//   * q == RN(a/b) iff |a/b - q| < half the spacing of doubles on a/b's side
//     of q, i.e. |a - b*q| < |b| * ulp(q)/2 (ulp(q)/4 when q is a power of two,
//     conservatively, so the narrower gap below 2^k is used on both sides);
//     an exact midpoint is impossible for a quotient of two doubles (away from
//     underflow), so the comparison is strict;
//   * a - b*q is exact in one FMA whenever |q - a/b| <= 1 ulp (the remainder is
//     a multiple of ulp(b)*ulp(q) of magnitude < |b|*ulp(q): it fits 53 bits);
//     a q off by more fails the test by a wide margin either way;
//   * the exponent guards keep every quantity above (q, b, b*ulp/2, the
//     remainder) normal and finite; outside them, or for NaN/inf/0, ok = false.
// The caller must redo the work with rdiv() when ok is false (the tiny kernel
// replays its group of RK4 steps; ~3e-4 of the quotients, see sto_selftest_div).
// IEEE division is unique, so the bits equal __ddiv_rn's.
// STO_DIV_SHORT (default): seed + FOUR DFMA (one correction with the seed
// itself); ~3e-4 of the quotients miss the last bit and fail the proof (replayed).
// 0: seed + five DFMA (a refined reciprocal), every RHS-domain quotient proved.
// N = 1: 2.44e6 vs 2.39e6 RK4 steps/s (profiles/r02k_division_variants.txt).
#ifndef STO_DIV_SHORT
#define STO_DIV_SHORT 1
#endif
__device__ __forceinline__ double rdiv_spec(double a, double b, bool &ok) {
    double r0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(b));
    const double e = __fma_rn(-b, r0, 1.0);
    const double ar0 = __dmul_rn(a, r0);
#if STO_DIV_SHORT
    // seed + four DFMA: q0 = a r0 (1 + e), one correction with the seed itself
    const double q0 = __fma_rn(ar0, e, ar0);
    const double rem = __fma_rn(-b, q0, a);
    const double q = __fma_rn(rem, r0, q0);
#else
    const double pe = __fma_rn(e, e, e);
    const double y = __fma_rn(r0, pe, r0);
    const double q0 = __fma_rn(ar0, pe, ar0);
    const double rem = __fma_rn(-b, q0, a);
    const double q = __fma_rn(rem, y, q0);
#endif
    // ---- proof of correct rounding (independent of the chain above) ----
    const double rem2 = __fma_rn(-b, q, a);
    const long long qb = __double_as_longlong(q);
    const long long bb = __double_as_longlong(b);
    const unsigned eq = (unsigned)(qb >> 52) & 0x7ffu;
    const unsigned eb = (unsigned)(bb >> 52) & 0x7ffu;
    // ulp(q)/2 as a double: exponent eq - 53 (eq - 54 for a power of two)
    const unsigned eh = eq - 53u - ((qb & 0xfffffffffffffLL) == 0 ? 1u : 0u);
    const double half_ulp = __longlong_as_double((long long)eh << 52);
    const double lim = __dmul_rn(fabs(b), half_ulp);
    ok = (eq - 400u < 1200u) & (eb - 823u < 400u) & (fabs(rem2) < lim);  // 2^-623 <= |q| < 2^577, 2^-200 <= |b| < 2^200
    return q;
}

struct Consts {
    double c_prec, c_damp, h_appl, h_aniso, pref, lam, a_cp, a_in, px, py, pz;
};

struct V3 {
    double x, y, z;
};

// dm/dt of one oscillator given its coupling row sum `cp` and input row sum
// `cin`.  cpu_jit.py:62-87 / model.py:239-301, operation for operation.
// Split in two: everything that depends only on the oscillator's own state
// (row_rhs_pre: m.p, the IEEE division for h_s, p x m, b_y, b_z, (m x b)_x)
// can be evaluated while the coupling GEMV / exchange is still in flight;
// row_rhs_post finishes once cp is known.  Same operations, same order.
struct RhsPre {
    V3 m;
    double hs_qx, by, bz, ax, ain_cin;
};

// kSpec: the division goes through rdiv_spec and `ok` collects its proof
// (the caller replays the step with kSpec = false when any proof failed).
template <bool kSpec = false>
__device__ __forceinline__ RhsPre row_rhs_pre(V3 m, double cin, const Consts &c, bool *ok = nullptr) {
    double md = radd(rmul(m.x, c.px), rmul(m.y, c.py));
    md = radd(md, rmul(m.z, c.pz));
    double hs;
    if constexpr (kSpec) {
        bool good;
        hs = rdiv_spec(c.pref, radd(1.0, rmul(c.lam, md)), good);
        *ok = *ok & good;
    } else {
        hs = rdiv(c.pref, radd(1.0, rmul(c.lam, md)));
    }
    const double qx = rsub(rmul(c.py, m.z), rmul(c.pz, m.y));
    const double qy = rsub(rmul(c.pz, m.x), rmul(c.px, m.z));
    const double qz = rsub(rmul(c.px, m.y), rmul(c.py, m.x));
    RhsPre r;
    r.m = m;
    r.hs_qx = rmul(hs, qx);
    r.by = rmul(hs, qy);
    r.bz = radd(radd(c.h_appl, rmul(c.h_aniso, m.z)), rmul(hs, qz));
    r.ax = rsub(rmul(m.y, r.bz), rmul(m.z, r.by));
    r.ain_cin = rmul(c.a_in, cin);
    return r;
}

__device__ __forceinline__ V3 row_rhs_post(const RhsPre &r, double cp, const Consts &c) {
    const V3 &m = r.m;
    const double bx = radd(radd(rmul(c.a_cp, cp), r.ain_cin), r.hs_qx);
    const double ay = rsub(rmul(m.z, bx), rmul(m.x, r.bz));
    const double az = rsub(rmul(m.x, r.by), rmul(m.y, bx));
    const double ex = rsub(rmul(m.y, az), rmul(m.z, ay));
    const double ey = rsub(rmul(m.z, r.ax), rmul(m.x, az));
    const double ez = rsub(rmul(m.x, ay), rmul(m.y, r.ax));
    V3 d;
    d.x = rsub(-rmul(c.c_prec, r.ax), rmul(c.c_damp, ex));
    d.y = rsub(-rmul(c.c_prec, ay), rmul(c.c_damp, ey));
    d.z = rsub(-rmul(c.c_prec, az), rmul(c.c_damp, ez));
    return d;
}

template <bool kSpec = false>
__device__ __forceinline__ V3 row_rhs(V3 m, double cp, double cin, const Consts &c, bool *ok = nullptr) {
    return row_rhs_post(row_rhs_pre<kSpec>(m, cin, c, ok), cp, c);
}

// s = m + k*h   (integrator.py:107-108, 110-111, 113-114)
__device__ __forceinline__ V3 stage_point(V3 m, V3 k, double h) {
    return V3{radd(m.x, rmul(k.x, h)), radd(m.y, rmul(k.y, h)), radd(m.z, rmul(k.z, h))};
}

// acc = k1 + k2*2   (integrator.py:117-118)
__device__ __forceinline__ V3 acc_k2(V3 k1, V3 k2) {
    return V3{radd(k1.x, rmul(k2.x, 2.0)), radd(k1.y, rmul(k2.y, 2.0)),
              radd(k1.z, rmul(k2.z, 2.0))};
}

// m + ((acc + (k3*2 + k4)) * dt_6)   (integrator.py:119-121)
__device__ __forceinline__ V3 rk4_final(V3 m, V3 acc, V3 k3, V3 k4, double dt6) {
    V3 r;
    r.x = radd(m.x, rmul(radd(acc.x, radd(rmul(k3.x, 2.0), k4.x)), dt6));
    r.y = radd(m.y, rmul(radd(acc.y, radd(rmul(k3.y, 2.0), k4.y)), dt6));
    r.z = radd(m.z, rmul(radd(acc.z, radd(rmul(k3.z, 2.0), k4.z)), dt6));
    return r;
}

__device__ __forceinline__ bool all_finite(V3 m) {
    return isfinite(m.x) && isfinite(m.y) && isfinite(m.z);
}

// Pinned adjacent-pairs tree of a[i]*b[i], i < w, streamed with a carry stack
// (binary counter): each completed aligned subtree is merged left+right as
// soon as its right sibling completes; the final fold adds the incomplete
// right edge (the padded region) exactly as the odd-tail carry does.
__device__ __forceinline__ double tree_dot_stream(const double *a, const double *b, int w) {
    double stk[32];
    unsigned cnt = 0;
    for (int i = 0; i < w; ++i) {
        double v = rmul(a[i], b[i]);
        int lvl = 0;
        while (cnt & (1u << lvl)) {
            v = radd(stk[lvl], v);
            ++lvl;
        }
        stk[lvl] = v;
        ++cnt;
    }
    double acc = 0.0;
    bool have = false;
    for (int lvl = 0; lvl < 32; ++lvl) {
        if (cnt & (1u << lvl)) {
            acc = have ? radd(stk[lvl], acc) : stk[lvl];
            have = true;
        }
    }
    return acc;
}

// In-place adjacent-pairs tree over buf[0:w] (cpu_jit.py:28-45 verbatim order).
__device__ __forceinline__ double tree_inplace(double *buf, int w) {
    while (w > 1) {
        const int half = w >> 1;
        for (int j = 0; j < half; ++j) buf[j] = radd(buf[2 * j], buf[2 * j + 1]);
        if (w & 1) {
            buf[half] = buf[w - 1];
            w = half + 1;
        } else {
            w = half;
        }
    }
    return buf[0];
}

// ----------------------------------------------------------------------------
// Column schedule of the device W layout ("lane-blocked" segments).
//
// A row is cut into segments of S = 32*C columns, C a power of two: first
// `nfull` segments of 512 (C = 16), then a tail of decreasing sizes from
// {256, 128, 64} plus one zero-padded 64 segment for the last < 64 columns.
// Sizes never increase, so every segment is an aligned node of the padded
// power-of-two tree.  Inside a segment, lane l owns the C contiguous
// columns [l*C, (l+1)*C); they are stored so that a warp-wide 16-byte load
// i delivers columns l*C + 2i, +1 to lane l:
//     offset(l, q) = ((q >> 1) * 32 + l) * 2 + (q & 1)
// Hence every load is perfectly coalesced (512 B per warp instruction), each
// lane reduces its chunk in registers, and a 5-level xor butterfly finishes
// the segment node -- all in the reference's tree order.
// ----------------------------------------------------------------------------
constexpr int kSegFull = 512;
constexpr int kMaxTail = 4;
constexpr int kMaxLeaves = 8;  // block_cols / 512 <= 8

struct ColSched {
    int n;        // real columns
    int ldw;      // padded physical width
    int nfull;    // 512-column segments
    int ntail;    // tail segments
    int tail_base[kMaxTail];
    int tail_c[kMaxTail];  // columns per lane in each tail segment
    int blk;      // columns per work block (512 * 2^r, r <= 3)
    int nblocks;  // ceil(ldw / blk)
};

__host__ __device__ inline int seg_offset(int l, int q) { return (((q >> 1) << 5) + l) * 2 + (q & 1); }

// physical position of logical column k
__host__ __device__ inline int col_perm(const ColSched &s, int k) {
    if (k < s.nfull * kSegFull) {
        const int q = k & (kSegFull - 1);
        return (k & ~(kSegFull - 1)) + seg_offset(q >> 4, q & 15);
    }
    for (int t = 0; t < s.ntail; ++t) {
        const int c = s.tail_c[t];
        const int base = s.tail_base[t];
        if (k < base + 32 * c) {
            const int q = k - base;
            return base + seg_offset(q / c, q % c);
        }
    }
    return -1;
}

// Load policies for W.
enum class WSrc { Shared, GlobalL2, GlobalStream };

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// `pol` is the L2 cache-hint policy of this row (global sources): the streaming
// kernel keeps a slice of W L2-resident (evict_last) and streams the rest
// (evict_first); see KParams::l2_keep_rows.
template <WSrc S>
__device__ __forceinline__ double2 load_w2(const double *p, uint64_t pol) {
    if constexpr (S == WSrc::Shared) {
        return *reinterpret_cast<const double2 *>(p);
    } else {
        double2 v;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                     : "=d"(v.x), "=d"(v.y)
                     : "l"(p), "l"(pol));
        return v;
    }
}

// Node of one segment (32*C columns).  wseg/xseg point at the segment start
// of the W row and of the staged X vector (same layout).
template <int C, WSrc S>
__device__ __forceinline__ double segment_node(const double *wseg, const double *xseg, int lane,
                                               uint64_t pol) {
    double p[C];
#pragma unroll
    for (int i = 0; i < C / 2; ++i) {
        const double2 w = load_w2<S>(wseg + ((i << 5) + lane) * 2, pol);
        const double2 x = *reinterpret_cast<const double2 *>(xseg + ((i << 5) + lane) * 2);
        p[2 * i] = rmul(w.x, x.x);
        p[2 * i + 1] = rmul(w.y, x.y);
    }
#pragma unroll
    for (int w = C; w > 1; w >>= 1) {
#pragma unroll
        for (int j = 0; j < w / 2; ++j) p[j] = radd(p[2 * j], p[2 * j + 1]);
    }
    double v = p[0];
#pragma unroll
    for (int mask = 1; mask < 32; mask <<= 1) v = radd(v, __shfl_xor_sync(0xffffffffu, v, mask));
    return v;
}

template <WSrc S>
__device__ __forceinline__ double tail_segment_node(int c, const double *wseg, const double *xseg,
                                                    int lane, uint64_t pol) {
    switch (c) {
        case 8: return segment_node<8, S>(wseg, xseg, lane, pol);
        case 4: return segment_node<4, S>(wseg, xseg, lane, pol);
        default: return segment_node<2, S>(wseg, xseg, lane, pol);
    }
}

// Node of one work block [b*blk, (b+1)*blk) of one row: its full 512-segment
// nodes are leaves; the tail (if the block holds it) is folded right to left
// (sizes decrease, so T = S0 + (S1 + (... + Sk))) into one 512-level leaf;
// the leaves then go through the pinned pairwise tree (width <= 8).
// wrow/xrow point at column 0 of the row / of the X window (x_base = first
// physical column held in the X window).
template <WSrc S>
__device__ __forceinline__ double block_node(const ColSched &cs, int b, const double *wrow,
                                             const double *xwin, int x_base, int lane, uint64_t pol) {
    const int c0 = b * cs.blk;
    const int seg0 = c0 / kSegFull;
    const int per = cs.blk / kSegFull;
    int nf = cs.nfull - seg0;
    nf = nf < 0 ? 0 : (nf > per ? per : nf);
    const bool has_tail = cs.ntail > 0 && cs.tail_base[0] >= c0 && cs.tail_base[0] < c0 + cs.blk;

    double leaf[kMaxLeaves];
#pragma unroll
    for (int j = 0; j < kMaxLeaves; ++j) {
        if (j < nf) {
            const int col = (seg0 + j) * kSegFull;
            leaf[j] = segment_node<16, S>(wrow + col, xwin + (col - x_base), lane, pol);
        }
    }
    int width = nf;
    if (has_tail) {
        double t = 0.0;
        for (int k = cs.ntail - 1; k >= 0; --k) {
            const int col = cs.tail_base[k];
            const double v = tail_segment_node<S>(cs.tail_c[k], wrow + col, xwin + (col - x_base), lane, pol);
            t = (k == cs.ntail - 1) ? v : radd(v, t);
        }
#pragma unroll
        for (int j = 0; j < kMaxLeaves; ++j)
            if (j == nf) leaf[j] = t;
        width = nf + 1;
    }
    // pinned pairwise tree over leaf[0:width], compile-time register indices
#pragma unroll
    for (int lvl = 0; lvl < 3; ++lvl) {
#pragma unroll
        for (int j = 0; j < (kMaxLeaves >> (lvl + 1)); ++j) {
            if (2 * j + 1 < width)
                leaf[j] = radd(leaf[2 * j], leaf[2 * j + 1]);
            else if (2 * j < width)
                leaf[j] = leaf[2 * j];
        }
        width = (width + 1) >> 1;
    }
    return leaf[0];
}

}  // namespace sto
