/*
 * sto_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the B200 kernels
 * and the timed CPU baseline of bench.py (cpu_baseline / --impl reference).
 * Only tests/, __graft_entry__.smoke() and bench.py may load it; the product
 * path (paper_2312_01121_b200) never does.
 *
 * It restates, operation for operation, the reference package `spinosc`:
 *   - tree_sum      <- backends/cpu_jit.py:28-45  (_tree_reduce), model.py:31-52
 *   - row_rhs       <- backends/cpu_jit.py:48-87  (_row_derivative), model.py:229-301
 *   - derivative    <- backends/cpu_jit.py:101-115 (_derivative_blocks: fixed
 *                      128-block row partition, so threads never change bits)
 *   - integrate     <- integrator.py:91-121 (rk4_step, pinned combination) and
 *                      integrator.py:131-187 (ZOH input, recording grid,
 *                      divergence check on the grid)
 * Build flags (Makefile) forbid FMA contraction and fast-math so every product
 * and sum is rounded separately, exactly as numpy / numba (no fastmath) do.
 *
 * Parity pinned: tests/test_oracle.py checks this file bit-for-bit against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py).
 */
#include "sto_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_ROW_BLOCKS 128 /* cpu_jit.py:25 */

/* In-place adjacent-pairs tree over buf[0:w]; odd tail carried (cpu_jit.py:28-45). */
double sto_oracle_tree_sum(double *buf, int64_t w) {
    if (w <= 0) return 0.0;
    while (w > 1) {
        int64_t half = w / 2;
        for (int64_t j = 0; j < half; ++j) buf[j] = buf[2 * j] + buf[2 * j + 1];
        if (w & 1) {
            buf[half] = buf[w - 1];
            w = half + 1;
        } else {
            w = half;
        }
    }
    return buf[0];
}

typedef struct {
    double c_prec, c_damp, h_appl, h_aniso, pref, lam, a_cp, a_in, px, py, pz;
} consts_t;

static consts_t unpack(const double *c) {
    consts_t k = {c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7], c[8], c[9], c[10]};
    return k;
}

/* First tree level fused with the products: prod[j] = w[2j]*x[2j] + w[2j+1]*x[2j+1]
 * (each product and the sum rounded separately -- the same values the
 * reference's product pass + first _tree_reduce pass produce), odd tail
 * carried; returns the width of the next level.  x is the contiguous m_x. */
#if defined(__GNUC__) && defined(__x86_64__) && !defined(__clang__)
__attribute__((target_clones("avx2", "default")))
#endif
static int64_t products_level1(const double *restrict wr, const double *restrict x,
                               double *restrict prod, int64_t n) {
    const int64_t half = n / 2;
    for (int64_t j = 0; j < half; ++j) prod[j] = wr[2 * j] * x[2 * j] + wr[2 * j + 1] * x[2 * j + 1];
    if (n & 1) {
        prod[half] = wr[n - 1] * x[n - 1];
        return half + 1;
    }
    return half;
}

/* dm/dt of oscillator k into out[3k..3k+2]; cpu_jit.py:48-87 / model.py:229-301.
 * mx = the contiguous x-components of m (gathered once per derivative). */
static void row_rhs(int64_t n, int64_t n_in, const double *w_cp, const double *w_in,
                    const double *m, const double *mx_all, const double *u, double *out,
                    double *prod_cp, double *prod_in, int64_t k, const consts_t *c) {
    const double *wr = w_cp + k * n;
    double cp = sto_oracle_tree_sum(prod_cp, products_level1(wr, mx_all, prod_cp, n));
    const double *wi = w_in + k * n_in;
    for (int64_t j = 0; j < n_in; ++j) prod_in[j] = wi[j] * u[j];
    double cin = sto_oracle_tree_sum(prod_in, n_in);

    double mx = m[3 * k], my = m[3 * k + 1], mz = m[3 * k + 2];
    double mdotp = mx * c->px + my * c->py;
    mdotp = mdotp + mz * c->pz;
    double hs = c->pref / (1.0 + c->lam * mdotp);

    double qx = c->py * mz - c->pz * my;
    double qy = c->pz * mx - c->px * mz;
    double qz = c->px * my - c->py * mx;

    double bx = (c->a_cp * cp + c->a_in * cin) + hs * qx;
    double by = hs * qy;
    double bz = (c->h_appl + c->h_aniso * mz) + hs * qz;

    double ax = my * bz - mz * by;
    double ay = mz * bx - mx * bz;
    double az = mx * by - my * bx;

    double ex = my * az - mz * ay;
    double ey = mz * ax - mx * az;
    double ez = mx * ay - my * ax;

    out[3 * k] = -(c->c_prec * ax) - c->c_damp * ex;
    out[3 * k + 1] = -(c->c_prec * ay) - c->c_damp * ey;
    out[3 * k + 2] = -(c->c_prec * az) - c->c_damp * ez;
}

typedef struct {
    int64_t n, n_in;
    const double *w_cp, *w_in;
    consts_t c;
    double *scratch; /* nthreads x (n + n_in) */
    double *mx;      /* n: contiguous m_x of the current stage */
    int threads;
} ctx_t;

/* One derivative (cpu_jit.py:101-115: 128 fixed row blocks, so the thread
 * count never changes bits).  Called by EVERY thread of an enclosing parallel
 * region (or outside one): gathers m_x, then the row blocks; both worksharing
 * loops end in an implicit barrier. */
static void derivative_in_team(const ctx_t *x, const double *m, const double *u, double *out) {
    const int64_t n = x->n, n_in = x->n_in;
    const int64_t chunk = (n + ORACLE_ROW_BLOCKS - 1) / ORACLE_ROW_BLOCKS;
#pragma omp for schedule(static)
    for (int64_t j = 0; j < n; ++j) x->mx[j] = m[3 * j];
#pragma omp for schedule(static)
    for (int b = 0; b < ORACLE_ROW_BLOCKS; ++b) {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double *prod_cp = x->scratch + (int64_t)tid * (n + n_in);
        double *prod_in = prod_cp + n;
        int64_t lo = (int64_t)b * chunk, hi = lo + chunk < n ? lo + chunk : n;
        for (int64_t k = lo; k < hi; ++k)
            row_rhs(n, n_in, x->w_cp, x->w_in, m, x->mx, u, out, prod_cp, prod_in, k, &x->c);
    }
}

/* Single-thread derivative with no OpenMP constructs (their per-call cost
 * dominates at small n): the same rows in the same order. */
static void derivative_serial(const ctx_t *x, const double *m, const double *u, double *out) {
    const int64_t n = x->n, n_in = x->n_in;
    for (int64_t j = 0; j < n; ++j) x->mx[j] = m[3 * j];
    for (int64_t k = 0; k < n; ++k)
        row_rhs(n, n_in, x->w_cp, x->w_in, m, x->mx, u, out, x->scratch, x->scratch + n, k, &x->c);
}

static void derivative(const ctx_t *x, const double *m, const double *u, double *out) {
    if (x->threads == 1) {
        derivative_serial(x, m, u, out);
        return;
    }
#pragma omp parallel num_threads(x->threads)
    derivative_in_team(x, m, u, out);
}

static int ctx_init(ctx_t *x, int64_t n, int64_t n_in, const double *w_cp,
                    const double *w_in, const double *consts, int threads) {
    if (threads < 1) threads = 1;
    x->n = n;
    x->n_in = n_in;
    x->w_cp = w_cp;
    x->w_in = w_in;
    x->c = unpack(consts);
    x->threads = threads;
    x->scratch = (double *)malloc(sizeof(double) * ((size_t)threads * (size_t)(n + n_in) + (size_t)n));
    x->mx = x->scratch ? x->scratch + (size_t)threads * (size_t)(n + n_in) : NULL;
    return x->scratch ? 0 : -1;
}

int sto_oracle_derivative(int64_t n, int64_t n_in, const double *w_cp, const double *w_in,
                          const double *consts, const double *m, const double *u,
                          double *out, int threads) {
    ctx_t x;
    if (n < 1 || n_in < 1) return STO_ORACLE_E_PARAM;
    if (ctx_init(&x, n, n_in, w_cp, w_in, consts, threads)) return STO_ORACLE_E_NOMEM;
    derivative(&x, m, u, out);
    free(x.scratch);
    return STO_ORACLE_OK;
}

static int64_t first_nonfinite_row(int64_t n, const double *m) {
    for (int64_t k = 0; k < n; ++k)
        if (!isfinite(m[3 * k]) || !isfinite(m[3 * k + 1]) || !isfinite(m[3 * k + 2]))
            return k;
    return -1;
}

/* integrator.py:91-187.  m holds m0 on entry and the last state on return.
 * states (n_record x n x 3) receives the recorded grid {0, s, 2s, ...} u {steps};
 * n_record must equal sto_oracle_n_records(steps, stride). */
int sto_oracle_integrate(int64_t n, int64_t n_in, const double *w_cp, const double *w_in,
                         const double *consts, double *m, const double *samples,
                         int64_t n_samples, int64_t steps_per_sample, double dt,
                         int64_t steps, int64_t stride, double *states,
                         int64_t *bad_oscillator, int64_t *bad_step, int threads) {
    if (n < 1 || n_in < 1 || steps < 1 || stride < 1 || n_samples < 1 ||
        steps_per_sample < 1 || !(dt > 0.0))
        return STO_ORACLE_E_PARAM;
    ctx_t x;
    if (ctx_init(&x, n, n_in, w_cp, w_in, consts, threads)) return STO_ORACLE_E_NOMEM;
    const size_t sz = (size_t)n * 3;
    double *buf = (double *)malloc(sizeof(double) * sz * 5);
    if (!buf) {
        free(x.scratch);
        return STO_ORACLE_E_NOMEM;
    }
    double *k1 = buf, *k2 = buf + sz, *k3 = buf + 2 * sz, *k4 = buf + 3 * sz, *s = buf + 4 * sz;
    const double h2 = dt * 0.5, dt_6 = dt / 6.0; /* integrator.py:103-104 */
    int rc = STO_ORACLE_OK;
    int64_t rec = 1;
    memcpy(states, m, sizeof(double) * sz);
    const int64_t isz = (int64_t)sz;
    if (x.threads == 1) { /* serial: no OpenMP constructs on the small-n path */
        for (int64_t step = 1; step <= steps; ++step) {
            const double *u =
                samples + (n_samples == 1 ? 0 : ((step - 1) / steps_per_sample)) * n_in;
            derivative_serial(&x, m, u, k1);
            for (int64_t i = 0; i < isz; ++i) s[i] = m[i] + k1[i] * h2;
            derivative_serial(&x, s, u, k2);
            for (int64_t i = 0; i < isz; ++i) s[i] = m[i] + k2[i] * h2;
            derivative_serial(&x, s, u, k3);
            for (int64_t i = 0; i < isz; ++i) s[i] = m[i] + k3[i] * dt;
            derivative_serial(&x, s, u, k4);
            for (int64_t i = 0; i < isz; ++i) {
                double t1 = k1[i] + k2[i] * 2.0;
                double t2 = k3[i] * 2.0 + k4[i];
                t1 = t1 + t2;
                t1 = t1 * dt_6;
                m[i] = m[i] + t1;
            }
            if (step % stride == 0 || step == steps) {
                int64_t bad = first_nonfinite_row(n, m);
                if (bad >= 0) {
                    if (bad_oscillator) *bad_oscillator = bad;
                    if (bad_step) *bad_step = step;
                    rc = STO_ORACLE_E_DIVERGED;
                    break;
                }
                memcpy(states + (size_t)rec * sz, m, sizeof(double) * sz);
                ++rec;
            }
        }
        free(buf);
        free(x.scratch);
        return rc;
    }
    /* one parallel region for the whole run (no fork/join per derivative); the
     * element-wise RK4 updates are worksharing loops -- same values per index */
#pragma omp parallel num_threads(x.threads)
    for (int64_t step = 1; step <= steps; ++step) {
        const double *u =
            samples + (n_samples == 1 ? 0 : ((step - 1) / steps_per_sample)) * n_in;
        derivative_in_team(&x, m, u, k1);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < isz; ++i) s[i] = m[i] + k1[i] * h2;
        derivative_in_team(&x, s, u, k2);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < isz; ++i) s[i] = m[i] + k2[i] * h2;
        derivative_in_team(&x, s, u, k3);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < isz; ++i) s[i] = m[i] + k3[i] * dt;
        derivative_in_team(&x, s, u, k4);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < isz; ++i) {
            double t1 = k1[i] + k2[i] * 2.0;
            double t2 = k3[i] * 2.0 + k4[i];
            t1 = t1 + t2;
            t1 = t1 * dt_6;
            m[i] = m[i] + t1;
        }
        if (step % stride == 0 || step == steps) {
#pragma omp single
            {
                int64_t bad = first_nonfinite_row(n, m);
                if (bad >= 0) {
                    if (bad_oscillator) *bad_oscillator = bad;
                    if (bad_step) *bad_step = step;
                    rc = STO_ORACLE_E_DIVERGED;
                } else {
                    memcpy(states + (size_t)rec * sz, m, sizeof(double) * sz);
                    ++rec;
                }
            } /* implicit barrier: every thread sees rc */
            if (rc != STO_ORACLE_OK) break;
        }
    }
    free(buf);
    free(x.scratch);
    return rc;
}

int64_t sto_oracle_n_records(int64_t steps, int64_t stride) {
    if (steps < 1 || stride < 1) return 0;
    return steps / stride + 1 + (steps % stride != 0);
}

int sto_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
