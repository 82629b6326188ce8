/* sto_oracle.h -- CPU parity oracle for the coupled-STO RK4 path.
 * TEST INFRASTRUCTURE ONLY (see sto_oracle.c). */
#ifndef STO_ORACLE_H
#define STO_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    STO_ORACLE_OK = 0,
    STO_ORACLE_E_PARAM = 2,
    STO_ORACLE_E_DIVERGED = 3,
    STO_ORACLE_E_NOMEM = 5,
};

/* consts[11] = c_prec, c_damp, h_appl, h_aniso, h_s_prefactor, lambda, a_cp, a_in, px, py, pz */
double sto_oracle_tree_sum(double *buf, int64_t w);
int sto_oracle_derivative(int64_t n, int64_t n_in, const double *w_cp, const double *w_in,
                          const double *consts, const double *m, const double *u,
                          double *out, int threads);
int sto_oracle_integrate(int64_t n, int64_t n_in, const double *w_cp, const double *w_in,
                         const double *consts, double *m, const double *samples,
                         int64_t n_samples, int64_t steps_per_sample, double dt,
                         int64_t steps, int64_t stride, double *states,
                         int64_t *bad_oscillator, int64_t *bad_step, int threads);
int64_t sto_oracle_n_records(int64_t steps, int64_t stride);
int sto_oracle_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
