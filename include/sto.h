/*
 * sto.h -- C ABI of the B200-native coupled spin-torque-oscillator simulator.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (`spinosc`, pure Python) has no FFI of its own; these entry points are what
 * its plugin layer binds (see INTEGRATION.md for the ctypes stub a spinosc
 * maintainer registers via `spinosc.backends.register_backend`):
 *
 *   sto_probe            <- backends/gpu.py:34-37        is_available()
 *   sto_plan_create      <- backends/gpu.py:55-77        TorchBackend.__init__ (W, W_in
 *                                                         resident on the device once)
 *   sto_derivative       <- backends/__init__.py:5-7,48-50  derivative(m, u, out) contract
 *                           (model.py:206-302 llg_derivative; gpu.py:83-119)
 *   sto_integrate        <- integrator.py:131-187 integrate() time loop with
 *                           integrator.py:91-121 rk4_step, fused into one
 *                           persistent kernel (no per-step launch)
 *   sto_tree_matvec      <- model.py:55-63 tree_matvec (pinned adjacent-pairs tree)
 *   status codes         <- errors.py (ParameterError, BackendUnavailableError,
 *                           IntegrationDivergedError(oscillator, step))
 *
 * Conventions: plain pointers and sizes only.  Pointers documented "device"
 * must be device (or managed) memory of the plan's device; "any" accepts host
 * or device memory (UVA, cudaMemcpyDefault).  `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream).  All state arrays are
 * row-major (n, 3) float64, exactly the numpy layout of the reference.
 * Every function returns STO_OK or an error code; sto_last_error() gives a
 * thread-local message for the last failure.  A plan is not thread-safe.
 */
#ifndef STO_H
#define STO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STO_ABI_VERSION 2

#if defined(__GNUC__)
#define STO_API __attribute__((visibility("default")))
#else
#define STO_API
#endif

enum sto_status_code {
    STO_OK = 0,
    STO_E_UNAVAILABLE = 1, /* no usable sm_100 device    -> BackendUnavailableError */
    STO_E_PARAM = 2,       /* bad sizes / pointers       -> ParameterError          */
    STO_E_DIVERGED = 3,    /* non-finite recorded state  -> IntegrationDivergedError */
    STO_E_CUDA = 4,        /* CUDA runtime failure       -> SpinoscError             */
    STO_E_NOMEM = 5        /* device allocation failed   -> SpinoscError             */
};

/* The 11 right-hand-side scalars, in the order of the reference's
 * `_scalar_pack` (backends/cpu_jit.py:118-122). */
enum sto_const_index {
    STO_C_PREC = 0, STO_C_DAMP, STO_H_APPL, STO_H_ANISO, STO_H_S_PREFACTOR,
    STO_LAMBDA, STO_A_CP, STO_A_IN, STO_PX, STO_PY, STO_PZ, STO_N_CONSTS
};

typedef struct sto_plan sto_plan;

typedef struct {
    int64_t n;            /* oscillators (rows and columns of W)                 */
    int64_t n_in;         /* input channels (columns of W_in)                    */
    const double *w_cp;   /* any: (n, ld_cp) row-major coupling W                */
    int64_t ld_cp;        /* row stride of w_cp in elements (>= n)               */
    const double *w_in;   /* any: (n, ld_in) row-major input weights             */
    int64_t ld_in;        /* row stride of w_in in elements (>= n_in)            */
    double consts[STO_N_CONSTS];
    int device;           /* CUDA device ordinal                                 */
    int flags;            /* STO_PLAN_* bits                                     */
    /* Row sharding (multi-GPU).  world <= 1: unsharded, the rest is ignored.
     * Otherwise this plan owns global rows [row_begin, row_begin + row_count)
     * and w_cp / w_in point at THOSE rows (w_cp still has n columns).        */
    int64_t row_begin;
    int64_t row_count;
    int32_t world;
    int32_t rank;
} sto_plan_desc;

/* Force a kernel family (testing / benchmarking); default = automatic. */
#define STO_PLAN_FORCE_STREAM   0x1  /* W streamed from HBM/L2 every stage        */
#define STO_PLAN_FORCE_RESIDENT 0x2  /* W slice held in shared memory per CTA     */
#define STO_PLAN_FORCE_SINGLE   0x4  /* one CTA, exchange through shared memory   */
#define STO_PLAN_NO_TINY        0x8  /* do not use the one-warp kernel for n<=32  */
#define STO_PLAN_FORCE_REG      0x10 /* W register-resident teams (n <= 1024)     */
#define STO_PLAN_NO_REG         0x20 /* do not use the register-resident kernel    */
#define STO_PLAN_FORCE_CLUSTER  0x40 /* one thread-block cluster, DSMEM exchange (n <= 512) */
#define STO_PLAN_NO_CLUSTER     0x80 /* do not use the cluster kernel              */

typedef struct {
    double *m;               /* device (n,3): initial state in, final state out    */
    const double *samples;   /* device (n_samples, n_in) zero-order-hold drive      */
    int64_t n_samples;
    int64_t steps_per_sample;
    double dt;               /* h2 = dt*0.5 and dt/6.0 are formed inside, in IEEE   */
    int64_t steps;
    int64_t record_stride;   /* grid {0, s, 2s, ...} u {steps} (integrator.py:124)  */
    double *states;          /* device (n_records, n, 3); states[0] = m0 is written */
} sto_run;

typedef struct {
    int32_t diverged;        /* 1 when a recorded state was non-finite              */
    int32_t reserved;
    int64_t oscillator;      /* first row with a non-finite component               */
    int64_t step;            /* recorded step at which it was seen                  */
} sto_status;

typedef struct {
    int32_t kernel;          /* 0 tiny, 1 single-CTA, 2 SMEM-resident grid, 3 streaming grid,
                                4 register-resident teams, 5 thread-block cluster */
    int32_t grid;            /* CTAs of the persistent kernel                        */
    int32_t threads;         /* threads per CTA                                      */
    int32_t smem_bytes;      /* dynamic shared memory per CTA                        */
    int64_t ldw;             /* padded row width of the device W layout              */
    int64_t block_cols;      /* columns per (row, block) work unit                   */
    int64_t w_bytes;         /* device bytes of the W layout                          */
    int64_t x_window_cols;   /* columns of x staged per shared-memory window (== ldw
                                unless the row is processed in several windows)     */
} sto_plan_info;

STO_API const char *sto_last_error(void);
STO_API int sto_abi_version(void);

/* 1 if `device` is an sm_100-class GPU this library can drive, else 0. */
STO_API int sto_probe(int device);
STO_API int64_t sto_n_records(int64_t steps, int64_t record_stride);

STO_API int sto_plan_create(sto_plan **plan, const sto_plan_desc *desc);
STO_API void sto_plan_destroy(sto_plan *plan);
STO_API int sto_plan_get_info(const sto_plan *plan, sto_plan_info *info);

/* out = dm/dt at state m under drive u.  m, u, out: device. Asynchronous. */
STO_API int sto_derivative(sto_plan *plan, const double *m, const double *u, double *out,
                   void *stream);

/* Whole RK4 run in one persistent launch.  If `status` is non-NULL the call
 * synchronises the stream, fills it and returns STO_E_DIVERGED on divergence;
 * with NULL it is asynchronous and sto_plan_last_status() reads it later. */
STO_API int sto_integrate(sto_plan *plan, const sto_run *run, sto_status *status, void *stream);
STO_API int sto_plan_last_status(sto_plan *plan, sto_status *status, void *stream);

/* Batched ensemble (BASELINE configs[3]): `batch` reservoirs sharing W and
 * W_in, each with its own 11 scalars (a parameter sweep) and optionally its
 * own drive.  The coupling of all members is one FP64 tensor-core GEMM per RK
 * stage (DMMA); tolerance parity (<= 1e-10 at 1e3 steps), not bit-exact.
 * On divergence: status->reserved = member, oscillator, step. */
typedef struct {
    int64_t batch;
    const double *consts;          /* device (batch, 11)                          */
    double *m;                     /* device (batch, n, 3): m0 in, final out       */
    const double *samples;         /* device; member b reads samples + b*stride    */
    int64_t n_samples;
    int64_t steps_per_sample;
    int64_t sample_member_stride;  /* elements between members' series (0 = shared) */
    double dt;
    int64_t steps;
    int64_t record_stride;
    double *states;                /* device (n_records, batch, n, 3) or NULL      */
} sto_ensemble_run;

STO_API int sto_integrate_ensemble(sto_plan *plan, const sto_ensemble_run *run,
                                   sto_status *status, void *stream);
/* The same run, bit-exact: every member's states equal integrate() / the
 * reference's pinned CPU path with that member's parameters and drive, at any
 * horizon (pinned adjacent-pairs tree on the CUDA cores, pinned RHS and RK4
 * order; sto_ensemble_exact.cuh).  n <= 8160.  Same arguments and status. */
STO_API int sto_integrate_ensemble_exact(sto_plan *plan, const sto_ensemble_run *run,
                                         sto_status *status, void *stream);

/* Row-sharded multi-GPU (one process per GPU).  Each rank exports the IPC
 * handle of its exchange buffer (64 bytes, cudaIpcMemHandle_t), the caller
 * all-gathers them (e.g. torch.distributed) and connects; sto_integrate then
 * runs this rank's rows and all-gathers the stage x-vector over NVLink inside
 * the persistent kernel (peer stores + epoch flags, no NCCL call per stage).
 * run->m must hold the full (n, 3) initial state on every rank; on return it
 * holds this rank's rows of the final state, and states (n_records, n, 3)
 * this rank's rows.  All ranks must call sto_integrate with the same run
 * parameters, and finish a run before any rank starts the next one.  A rank
 * whose peer does not raise its epoch flag within STO_PEER_TIMEOUT_S seconds
 * (default 120; the peer died or never launched) stops the run and returns
 * STO_E_CUDA (status needed); the plan then refuses further runs. */
STO_API int sto_plan_exchange_handle(sto_plan *plan, void *handle_out, int64_t handle_bytes);
STO_API int sto_plan_connect(sto_plan *plan, const void *handles, int32_t world);

/* Test / single-GPU mode: `world` sharded plans of ONE device act as logical
 * ranks of one persistent launch, exchanging through plain device buffers
 * with exactly the multi-GPU protocol. */
STO_API int sto_plan_connect_local(sto_plan **plans, int32_t world);
STO_API int sto_integrate_group(sto_plan **plans, int32_t world, const sto_run *run,
                                sto_status *status, void *stream);

/* Host-buffer variant (the e2e path): m, samples, states are HOST pointers;
 * copies in and out are done inside (pinned staging), then synchronises. */
STO_API int sto_integrate_host(sto_plan *plan, double *m, const double *samples, int64_t n_samples,
                       int64_t steps_per_sample, double dt, int64_t steps,
                       int64_t record_stride, double *states, sto_status *status);

/* out[r] = pinned-tree sum_j a[r, j] * x[j] (model.py:55-63).
 * a: any (rows, lda); x: any (cols); out: any (rows).  Synchronous. */
STO_API int sto_tree_matvec(int device, int64_t rows, int64_t cols, const double *a, int64_t lda,
                    const double *x, double *out);

/* out[r] = pinned-tree sum_j W[r][j] * x[j] with the plan's resident W layout
 * (model.py:176-180 coupling_field_x without the a_cp factor): no W upload per
 * call.  x (n), out (n): device pointers; asynchronous on `stream`. */
STO_API int sto_plan_matvec(sto_plan *plan, const double *x, double *out, void *stream);

/* Reservoir construction on the device (topology.py:27-54 RngStream,
 * :241-273 generate_coupling / generate_input_weights, :146-238 spectral_radius
 * matvecs).  pcg = {state_hi, state_lo, inc_hi, inc_lo} of numpy's PCG64(seed)
 * (bit_generator.state).  sto_pcg64_fill writes draws offset .. offset+count-1
 * of Generator(PCG64).random() mapped to 2u - 1 -- bit-identical to
 * RngStream.uniform_pm1 -- into out[0..count) or, when diag_n > 0, draws
 * 0 .. n(n-1)-1 row-major onto the off-diagonal of the (n, ld) matrix out
 * (diagonal set to 0).  All pointers device; asynchronous on `stream`. */
STO_API int sto_pcg64_fill(int device, double *out, int64_t count, int64_t offset,
                           const uint64_t pcg[4], int64_t diag_n, int64_t ld, void *stream);
/* y = W x (row-major (rows, ld), device), unpinned summation order: the
 * Arnoldi matvecs of the spectral-radius estimate.  Asynchronous. */
STO_API int sto_gemv(int device, const double *w, int64_t rows, int64_t cols, int64_t ld,
                     const double *x, double *y, void *stream);
/* a[i] /= divisor (IEEE), device, asynchronous: `entries /= rho`. */
STO_API int sto_scale_div(int device, double *a, int64_t count, double divisor, void *stream);

/* out[b] = max over records r and oscillators k of | |states[r][b][k]| - 1 |
 * for recorded states (outer, members, n, 3): Trajectory.max_norm_drift
 * (integrator.py:184-185, np.linalg.norm order, bit-identical) computed on the
 * device, so a densely recorded run does not pay a host pass over its states.
 * Device pointers (out: `members` doubles), asynchronous. */
STO_API int sto_norm_drift(int device, const double *states, int64_t outer, int64_t members, int64_t n,
                           double *out, void *stream);

/* Self-test of the kernels' speculative division (sto_device.cuh rdiv_spec, used
 * for h_s = pref / (1 + lambda m.p), model.py:250 / cpu_jit.py:68): for each i,
 * q[i] = rdiv_spec(a[i], b[i]) and ok[i] = its proof of correct rounding, and
 * ref[i] = __ddiv_rn(a[i], b[i]).  Test hook only (tests/test_gpu_division.py):
 * ok[i] = 1 must imply q[i] == ref[i] bit for bit.  Device pointers, async. */
STO_API int sto_selftest_div(int device, const double *a, const double *b, int64_t count, double *q,
                             int32_t *ok, double *ref, void *stream);

/* Recorded states as CSV text (integrator.py:217-225 write_trajectory_csv):
 * header "t,k,mx,my,mz", then one row per (record i, oscillator k) in that
 * order, every float as Python's f"{x:.17g}" (byte-identical), formatted by
 * `threads` host threads (<= 0: all cores).  times (n_records,), states
 * (n_records, n, 3): HOST pointers.  STO_E_PARAM on bad arguments / IO error. */
STO_API int sto_write_trajectory_csv(const char *path, const double *times, const double *states,
                                     int64_t n_records, int64_t n, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* STO_H */
