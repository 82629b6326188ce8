// sto_b200.cu -- C-ABI implementation (include/sto.h) of the B200-native
// coupled spin-torque-oscillator RK4 path.  Build: see csrc/Makefile
// (nvcc -gencode arch=compute_100a,code=sm_100a -fmad=false -lineinfo).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/sto.h"
#include "sto_kernels.cuh"
#include "sto_reg_kernel.cuh"
#include "sto_cluster_kernel.cuh"
#include "sto_ensemble_kernel.cuh"
#include "sto_ensemble_exact.cuh"
#include "sto_build.cuh"

using namespace sto;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

// Peer watchdog of the sharded exchange (sto_kernels.cuh::multi_sync): the
// longest a rank waits for one peer's epoch flag before it stops the run and
// reports the peer lost.  STO_PEER_TIMEOUT_S overrides the 120 s default.
unsigned long long peer_timeout_ns() {
    double sec = 120.0;
    if (const char *v = std::getenv("STO_PEER_TIMEOUT_S")) {
        const double t = std::atof(v);
        if (t > 0) sec = t;
    }
    return (unsigned long long)(sec * 1e9);
}

#define STO_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                               \
            return fail(_e == cudaErrorMemoryAllocation ? STO_E_NOMEM : STO_E_CUDA,          \
                        std::string(#call) + ": " + cudaGetErrorString(_e));                 \
    } while (0)

constexpr int kThreads = 512;
constexpr size_t kSmemBudget = 220 * 1024;  // of 227 KB opt-in per CTA

// Column schedule for `n` logical columns (see sto_device.cuh).
ColSched make_sched(int n, int blk_hint) {
    ColSched s{};
    s.n = n;
    s.nfull = n / kSegFull;
    int rem = n - s.nfull * kSegFull;
    int pos = s.nfull * kSegFull;
    const int sizes[3] = {256, 128, 64};
    for (int i = 0; i < 3; ++i) {
        if (rem >= sizes[i]) {
            s.tail_base[s.ntail] = pos;
            s.tail_c[s.ntail] = sizes[i] / 32;
            ++s.ntail;
            pos += sizes[i];
            rem -= sizes[i];
        }
    }
    if (rem > 0) {
        s.tail_base[s.ntail] = pos;
        s.tail_c[s.ntail] = 2;
        ++s.ntail;
        pos += 64;
    }
    s.ldw = pos;
    int blk = kSegFull;
    while (blk < blk_hint && blk < kSegFull * kMaxLeaves) blk <<= 1;
    s.blk = blk;
    s.nblocks = (s.ldw + blk - 1) / blk;
    return s;
}

// physical -> logical column (inverse of col_perm); -1 for padding
__host__ __device__ inline int col_unperm(const ColSched &s, int p) {
    int base, c;
    if (p < s.nfull * kSegFull) {
        base = p & ~(kSegFull - 1);
        c = 16;
    } else {
        base = -1;
        c = 2;
        for (int t = 0; t < s.ntail; ++t)
            if (p >= s.tail_base[t] && p < s.tail_base[t] + 32 * s.tail_c[t]) {
                base = s.tail_base[t];
                c = s.tail_c[t];
            }
        if (base < 0) return -1;
    }
    const int o = p - base;
    const int vec = o >> 1, half = o & 1;
    const int l = vec & 31, i = vec >> 5;
    const int k = base + l * c + 2 * i + half;
    return k < s.n ? k : -1;
}

__global__ void permute_rows_kernel(const double *__restrict__ src, long long lds,
                                    double *__restrict__ dst, int rows, ColSched cs) {
    const long long total = (long long)rows * cs.ldw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / cs.ldw);
        const int pcol = (int)(i - (long long)r * cs.ldw);
        const int k = col_unperm(cs, pcol);
        dst[i] = k >= 0 ? src[(long long)r * lds + k] : -0.0;  // -0.0: exact identity
    }
}

constexpr int kMaxFlags = 1024;
constexpr int kClusterMaxN = 512;  // cluster kernel: W of n <= 512 fits 16 SMs' registers

// logical row-major (zero padded to np x np) copy of W from the device layout
// Ensemble W in DMMA fragment order for row tiles of TR = 8U rows
// (sto_ensemble_kernel.cuh, ens layout comment); zero outside n x n.
__global__ void ens_layout_kernel(const double *__restrict__ src, double *__restrict__ dst, int n,
                                  int kp, int tr, int n_rt, ColSched cs) {
    const long long tile = (long long)tr * kp, total = tile * n_rt;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int rt = (int)(i / tile);
        const int rem = (int)(i - (long long)rt * tile);
        const int ch = rem / (tr * kEnsKC);
        const int within = rem - ch * tr * kEnsKC;
        const int nk = min(kEnsKC, kp - ch * kEnsKC) >> 2;
        const int ru = within / (nk * 32), ks = (within / 32) % nk, lane = within & 31;
        const int row = rt * tr + 8 * ru + (lane >> 2), col = ch * kEnsKC + 4 * ks + (lane & 3);
        dst[i] = (row < n && col < n) ? src[(long long)row * cs.ldw + col_perm(cs, col)] : 0.0;
    }
}

// Exact-ensemble W: row-major np x kp, logical columns, -0.0 outside n x n
// (sto_ensemble_exact.cuh: the padding identity of the pinned tree).
__global__ void ex_layout_kernel(const double *__restrict__ src, double *__restrict__ dst, int n, int np,
                                 int kp, ColSched cs) {
    const long long total = (long long)np * kp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / kp), col = (int)(i - (long long)row * kp);
        dst[i] = (row < n && col < n) ? src[(long long)row * cs.ldw + col_perm(cs, col)] : -0.0;
    }
}

__global__ void reset_status_kernel(StatusDev *st, unsigned long long *bar, unsigned *flags) {
    for (int i = threadIdx.x; i < kMaxFlags; i += blockDim.x) flags[i] = 0u;
    if (threadIdx.x == 0) {
        st->flag = 0;
        st->key = 0x7fffffffffffffffLL;
        *bar = 0ull;
    }
}

struct Layout {
    ColSched cs{};
    int rows = 0;
    double *w = nullptr;
};

// Big buffers (the W layout, its staging copy) come from the device's
// stream-ordered pool with an unbounded release threshold, so destroying a
// plan and building the next one (the e2e path: one plan per integrate())
// reuses the memory instead of paying cudaMalloc/cudaFree of ~1 GB each time.
void keep_pool_memory() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
}

bool is_device_pointer(const void *p) {
    cudaPointerAttributes attr;
    int dev = -1;
    const bool ok = cudaPointerGetAttributes(&attr, p) == cudaSuccess && cudaGetDevice(&dev) == cudaSuccess &&
                    (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) &&
                    attr.device == dev;
    cudaGetLastError();
    return ok;
}

int upload_layout(Layout &L, int rows, int cols, const double *a, long long lda, int blk_hint,
                  cudaStream_t stream) {
    L.rows = rows;
    L.cs = make_sched(cols, blk_hint);
    keep_pool_memory();
    const size_t bytes = (size_t)rows * L.cs.ldw * sizeof(double);
    STO_CUDA(cudaMallocAsync(&L.w, bytes, stream));
    if (is_device_pointer(a)) {  // device-built W: permute in place, no staging copy
        permute_rows_kernel<<<1184, 256, 0, stream>>>(a, lda, L.w, rows, L.cs);
        STO_CUDA(cudaGetLastError());
    } else {
        double *stage = nullptr;
        STO_CUDA(cudaMallocAsync(&stage, (size_t)rows * cols * sizeof(double), stream));
        STO_CUDA(cudaMemcpy2DAsync(stage, (size_t)cols * sizeof(double), a, (size_t)lda * sizeof(double),
                                   (size_t)cols * sizeof(double), rows, cudaMemcpyDefault, stream));
        permute_rows_kernel<<<1184, 256, 0, stream>>>(stage, cols, L.w, rows, L.cs);
        STO_CUDA(cudaGetLastError());
        STO_CUDA(cudaFreeAsync(stage, stream));
    }
    STO_CUDA(cudaStreamSynchronize(stream));
    return STO_OK;
}

enum KernelKind { kTiny = 0, kSingle = 1, kResident = 2, kStream = 3, kReg = 4, kCluster = 5 };

}  // namespace

struct sto_plan {
    int device = 0;
    int sm_count = 0;
    long long l2_bytes = 0;
    int n = 0, n_in = 0;
    Consts c{};
    Layout L;
    double *w_in = nullptr;
    double *xbuf = nullptr;
    unsigned long long *bar = nullptr;
    unsigned *flags = nullptr;
    uint4 *ll = nullptr;  // kReg: [2][n] LL words
    StatusDev *status = nullptr;
    // integrate launch configuration
    int kind = kStream;
    bool stream_evict_first = true;
    int l2_keep_rows = 0;             // streaming kernel: rows per CTA kept L2-resident
    int grid = 1;
    int rows_cap = 1;
    int chunk_cols = 0;
    size_t smem = 0;
    int threads = 512;
    int team = 0;  // kReg: threads per row
    int rows_per_team = 1;
    int clu_cols = 0;  // kCluster: W columns per thread (grid = cluster size)
    int grid_threads = kThreads;  // kStream (HBM-streaming, unsharded): 512 or 640
    bool clu_hyb = true;  // kCluster: teams finish their rows (clu_hyb_kernel)
    // row sharding (world > 1)
    int world = 1, rank = 0;
    long long row_begin = 0;
    int rows = 0;                       // rows owned (== n unsharded)
    double *exch = nullptr;             // [2][ldw] receive buffer + flags (IPC-exportable)
    unsigned long long *exch_flags = nullptr;
    double *xbuf_of[kMaxRanks] = {};
    unsigned long long *flags_of[kMaxRanks] = {};
    void *ipc_opened[kMaxRanks] = {};
    bool connected = false;
    unsigned long long epoch_base = 0;  // monotonic epochs across launches
    bool peer_lost = false;             // a run hit the peer watchdog: epochs out of step
    // ensemble resources (allocated on first sto_integrate_ensemble)
    double *ens_w = nullptr;           // np x np row-major, zero padded
    int ens_np = 0;
    int ens_u = 0;                     // tile height ens_w is laid out for
    double *ens_x = nullptr, *ens_st = nullptr;
    size_t ens_bp = 0;                 // member capacity of ens_x / ens_st
    unsigned long long *ens_bar = nullptr;
    // exact (CUDA-core, pinned-tree) ensemble resources
    double *ex_w = nullptr;            // ex_np x ex_kp row-major, -0.0 padded
    double *ex_x = nullptr, *ex_st = nullptr;
    size_t ex_bp = 0;                  // member capacity of ex_x / ex_st
    unsigned long long *ex_bar = nullptr;
};

namespace {

size_t grid_smem(int rows_cap, const ColSched &cs, int chunk_cols, bool resident) {
    size_t d = (size_t)chunk_cols + (resident ? (size_t)rows_cap * cs.ldw : 0) +
               (size_t)rows_cap * cs.nblocks + 13 * (size_t)rows_cap + 2;
    return d * sizeof(double);
}

int choose_chunk(const ColSched &cs, int rows_cap, bool resident) {
    // STO_CHUNK_COLS (tests): force x windows of that many physical columns
    // (rounded down to whole blocks) even when the row fits one window, so the
    // chunked block loop that N >~ 2.4e4 takes is exercised at small N.
    if (const char *e = getenv("STO_CHUNK_COLS")) {
        const int c = atoi(e) / cs.blk * cs.blk;
        if (c >= cs.blk && c < cs.ldw && grid_smem(rows_cap, cs, c, resident) <= kSmemBudget) return c;
    }
    if (grid_smem(rows_cap, cs, cs.ldw, resident) <= kSmemBudget) return cs.ldw;
    int chunk = 16384;
    while (chunk > cs.blk && grid_smem(rows_cap, cs, chunk, resident) > kSmemBudget) chunk >>= 1;
    return std::max(chunk, cs.blk);
}

template <WSrc S, bool SINGLE, int NT = kThreads>
int launch_grid(const KParams &p, int grid, size_t smem, bool cooperative, cudaStream_t stream) {
    auto fn = grid_rk4_kernel<S, SINGLE, false, NT>;
    STO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (cooperative) {
        void *args[] = {(void *)&p};
        STO_CUDA(cudaLaunchCooperativeKernel((void *)fn, dim3(grid), dim3(NT), args, smem,
                                             stream));
    } else {
        fn<<<grid, NT, smem, stream>>>(p);
        STO_CUDA(cudaGetLastError());
    }
    return STO_OK;
}

// Threads per CTA of the HBM-streaming kernel: 20 warps (640 threads, <= 96
// registers) keep more 16-byte loads in flight per SM than 16; measured
// (bench n1e4 on two boxes, tools/midsize_sweep.py), relative to 16 warps:
//   warps   17     18     20     24     32
//   n1e4  +1.5%  +2.5%  +3.7%  +2.6%  -1.2%   (N = 5000 / 7000 / 15000 at 20:
//   +5.6 / +7.5 / +5.7 %, at 24 slightly more); N = 4e4, where x is staged in
// chunks: within +-1 %.  So 640 when one x window covers the row, else 512.
// STO_GRID_WARPS=16/20 forces either.
int stream_threads(const ColSched &cs, int chunk_cols) {
    if (const char *e = getenv("STO_GRID_WARPS")) return atoi(e) == 20 ? 640 : kThreads;
    return chunk_cols >= cs.ldw ? 640 : kThreads;
}

template <WSrc S>
int launch_multi(const KParams &p, int grid, size_t smem, cudaStream_t stream) {
    auto fn = grid_rk4_kernel<S, false, true>;
    STO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    void *args[] = {(void *)&p};
    STO_CUDA(cudaLaunchCooperativeKernel((void *)fn, dim3(grid), dim3(kThreads), args, smem, stream));
    return STO_OK;
}

ShardInfo shard_info(const sto_plan *P) {
    ShardInfo s{};
    s.w = P->L.w;
    s.w_in = P->w_in;
    s.row_begin = P->row_begin;
    s.rows = P->rows;
    s.bar = P->bar;
    s.xbuf = P->exch;
    s.flags = P->exch_flags;
    return s;
}

template <int T, int C, int R, bool SINGLE>
int launch_reg_t(const RegParams &rp, int grid, int threads, size_t smem, cudaStream_t stream) {
    auto fn = reg_rk4_kernel<T, C, R, SINGLE>;
    STO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (SINGLE) {
        fn<<<1, threads, smem, stream>>>(rp);
        STO_CUDA(cudaGetLastError());
    } else {
        void *args[] = {(void *)&rp};
        STO_CUDA(cudaLaunchCooperativeKernel((void *)fn, dim3(grid), dim3(threads), args, smem,
                                             stream));
    }
    return STO_OK;
}

// (team T, columns per thread C, rows per team R): n <= 128 uses C = 32 in
// one CTA; larger n uses C = 16 over the grid, R = 2 rows per team for the
// 64-thread teams (each shared-memory x load then feeds two rows).
template <int T, int C>
int launch_clu_t(const KParams &p, bool hyb, int K, int threads, size_t smem, cudaStream_t stream) {
    auto fn = hyb ? clu_hyb_kernel<T, C> : clu_rk4_kernel<T, C>;
    STO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (K > 8) STO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(K);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    STO_CUDA(cudaLaunchKernelEx(&cfg, fn, p));
    return STO_OK;
}

// clusters of K CTAs of the cluster kernel that can be resident at once
int clu_max_clusters(bool hyb, int team, int cols, int K, int threads, size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(K);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    auto q = [&](auto fn) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
            (K > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) ||
            cudaOccupancyMaxActiveClusters(&nc, fn, &cfg) != cudaSuccess)
            nc = 0;
    };
#define STO_CLU_Q(T_, C_) q(hyb ? clu_hyb_kernel<T_, C_> : clu_rk4_kernel<T_, C_>)
    if (cols == 64) {
        STO_CLU_Q(8, 64);
    } else if (cols == 32) {
        if (team == 2) STO_CLU_Q(2, 32);
        else if (team == 4) STO_CLU_Q(4, 32);
        else STO_CLU_Q(8, 32);
    } else {
        if (team == 4) STO_CLU_Q(4, 16);
        else if (team == 8) STO_CLU_Q(8, 16);
        else STO_CLU_Q(16, 16);
    }
#undef STO_CLU_Q
    cudaGetLastError();
    return nc;
}

// (team T, columns per thread C) of the cluster kernel; P = T*C padded row
int launch_clu(const KParams &p, bool hyb, int team, int cols, int K, int threads, size_t smem,
               cudaStream_t s) {
    if (cols == 64) return launch_clu_t<8, 64>(p, hyb, K, threads, smem, s);
    if (cols == 32) {
        switch (team) {
            case 2: return launch_clu_t<2, 32>(p, hyb, K, threads, smem, s);
            case 4: return launch_clu_t<4, 32>(p, hyb, K, threads, smem, s);
            default: return launch_clu_t<8, 32>(p, hyb, K, threads, smem, s);
        }
    }
    switch (team) {
        case 4: return launch_clu_t<4, 16>(p, hyb, K, threads, smem, s);
        case 8: return launch_clu_t<8, 16>(p, hyb, K, threads, smem, s);
        default: return launch_clu_t<16, 16>(p, hyb, K, threads, smem, s);
    }
}

int launch_reg(const RegParams &rp, int team, int rows_per_team, bool single, int grid,
               int threads, size_t smem, cudaStream_t s) {
    if (single) {
        switch (team) {
            case 1: return launch_reg_t<1, 32, 1, true>(rp, grid, threads, smem, s);
            case 2: return launch_reg_t<2, 32, 1, true>(rp, grid, threads, smem, s);
            default: return launch_reg_t<4, 32, 1, true>(rp, grid, threads, smem, s);
        }
    }
    switch (team) {
        case 2: return launch_reg_t<2, 16, 1, false>(rp, grid, threads, smem, s);
        case 4: return launch_reg_t<4, 16, 1, false>(rp, grid, threads, smem, s);
        case 8: return launch_reg_t<8, 16, 1, false>(rp, grid, threads, smem, s);
        case 16: return launch_reg_t<16, 16, 1, false>(rp, grid, threads, smem, s);
        case 32: return launch_reg_t<32, 16, 1, false>(rp, grid, threads, smem, s);
        default:
            return rows_per_team == 2 ? launch_reg_t<64, 16, 2, false>(rp, grid, threads, smem, s)
                                      : launch_reg_t<64, 16, 1, false>(rp, grid, threads, smem, s);
    }
}

int launch_tiny(const KParams &p, int n, cudaStream_t stream) {
    if (n <= 1) tiny_rk4_kernel<1><<<1, 32, 0, stream>>>(p);
    else if (n <= 2) tiny_rk4_kernel<2><<<1, 32, 0, stream>>>(p);
    else if (n <= 4) tiny_rk4_kernel<4><<<1, 32, 0, stream>>>(p);
    else if (n <= 8) tiny_rk4_kernel<8><<<1, 32, 0, stream>>>(p);
    else if (n <= 16) tiny_rk4_kernel<16><<<1, 32, 0, stream>>>(p);
    else tiny_rk4_kernel<32><<<1, 32, 0, stream>>>(p);
    STO_CUDA(cudaGetLastError());
    return STO_OK;
}

// Streaming W (> 0.6 L2): a fixed slice of every CTA's rows is loaded with
// evict_last and stays L2-resident across stages, so each stage reads that
// slice from L2 and only the rest from HBM.  Budget: kL2KeepFrac of L2
// (STO_L2_KEEP_MB overrides, 0 disables), spread evenly over the CTAs so the
// per-stage work stays balanced.
constexpr double kL2KeepFrac = 0.5;
int l2_keep_rows_for(int l2_bytes, int ctas, int ldw) {
    double budget = kL2KeepFrac * (double)l2_bytes;
    if (const char *e = getenv("STO_L2_KEEP_MB")) budget = atof(e) * 1048576.0;
    const double row_bytes = (double)ldw * sizeof(double);
    return std::max(0, (int)(budget / (row_bytes * std::max(1, ctas))));
}

KParams base_params(const sto_plan *P) {
    KParams p{};
    p.cs = P->L.cs;
    p.c = P->c;
    p.rows = P->n;
    p.n_in = P->n_in;
    p.w = P->L.w;
    p.w_in = P->w_in;
    p.xbuf = P->xbuf;
    p.bar = P->bar;
    p.status = P->status;
    p.l2_keep_rows = P->l2_keep_rows;
    p.x_stride = 1;
    p.n_samples = 1;
    p.sps = 1;
    p.steps = 1;
    p.stride = 1;
    return p;
}

int check_device(int device, cudaDeviceProp *prop) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count)
        return fail(STO_E_UNAVAILABLE, "no CUDA device " + std::to_string(device));
    // properties cached per device (cudaGetDeviceProperties costs ~8 ms per call)
    static std::mutex mu;
    static std::map<int, cudaDeviceProp> cache;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(device);
        if (it == cache.end()) {
            cudaDeviceProp p;
            STO_CUDA(cudaGetDeviceProperties(&p, device));
            it = cache.emplace(device, p).first;
        }
        *prop = it->second;
    }
    if (prop->major != 10)
        return fail(STO_E_UNAVAILABLE, std::string("device is not sm_100-class: ") + prop->name);
    return STO_OK;
}

}  // namespace

extern "C" {

const char *sto_last_error(void) { return g_err.c_str(); }

int sto_abi_version(void) { return STO_ABI_VERSION; }

int sto_probe(int device) {
    int count = 0, major = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) return 0;
    // one attribute query (cudaGetDeviceProperties costs ~8 ms per call)
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) return 0;
    return major == 10 ? 1 : 0;
}

int64_t sto_n_records(int64_t steps, int64_t record_stride) {
    if (steps < 1 || record_stride < 1) return 0;
    return steps / record_stride + 1 + (steps % record_stride != 0 ? 1 : 0);
}

int sto_plan_create(sto_plan **out, const sto_plan_desc *d) {
    if (!out || !d) return fail(STO_E_PARAM, "null plan or descriptor");
    *out = nullptr;
    if (d->n < 1 || d->n_in < 1 || d->n > (1 << 24) || d->n_in > (1 << 20))
        return fail(STO_E_PARAM, "n and n_in must be >= 1");
    const bool sharded = d->world > 1;
    if (sharded && (d->world > kMaxRanks || d->rank < 0 || d->rank >= d->world ||
                    d->row_begin < 0 || d->row_count < 1 || d->row_begin + d->row_count > d->n))
        return fail(STO_E_PARAM, "bad row shard (world <= 8, 0 <= rank < world, rows inside n)");
    if (!d->w_cp || !d->w_in || d->ld_cp < d->n || d->ld_in < d->n_in)
        return fail(STO_E_PARAM, "bad W / W_in pointers or leading dimensions");
    cudaDeviceProp prop;
    if (int rc = check_device(d->device, &prop)) return rc;
    STO_CUDA(cudaSetDevice(d->device));

    sto_plan *P = new sto_plan();
    P->device = d->device;
    P->sm_count = prop.multiProcessorCount;
    P->l2_bytes = prop.l2CacheSize;
    P->n = (int)d->n;
    P->n_in = (int)d->n_in;
    P->world = sharded ? d->world : 1;
    P->rank = sharded ? d->rank : 0;
    P->row_begin = sharded ? d->row_begin : 0;
    P->rows = sharded ? (int)d->row_count : (int)d->n;
    const double *k = d->consts;
    P->c = Consts{k[0], k[1], k[2], k[3], k[4], k[5], k[6], k[7], k[8], k[9], k[10]};

    auto bail = [&](int rc) {
        sto_plan_destroy(P);
        return rc;
    };
    cudaStream_t s = nullptr;
    const int n = P->n;
    int blk_hint = n >= 8192 ? 2048 : 512;
    if (const char *e = getenv("STO_BLK")) blk_hint = std::max(512, atoi(e));  // (row, block) unit width
    if (int rc = upload_layout(P->L, P->rows, n, d->w_cp, d->ld_cp, blk_hint, s)) return bail(rc);
    const ColSched &cs = P->L.cs;
    if (sharded) {
        const size_t xb = sizeof(double) * 2 * (size_t)cs.ldw;
        const size_t fb = sizeof(unsigned long long) * kMaxRanks * kFlagSlot;
        if (cudaMalloc(&P->exch, xb + fb) != cudaSuccess)
            return bail(fail(STO_E_NOMEM, "exchange buffer allocation failed"));
        if (cudaMemset(P->exch, 0, xb + fb) != cudaSuccess)
            return bail(fail(STO_E_CUDA, "exchange buffer init failed"));
        P->exch_flags = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(P->exch) + xb);
        P->xbuf_of[P->rank] = P->exch;
        P->flags_of[P->rank] = P->exch_flags;
    }
    if (cudaMalloc(&P->w_in, sizeof(double) * (size_t)P->rows * d->n_in) != cudaSuccess ||
        cudaMalloc(&P->xbuf, sizeof(double) * 2 * (size_t)cs.ldw) != cudaSuccess ||
        cudaMalloc(&P->bar, 64) != cudaSuccess ||
        cudaMalloc(&P->flags, sizeof(unsigned) * kMaxFlags) != cudaSuccess ||
        cudaMalloc(&P->ll, sizeof(uint4) * 2 * (size_t)n) != cudaSuccess ||
        cudaMalloc(&P->status, sizeof(StatusDev)) != cudaSuccess)
        return bail(fail(STO_E_NOMEM, "device allocation failed"));
    if (cudaMemcpy2D(P->w_in, sizeof(double) * d->n_in, d->w_in, sizeof(double) * d->ld_in,
                     sizeof(double) * d->n_in, P->rows, cudaMemcpyDefault) != cudaSuccess ||
        cudaMemset(P->xbuf, 0, sizeof(double) * 2 * (size_t)cs.ldw) != cudaSuccess)
        return bail(fail(STO_E_CUDA, "W_in upload failed"));

    // ---- choose the integrate kernel ------------------------------------
    const int fl = d->flags;
    const int forced = fl & (STO_PLAN_FORCE_STREAM | STO_PLAN_FORCE_RESIDENT |
                             STO_PLAN_FORCE_SINGLE | STO_PLAN_FORCE_REG | STO_PLAN_FORCE_CLUSTER);
    const size_t single_smem = grid_smem(n, cs, cs.ldw, true);
    int pw = 32;
    while (pw < n) pw <<= 1;
    // cluster kernel configuration (CTA b owns the SEG = P/K rows whose x positions
    // are [b*SEG, (b+1)*SEG): one owner warp per CTA, SEG <= 32, K a power of two).
    // Fastest measured (tools/clu_sweep.py, padded row P -> kernel, K, C):
    //   P =  64 -> teams finish rows (clu_hyb_kernel), K = 2,  C = 32
    //   P = 128 -> clu_hyb_kernel, K = 8,  C = 32
    //   P = 256 -> owner warp (clu_rk4_kernel), K = 16, C = 32  (K = 8)
    //   P = 512 -> clu_rk4_kernel, K = 16, C = 64  (register kernel without 16-CTA clusters)
    // K = 16 is B200's non-portable cluster size: it needs 16 free SMs in one GPC.
    struct {
        int pc = 0, cols = 0, K = 0, team = 0, rows = 0, threads = 0;
        bool fits = false, hyb = true;
    } clu;
    if (n <= kClusterMaxN) {
        clu.pc = std::max(pw, 64);
        clu.hyb = clu.pc <= 128;
        if (const char *e = getenv("STO_CLU_HYB")) clu.hyb = atoi(e) != 0;
        clu.cols = clu.pc == 512 ? 64 : 32;
        clu.K = clu.pc == 64 ? 2 : clu.pc == 128 ? 8 : 16;
        if (const char *e = getenv("STO_CLU_C")) clu.cols = atoi(e) == 16 ? 16 : atoi(e) == 64 ? 64 : 32;
        if (const char *e = getenv("STO_CLU_K")) clu.K = std::max(1, std::min(atoi(e), kCluMaxK));
        clu.team = clu.pc / clu.cols;
        auto smem_of = [&] { return clu.hyb ? clu_hyb_smem_bytes(clu.pc) : clu_smem_bytes(clu.pc); };
        if (clu.K > 8 && (clu.cols != 64 || clu.team == 8) &&
            clu_max_clusters(clu.hyb, clu.team, clu.cols, clu.K, clu_threads(clu.pc / clu.K, clu.team),
                             smem_of()) < 1) {
            clu.K = 8;  // the portable size
        }
        clu.rows = clu.pc / clu.K;
        clu.threads = clu_threads(clu.rows, clu.team);
        clu.fits = !(clu.K & (clu.K - 1)) && clu.rows <= 32 && clu.team >= 1 && clu.team <= 32 &&
                   (clu.cols != 64 || clu.team == 8) && clu.threads <= (clu.cols == 16 ? 576 : 288);
    }

    if (sharded) {
        // sharded plans always use the grid kernel (MULTI); rows = this shard
        const int g = std::min(P->sm_count, P->rows);
        P->rows_cap = (P->rows + g - 1) / g;
        const size_t res_smem = grid_smem(P->rows_cap, cs, cs.ldw, true);
        if (!(fl & STO_PLAN_FORCE_STREAM) && res_smem <= kSmemBudget) {
            P->kind = kResident;
            P->chunk_cols = cs.ldw;
            P->smem = res_smem;
        } else {
            P->kind = kStream;
            P->chunk_cols = choose_chunk(cs, P->rows_cap, false);
            P->smem = grid_smem(P->rows_cap, cs, P->chunk_cols, false);
            const double wbytes = (double)P->rows * cs.ldw * sizeof(double);
            P->stream_evict_first = wbytes > 0.75 * (double)P->l2_bytes;
            if (P->stream_evict_first) {
                P->l2_keep_rows = l2_keep_rows_for(P->l2_bytes, g, cs.ldw);
                P->grid_threads = stream_threads(cs, P->chunk_cols);
            }
        }
        P->grid = g;
    } else if (n <= 32 && !(fl & STO_PLAN_NO_TINY) && !forced) {
        P->kind = kTiny;
        P->grid = 1;
        P->threads = 32;
    } else if ((fl & STO_PLAN_FORCE_CLUSTER) ||
               (!forced && !(fl & STO_PLAN_NO_CLUSTER) && n <= kClusterMaxN && clu.fits)) {
        if (!clu.fits)
            return bail(fail(STO_E_PARAM, "cluster kernel does not fit (n <= 512, K a power of two, "
                                          "P/K <= 32 rows per CTA, 16-CTA clusters resident for n > 256)"));
        P->kind = kCluster;
        P->team = clu.team;
        P->clu_cols = clu.cols;
        P->grid = clu.K;
        P->rows_cap = clu.rows;
        P->threads = clu.threads;
        P->clu_hyb = clu.hyb;
        P->smem = clu.hyb ? clu_hyb_smem_bytes(clu.pc) : clu_smem_bytes(clu.pc);
    } else if ((fl & STO_PLAN_FORCE_REG) || (!forced && !(fl & STO_PLAN_NO_REG) && n <= 1024)) {
        if (n > 1024) return bail(fail(STO_E_PARAM, "register-resident kernel needs n <= 1024"));
        P->kind = kReg;
        const bool single = n <= 128;
        const int cols = single ? 32 : 16;  // W columns per thread (registers)
        const int team = std::max(single ? 1 : 2, pw / cols);
        P->team = team;
        int g = 1;
        if (!single) {
            // ~512 threads per CTA, at most one CTA per SM
            g = (int)std::min<long long>(P->sm_count, ((long long)n * team + 511) / 512);
            if (const char *e = getenv("STO_REG_GRID")) g = std::max(1, std::min(atoi(e), P->sm_count));
            g = std::max(g, (n * team + 511) / 512);
        }
        P->grid = g;
        P->rows_cap = (n + g - 1) / g;
        P->rows_per_team = (!single && team == 64 && !getenv("STO_REG_R1")) ? 2 : 1;
        int teams = (P->rows_cap + P->rows_per_team - 1) / P->rows_per_team;
        if (P->rows_per_team == 2 && teams * team > 256) {  // R = 2 kernel is built for 256 threads
            P->rows_per_team = 1;
            teams = P->rows_cap;
        }
        P->threads = std::max(((teams * team + 31) / 32) * 32, ((P->rows_cap + 31) / 32) * 32);
        P->chunk_cols = single ? 1 : 0;  // marks SINGLE for the launcher
        P->smem = sizeof(double) * ((size_t)team * cols + 2 * (size_t)P->rows_per_team *
                                    (P->threads / team) + 8);
        if (P->threads > 512 || g > kMaxFlags)
            return bail(fail(STO_E_PARAM, "register-resident kernel does not fit"));
    } else if ((fl & STO_PLAN_FORCE_SINGLE) ||
               (!forced && n <= 128 && single_smem <= kSmemBudget)) {
        if (single_smem > kSmemBudget)
            return bail(fail(STO_E_PARAM, "single-CTA kernel does not fit shared memory"));
        P->kind = kSingle;
        P->grid = 1;
        P->rows_cap = n;
        P->chunk_cols = cs.ldw;
        P->smem = single_smem;
    } else {
        int g = std::min(P->sm_count, n);
        P->rows_cap = (n + g - 1) / g;
        const size_t res_smem = grid_smem(P->rows_cap, cs, cs.ldw, true);
        const bool want_res = (fl & STO_PLAN_FORCE_RESIDENT) ||
                              (!(fl & STO_PLAN_FORCE_STREAM) && res_smem <= kSmemBudget);
        if (want_res) {
            if (res_smem > kSmemBudget)
                return bail(fail(STO_E_PARAM, "resident kernel does not fit shared memory"));
            P->kind = kResident;
            P->chunk_cols = cs.ldw;
            P->smem = res_smem;
        } else {
            P->kind = kStream;
            P->chunk_cols = choose_chunk(cs, P->rows_cap, false);
            P->smem = grid_smem(P->rows_cap, cs, P->chunk_cols, false);
            const double wbytes = (double)n * cs.ldw * sizeof(double);
            P->stream_evict_first = wbytes > 0.75 * (double)P->l2_bytes;
            if (P->stream_evict_first) {
                P->l2_keep_rows = l2_keep_rows_for(P->l2_bytes, g, cs.ldw);
                P->grid_threads = stream_threads(cs, P->chunk_cols);
            }
        }
        P->grid = g;
    }
    *out = P;
    return STO_OK;
}

void sto_plan_destroy(sto_plan *P) {
    if (!P) return;
    cudaSetDevice(P->device);
    cudaDeviceSynchronize();  // no launch may still read the plan's buffers
    for (int q = 0; q < kMaxRanks; ++q)
        if (P->ipc_opened[q]) cudaIpcCloseMemHandle(P->ipc_opened[q]);
    cudaFree(P->exch);
    cudaFreeAsync(P->L.w, nullptr);
    cudaFree(P->w_in);
    cudaFree(P->xbuf);
    cudaFree(P->bar);
    cudaFree(P->flags);
    cudaFree(P->ll);
    cudaFree(P->ens_w);
    cudaFree(P->ens_x);
    cudaFree(P->ens_st);
    cudaFree(P->ens_bar);
    cudaFree(P->ex_w);
    cudaFree(P->ex_x);
    cudaFree(P->ex_st);
    cudaFree(P->ex_bar);
    cudaFree(P->status);
    delete P;
}

int sto_plan_get_info(const sto_plan *P, sto_plan_info *info) {
    if (!P || !info) return fail(STO_E_PARAM, "null plan or info");
    info->kernel = P->kind;
    info->grid = P->grid;
    info->threads = (P->kind == kTiny || P->kind == kReg || P->kind == kCluster) ? P->threads
                    : P->kind == kStream                                          ? P->grid_threads
                                                                                  : kThreads;
    info->smem_bytes = (int)P->smem;
    info->ldw = P->L.cs.ldw;
    info->block_cols = P->L.cs.blk;
    info->w_bytes = (int64_t)P->rows * P->L.cs.ldw * (int64_t)sizeof(double);
    info->x_window_cols = (P->kind == kStream || P->kind == kResident) ? P->chunk_cols : P->L.cs.ldw;
    return STO_OK;
}

int sto_derivative(sto_plan *P, const double *m, const double *u, double *out, void *stream) {
    if (!P || !m || !u || !out) return fail(STO_E_PARAM, "null argument");
    if (P->world > 1) return fail(STO_E_PARAM, "sto_derivative needs an unsharded plan");
    STO_CUDA(cudaSetDevice(P->device));
    cudaStream_t s = (cudaStream_t)stream;
    KParams p = base_params(P);
    p.mode = kDerivative;
    p.m = const_cast<double *>(m);
    p.samples = u;
    p.out = out;
    const int g = std::min(P->sm_count, P->n);
    p.rows_cap = (P->n + g - 1) / g;
    p.chunk_cols = choose_chunk(P->L.cs, p.rows_cap, false);
    const size_t smem = grid_smem(p.rows_cap, P->L.cs, p.chunk_cols, false);
    return launch_grid<WSrc::GlobalL2, false>(p, g, smem, false, s);
}

int sto_integrate(sto_plan *P, const sto_run *r, sto_status *status, void *stream) {
    if (!P || !r) return fail(STO_E_PARAM, "null plan or run");
    if (!r->m || !r->samples || r->n_samples < 1 || r->steps_per_sample < 1 || r->steps < 1 ||
        r->record_stride < 1 || !(r->dt > 0.0))
        return fail(STO_E_PARAM, "bad run descriptor");
    if (r->n_samples > 1 && !((r->n_samples - 1) * r->steps_per_sample < r->steps &&
                              r->steps <= r->n_samples * r->steps_per_sample))
        return fail(STO_E_PARAM, "input series does not cover the run (model.py:128-143)");
    STO_CUDA(cudaSetDevice(P->device));
    cudaStream_t s = (cudaStream_t)stream;
    KParams p = base_params(P);
    p.mode = kIntegrate;
    p.m = r->m;
    p.samples = r->samples;
    p.n_samples = r->n_samples;
    p.sps = r->steps_per_sample;
    p.dt = r->dt;
    p.h2 = r->dt * 0.5;   // integrator.py:103
    p.dt6 = r->dt / 6.0;  // integrator.py:104 (IEEE division, as in Python)
    p.steps = r->steps;
    p.stride = r->record_stride;
    p.n_records = sto_n_records(r->steps, r->record_stride);
    p.states = r->states;
    p.rows_cap = P->rows_cap;
    p.chunk_cols = P->chunk_cols;
    reset_status_kernel<<<1, 256, 0, s>>>(P->status, P->bar, P->flags);
    STO_CUDA(cudaGetLastError());
    int rc = STO_OK;
    if (P->world > 1) {
        if (!P->connected) return fail(STO_E_PARAM, "sharded plan is not connected to its peers");
        if (P->peer_lost) return fail(STO_E_CUDA, "sharded plan lost a peer in an earlier run; destroy it");
        p.mp.world = P->world;
        p.mp.timeout_ns = peer_timeout_ns();
        p.mp.rank_base = P->rank;
        p.mp.ctas_per_rank = P->grid;
        p.mp.epoch_base = P->epoch_base;
        p.mp.sh[0] = shard_info(P);
        for (int q = 0; q < P->world; ++q) {
            p.mp.xbuf_of[q] = P->xbuf_of[q];
            p.mp.flags_of[q] = P->flags_of[q];
        }
        rc = P->kind == kResident ? launch_multi<WSrc::Shared>(p, P->grid, P->smem, s)
             : P->stream_evict_first ? launch_multi<WSrc::GlobalStream>(p, P->grid, P->smem, s)
                                     : launch_multi<WSrc::GlobalL2>(p, P->grid, P->smem, s);
        P->epoch_base += 4ull * (unsigned long long)r->steps;
        if (rc) return rc;
        if (status) return sto_plan_last_status(P, status, stream);
        return STO_OK;
    }
    switch (P->kind) {
        case kTiny: rc = launch_tiny(p, P->n, s); break;
        case kReg: {
            RegParams rp{p, P->ll, 0u};
            // test knob: start the 31-bit LL epoch near its wrap (STO_REG_EPOCH0, even)
            if (const char *e = getenv("STO_REG_EPOCH0")) rp.epoch0 = (unsigned)strtoul(e, nullptr, 0) & 0x7ffffffeu;
            STO_CUDA(cudaMemsetAsync(P->ll, 0, sizeof(uint4) * 2 * (size_t)P->n, s));
            rc = launch_reg(rp, P->team, P->rows_per_team, P->chunk_cols == 1, P->grid, P->threads,
                            P->smem, s);
            break;
        }
        case kCluster:
            rc = launch_clu(p, P->clu_hyb, P->team, P->clu_cols, P->grid, P->threads, P->smem, s);
            break;
        case kSingle: rc = launch_grid<WSrc::Shared, true>(p, 1, P->smem, false, s); break;
        case kResident: rc = launch_grid<WSrc::Shared, false>(p, P->grid, P->smem, true, s); break;
        default:
            rc = P->stream_evict_first
                     ? (P->grid_threads == 640
                            ? launch_grid<WSrc::GlobalStream, false, 640>(p, P->grid, P->smem, true, s)
                            : launch_grid<WSrc::GlobalStream, false>(p, P->grid, P->smem, true, s))
                     : launch_grid<WSrc::GlobalL2, false>(p, P->grid, P->smem, true, s);
    }
    if (rc) return rc;
    if (status) return sto_plan_last_status(P, status, stream);
    return STO_OK;
}

}  // extern "C"

namespace {
template <int U>
int launch_ens(const EnsParams &e, int grid, cudaStream_t s) {
    const size_t smem = ens_smem_bytes(U);
    STO_CUDA(cudaFuncSetAttribute(ens_rk4_kernel<U>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    void *args[] = {(void *)&e};
    STO_CUDA(cudaLaunchCooperativeKernel((void *)ens_rk4_kernel<U>, dim3(grid), dim3(kEnsThreads),
                                         args, smem, s));
    return STO_OK;
}
int launch_ens_u(int u, const EnsParams &e, int grid, cudaStream_t s) {
    switch (u) {
        case 1: return launch_ens<1>(e, grid, s);
        case 2: return launch_ens<2>(e, grid, s);
        case 3: return launch_ens<3>(e, grid, s);
        case 4: return launch_ens<4>(e, grid, s);
        case 5: return launch_ens<5>(e, grid, s);
        case 6: return launch_ens<6>(e, grid, s);
        default: return launch_ens<7>(e, grid, s);
    }
}
}  // namespace

extern "C" {

int sto_integrate_ensemble(sto_plan *P, const sto_ensemble_run *r, sto_status *status,
                           void *stream) {
    if (!P || !r) return fail(STO_E_PARAM, "null plan or run");
    if (r->batch < 1 || !r->consts || !r->m || !r->samples || r->n_samples < 1 ||
        r->steps_per_sample < 1 || r->steps < 1 || r->record_stride < 1 || !(r->dt > 0.0) ||
        r->batch >= (1 << 20) || P->n >= (1 << 20) || r->steps >= (1LL << 23))
        return fail(STO_E_PARAM, "bad ensemble run descriptor");
    STO_CUDA(cudaSetDevice(P->device));
    cudaStream_t s = (cudaStream_t)stream;
    // Tile choice: TR = 8U rows x 64 members per CTA.  Minimise the per-SM
    // work U * (number of launches) over U = 1..8 (ties -> larger U: fewer
    // row tiles re-reading X).
    const int nu = (P->n + 7) / 8;  // 8-row units
    const int total_cols = (int)((r->batch + kEnsBT - 1) / kEnsBT);
    int best_u = 0, best_launch_cols = 0;
    long long best_cost = 0;
    for (int u = 1; u <= kEnsMaxU; ++u) {
        const int n_rt = (nu + u - 1) / u;
        if (n_rt > P->sm_count) continue;
        const int cols = std::min(total_cols, P->sm_count / n_rt);
        const long long cost = (long long)u * ((total_cols + cols - 1) / cols);
        if (!best_u || cost <= best_cost) {
            best_u = u;
            best_cost = cost;
            best_launch_cols = cols;
        }
    }
    if (!best_u) return fail(STO_E_PARAM, "ensemble needs n <= 64 * SM count");
    if (const char *ev = getenv("STO_ENS_U")) {  // tuning override
        const int u = atoi(ev);
        if (u >= 1 && u <= kEnsMaxU && (nu + u - 1) / u <= P->sm_count) {
            best_u = u;
            best_launch_cols = std::min(total_cols, P->sm_count / ((nu + u - 1) / u));
        }
    }
    const int U = best_u, TR = 8 * U;
    const int n_rt = (nu + U - 1) / U;
    const int cols_per_launch = best_launch_cols;
    const int kp = ((P->n + kEnsKAlign - 1) / kEnsKAlign) * kEnsKAlign;
    const int np_alloc = nu * 8 + 8 * kEnsMaxU;  // any n_rt * TR fits
    const size_t bp = (size_t)cols_per_launch * kEnsBT;
    if (!P->ens_w) {
        STO_CUDA(cudaMalloc(&P->ens_w, sizeof(double) * (size_t)np_alloc * kp));
        P->ens_np = np_alloc;
        STO_CUDA(cudaMalloc(&P->ens_bar, sizeof(unsigned long long) * 32 * 1024));
    }
    if (P->ens_u != U) {  // W in fragment order for this tile height
        ens_layout_kernel<<<1184, 256, 0, s>>>(P->L.w, P->ens_w, P->n, kp, TR, n_rt, P->L.cs);
        STO_CUDA(cudaGetLastError());
        P->ens_u = U;
    }
    if (P->ens_bp < bp) {
        cudaFree(P->ens_x);
        cudaFree(P->ens_st);
        P->ens_x = P->ens_st = nullptr;
        STO_CUDA(cudaMalloc(&P->ens_x, sizeof(double) * 2 * kp * bp));
        STO_CUDA(cudaMalloc(&P->ens_st, sizeof(double) * kEnsState * np_alloc * bp));
        P->ens_bp = bp;
    }
    reset_status_kernel<<<1, 256, 0, s>>>(P->status, P->bar, P->flags);
    STO_CUDA(cudaGetLastError());
    for (int c0 = 0; c0 < total_cols; c0 += cols_per_launch) {
        const int ncols = std::min(cols_per_launch, total_cols - c0);
        EnsParams e{};
        e.n = P->n;
        e.np = np_alloc;
        e.kp = kp;
        e.n_rt = n_rt;
        e.batch = (int)r->batch;
        e.bp = (int)bp;
        e.member0 = c0 * kEnsBT;
        e.n_in = P->n_in;
        e.w = P->ens_w;
        e.w_in = P->w_in;
        e.consts = r->consts;
        e.m = r->m;
        e.samples = r->samples;
        e.sample_member_stride = r->sample_member_stride;
        e.n_samples = r->n_samples;
        e.sps = r->steps_per_sample;
        e.dt = r->dt;
        e.h2 = r->dt * 0.5;
        e.dt6 = r->dt / 6.0;
        e.steps = r->steps;
        e.stride = r->record_stride;
        e.n_records = sto_n_records(r->steps, r->record_stride);
        e.states = r->states;
        e.x = P->ens_x;
        e.st = P->ens_st;
        e.bar = P->ens_bar;
        e.status = P->status;
        e.debug_solo = getenv("STO_ENS_DEBUG_SOLO") ? 1 : 0;
        e.gate_frac = getenv("STO_ENS_GATE") ? (float)atof(getenv("STO_ENS_GATE")) : 0.5f;
        STO_CUDA(cudaMemsetAsync(P->ens_x, 0, sizeof(double) * 2 * kp * bp, s));
        STO_CUDA(cudaMemsetAsync(P->ens_bar, 0, sizeof(unsigned long long) * 32 * 1024, s));
        const int rc = launch_ens_u(U, e, n_rt * ncols, s);
        if (rc) return rc;
    }
    if (!status) return STO_OK;
    StatusDev h{};
    STO_CUDA(cudaMemcpyAsync(&h, P->status, sizeof(h), cudaMemcpyDeviceToHost, s));
    STO_CUDA(cudaStreamSynchronize(s));
    status->diverged = h.flag;
    status->reserved = h.flag ? (int32_t)((h.key >> 20) & 0xfffff) : -1;  // member
    status->oscillator = h.flag ? (h.key & 0xfffff) : -1;
    status->step = h.flag ? (h.key >> 40) : -1;
    if (h.flag)
        return fail(STO_E_DIVERGED, "member " + std::to_string(status->reserved) +
                                        ": non-finite state for oscillator " +
                                        std::to_string(status->oscillator) + " at step " +
                                        std::to_string(status->step));
    return STO_OK;
}

}  // extern "C"

namespace {
template <int BV>
const void *ex_kernel_bv(int u) {
    switch (u) {
        case 1: return (const void *)ens_exact_kernel<1, BV>;
        case 2: return (const void *)ens_exact_kernel<2, BV>;
        case 3: return (const void *)ens_exact_kernel<3, BV>;
        case 4: return (const void *)ens_exact_kernel<4, BV>;
        case 5: return (const void *)ens_exact_kernel<5, BV>;
        case 6: return (const void *)ens_exact_kernel<6, BV>;
        default: return (const void *)ens_exact_kernel<7, BV>;
    }
}
const void *ex_kernel_of(int u, int bv) {
    return bv == 4 ? ex_kernel_bv<4>(u) : (bv == 2 ? ex_kernel_bv<2>(u) : ex_kernel_bv<1>(u));
}
}  // namespace

extern "C" {

int sto_integrate_ensemble_exact(sto_plan *P, const sto_ensemble_run *r, sto_status *status,
                                 void *stream) {
    if (!P || !r) return fail(STO_E_PARAM, "null plan or run");
    if (r->batch < 1 || !r->consts || !r->m || !r->samples || r->n_samples < 1 ||
        r->steps_per_sample < 1 || r->steps < 1 || r->record_stride < 1 || !(r->dt > 0.0) ||
        r->batch >= (1 << 20) || P->n >= (1 << 20) || r->steps >= (1LL << 23))
        return fail(STO_E_PARAM, "bad ensemble run descriptor");
    if (P->world > 1) return fail(STO_E_PARAM, "ensemble needs an unsharded plan");
    const int kp = ((P->n + kExKC - 1) / kExKC) * kExKC;
    const int n_leaves = (kp / kExKC + 1) / 2;  // 64-column leaves
    int levels = 1;
    while ((1 << levels) <= n_leaves) ++levels;  // bit length of the leaf count
    if (levels > kExMaxLevels) return fail(STO_E_PARAM, "exact ensemble supports n <= 16320");
    STO_CUDA(cudaSetDevice(P->device));
    cudaStream_t s = (cudaStream_t)stream;
    // Tile = 8U oscillators x 64 members, one CTA per SM, several tiles per CTA:
    // minimise the per-CTA work U * ceil(tiles / grid) (ties -> larger U), among
    // the U whose leaf stack fits shared memory.
    // members per thread: BV = 2 (tiles of 64 members) unless STO_EX_BV says otherwise
    int BV = kExDefaultBV;
    if (const char *ev = getenv("STO_EX_BV")) BV = atoi(ev) == 1 ? 1 : (atoi(ev) == 4 ? 4 : 2);
    const int TB = ex_tile_members(BV);
    const int nu = (P->n + 7) / 8;
    const int total_ct = (int)((r->batch + TB - 1) / TB);
    int U = 0;
    long long best = 0;
    for (int u = 1; u <= kExMaxU; ++u) {
        if (ex_smem_bytes(u, BV, levels) > kExSmemBudget) continue;
        const long long tiles = (long long)((nu + u - 1) / u) * total_ct;
        const long long cost = (long long)u * ((tiles + P->sm_count - 1) / P->sm_count);
        if (!U || cost <= best) {
            U = u;
            best = cost;
        }
    }
    if (!U) return fail(STO_E_PARAM, "exact ensemble: no tile fits shared memory");
    if (const char *ev = getenv("STO_EX_U")) {  // test knob: force a tile height
        const int u = atoi(ev);
        if (u >= 1 && u <= kExMaxU && ex_smem_bytes(u, BV, levels) <= kExSmemBudget) U = u;
    }
    const int TR = 8 * U;
    const int n_rt = (P->n + TR - 1) / TR;
    const int np_alloc = nu * 8 + 8 * kExMaxU;  // any n_rt * TR fits
    const int grid = std::min(P->sm_count, n_rt * total_ct);
    // member tiles per launch: at most kExMaxTiles tiles per CTA
    int ct_per_launch = std::max(1, std::min(total_ct, (kExMaxTiles * grid) / n_rt));
    if (const char *ev = getenv("STO_EX_CT_PER_LAUNCH"))  // test knob: force several launches
        ct_per_launch = std::max(1, std::min(ct_per_launch, atoi(ev)));
    if (ct_per_launch > 4096) return fail(STO_E_PARAM, "too many member tiles");
    const size_t bp = (size_t)ct_per_launch * TB;
    if (!P->ex_w) {
        STO_CUDA(cudaMalloc(&P->ex_w, sizeof(double) * (size_t)np_alloc * kp));
        STO_CUDA(cudaMalloc(&P->ex_bar, sizeof(unsigned long long) * 32 * 4096));
        ex_layout_kernel<<<1184, 256, 0, s>>>(P->L.w, P->ex_w, P->n, np_alloc, kp, P->L.cs);
        STO_CUDA(cudaGetLastError());
    }
    if (P->ex_bp < bp) {
        cudaFree(P->ex_x);
        cudaFree(P->ex_st);
        P->ex_x = P->ex_st = nullptr;
        STO_CUDA(cudaMalloc(&P->ex_x, sizeof(double) * 2 * kp * bp));
        STO_CUDA(cudaMalloc(&P->ex_st, sizeof(double) * kExPlanes * np_alloc * bp));
        P->ex_bp = bp;
    }
    const size_t smem = ex_smem_bytes(U, BV, levels);
    const void *fn = ex_kernel_of(U, BV);
    STO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    reset_status_kernel<<<1, 256, 0, s>>>(P->status, P->bar, P->flags);
    STO_CUDA(cudaGetLastError());
    for (int c0 = 0; c0 < total_ct; c0 += ct_per_launch) {
        const int nct = std::min(ct_per_launch, total_ct - c0);
        ExParams e{};
        e.n = P->n;
        e.np = np_alloc;
        e.kp = kp;
        e.n_rt = n_rt;
        e.n_ct = nct;
        e.member0 = c0 * TB;
        e.batch = (int)std::min<int64_t>((int64_t)nct * TB, r->batch - e.member0);
        e.batch_total = (int)r->batch;
        e.bp = (int)bp;
        e.n_in = P->n_in;
        e.levels = levels;
        e.w = P->ex_w;
        e.w_in = P->w_in;
        e.consts = r->consts;
        e.m = r->m;
        e.samples = r->samples;
        e.sample_member_stride = r->sample_member_stride;
        e.n_samples = r->n_samples;
        e.sps = r->steps_per_sample;
        e.dt = r->dt;
        e.h2 = r->dt * 0.5;
        e.dt6 = r->dt / 6.0;
        e.steps = r->steps;
        e.stride = r->record_stride;
        e.n_records = sto_n_records(r->steps, r->record_stride);
        e.states = r->states;
        e.x = P->ex_x;
        e.st = P->ex_st;
        e.bar = P->ex_bar;
        e.status = P->status;
        STO_CUDA(cudaMemsetAsync(P->ex_x, 0, sizeof(double) * 2 * kp * bp, s));
        STO_CUDA(cudaMemsetAsync(P->ex_bar, 0, sizeof(unsigned long long) * 32 * nct, s));
        const int g = std::min(grid, n_rt * nct);
        void *args[] = {(void *)&e};
        STO_CUDA(cudaLaunchCooperativeKernel(fn, dim3(g), dim3(kExThreads), args, smem, s));
    }
    if (!status) return STO_OK;
    StatusDev h{};
    STO_CUDA(cudaMemcpyAsync(&h, P->status, sizeof(h), cudaMemcpyDeviceToHost, s));
    STO_CUDA(cudaStreamSynchronize(s));
    status->diverged = h.flag;
    status->reserved = h.flag ? (int32_t)((h.key >> 20) & 0xfffff) : -1;  // member
    status->oscillator = h.flag ? (h.key & 0xfffff) : -1;
    status->step = h.flag ? (h.key >> 40) : -1;
    if (h.flag)
        return fail(STO_E_DIVERGED, "member " + std::to_string(status->reserved) +
                                        ": non-finite state for oscillator " +
                                        std::to_string(status->oscillator) + " at step " +
                                        std::to_string(status->step));
    return STO_OK;
}

int sto_plan_exchange_handle(sto_plan *P, void *out, int64_t bytes) {
    if (!P || !out || bytes < (int64_t)sizeof(cudaIpcMemHandle_t) || P->world < 2)
        return fail(STO_E_PARAM, "exchange handle needs a sharded plan and a 64-byte buffer");
    STO_CUDA(cudaSetDevice(P->device));
    cudaIpcMemHandle_t h;
    STO_CUDA(cudaIpcGetMemHandle(&h, P->exch));
    std::memcpy(out, &h, sizeof(h));
    return STO_OK;
}

int sto_plan_connect(sto_plan *P, const void *handles, int32_t world) {
    if (!P || !handles || world != P->world) return fail(STO_E_PARAM, "bad connect arguments");
    STO_CUDA(cudaSetDevice(P->device));
    const size_t xb = sizeof(double) * 2 * (size_t)P->L.cs.ldw;
    for (int q = 0; q < world; ++q) {
        if (q == P->rank) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char *>(handles) + q * sizeof(h), sizeof(h));
        void *ptr = nullptr;
        STO_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        P->ipc_opened[q] = ptr;
        P->xbuf_of[q] = static_cast<double *>(ptr);
        P->flags_of[q] = reinterpret_cast<unsigned long long *>(static_cast<char *>(ptr) + xb);
    }
    P->connected = true;
    return STO_OK;
}

int sto_plan_connect_local(sto_plan **plans, int32_t world) {
    if (!plans || world < 2 || world > kMaxRanks) return fail(STO_E_PARAM, "bad local group");
    for (int q = 0; q < world; ++q) {
        if (!plans[q] || plans[q]->world != world || plans[q]->rank != q ||
            plans[q]->device != plans[0]->device || plans[q]->n != plans[0]->n ||
            plans[q]->L.cs.ldw != plans[0]->L.cs.ldw)
            return fail(STO_E_PARAM, "local group plans must be ranks 0..world-1 of one device");
    }
    for (int q = 0; q < world; ++q) {
        for (int o = 0; o < world; ++o) {
            plans[q]->xbuf_of[o] = plans[o]->exch;
            plans[q]->flags_of[o] = plans[o]->exch_flags;
        }
        plans[q]->connected = true;
    }
    return STO_OK;
}

int sto_integrate_group(sto_plan **plans, int32_t world, const sto_run *r, sto_status *status,
                        void *stream) {
    if (!plans || world < 2 || world > kMaxRanks || !r) return fail(STO_E_PARAM, "bad group");
    sto_plan *P0 = plans[0];
    for (int q = 0; q < world; ++q)
        if (!plans[q] || !plans[q]->connected || plans[q]->world != world ||
            plans[q]->kind != P0->kind || plans[q]->smem > P0->smem ||
            plans[q]->stream_evict_first != P0->stream_evict_first ||
            plans[q]->chunk_cols != P0->chunk_cols)
            return fail(STO_E_PARAM, "group plans must be connected shards with one kernel family");
    if (!r->m || !r->samples || r->n_samples < 1 || r->steps_per_sample < 1 || r->steps < 1 ||
        r->record_stride < 1 || !(r->dt > 0.0))
        return fail(STO_E_PARAM, "bad run descriptor");
    STO_CUDA(cudaSetDevice(P0->device));
    cudaStream_t s = (cudaStream_t)stream;
    KParams p = base_params(P0);
    p.mode = kIntegrate;
    p.m = r->m;
    p.samples = r->samples;
    p.n_samples = r->n_samples;
    p.sps = r->steps_per_sample;
    p.dt = r->dt;
    p.h2 = r->dt * 0.5;
    p.dt6 = r->dt / 6.0;
    p.steps = r->steps;
    p.stride = r->record_stride;
    p.n_records = sto_n_records(r->steps, r->record_stride);
    p.states = r->states;
    int cap = 1;
    const int per = P0->sm_count / world;  // CTAs per logical rank
    for (int q = 0; q < world; ++q) cap = std::max(cap, (plans[q]->rows + per - 1) / per);
    p.rows_cap = cap;
    p.chunk_cols = P0->chunk_cols;
    const size_t smem = grid_smem(cap, P0->L.cs, p.chunk_cols, P0->kind == kResident);
    if (smem > kSmemBudget)
        return fail(STO_E_PARAM, "group shard does not fit shared memory");
    p.mp.world = world;
    p.mp.rank_base = 0;
    p.mp.ctas_per_rank = per;
    p.mp.epoch_base = P0->epoch_base;
    p.mp.timeout_ns = peer_timeout_ns();
    for (int q = 0; q < world; ++q) {
        p.mp.sh[q] = shard_info(plans[q]);
        p.mp.xbuf_of[q] = plans[q]->exch;
        p.mp.flags_of[q] = plans[q]->exch_flags;
        if (plans[q]->epoch_base != P0->epoch_base) return fail(STO_E_PARAM, "group epochs differ");
        reset_status_kernel<<<1, 256, 0, s>>>(plans[q]->status, plans[q]->bar, plans[q]->flags);
    }
    p.status = P0->status;
    int rc = P0->kind == kResident ? launch_multi<WSrc::Shared>(p, per * world, smem, s)
             : P0->stream_evict_first ? launch_multi<WSrc::GlobalStream>(p, per * world, smem, s)
                                      : launch_multi<WSrc::GlobalL2>(p, per * world, smem, s);
    for (int q = 0; q < world; ++q) plans[q]->epoch_base += 4ull * (unsigned long long)r->steps;
    if (rc) return rc;
    if (status) return sto_plan_last_status(P0, status, stream);
    return STO_OK;
}

int sto_plan_last_status(sto_plan *P, sto_status *status, void *stream) {
    if (!P || !status) return fail(STO_E_PARAM, "null plan or status");
    STO_CUDA(cudaSetDevice(P->device));
    StatusDev h{};
    STO_CUDA(cudaMemcpyAsync(&h, P->status, sizeof(h), cudaMemcpyDeviceToHost,
                             (cudaStream_t)stream));
    STO_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (h.flag == 2) {
        P->peer_lost = true;
        status->diverged = 0;
        status->reserved = 0;
        status->oscillator = -1;
        status->step = -1;
        return fail(STO_E_CUDA, "rank " + std::to_string(h.key) +
                                    " did not reach the x exchange within the peer watchdog limit "
                                    "(STO_PEER_TIMEOUT_S); the run stopped early and the plan is unusable");
    }
    status->diverged = h.flag;
    status->reserved = 0;
    status->oscillator = h.flag ? (h.key & 0xffffff) : -1;
    status->step = h.flag ? (h.key >> 24) : -1;
    if (h.flag)
        return fail(STO_E_DIVERGED, "non-finite state for oscillator " +
                                        std::to_string(status->oscillator) + " at step " +
                                        std::to_string(status->step));
    return STO_OK;
}

int sto_integrate_host(sto_plan *P, double *m, const double *samples, int64_t n_samples,
                       int64_t steps_per_sample, double dt, int64_t steps, int64_t record_stride,
                       double *states, sto_status *status) {
    if (!P || !m || !samples || !states || !status) return fail(STO_E_PARAM, "null argument");
    STO_CUDA(cudaSetDevice(P->device));
    const int64_t nrec = sto_n_records(steps, record_stride);
    if (nrec < 1 || n_samples < 1) return fail(STO_E_PARAM, "bad run sizes");
    const size_t mb = sizeof(double) * 3 * (size_t)P->n;
    const size_t sb = sizeof(double) * (size_t)n_samples * P->n_in;
    double *dm = nullptr, *ds = nullptr, *dst = nullptr;
    STO_CUDA(cudaMalloc(&dm, mb));
    STO_CUDA(cudaMalloc(&ds, sb));
    STO_CUDA(cudaMalloc(&dst, mb * nrec));
    int rc = STO_OK;
    if (cudaMemcpy(dm, m, mb, cudaMemcpyDefault) != cudaSuccess ||
        cudaMemcpy(ds, samples, sb, cudaMemcpyDefault) != cudaSuccess) {
        rc = fail(STO_E_CUDA, "host to device copy failed");
    } else {
        sto_run r{dm, ds, n_samples, steps_per_sample, dt, steps, record_stride, dst};
        rc = sto_integrate(P, &r, status, nullptr);
        if (rc == STO_OK || rc == STO_E_DIVERGED) {
            const int keep = rc;
            if (cudaMemcpy(states, dst, mb * nrec, cudaMemcpyDefault) != cudaSuccess ||
                cudaMemcpy(m, dm, mb, cudaMemcpyDefault) != cudaSuccess)
                rc = fail(STO_E_CUDA, "device to host copy failed");
            else
                rc = keep;
        }
    }
    cudaFree(dm);
    cudaFree(ds);
    cudaFree(dst);
    return rc;
}

int sto_tree_matvec(int device, int64_t rows, int64_t cols, const double *a, int64_t lda,
                    const double *x, double *out) {
    if (rows < 1 || cols < 1 || lda < cols || !a || !x || !out)
        return fail(STO_E_PARAM, "bad matvec arguments");
    cudaDeviceProp prop;
    if (int rc = check_device(device, &prop)) return rc;
    STO_CUDA(cudaSetDevice(device));
    Layout L;
    int rc = upload_layout(L, (int)rows, (int)cols, a, lda, cols >= 8192 ? 2048 : 512, nullptr);
    double *dx = nullptr, *dout = nullptr;
    if (rc == STO_OK) {
        if (cudaMalloc(&dx, sizeof(double) * cols) != cudaSuccess ||
            cudaMalloc(&dout, sizeof(double) * rows) != cudaSuccess ||
            cudaMemcpy(dx, x, sizeof(double) * cols, cudaMemcpyDefault) != cudaSuccess) {
            rc = fail(STO_E_CUDA, "matvec staging failed");
        } else {
            KParams p{};
            p.cs = L.cs;
            p.rows = (int)rows;
            p.mode = kMatvec;
            p.w = L.w;
            p.xsrc = dx;
            p.x_stride = 1;
            p.out = dout;
            const int g = (int)std::min<int64_t>(prop.multiProcessorCount, rows);
            p.rows_cap = (int)((rows + g - 1) / g);
            p.chunk_cols = choose_chunk(L.cs, p.rows_cap, false);
            const size_t smem = grid_smem(p.rows_cap, L.cs, p.chunk_cols, false);
            rc = launch_grid<WSrc::GlobalL2, false>(p, g, smem, false, nullptr);
            if (rc == STO_OK &&
                cudaMemcpy(out, dout, sizeof(double) * rows, cudaMemcpyDefault) != cudaSuccess)
                rc = fail(STO_E_CUDA, "matvec result copy failed");
        }
    }
    cudaFree(dx);
    cudaFree(dout);
    cudaDeviceSynchronize();
    cudaFreeAsync(L.w, nullptr);
    return rc;
}

int sto_plan_matvec(sto_plan *P, const double *x, double *out, void *stream) {
    if (!P || !x || !out) return fail(STO_E_PARAM, "bad plan matvec arguments");
    if (P->world > 1) return fail(STO_E_PARAM, "plan matvec needs an unsharded plan");
    STO_CUDA(cudaSetDevice(P->device));
    KParams p{};
    p.cs = P->L.cs;
    p.rows = P->n;
    p.mode = kMatvec;
    p.w = P->L.w;
    p.xsrc = x;
    p.x_stride = 1;
    p.out = out;
    const int g = std::min(P->sm_count, P->n);
    p.rows_cap = (P->n + g - 1) / g;
    p.chunk_cols = choose_chunk(P->L.cs, p.rows_cap, false);
    const size_t smem = grid_smem(p.rows_cap, P->L.cs, p.chunk_cols, false);
    return launch_grid<WSrc::GlobalL2, false>(p, g, smem, false, (cudaStream_t)stream);
}

#ifdef STO_TIMELINE
STO_API int sto_debug_ens_timeline(unsigned long long *out, int count) {
    STO_CUDA(cudaMemcpyFromSymbol(out, g_ens_timeline, sizeof(unsigned long long) * count));
    return STO_OK;
}
STO_API int sto_debug_grid_cta_block(unsigned long long *out, int count) {
    STO_CUDA(cudaMemcpyFromSymbol(out, g_grid_cta_block, sizeof(unsigned long long) * count));
    return STO_OK;
}
STO_API int sto_debug_grid_timeline(unsigned long long *out, int count) {
    STO_CUDA(cudaMemcpyFromSymbol(out, g_grid_timeline, sizeof(unsigned long long) * count));
    return STO_OK;
}
STO_API int sto_debug_multi_timeline(unsigned long long *out, int count) {
    STO_CUDA(cudaMemcpyFromSymbol(out, g_multi_timeline, sizeof(unsigned long long) * count));
    return STO_OK;
}
STO_API int sto_debug_timeline(unsigned long long *out, int count) {
    STO_CUDA(cudaMemcpyFromSymbol(out, g_timeline, sizeof(unsigned long long) * count));
    return STO_OK;
}
#endif

// ---- reservoir construction on the device (sto_build.cuh) ------------------
int sto_pcg64_fill(int device, double *out, int64_t count, int64_t offset, const uint64_t pcg[4],
                   int64_t diag_n, int64_t ld, void *stream) {
    if (!out || !pcg || count < 0 || offset < 0 || (diag_n > 0 && (count != diag_n * (diag_n - 1) || ld < diag_n)))
        return fail(STO_E_PARAM, "sto_pcg64_fill: bad arguments");
    STO_CUDA(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    Pcg64 g;
    g.state = ((u128)pcg[0] << 64) | (u128)pcg[1];
    g.inc = ((u128)pcg[2] << 64) | (u128)pcg[3];
    u128 a32, c32;
    pcg_jump_coeffs(g.inc, 32, a32, c32);
    if (diag_n > 0) {
        zero_diag_kernel<<<256, 256, 0, s>>>(out, diag_n, ld);
        STO_CUDA(cudaGetLastError());
    }
    if (count > 0) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const long long warps_needed = (count + 4095) / 4096;  // >= 128 draws per lane
        const int blocks = (int)std::max<long long>(1, std::min<long long>(8LL * sms, (warps_needed + 7) / 8));
        pcg64_fill_kernel<<<blocks, 256, 0, s>>>(out, count, offset, g, diag_n, ld, a32, c32);
        STO_CUDA(cudaGetLastError());
    }
    return STO_OK;
}

int sto_gemv(int device, const double *w, int64_t rows, int64_t cols, int64_t ld, const double *x,
             double *y, void *stream) {
    if (!w || !x || !y || rows < 0 || cols < 0 || ld < cols) return fail(STO_E_PARAM, "sto_gemv: bad arguments");
    STO_CUDA(cudaSetDevice(device));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = (int)std::max<long long>(1, std::min<long long>(4LL * sms, (rows + 7) / 8));
    gemv_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(w, rows, cols, ld, x, y);
    STO_CUDA(cudaGetLastError());
    return STO_OK;
}

int sto_scale_div(int device, double *a, int64_t count, double divisor, void *stream) {
    if (!a || count < 0) return fail(STO_E_PARAM, "sto_scale_div: bad arguments");
    STO_CUDA(cudaSetDevice(device));
    scale_div_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(a, count, divisor);
    STO_CUDA(cudaGetLastError());
    return STO_OK;
}

int sto_norm_drift(int device, const double *states, int64_t outer, int64_t members, int64_t n,
                   double *out, void *stream) {
    if (!states || !out || outer < 0 || members < 1 || n < 1 || members >= (1 << 30))
        return fail(STO_E_PARAM, "sto_norm_drift: bad arguments");
    STO_CUDA(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    STO_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * members, s));
    const long long total = outer * members * n;
    const int blocks = (int)std::max<long long>(1, std::min<long long>(1184, (total + 255) / 256));
    norm_drift_kernel<<<blocks, 256, 0, s>>>(states, outer, (int)members, n,
                                             reinterpret_cast<unsigned long long *>(out));
    STO_CUDA(cudaGetLastError());
    return STO_OK;
}

int sto_selftest_div(int device, const double *a, const double *b, int64_t count, double *q,
                     int32_t *ok, double *ref, void *stream) {
    if (!a || !b || !q || !ok || !ref || count < 0) return fail(STO_E_PARAM, "sto_selftest_div: bad arguments");
    STO_CUDA(cudaSetDevice(device));
    selftest_div_kernel<<<1184, 256, 0, (cudaStream_t)stream>>>(a, b, count, q, ok, ref);
    STO_CUDA(cudaGetLastError());
    return STO_OK;
}

}  // extern "C"
