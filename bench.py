#!/usr/bin/env python
"""Benchmark: oscillator-steps/s of the coupled-STO RK4 path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]

One bench "step" = one whole integrate() run of the workload (BASELINE.json
configs): N oscillators x S RK4 steps, recorded initial + final
(record_stride = S, as the reference's run_benchmark does, bench.py:291).
Metric = N * S / seconds per run (oscillator-steps/s), summed over ranks.

Default workload "n1e4" = configs[4] at N = 1e4 (the largest N of the
metric's N=1..1e4 range that fits one GPU; W = 800 MB > L2, so no L2 flush
is needed between runs). Other workloads: n1 (configs[1]), n100
(configs[0]), n1000 (configs[2]), n4e4.

Arms
  ours (default)  value: device-resident inputs, CUDA events around K runs of
                  sto_integrate (persistent kernel), max over ranks.
                  e2e: the public API `integrate(topology, params, config)` from
                  pinned host buffers: W/W_in/m0/drive uploaded, run, states read
                  back -- every step.
  reference       the reference's CPU path restated in C (oracle/, kind
                  "port": the reference is pure Python/numba, nothing to
                  compile) on all host cores, bounded sample of the workload.

Multi-GPU (torchrun): n1e4 / n4e4 shard the ONE trajectory's rows over the
ranks (peer-store all-gather of x inside the persistent kernel; "scaling":
"strong"); ens512 shards members (no communication); n1 / n100 / n1000 run
replicas ("weak").
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (n, rk4 steps per run, description, random drive)
    "n1e4": (10_000, 1000, "configs[4]: N=1e4 coupled STOs, single trajectory, 1e3 RK4 steps", False),
    "n4e4": (40_000, 50, "configs[4]: N=4e4 coupled STOs, single trajectory, 50 RK4 steps", False),
    "n1000": (1000, 100_000, "configs[2]: N=1000, single trajectory, 1e5 RK4 steps", False),
    "n100": (100, 10_000, "configs[0]: N=100, 1e4 RK4 steps, random drive", True),
    "n1": (1, 1_000_000, "configs[1]: N=1 single STO, 1e6 RK4 steps", False),
    "ens512": (1000, 10_000, "configs[3]: N=1000 x B=512 ensemble (current sweep 2.0-3.0 mA), "
               "1e4 RK4 steps, FP64 tensor-core (DMMA) coupling GEMM", False),
}
# dense recording (the reservoir-readout case, integrator.py:171-181): every
# record_stride-th state is written to HBM in-kernel and read back in e2e
WORKLOADS["n100_rec1"] = (100, 10_000, "configs[0] with record_stride=1: N=100, 1e4 RK4 steps, random "
                          "drive, every state recorded (24 MB of states per run)", True)
WORKLOADS["n1e4_rec10"] = (10_000, 1000, "configs[4] with record_stride=10: N=1e4, 1e3 RK4 steps, "
                           "every 10th state recorded (24 MB of states per run)", False)
WORKLOADS["ens512_exact"] = (1000, 10_000, "configs[3] bit-exact mode: N=1000 x B=512 ensemble (current "
                             "sweep 2.0-3.0 mA), 1e4 RK4 steps, pinned-tree coupling on the FP64 CUDA cores",
                             False)
RECORD_STRIDE = {"n100_rec1": 1, "n1e4_rec10": 10}
ENSEMBLE_BATCH = {"ens512": 512, "ens512_exact": 512}
EXACT_ENSEMBLE = ("ens512_exact",)
SHARDED_WORKLOADS = ("n1e4", "n4e4", "n1e4_rec10")  # row-sharded over GPUs when --gpus > 1
# FP64 peaks measured on this pool's B200 (tools/fp64_peak.cu; MEASURED_PEAKS.json has
# none): DMMA m8n8k4 37.1 TFLOP/s, DFMA 34.0, cuBLAS DGEMM 8192^3 35.5.
FP64_TENSOR_PEAK_TFLOPS = 37.1
# the bit-exact mode issues every product and sum separately (no FMA: the pinned
# order), so its ceiling is the FP64 pipe's instruction rate = half the DFMA flops
FP64_MULADD_PEAK_TFLOPS = 34.0 / 2
DT = 1e-11


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# Dependent fp64 chain of one RK4 step in the pinned order (sto_device.cuh): 15
# dependent DMUL/DADD between two h_s divisions in stages 1-3 (m.p, 1 + lam*md,
# then h_s*q_z -> b_z -> a_y -> e_x -> dm/dt -> stage point) and 17 around the
# RK4 combination, i.e. 62 x 8.4 cycles, plus 4 speculative divisions at 68.5
# cycles (tools/microbench.cu: dadd 8.44, dmul 8.38, ddiv_spec 68.5 with the
# four-DFMA quotient, profiles/r02k_division_variants.txt; __ddiv_rn was 113.5)
# = 795 cycles.
RK4_CHAIN_CYCLES = 62 * 8.4 + 4 * 68.5


def measured_peaks() -> dict:
    """Roofline denominators: the driver-written MEASURED_PEAKS.json (hbm_gbs = STREAM
    copy on this pool's B200s), else the profiling recipe's fallback 6.65 TB/s."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            v = d.get("hbm_gbs")
            if isinstance(v, dict):  # tolerate {"value": ...} entries
                v = v.get("value")
            if v:
                return {"hbm_gbs": float(v), "fallback": False}
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "fallback": True}


def device_topology(n: int, seed: int = 0):
    """N > 2e4: the host Arnoldi of build_topology would take ~20 min,
    so the reservoir is built on the GPU (build_topology_device: the same PCG64
    draws bit for bit, rho from device matvecs, ~14 s at N = 4e4)."""
    import paper_2312_01121_b200 as sto

    top = sto.build_topology_device(n, n_in=1, seed=seed)
    return sto.Topology(sto.CouplingMatrix(top.coupling.entries), top.input_weights)


def cached_topology(n: int, seed: int = 0):
    """build_topology(n, seed) with a /dev/shm cache (same box, both arms)."""
    import paper_2312_01121_b200 as sto

    if n > 20000:
        return device_topology(n, seed)

    cache = Path("/dev/shm") / f"sto_topology_n{n}_s{seed}.npz"
    if cache.exists():
        try:
            with np.load(cache) as z:
                return sto.Topology(sto.CouplingMatrix(z["w"]), sto.InputWeights(z["w_in"]))
        except Exception:
            pass
    top = sto.build_topology(n, n_in=1, seed=seed)
    try:
        tmp = cache.with_suffix(f".tmp{os.getpid()}.npz")  # torchrun ranks write concurrently
        np.savez(tmp, w=top.coupling.entries, w_in=top.input_weights.entries)
        os.replace(tmp, cache)
    except OSError:
        pass
    return top


def drive_for(name: str, n_in: int = 1):
    n, steps, _, random_drive = WORKLOADS[name]
    if name in ENSEMBLE_BATCH:
        return np.zeros((1, n_in)), 1
    if random_drive:
        return np.random.default_rng(1).uniform(-1, 1, (steps, n_in)), 1
    return np.zeros((1, n_in)), 1


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def oracle_sample(top, name: str, rk4_steps: int, threads: int):
    """Time the CPU oracle (reference path restated in C) on `rk4_steps` steps."""
    import paper_2312_01121_b200 as sto
    from oracle import oracle

    n = top.n
    samples, sps = drive_for(name)
    samples = samples[:max(1, min(samples.shape[0], rk4_steps))]
    consts = sto.kernel_scalars(sto.PhysicalParams())
    m0 = sto.initial_state(n)
    t0 = time.perf_counter()
    oracle.integrate(top.coupling.entries, top.input_weights.entries, consts, m0, samples, sps,
                     DT, rk4_steps, rk4_steps, threads=threads)
    return time.perf_counter() - t0


def cpu_sample_steps(n: int) -> int:
    """RK4 steps for a ~10-20 s oracle sample (about 1e10 osc-steps*N work)."""
    return int(max(2, min(200_000, 4e10 / max(1.0, float(n) * n * 4) / 2)))


def best_threads(top, name: str, sample: int) -> int:
    """The reference picks its best CPU engine per size (fused = 1 thread vs
    parallel = all cores); do the same on a short probe."""
    cores = os.cpu_count() or 1
    if cores == 1:
        return 1
    if top.n > 2000:
        return cores  # a single thread is never competitive at large N
    probe = max(2, sample // 4)
    oracle_sample(top, name, min(probe, 2), cores)  # page in W
    t_all = min(oracle_sample(top, name, probe, cores) for _ in range(2))
    t_one = min(oracle_sample(top, name, probe, 1) for _ in range(2))
    return 1 if t_one < t_all else cores


def gpu_and_backend(local_rank: int):
    """One process per GPU over NCCL.  STO_BENCH_SHARE_GPU=1 (tests only) puts every
    rank on cuda:0 with gloo, so the multi-rank code path (IPC handle exchange,
    in-kernel all-gather, max-over-ranks timing) runs on a one-GPU box."""
    if os.environ.get("STO_BENCH_SHARE_GPU") == "1":
        return 0, "gloo"
    return local_rank, "nccl"


def run_reference(args, rank, world):
    if rank != 0:
        return
    name = args.workload
    n, steps, desc, _ = WORKLOADS[name]
    top = cached_topology(n)
    sample = min(steps, cpu_sample_steps(n))
    threads = best_threads(top, name, sample)
    oracle_sample(top, name, min(sample, 2), threads)  # warm caches / page in W
    times = []
    for i in range(args.warmup + args.steps):
        dt = oracle_sample(top, name, sample, threads)
        if i >= args.warmup:
            times.append(dt)
    sec = float(np.mean(times))
    value = n * sample / sec
    line = {
        "impl": "reference", "metric": "oscillator-steps/s", "value": value,
        "unit": "osc-steps/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (build_topology seed 0)",
        "config": {"workload": desc, "n": n, "rk4_steps_per_sample": sample, "dt": DT,
                   "parallelism": f"{threads} of {os.cpu_count()} host threads (OpenMP, 128 "
                                  f"fixed row blocks; best of 1 vs all, like fused vs parallel)"},
        "cpu_baseline": {"value": value, "unit": "osc-steps/s", "cores": threads,
                         "kind": "port",
                         "sample": f"N={n}, {sample} RK4 steps per bench step (reference "
                                   f"rk4_step/_row_derivative restated in C, oracle/)"},
        "e2e": {"value": value, "unit": "osc-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def traffic_per_launch(name: str, rk4_steps: int):
    """DRAM bytes (read + write) per persistent-kernel launch, from the committed
    ncu capture (profiles/ncu_traffic.json, normalised per RK4 step)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        entry = json.loads(p.read_text()).get(name)
        return float(entry["bytes_per_rk4_step"]) * rk4_steps if entry else None
    except Exception:
        return None


def run_ours_ensemble(args, rank, world, local_rank):
    """configs[3]: B members sharing W, batch-sharded over ranks (no communication)."""
    import torch

    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200.backends.b200 import B200Backend

    dev, backend_name = gpu_and_backend(local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend_name == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend_name)
    name = args.workload
    n, steps, desc, _ = WORKLOADS[name]
    if args.rk4_steps:
        steps = args.rk4_steps
    batch_total = ENSEMBLE_BATCH[name]
    exact = name in EXACT_ENSEMBLE
    currents = np.linspace(2.0e-3, 3.0e-3, batch_total)
    from paper_2312_01121_b200.sharding import shard_members

    mine = shard_members(batch_total, world, rank)   # batch sharding (no communication)
    params_all = [sto.PhysicalParams(current=float(c)) for c in currents]
    params = [params_all[i] for i in mine]
    top = cached_topology(n)
    backend = B200Backend(top, params[0], device=dev)
    consts = np.array([sto.kernel_scalars(p) for p in params])
    batch = len(params)
    stride = steps
    from paper_2312_01121_b200 import _native

    nrec = _native.n_records(steps, stride)
    c_d = torch.as_tensor(consts, device="cuda")
    m0 = torch.as_tensor(np.tile(sto.initial_state(n)[None], (batch, 1, 1)), device="cuda")
    m_d = torch.empty_like(m0)
    s_d = torch.zeros((1, 1), dtype=torch.float64, device="cuda")
    states_d = torch.empty((nrec, batch, n, 3), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def one_run():
        m_d.copy_(m0)
        backend._plan.integrate_ensemble_dev(m_d, c_d, s_d, 1, 0, DT, steps, stride, states_d,
                                             exact=exact)

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clocks:
        t0e.record(stream)
        for _ in range(args.steps):
            one_run()
        t1e.record(stream)
        torch.cuda.synchronize()
    total_s = t0e.elapsed_time(t1e) / 1e3
    if dist:
        t = torch.tensor([total_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = float(t.item())
    value = batch_total * n * steps * args.steps / total_s
    kernel_s = total_s / args.steps
    flops = 8.0 * n * n * batch * steps  # 4 stages x 2N MACs per oscillator-step
    achieved = flops / kernel_s / 1e12

    # e2e through the public API, host buffers, each step; with N ranks the
    # batch-sharded integrate_ensemble(group=) returns every member on every rank
    cfg = sto.RunConfig(n=n, steps=steps, dt=DT, record_stride=stride, gpu_device=dev)
    group = "world" if dist else None
    sto.integrate_ensemble(top, params_all, cfg, backend=backend, group=group, exact=exact)
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 2))
    for _ in range(e2e_steps):
        ens = sto.integrate_ensemble(top, params_all, cfg, backend=backend, group=group,
                                     exact=exact)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = min(steps, cpu_sample_steps(n))
        oracle_sample(top, "n1000", min(sample, 2), threads)
        sec = oracle_sample(top, "n1000", sample, threads)
        cpu = {"value": n * sample / sec, "unit": "osc-steps/s", "cores": threads, "kind": "port",
               "sample": f"1 member of {batch_total}, N={n}, {sample} RK4 steps (members run "
                         f"sequentially on the CPU, so the ensemble rate equals this rate)"}
    if rank == 0:
        line = {
            "metric": "oscillator-steps/s", "value": value, "unit": "osc-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_s * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (build_topology(1000, seed=0), u=0, current sweep)",
            "config": {"workload": desc, "n": n, "batch": batch_total, "rk4_steps_per_run": steps,
                       "record_stride": stride, "dt": DT,
                       "parallelism": f"batch-sharded x{world}" if world > 1 else "1 GPU",
                       "kernel": ("ens_exact_kernel (pinned tree, DMUL+DADD, bit-exact per member)" if exact
                                  else "ens_rk4_kernel (DMMA m8n8k4 f64)"),
                       "l2": ("W 8 MB + stage x 8 MB + RK state planes L2-resident; one launch per run" if exact
                              else "W 8 MB + stage x 8 MB L2-resident (fragment order), RK state in TMEM; "
                                   "one launch per run")},
            "e2e": {"value": batch_total * n * steps / e2e_s, "unit": "osc-steps/s",
                    "h2d_bytes_per_step": 8 * (n * n + n + batch * 3 * n + batch * 11),
                    "d2h_bytes_per_step": 8 * ens.states.size // world},
            "gpu_launches": 2 * args.steps,
            "roofline": ({"bound": "fp64", "achieved": achieved, "peak": FP64_MULADD_PEAK_TFLOPS,
                          "unit": "TFLOP/s", "frac": achieved / FP64_MULADD_PEAK_TFLOPS,
                          "traffic": traffic_per_launch("ens512_exact", steps),
                          "peak_source": "FP64 CUDA-core mul/add issue rate: half the measured DFMA "
                                         "34.0 TFLOP/s (tools/fp64_peak.cu); the pinned order forbids FMA",
                          "kernel": "ens_exact_kernel"} if exact else
                         {"bound": "tensor", "achieved": achieved, "peak": FP64_TENSOR_PEAK_TFLOPS,
                          "unit": "TFLOP/s", "frac": achieved / FP64_TENSOR_PEAK_TFLOPS,
                          "traffic": traffic_per_launch("ens512", steps),
                          "peak_source": "measured here: DMMA f64 microbenchmark (tools/fp64_peak.cu)",
                          "kernel": "ens_rk4_kernel"}),
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2312_01121_b200 as sto
    from paper_2312_01121_b200 import _native
    from paper_2312_01121_b200.backends.b200 import B200Backend

    dev, backend_name = gpu_and_backend(local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend_name == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend_name)

    name = args.workload
    n, steps, desc, _ = WORKLOADS[name]
    if args.rk4_steps:
        steps = args.rk4_steps
    stride = min(steps, RECORD_STRIDE.get(name, steps))
    params = sto.PhysicalParams()
    if world > 1 and rank != 0:
        dist.barrier()
    top = cached_topology(n)
    if world > 1 and rank == 0:
        dist.barrier()
    samples, sps = drive_for(name)
    samples = samples[:steps] if samples.shape[0] > 1 else samples

    # ------------------------------------------------------------ value ----
    # N > 1 GPUs: the single trajectory is row-sharded (NVLink all-gather of x
    # inside the kernel) for the large-N workloads; small N runs replicas.
    sharded = world > 1 and name in SHARDED_WORKLOADS
    if sharded:
        from paper_2312_01121_b200.sharding import ShardedB200Backend

        backend = ShardedB200Backend(top, params, device=dev)
        rows_mine = backend.shards[rank][1]
        info = {"kernel_name": "stream-sharded", "grid": torch.cuda.get_device_properties(dev)
                .multi_processor_count, "w_bytes": 8 * rows_mine * n}
    else:
        backend = B200Backend(top, params, device=dev)
        info = backend.plan_info
        rows_mine = n
    nrec = _native.n_records(steps, stride)
    m0 = torch.as_tensor(sto.initial_state(n), device="cuda")
    samples_d = torch.as_tensor(samples, device="cuda")
    m_d = torch.empty_like(m0)
    states_d = torch.empty((nrec, n, 3), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def launch():
        backend._plan.integrate_dev(m_d, samples_d, sps, DT, steps, stride, states_d, sync=False)

    for _ in range(args.warmup):
        m_d.copy_(m0)
        launch()
    backend._plan.last_status()
    torch.cuda.synchronize()
    kstart = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kstop = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_start, t_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clocks:
        t_start.record(stream)
        for i in range(args.steps):
            m_d.copy_(m0)
            kstart[i].record(stream)
            launch()
            kstop[i].record(stream)
        t_stop.record(stream)
        torch.cuda.synchronize()
    backend._plan.last_status()
    total_s = t_start.elapsed_time(t_stop) / 1e3
    per_run_ms = [a.elapsed_time(b) for a, b in zip(kstart, kstop)]
    kernel_s = float(np.mean(per_run_ms)) / 1e3
    if dist:
        t = torch.tensor([total_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = float(t.item())
    # sharded: the whole job is ONE trajectory of n oscillators (strong scaling);
    # replicas: every rank integrates its own copy (weak scaling)
    value = (1 if sharded else world) * n * steps * args.steps / total_s
    launches = 2 * args.steps  # reset_status_kernel + persistent RK4 kernel per run

    # -------------------------------------------------------------- e2e ----
    # pinned host copies of every input; public API call each step
    w_pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    w_pin.numpy()[...] = top.coupling.entries
    win_pin = torch.empty((n, 1), dtype=torch.float64, pin_memory=True)
    win_pin.numpy()[...] = top.input_weights.entries
    top_pinned = sto.Topology(sto.CouplingMatrix(w_pin.numpy()), sto.InputWeights(win_pin.numpy()))
    series = sto.InputSeries(samples, sps)
    cfg = sto.RunConfig(n=n, steps=steps, dt=DT, record_stride=stride, input_series=series,
                        backend="gpu", gpu_device=dev)

    def e2e_once():
        if sharded:
            be = ShardedB200Backend(top_pinned, params, device=dev)  # W shard upload
            try:
                return sto.integrate(top_pinned, params, cfg, backend=be)
            finally:
                be.close()
        return sto.integrate(top_pinned, params, cfg)

    e2e_steps = max(1, min(args.steps, 3))
    e2e_once()  # warm
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        traj = e2e_once()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = 8 * (rows_mine * n + n * 1 + 3 * n + samples.size)
    d2h = 8 * (traj.states.size + 3 * n)

    # -------------------------------------------------------- roofline ----
    peaks = measured_peaks()
    alg_bytes = 32.0 * rows_mine * n * steps  # one f64 W row per RK stage per (own) osc-step
    achieved = alg_bytes / kernel_s / 1e9
    clu_hyb = max(64, 1 << (n - 1).bit_length()) <= 128 and os.environ.get("STO_CLU_HYB") != "0"
    kname = {"tiny": "tiny_rk4_kernel", "reg": "reg_rk4_kernel",
             "cluster": "clu_hyb_kernel" if clu_hyb else "clu_rk4_kernel",
             "single": "grid_rk4_kernel[Shared,single]",
             "resident": "grid_rk4_kernel[Shared]",
             "stream": "grid_rk4_kernel[GlobalStream]"}.get(info["kernel_name"], info["kernel_name"])
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "traffic": traffic_per_launch(name, steps),
                "peak_source": "fallback" if peaks.get("fallback") else "measured",
                "kernel": kname}
    if roofline["traffic"]:
        share = roofline["traffic"] / (32.0 * rows_mine * n * steps)
        if info["kernel_name"].startswith("stream") and share < 1.0:
            roofline["note"] = ("achieved counts algorithmic W bytes; DRAM traffic is %.3f of them (a "
                                "slice of W stays L2-resident across stages), so frac can exceed 1" % share)
        elif info["kernel_name"] in ("reg", "resident"):
            roofline["note"] = ("W is held on chip (registers / shared memory): HBM-equivalent roofline "
                                "(SURVEY 8(d)); DRAM traffic is %.2g of the algorithmic bytes" % share)
    if n < 1000:
        # W is a few KB: no HBM/tensor roofline applies.  The bound is the dependent
        # fp64 chain of one RK4 step (4 RHS evaluations, divisions included):
        # RK4_CHAIN_CYCLES, from the latencies tools/microbench.cu measures.
        clk = clocks.summary().get("sm_mhz") or 1965.0
        peak_steps = clk * 1e6 / RK4_CHAIN_CYCLES
        got = steps / kernel_s
        roofline = {"bound": "latency", "achieved": got, "peak": peak_steps, "unit": "RK4 steps/s",
                    "frac": got / peak_steps, "traffic": traffic_per_launch(name, steps),
                    "peak_source": f"dependent-chain bound ({RK4_CHAIN_CYCLES:.0f} cycles per RK4 step = 62 "
                                   f"dependent DMUL/DADD + 4 speculative divisions, latencies measured "
                                   f"by tools/microbench.cu; at {clk:.0f} MHz)",
                    "kernel": kname}

    # ----------------------------------------------------- cpu baseline ----
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        sample = min(steps, cpu_sample_steps(n))
        threads = best_threads(top, name, sample)
        oracle_sample(top, name, min(sample, 2), threads)
        sec = oracle_sample(top, name, sample, threads)
        cpu = {"value": n * sample / sec, "unit": "osc-steps/s", "cores": threads,
               "kind": "port",
               "sample": f"N={n}, {sample} RK4 steps (reference path restated in C, oracle/)"}

    if rank == 0:
        line = {
            "metric": "oscillator-steps/s", "value": value, "unit": "osc-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_s * 1e3 / args.steps,
            "ms_per_step_std": float(np.std(per_run_ms)),  # population std of the K runs (ref bench.py:196)
            "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic (build_topology_device(n, seed=0): reference draws, rho from device "
                     "matvecs)" if n > 20000 else "synthetic (build_topology(n, seed=0), u=0 / "
                     "seeded uniform drive)"),
            "config": {"workload": desc, "n": n, "rk4_steps_per_run": steps,
                       "record_stride": stride, "dt": DT,
                       "parallelism": (f"row-sharded x{world} (in-kernel NVLink all-gather)"
                                       if sharded else f"replicas x{world}" if world > 1
                                       else "1 GPU"),
                       "kernel": info["kernel_name"], "grid": info["grid"],
                       "cta_threads": info.get("threads"),
                       "l2": ("inputs larger than L2 (W %.0f MB)" % (info["w_bytes"] / 1e6))
                       if info["w_bytes"] > 126e6 else
                       "W on-chip/L2-resident by design (persistent kernel; one launch per run)"},
            "e2e": {"value": (1 if sharded else world) * n * steps / e2e_s, "unit": "osc-steps/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def spawn_ranks(gpus: int) -> int:
    """`python bench.py --gpus N` without torchrun: launch the N ranks (one
    process per GPU) through torch.distributed.run on this node, exactly as
    the driver's torchrun form would, and pass rank 0's JSON line through."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(gpus), "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="n1e4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rk4-steps", type=int, default=0, help="override RK4 steps per run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank, world, local_rank = env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload in ENSEMBLE_BATCH:
        run_ours_ensemble(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
