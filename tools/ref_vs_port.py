"""The reference's own CPU engines (spinosc, installed offline in baseline/_ref)
beside the C restatement bench.py uses as its CPU baseline (oracle/, kind
"port"), on the same host, the same W and the same horizon.

Protocol of the reference's `time_integration` (bench.py:171-206): backend
constructed once, one untimed warm-up, 3 timed runs, mean of
`Trajectory.elapsed_seconds`.  The port is timed the same way (wall clock of
oracle.integrate, all host threads and 1 thread).  Prints one JSON line per
(N, engine) and checks that the port's final state equals the reference's bit
for bit.  Usage: python tools/ref_vs_port.py [N ...]
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_sto")

import spinosc  # noqa: E402
import paper_2312_01121_b200 as sto  # noqa: E402
from oracle import oracle  # noqa: E402

HORIZON = {100: 1000, 1000: 100, 10000: 4}
REPS = 3


def main():
    ns = [int(a) for a in sys.argv[1:]] or [100, 1000, 10000]
    cores = os.cpu_count() or 1
    oracle.build()
    for n in ns:
        steps = HORIZON.get(n, max(2, int(4e8 / (n * n))))
        top = sto.build_topology(n, seed=0)
        w = top.coupling.entries
        w_in = top.input_weights.entries
        rtop = spinosc.Topology(spinosc.CouplingMatrix(w), spinosc.InputWeights(w_in))
        params = spinosc.PhysicalParams()
        want = None
        engines = ["fused", "parallel"] + (["reference"] if n <= 1000 else [])
        for eng in engines:
            cfg = spinosc.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=steps, backend=eng)
            be = spinosc.create_backend(eng, rtop, params)
            spinosc.integrate(rtop, params, cfg, backend=be)  # warm-up (JIT compile)
            ts, traj = [], None
            for _ in range(REPS):
                traj = spinosc.integrate(rtop, params, cfg, backend=be)
                ts.append(traj.elapsed_seconds)
            want = traj.states[-1] if want is None else want
            t = statistics.fmean(ts)
            print(json.dumps({"n": n, "steps": steps, "engine": f"spinosc {eng}",
                              "threads": cores if eng == "parallel" else 1,
                              "mean_s": t, "std_s": statistics.pstdev(ts),
                              "osc_steps_per_s": n * steps / t}), flush=True)
        consts = sto.kernel_scalars(sto.PhysicalParams())
        for threads in (cores, 1):
            if threads == 1 and n > 2000:
                continue
            m0 = sto.initial_state(n)
            args = (w, w_in, consts, m0, np.zeros((1, 1)), 1, 1e-11, steps, steps)
            oracle.integrate(*args, threads=threads)
            ts = []
            for _ in range(REPS):
                t0 = time.perf_counter()
                got, _ = oracle.integrate(*args, threads=threads)
                ts.append(time.perf_counter() - t0)
            t = statistics.fmean(ts)
            print(json.dumps({"n": n, "steps": steps, "engine": "C port (oracle/, bench cpu_baseline)",
                              "threads": threads, "mean_s": t, "std_s": statistics.pstdev(ts),
                              "osc_steps_per_s": n * steps / t,
                              "bit_equal_to_reference": bool(np.array_equal(
                                  got[-1].view(np.uint64), want.view(np.uint64)))}), flush=True)


if __name__ == "__main__":
    main()
