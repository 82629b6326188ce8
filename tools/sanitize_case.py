"""One small invocation of one kernel family, for compute-sanitizer (tools/sanitize.sh).

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
        python tools/sanitize_case.py CASE

Each case runs a few RK4 steps at a small size through the C ABI (so the
sanitizer sees exactly the product kernels) and checks the result against the
pinned oracle, printing "CASE ok" -- a sanitizer run is only meaningful if the
kernel also produced the right bits.  Knobs are set through the same
environment variables the tests use (STO_CLU_K, STO_CLU_HYB, STO_ENS_U, ...).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

FORCE = {"auto": 0, "single": 0x4 | 0x8, "resident": 0x2 | 0x8, "stream": 0x1 | 0x8,
         "reg": 0x10 | 0x8, "cluster": 0x40 | 0x8}

# name: (family, n, steps, stride, env)
CASES = {
    "tiny_n7": ("auto", 7, 6, 2, {}),
    "cluster_hyb_k2_n50": ("cluster", 50, 4, 2, {"STO_CLU_HYB": "1"}),
    "cluster_hyb_k8_n100": ("cluster", 100, 4, 2, {"STO_CLU_HYB": "1"}),
    "cluster_own_k8_n100": ("cluster", 100, 4, 2, {"STO_CLU_HYB": "0"}),
    "cluster_own_k16_n200": ("cluster", 200, 4, 2, {"STO_CLU_HYB": "0", "STO_CLU_K": "16"}),
    "cluster_hyb_k16_n200": ("cluster", 200, 4, 2, {"STO_CLU_HYB": "1", "STO_CLU_K": "16"}),
    "cluster_c64_n400": ("cluster", 400, 3, 1, {}),
    # the record-step stop path (divergence words on the mbarrier, no cluster barrier)
    "cluster_hyb_k8_n100_div": ("cluster", 100, 6, 1, {"STO_CLU_HYB": "1", "SAN_DIVERGE": "1"}),
    "cluster_own_k16_n200_div": ("cluster", 200, 6, 1, {"STO_CLU_HYB": "0", "STO_CLU_K": "16",
                                                        "SAN_DIVERGE": "1"}),
    "reg_single_n100": ("reg", 100, 4, 2, {}),
    "reg_grid_n700": ("reg", 700, 3, 1, {}),
    "single_n60": ("single", 60, 4, 2, {}),
    "resident_n1500": ("resident", 1500, 2, 1, {}),
    "stream_l2_n3000": ("stream", 3000, 2, 1, {}),
    "stream_chunked_n3000": ("stream", 3000, 2, 1, {"STO_CHUNK_COLS": "1024"}),
    "stream_hbm_n3600": ("stream", 3600, 2, 1, {}),
    "multi_w2_n600": ("multi2", 600, 3, 1, {}),
    "multi_w4_n1500_chunked": ("multi4", 1500, 2, 1, {"STO_CHUNK_COLS": "512"}),
    "ensemble_u1": ("ens", 200, 3, 1, {"STO_ENS_U": "1"}),
    "ensemble_u7": ("ens", 200, 3, 1, {"STO_ENS_U": "7"}),
    "ensemble_exact": ("ensx", 200, 3, 1, {}),
    "ensemble_exact_2launch": ("ensx", 100, 2, 1, {"STO_EX_CT_PER_LAUNCH": "1"}),
    "ensemble_exact_multitile": ("ensx", 600, 2, 1, {"STO_EX_U": "1"}),
    "derivative_k0": ("deriv", 900, 0, 0, {}),
    "tiny_n1_spec": ("auto", 1, 40, 10, {}),
    "device_build": ("build", 300, 0, 0, {}),
}


def main(name: str) -> None:
    fam, n, steps, stride, env = CASES[name]
    os.environ.update(env)
    import torch

    import paper_2312_01121_b200 as sto
    from oracle import oracle

    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0)
    np.fill_diagonal(w, 0.0)
    w_in = g.uniform(-1, 1, (n, 1))
    p = sto.PhysicalParams()
    consts = sto.kernel_scalars(p)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
    drive = g.uniform(-1, 1, (max(steps, 1), 1))
    m0 = sto.initial_state(n)

    if fam == "deriv":
        from paper_2312_01121_b200.backends.b200 import B200Backend

        m = g.standard_normal((n, 3))
        out = np.empty((n, 3))
        B200Backend(top, p).derivative(m, drive[0], out)
        want = oracle.derivative(w, w_in, consts, m, drive[0])
        assert np.array_equal(out.view(np.uint64), want.view(np.uint64))
    elif fam == "build":
        top_d = sto.build_topology_device(n, n_in=1, seed=3)
        top_h = sto.build_topology(n, n_in=1, seed=3)
        got = top_d.coupling.entries
        got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
        assert np.allclose(got, top_h.coupling.entries, rtol=1e-12, atol=0)
    elif fam in ("ens", "ensx"):
        currents = np.linspace(2.0e-3, 3.0e-3, 70)
        params = [sto.PhysicalParams(current=float(c)) for c in currents]
        cfg = sto.RunConfig(n=n, steps=steps, dt=1e-11, record_stride=stride)
        ens = sto.integrate_ensemble(top, params, cfg, exact=fam == "ensx")
        for b in (0, 33, 69):
            want, _ = oracle.integrate(w, w_in, sto.kernel_scalars(params[b]), m0, np.zeros((1, 1)),
                                       1, 1e-11, steps, stride)
            if fam == "ensx":
                assert np.array_equal(ens.states[:, b].view(np.uint64), want.view(np.uint64))
            else:
                assert np.abs(ens.states[:, b] - want).max() <= 1e-12
    elif fam.startswith("multi"):
        from paper_2312_01121_b200.sharding import integrate_logical

        world = int(fam[5:])
        m = m0.copy()
        got = integrate_logical(top, p, m, drive, 1, 1e-11, steps, stride, world, flags=0x1)
        want, _ = oracle.integrate(w, w_in, consts, m0, drive, 1, 1e-11, steps, stride)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    else:
        from paper_2312_01121_b200.backends.b200 import B200Backend

        be = B200Backend(top, p, device=0, flags=FORCE[fam])
        if os.environ.get("SAN_DIVERGE") == "1":  # a bad oscillator: every CTA must stop
            bad = m0.copy()
            bad[n // 2] = (1e200, 1e200, 1e200)
            try:
                oracle.integrate(w, w_in, consts, bad, drive, 1, 1e-11, steps, stride)
                raise AssertionError("oracle did not diverge")
            except oracle.OracleDiverged as e:
                want_div = (e.oscillator, e.step)
            try:
                be.integrate_run(bad, drive, 1, 1e-11, steps, stride)
                raise AssertionError("no divergence reported")
            except sto.IntegrationDivergedError as e:
                assert (e.oscillator, e.step) == want_div, ((e.oscillator, e.step), want_div)
        m = m0.copy()
        got = be.integrate_run(m, drive, 1, 1e-11, steps, stride)
        want, _ = oracle.integrate(w, w_in, consts, m0, drive, 1, 1e-11, steps, stride)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), be.plan_info
        print(name, be.plan_info)
    torch.cuda.synchronize()
    print(name, "ok", flush=True)


if __name__ == "__main__":
    if len(sys.argv) != 2 or sys.argv[1] not in CASES:
        print("cases:", " ".join(CASES))
        sys.exit(2)
    main(sys.argv[1])
