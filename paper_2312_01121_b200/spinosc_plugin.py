"""Plug the B200 path into the reference package `spinosc` itself.

`register()` does, at run time, what INTEGRATION.md §2 asks a `spinosc`
maintainer to do in source:

1. registers the B200 backend under the reference's own id ``"gpu"`` in
   `spinosc.backends` (replacing the torch `TorchBackend`, which the
   registry allows, `backends/__init__.py:43-54`), with the same factory
   signature `factory(topology, params, workers=, gpu_device=)`; the object
   it returns keeps the plugin contract `derivative(m, u, out)` (one K0
   launch) and adds `integrate_run`;
2. installs the whole-run hook: `spinosc.integrator.integrate` (and the
   names `spinosc`, `spinosc.cli` and `spinosc.bench` bound to it at import,
   including `time_integration`'s default `runner`) is wrapped so that a
   backend with `integrate_run` executes the whole time loop in one
   persistent launch.  Everything else -- validation of arguments, the
   recording grid `record_at * dt`, the drift definition, the returned
   `spinosc.integrator.Trajectory`, `IntegrationDivergedError(oscillator,
   step)` -- follows `integrator.py:131-187`; backends without
   `integrate_run` go through the untouched original.

After `register()`, the reference's own tooling sees the B200 backend:
``spinosc validate`` checks it against the numpy reference at the
reference's gpu tolerance (`cli.py:232`: it is in fact bit-identical),
``spinosc bench`` puts it in the speedup table, ``spinosc scaling`` times
its derivative.  `python -m paper_2312_01121_b200.spinosc_plugin <args>`
runs the reference CLI with the backend registered.
"""

from __future__ import annotations

import sys
import time

import numpy as np

KIND = "B200 persistent RK4 (sm_100a)"
REQUIRES = "paper_2312_01121_b200 + sm_100 GPU"


def _probe() -> bool:  # the registry's probe must never raise
    try:
        from .backends.b200 import is_available

        return bool(is_available())
    except Exception:
        return False


def _factory(topology, params, workers=None, gpu_device=None):
    from .backends.b200 import B200Backend

    return B200Backend(topology, params, device=gpu_device)


def _whole_run_integrate(original):
    """`spinosc.integrator.integrate` with the INTEGRATION.md §2 hook."""
    import spinosc.integrator as ref

    def integrate(topology, params, config, backend=None):
        if topology.n != config.n:  # the reference's checks come first (integrator.py:139-150)
            return original(topology, params, config, backend=backend)
        if backend is None:
            from spinosc.backends import create_backend

            backend = create_backend(config.backend, topology, params, workers=config.workers,
                                     gpu_device=config.gpu_device)
        if not hasattr(backend, "integrate_run"):
            return original(topology, params, config, backend=backend)
        if getattr(backend, "n", config.n) != config.n:
            raise ref.ParameterError(
                f"backend is for {backend.n} oscillators, config.n is {config.n}")
        series = config.input_series
        if series is None:
            series = ref.InputSeries.zeros(topology.n_in)
        if series.n_in != topology.n_in:
            raise ref.ParameterError(
                f"input series has {series.n_in} channels, topology expects {topology.n_in}")
        series.check_steps(config.steps)
        m = ref.initial_state(config.n, config.phi0)
        record_at = ref._recorded_steps(config.steps, config.record_stride)
        start = time.perf_counter()
        try:
            states = backend.integrate_run(m, np.asarray(series.samples, dtype=np.float64),
                                           series.steps_per_sample, config.dt, config.steps,
                                           config.record_stride)
        except Exception as exc:  # map our divergence error onto the reference's class
            if type(exc).__name__ == "IntegrationDivergedError":
                raise ref.IntegrationDivergedError(oscillator=exc.oscillator,
                                                   step=exc.step) from None
            raise
        elapsed = time.perf_counter() - start
        norms = np.linalg.norm(states, axis=2)
        return ref.Trajectory(times=record_at * config.dt, states=states,
                              max_norm_drift=float(np.abs(norms - 1.0).max()), config=config,
                              elapsed_seconds=elapsed)

    integrate.__wrapped__ = original
    integrate.__doc__ = original.__doc__
    return integrate


def register(hook_integrate: bool = True) -> None:
    """Register the B200 backend as spinosc's "gpu" and install the whole-run hook.
    Idempotent."""
    import spinosc
    import spinosc.backends as backends
    import spinosc.integrator as integrator

    backends.register_backend("gpu", kind=KIND, requires=REQUIRES, probe=_probe,
                              factory=_factory)
    if not hook_integrate or getattr(integrator.integrate, "__wrapped__", None) is not None:
        return
    original = integrator.integrate
    hooked = _whole_run_integrate(original)
    integrator.integrate = hooked
    for modname in ("spinosc", "spinosc.cli", "spinosc.bench"):
        mod = sys.modules.get(modname)
        if mod is None:
            try:
                __import__(modname)
                mod = sys.modules[modname]
            except ImportError:
                continue
        if getattr(mod, "integrate", None) is original:
            mod.integrate = hooked
    bench = sys.modules.get("spinosc.bench")
    ti = getattr(bench, "time_integration", None)
    if ti is not None and ti.__defaults__:
        ti.__defaults__ = tuple(hooked if d is original else d for d in ti.__defaults__)
    del spinosc


def main(argv=None) -> int:
    """The reference CLI (`spinosc.cli.main`) with the B200 backend registered."""
    register()
    from spinosc.cli import main as cli_main

    return cli_main(argv)


if __name__ == "__main__":
    sys.exit(main())
