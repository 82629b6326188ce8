"""Ad-hoc parity probe: derivative / matvec / 1-step integrate at one size."""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.backends.b200 import B200Backend
from oracle import oracle

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = np.random.default_rng(0)
w = g.uniform(-1, 1, (n, n)); np.fill_diagonal(w, 0.0)
w_in = g.uniform(-1, 1, (n, 1))
m = g.standard_normal((n, 3)); m /= np.linalg.norm(m, axis=1, keepdims=True)
u = np.array([0.3])
consts = sto.kernel_scalars(sto.PhysicalParams())
top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(w_in))
want_cp = np.array([oracle.tree_sum(w[k] * m[:, 0]) for k in range(n)])
got_cp = sto.tree_matvec(w, m[:, 0].copy())
print("matvec bad:", int((got_cp != want_cp).sum()), np.abs(got_cp - want_cp).max())
want_d = oracle.derivative(w, w_in, consts, m, u)
for flags, name in [(0, 'auto'), (1 | 8, 'stream'), (2 | 8, 'resident'), (4 | 8, 'single')]:
    try:
        be = B200Backend(top, None, device=0, flags=flags, consts=consts)
    except Exception as e:
        print(name, 'skip', e); continue
    out = np.empty((n, 3)); be.derivative(m, u, out)
    print(name, be.plan_info['kernel_name'], "deriv bad:", int((out != want_d).sum()))
    for steps in (1, 2, 5):
        want, _ = oracle.integrate(w, w_in, consts, sto.initial_state(n), np.array([[0.3]]), 1, 1e-11, steps, 1)
        mm = sto.initial_state(n)
        st = be.integrate_run(mm, np.array([[0.3]]), 1, 1e-11, steps, 1)
        bad = (st != want)
        print(f"  steps={steps} bad={int(bad.sum())} maxdiff={np.abs(st-want).max():.3e} first bad rec/row:",
              np.argwhere(bad)[:3].tolist())
