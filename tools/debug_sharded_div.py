"""Debug: sharded divergence across processes (torchrun, one GPU, gloo)."""
import os, sys, traceback
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_01121_b200 as sto
from paper_2312_01121_b200.sharding import ShardedB200Backend, RUN_OK

def main():
    n = int(sys.argv[1]); steps = int(sys.argv[2]); badrow = int(sys.argv[3])
    dist.init_process_group("gloo"); torch.cuda.set_device(0)
    r = dist.get_rank()
    g = np.random.default_rng(n)
    w = g.uniform(-1, 1, (n, n)) / np.sqrt(n / 3.0); np.fill_diagonal(w, 0.0)
    top = sto.Topology(sto.CouplingMatrix(w), sto.InputWeights(g.uniform(-1, 1, (n, 1))))
    be = ShardedB200Backend(top, sto.PhysicalParams(), device=0)
    print(r, "kernel", be._plan.info, flush=True)
    for trial in range(2):
        bad = sto.initial_state(n)
        if badrow >= 0: bad[badrow, 1] = np.nan
        # raw launch to see each rank's own status
        dev = torch.device("cuda", 0)
        m_d = torch.as_tensor(bad).to(dev); s_d = torch.zeros((1, 1), dtype=torch.float64, device=dev)
        st = torch.zeros((steps + 2, n, 3), dtype=torch.float64, device=dev)
        dist.barrier()
        try:
            s = be._plan.integrate_dev(m_d, s_d, 1, 1e-11, steps, 1, st, sync=True)
            print(r, trial, "OK", s.diverged, s.oscillator, s.step, flush=True)
        except Exception as e:
            print(r, trial, "EXC", type(e).__name__, e, flush=True)
    dist.barrier(); be.close(); dist.destroy_process_group()

main()
