"""Dev tool: aggregate throughput of 1 vs 2 concurrent c3 marches (latency-hiding headroom)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.batch import march_many
from paper_1410_2788_b200.configs import CONFIGS, synthetic_atoms, cubic_box, kappa_bar
from paper_1410_2788_b200.problem import assemble_on_grid
from paper_1410_2788_b200.schemes import device_problem
key = sys.argv[1] if len(sys.argv) > 1 else "c3"
c = CONFIGS[key]
atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
lo, hi = cubic_box(atoms, c.n, c.h)
probs = []
for _ in range(2):
    p = assemble_on_grid(pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms]),
                         pb.make_grid(lo, hi, c.h), kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    device_problem(p)
    probs.append(p)
torch.cuda.synchronize()
n = 50
nint = (c.n - 2) ** 3
for k in (1, 2):
    jobs = [((i,), probs[i], pb.MarchConfig(dt=c.dt, T=c.dt * n, variant="LODIE2")) for i in range(k)]
    march_many(jobs, streams=k); torch.cuda.synchronize()
    t0 = time.perf_counter(); march_many(jobs, streams=k); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(key, "concurrent marches", k, f"{k*n*nint/dt/1e9:.1f} Gupd/s aggregate")
