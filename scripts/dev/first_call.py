import sys, os, time
sys.path.insert(0, "/root/repo")
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.configs import CONFIGS, synthetic_atoms, cubic_box, kappa_bar
from paper_1410_2788_b200.problem import assemble_on_grid
import torch
c = CONFIGS["c2"]
atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
lo, hi = cubic_box(atoms, c.n, c.h)
g = pb.make_grid(lo, hi, c.h)
t0=time.perf_counter()
p = assemble_on_grid(pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms]), g, kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
torch.cuda.synchronize(); print("assembly", time.perf_counter()-t0)
for v in ["LODIE2", "LODIE2", "AOSIE1", "AOSIE1"]:
    t0=time.perf_counter()
    rep = pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 2, variant=v))
    print(v, "wall", time.perf_counter()-t0, "dev", rep.wall_time)
