"""Minimal profiling driver: assemble a config, march a few steps (dev tool for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.configs import CONFIGS, synthetic_atoms, cubic_box, kappa_bar
from paper_1410_2788_b200.problem import assemble_on_grid

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
variant = sys.argv[2] if len(sys.argv) > 2 else "LODIE2"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = CONFIGS[key]
atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
lo, hi = cubic_box(atoms, c.n, c.h)
g = pb.make_grid(lo, hi, c.h)
p = assemble_on_grid(pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms]), g,
                     kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
rep = pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * steps, variant=variant))
print("steps", rep.steps_taken, "ms/step", rep.wall_time / rep.steps_taken * 1e3)
