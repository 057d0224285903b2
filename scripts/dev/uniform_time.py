"""Dev tool: per-kernel timing on the vacuum (uniform dielectric) version of a config, to
separate the cost of general (dielectric-crossing) segments from the uniform path."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200 import _native as nat
from paper_1410_2788_b200.configs import CONFIGS, synthetic_atoms, cubic_box, kappa_bar
from paper_1410_2788_b200.problem import assemble_on_grid, make_vacuum_problem

for key in sys.argv[1:] or ["c3"]:
    c = CONFIGS[key]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    g = pb.make_grid(lo, hi, c.h)
    p = assemble_on_grid(pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms]), g,
                         kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    for name, prob in (("protein", p), ("vacuum", make_vacuum_problem(p))):
        for v in ("LODIE1",):
            pb.march(prob, pb.MarchConfig(dt=c.dt, T=c.dt * 3, variant=v))
            lib = nat.lib(); lib.pbg_set_profiling(1)
            rep = pb.march(prob, pb.MarchConfig(dt=c.dt, T=c.dt * 10, variant=v))
            ms = (ctypes.c_double * 3)(); n = (ctypes.c_int64 * 3)(); lib.pbg_get_profile(ms, n)
            lib.pbg_set_profiling(0)
            print(key, name, v, "kernels us", [round(ms[a] / max(1, n[a]) * 1e3, 1) for a in range(3)])
