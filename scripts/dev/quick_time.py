"""Quick device timing of the step and of each sweep kernel at config sizes (dev tool)."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200 import _native as nat
from paper_1410_2788_b200.configs import CONFIGS, synthetic_atoms, cubic_box, kappa_bar
from paper_1410_2788_b200.problem import assemble_on_grid

variants = os.environ.get("VARIANTS", "LODIE2,LODIE1,AOSIE1,LODCN2").split(",")
for key in sys.argv[1:] or ["c3"]:
    c = CONFIGS[key]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    g = pb.make_grid(lo, hi, c.h)
    t0 = time.perf_counter()
    system = pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms])
    p = assemble_on_grid(system, g, kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    import torch; torch.cuda.synchronize()
    t1 = time.perf_counter()
    nint = (c.n - 2) ** 3
    for v in variants:
        pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 3, variant=v))
        rep = pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 20, variant=v))
        per = rep.wall_time / rep.steps_taken
        lib = nat.lib(); lib.pbg_set_profiling(1)
        pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 10, variant=v))
        ms = (ctypes.c_double * 3)(); n = (ctypes.c_int64 * 3)(); lib.pbg_get_profile(ms, n)
        lib.pbg_set_profiling(0)
        ks = [ms[a] / max(1, n[a]) * 1e3 for a in range(3)]
        B = 48 if v.startswith("LOD") else 64
        print(f"{key} n={c.n} {v}: {per*1e6:.1f} us/step  {nint/per/1e9:.2f} Gupd/s  "
              f"{B*nint/per/1e9:.0f} GB/s | kernels us {ks[0]:.0f} {ks[1]:.0f} {ks[2]:.0f} "
              f"(16B/node: {16*nint/ks[0]/1e3:.0f} {16*nint/ks[1]/1e3:.0f} {16*nint/ks[2]/1e3:.0f} GB/s)"
              f"  (assembly {t1-t0:.2f}s)", flush=True)
