"""Small-grid workload for compute-sanitizer (memcheck / racecheck / synccheck): every
sweep kernel family once -- column tiles, row-warp (cp.async and TMA) at each line shape,
staged strided tiles (CN / AOS / MAOS), ADI / Euler, assembly, energy, DST vacuum, slab
partitions (dev tool; see profiles/sanitizer_r02.md)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.configs import synthetic_atoms

atoms = synthetic_atoms(12, 3.0, 41)
system = pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms], label="san")
p = pb.protein_problem(system, h=0.5, padding=4.0, kappa_bar=1.1283, eps_m=2.0, eps_s=80.0)
for v in pb.SCHEME_NAMES:
    dt = 2e-4 if v == "ExplicitEuler" else 0.5
    pb.march(p, pb.MarchConfig(dt=dt, T=2 * dt, variant=v))
pb.energy_pipeline(p, pb.MarchConfig(dt=0.5, T=1.0, variant="LODIE2"), "REplusV")
pb.energy_pipeline(p, pb.MarchConfig(dt=0.5, T=1.0, variant="LODIE2"), "Plain")
for n2 in (513, 257, 129, 97):  # row-warp line shapes, ragged line counts
    g = pb.make_grid((0, 0, 0), (0.25 * 4, 0.25 * 5, 0.25 * (n2 - 1)), 0.25)
    rng = np.random.default_rng(n2)
    b = rng.standard_normal(g.shape)
    region = pb.build_region_maps(g, pb.AnalyticSphere(0.6), 2.0, 80.0, 1.0)
    rho = np.zeros(g.shape)
    rho[1:-1, 1:-1, 1:-1] = rng.standard_normal(tuple(s - 2 for s in g.shape))
    q = pb.NPBProblem(grid=g, region=region, rho=pb.ScalarField(g, rho),
                      qfrac=pb.ScalarField.zeros(g), boundary=pb.BoundarySpec(g, b), alpha=1.0,
                      initial=pb.ScalarField(g, b.copy()))
    for v in ("LODIE2", "LODIE1", "AOSIE1", "LODCN2"):
        pb.march(q, pb.MarchConfig(dt=0.2, T=0.4, variant=v))
from paper_1410_2788_b200.slab import march_partitioned
march_partitioned(p, pb.MarchConfig(dt=0.5, T=1.0, variant="LODIE2"), 3)
print("sanitize workload done")
