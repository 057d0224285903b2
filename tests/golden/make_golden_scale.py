"""Golden fixtures at the MEASURED scales (configs 3, 4 and 5), from the REAL reference.

Run in the build container (the reference is importable there, not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden_scale.py c3 c4 c5

Recipe: the cubic-box grid of configs.py, the region maps from the oracle's
bbox-culled classification (bit-identical to `build_region_maps`, checked again below on a
config-5 protein against the reference's own `build_region_maps`), everything else from the
reference's public API -- `deposit_charges`, `BoundarySpec.from_function` +
`coulomb_screened_values`, `NPBProblem`, `march` (schemes.py:399-425) and
`energy_pipeline` (energy.py:109-164).  Only compact summaries are committed: hashes of the
assembled maps, mid-planes, a seeded node sample, field statistics, dG and the reference's
own `MarchReport.wall_time`.

Outputs: scale_c3.npz, scale_c4.npz, scale_c5.npz next to this script.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

import pbsplit as pb  # noqa: E402
from pbsplit.problem import coulomb_screened_values  # noqa: E402
from pbsplit.schemes import MarchConfig, march  # noqa: E402

from oracle import pbs_oracle as O  # noqa: E402
from tests.golden.scale_common import (SAMPLE_SEED, SAMPLE_N, mask_digest, sample_index,  # noqa: E402
                                       field_stats, load_configs)

C = load_configs()


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


def save(name, **kw):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **kw)
    log(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def system_of(atoms, label):
    return pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms], label=label)


def reference_problem(atoms, n, h, eps_m, eps_s, kbar, label):
    """NPBProblem on the cubic box: culled oracle masks + reference deposit/faces."""
    lo, hi = C.cubic_box(atoms, n, h)
    grid = pb.make_grid(lo, hi, h)
    og = O.OGrid(grid.lo, grid.h, grid.shape)
    masks = [O.union_of_spheres_mask(og, atoms, 0.0, ha) for ha in (None, 0, 1, 2)]
    node, hx, hy, hz = masks
    eps_node = np.where(node, eps_m, eps_s)
    kappa2 = np.where(eps_node == eps_m, 0.0, kbar ** 2)  # geometry.py:148
    region = pb.RegionMap(grid=grid, eps_node=pb.ScalarField(grid, eps_node),
                          eps_half_x=np.where(hx, eps_m, eps_s),
                          eps_half_y=np.where(hy, eps_m, eps_s),
                          eps_half_z=np.where(hz, eps_m, eps_s),
                          kappa2=pb.ScalarField(grid, kappa2))
    system = system_of(atoms, label)
    qfrac, rho = pb.deposit_charges(system, grid)
    boundary = pb.BoundarySpec.from_function(
        grid, lambda pts: coulomb_screened_values(pts, system, eps_s, kbar))
    initial = np.zeros(grid.shape)
    boundary.apply(initial)
    prob = pb.NPBProblem(grid=grid, region=region, rho=rho, qfrac=qfrac, boundary=boundary,
                         alpha=1.0, initial=pb.ScalarField(grid, initial), eps_m=eps_m,
                         eps_s=eps_s, kappa_bar=kbar, system=system, label=label)
    asm = dict(lo=np.array(grid.lo), h=grid.h, shape=np.array(grid.shape),
               dig_node=mask_digest(node), dig_hx=mask_digest(hx), dig_hy=mask_digest(hy),
               dig_hz=mask_digest(hz), n_node=int(node.sum()), n_hx=int(hx.sum()),
               n_hy=int(hy.sum()), n_hz=int(hz.sum()),
               dig_qfrac=hashlib.sha256(qfrac.data.tobytes()).hexdigest(),
               dig_rho=hashlib.sha256(rho.data.tobytes()).hexdigest(),
               faces_stats=field_stats(boundary.values))
    return prob, asm


def summarize(prefix, u, out):
    out[prefix + "_stats"] = field_stats(u)
    out[prefix + "_plane"] = u[u.shape[0] // 2]
    out[prefix + "_sample"] = u.ravel()[sample_index(u.shape)]


def case_c3():
    """Config 3: REplusV energy pipeline (4 marches) at 257^3, T = 50 (100 + 200 steps)."""
    c = C.CONFIGS["c3"]
    atoms = C.synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    kbar = C.kappa_bar(c.ionic_strength)
    t0 = time.time()
    prob, asm = reference_problem(atoms, c.n, c.h, c.eps_m, c.eps_s, kbar, "c3")
    log("c3 assembled", time.time() - t0)
    T = 50.0
    res = pb.energy_pipeline(prob, MarchConfig(dt=c.dt, T=T, variant=c.variant), "REplusV")
    log("c3 energy", res.delta_g, res.wall_time)
    out = dict(asm, T=T, dt=c.dt, delta_g=res.delta_g, wall_time=res.wall_time,
               diverged=res.diverged)
    summarize("phim", res.phi_m.data, out)
    summarize("phi0", res.phi_0.data, out)
    save("scale_c3", **out)


def case_c4():
    """Config 4: 513^3, 10,000 atoms, LODIE2 dt 0.5, 50 steps."""
    c = C.CONFIGS["c4"]
    atoms = C.synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    kbar = C.kappa_bar(c.ionic_strength)
    t0 = time.time()
    prob, asm = reference_problem(atoms, c.n, c.h, c.eps_m, c.eps_s, kbar, "c4")
    log("c4 assembled", time.time() - t0)
    rep = march(prob, MarchConfig(dt=c.dt, T=c.dt * c.steps, variant=c.variant))
    log("c4 march", rep.steps_taken, rep.wall_time)
    out = dict(asm, dt=c.dt, steps=rep.steps_taken, wall_time=rep.wall_time,
               diverged=rep.diverged)
    summarize("u", rep.final.data, out)
    save("scale_c4", **out)


def _c5_worker(idx):
    sizes = C.batch_sizes()
    cfg = C.batch_config(idx, sizes[idx])
    atoms = C.synthetic_atoms(cfg.n_atoms, cfg.ball_radius, cfg.seed)
    kbar = C.kappa_bar(cfg.ionic_strength)
    prob, asm = reference_problem(atoms, cfg.n, cfg.h, cfg.eps_m, cfg.eps_s, kbar, f"c5-{idx}")
    res = {"asm": asm}
    for v in ("AOSIE1", "LODIE2"):
        rep = march(prob, MarchConfig(dt=cfg.dt, T=cfg.dt * cfg.steps, variant=v))
        u = rep.final.data
        res[v] = (field_stats(u), u.ravel()[sample_index(u.shape)], rep.wall_time,
                  rep.steps_taken)
    if idx == 0:  # the culled classification against the reference's own classifier
        region = pb.build_region_maps(prob.grid, pb.UnionOfSpheres(prob.system, 0.0),
                                      cfg.eps_m, cfg.eps_s, kbar ** 2)
        assert np.array_equal(region.eps_node.data, prob.region.eps_node.data)
        for a in range(3):
            assert np.array_equal(region.eps_half(a), prob.region.eps_half(a))
        res["culled_checked"] = True
    return idx, res


def case_c5(workers=6):
    """Config 5: all 64 proteins x {AOSIE1, LODIE2}, 100 steps at dt 0.5 on 97^3."""
    from multiprocessing import Pool

    count = 64
    with Pool(workers) as pool:
        results = dict(pool.imap_unordered(_c5_worker, range(count)))
    assert results[0].get("culled_checked")
    out = dict(count=count, sizes=np.array(C.batch_sizes()))
    for v in ("AOSIE1", "LODIE2"):
        out[v + "_stats"] = np.array([results[i][v][0] for i in range(count)])
        out[v + "_sample"] = np.array([results[i][v][1] for i in range(count)])
        out[v + "_wall"] = np.array([results[i][v][2] for i in range(count)])
        out[v + "_steps"] = np.array([results[i][v][3] for i in range(count)])
    for key in ("dig_node", "dig_hx", "dig_hy", "dig_hz", "dig_qfrac", "dig_rho"):
        out[key] = np.array([results[i]["asm"][key] for i in range(count)])
    out["faces_stats"] = np.array([results[i]["asm"]["faces_stats"] for i in range(count)])
    save("scale_c5", **out)


if __name__ == "__main__":
    cases = {"c3": case_c3, "c4": case_c4, "c5": case_c5}
    for name in sys.argv[1:] or list(cases):
        cases[name]()
