"""Generate the golden fixtures by running the REAL reference (`pbsplit`).

Run in the build container, where the read-only reference is importable:

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py

It writes small `.npz` files next to this script.  The GPU box has no /root/reference, so
the fixtures are committed; `tests/test_oracle_golden.py` pins the CPU oracle against them
and the GPU tests compare the device path against both.  Inputs are seeded and regenerated
from the parameters stored in each file.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

import pbsplit as pb  # noqa: E402
from pbsplit.schemes import MarchConfig, march, step  # noqa: E402

from paper_1410_2788_b200.configs import KIRKWOOD, synthetic_atoms  # noqa: E402

VARIANTS = ["LODIE1", "LODIE2", "LODCN1", "LODCN2", "AOSIE1", "AOSIE2", "AOSCN1", "AOSCN2",
            "MAOSIE", "MAOSCN"]


def system_of(atoms, label="golden"):
    return pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms], label=label)


def faces(arr):
    """Pack the six faces (x-lo, x-hi, y-lo, y-hi, z-lo, z-hi)."""
    return np.concatenate([arr[0].ravel(), arr[-1].ravel(), arr[:, 0].ravel(),
                           arr[:, -1].ravel(), arr[:, :, 0].ravel(), arr[:, :, -1].ravel()])


def grid_meta(g):
    return dict(lo=np.array(g.lo), hi=np.array(g.hi), h=g.h, shape=np.array(g.shape))


def save(name, **kw):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def assembly_case(tag, n_atoms, radius, seed, h, padding, probe, kbar):
    atoms = synthetic_atoms(n_atoms, radius, seed)
    prob = pb.protein_problem(system_of(atoms), h=h, padding=padding, kappa_bar=kbar,
                              eps_m=2.0, eps_s=80.0, probe_inflation=probe)
    r = prob.region
    save(f"assembly_{tag}", atoms=np.array(atoms), probe=probe, kappa_bar=kbar, padding=padding,
         eps_m=2.0, eps_s=80.0, **grid_meta(prob.grid),
         node_solute=r.eps_node.data == 2.0, hx=r.eps_half_x == 2.0, hy=r.eps_half_y == 2.0,
         hz=r.eps_half_z == 2.0, kappa2=r.kappa2.data, qfrac=prob.qfrac.data,
         rho=prob.rho.data, faces=faces(prob.boundary.values))
    return atoms, prob


def march_cases():
    atoms = synthetic_atoms(8, 2.5, 21)
    prob = pb.protein_problem(system_of(atoms), h=0.5, padding=3.0, kappa_bar=1.0,
                              eps_m=2.0, eps_s=80.0)
    out = dict(atoms=np.array(atoms), padding=3.0, kappa_bar=1.0, eps_m=2.0, eps_s=80.0,
               dt=0.3, T=1.5, **grid_meta(prob.grid))
    for v in VARIANTS:
        rep = march(prob, MarchConfig(dt=0.3, T=1.5, variant=v))
        out[v] = rep.final.data
    for v in ("AOSIE1", "AOSCN2"):
        rep = march(prob, MarchConfig(dt=0.3, T=1.5, variant=v, aos_nonlinear="literal"))
        out[v + "_literal"] = rep.final.data
    # alpha override and a diverging run (threshold forces a stop at the first bad step)
    rep = march(prob, MarchConfig(dt=0.3, T=1.5, variant="LODIE2", alpha=0.5))
    out["LODIE2_alpha05"] = rep.final.data
    rep = march(prob, MarchConfig(dt=0.3, T=3.0, variant="LODIE1", divergence_threshold=2.0e3))
    out["div_final"] = rep.final.data
    out["div_steps"] = rep.steps_taken
    out["div_step"] = -1 if rep.diverged_step is None else rep.diverged_step
    save("march_variants", **out)


def kirkwood_case():
    sysk = pb.MolecularSystem([pb.Atom((0.0, 0.0, 0.0), 1.0, 2.0)], label="kirkwood")
    kw = KIRKWOOD
    prob = pb.protein_problem(sysk, h=kw["h"], padding=kw["padding"], kappa_bar=kw["kappa_bar"],
                              eps_m=kw["eps_m"], eps_s=kw["eps_s"])
    out = dict(**grid_meta(prob.grid))
    for v in ("LODIE1", "LODIE2"):
        rep = march(prob, MarchConfig(dt=kw["dt"], T=kw["T"], variant=v))
        u = rep.final.data
        out[v + "_plane"] = u[u.shape[0] // 2]
        out[v + "_stats"] = np.array([np.max(np.abs(u)), np.sum(u), np.sum(u * u)])
        out[v + "_wall"] = rep.wall_time
    res = pb.energy_pipeline(prob, MarchConfig(dt=kw["dt"], T=kw["T"], variant="LODIE2"),
                             "REplusV")
    out["dg_replusv_lodie2"] = res.delta_g
    out["phim_plane"] = res.phi_m.data[32]
    out["phi0_plane"] = res.phi_0.data[32]
    save("kirkwood", **out)


def small_api_cases():
    out = {}
    # sweeps on a heterogeneous sphere-cut grid (the shape of test_schemes.small_setup)
    g = pb.make_grid((0, 0, 0), (2, 2, 2), 0.5)
    region = pb.build_region_maps(g, pb.AnalyticSphere(0.8), 1.0, 80.0, 1.0)
    rng = np.random.default_rng(77)
    bvals = rng.standard_normal(g.shape)
    b = pb.BoundarySpec(g, bvals)
    rhs = rng.standard_normal(g.shape)
    out["sweep_bvals"] = bvals
    out["sweep_rhs"] = rhs
    for axis in range(3):
        out[f"ie_{axis}"] = pb.ie_sweep(axis, pb.ScalarField(g, rhs), 3.0, 0.21, 1.7, region,
                                        b).data
        out[f"cn_{axis}"] = pb.cn_sweep(axis, pb.ScalarField(g, rhs), 4.0, 0.15, 0.8, region,
                                        b).data
    # larger sweep (lines longer than one warp segment) on a 2-valued union region
    atoms = synthetic_atoms(30, 5.0, 31)
    prob = pb.protein_problem(system_of(atoms), h=0.5, padding=3.0, kappa_bar=1.0, eps_m=2.0,
                              eps_s=80.0)
    gg = prob.grid
    rhs2 = np.random.default_rng(78).standard_normal(gg.shape)  # regenerated by the tests
    out["big_atoms"] = np.array(atoms)
    out["big_lo"] = np.array(gg.lo)
    out["big_hi"] = np.array(gg.hi)
    out["big_shape"] = np.array(gg.shape)
    for axis in range(3):
        out[f"big_ie_{axis}"] = pb.ie_sweep(axis, pb.ScalarField(gg, rhs2), 1.0, 0.5, 1.0,
                                            prob.region, prob.boundary).data
        out[f"big_cn_{axis}"] = pb.cn_sweep(axis, pb.ScalarField(gg, rhs2), 1.0, 0.5, 1.0,
                                            prob.region, prob.boundary).data
    # nonlinear flow with per-element kappa2
    w = rng.uniform(-60, 60, 500)
    w[:4] = [-5000.0, -750.0, 750.0, 5000.0]
    k2 = np.where(rng.uniform(size=500) < 0.3, 0.0, rng.uniform(0.05, 4.0, 500))
    out["flow_w"] = w
    out["flow_k2"] = k2
    out["flow_out"] = pb.nonlinear_step(w, k2, 0.37, 1.3)
    out["flow_out_pm4"] = pb.nonlinear_step(w, k2, 0.37, 1.3, premultiplier=4.0)
    out["flow_out_rate4"] = pb.nonlinear_step(w, k2, 0.37, 1.3, rate=4.0)
    # single step() with an AOS axis-order permutation
    g3 = pb.make_grid((0, 0, 0), (2, 2, 2), 0.25)
    reg3 = pb.build_region_maps(g3, pb.AnalyticSphere(1.1), 1.0, 80.0, 1.0)
    b3 = rng.standard_normal(g3.shape)
    s3 = rng.standard_normal(g3.shape)
    rho3 = np.zeros(g3.shape)
    rho3[1:-1, 1:-1, 1:-1] = rng.standard_normal((7, 7, 7))
    p3 = pb.NPBProblem(grid=g3, region=reg3, rho=pb.ScalarField(g3, rho3),
                       qfrac=pb.ScalarField.zeros(g3), boundary=pb.BoundarySpec(g3, b3),
                       alpha=1.0, initial=pb.ScalarField(g3, s3), eps_m=1.0, eps_s=80.0,
                       kappa_bar=1.0, label="perm")
    out["step_b"] = b3
    out["step_s"] = s3
    out["step_rho"] = rho3
    for v in VARIANTS:
        out[f"step_{v}"] = step(v, pb.ScalarField(g3, s3), p3, dt=0.2).data
    save("small_api", **out)


def sphere_case():
    g = pb.default_sphere_grid(0.5)
    prob = pb.sphere_benchmark(g, H=1.0)
    out = dict(h=0.5)
    for v in ("LODIE1", "AOSCN2", "MAOSIE"):
        rep = march(prob, MarchConfig(dt=0.0125, T=1.0, variant=v))
        out[v] = rep.final.data
    out["rho"] = prob.rho.data
    out["initial"] = prob.initial.data
    out["bvals"] = prob.boundary.values
    save("sphere", **out)


def energy_case():
    atoms = synthetic_atoms(12, 3.0, 41)
    prob = pb.protein_problem(system_of(atoms), h=0.5, padding=4.0, kappa_bar=1.1283,
                              eps_m=2.0, eps_s=80.0)
    out = dict(atoms=np.array(atoms), padding=4.0, kappa_bar=1.1283, eps_m=2.0, eps_s=80.0,
               **grid_meta(prob.grid))
    for v in ("LODIE2", "AOSIE1"):
        res = pb.energy_pipeline(prob, MarchConfig(dt=0.5, T=5.0, variant=v), "REplusV")
        out[f"dg_{v}"] = res.delta_g
        out[f"phim_{v}"] = res.phi_m.data
        out[f"phi0_{v}"] = res.phi_0.data
    save("energy", **out)


def vacuum_case():
    """DST-I vacuum solver and the Plain / RE energies (energy.py:46-85, 109-164)."""
    from pbsplit.energy import vacuum_potential_fast
    from pbsplit.problem import make_vacuum_problem

    atoms = synthetic_atoms(12, 3.0, 41)  # the energy_case problem
    prob = pb.protein_problem(system_of(atoms), h=0.5, padding=4.0, kappa_bar=1.1283,
                              eps_m=2.0, eps_s=80.0)
    vac = make_vacuum_problem(prob)
    out = dict(atoms=np.array(atoms), padding=4.0, kappa_bar=1.1283, eps_m=2.0, eps_s=80.0,
               **grid_meta(prob.grid))
    out["phi0_fast"] = vacuum_potential_fast(prob.rho, prob.grid, prob.eps_m,
                                             vac.boundary).data
    for v in ("LODIE2", "AOSIE1"):
        for ev in ("Plain", "RE"):
            res = pb.energy_pipeline(prob, MarchConfig(dt=0.5, T=5.0, variant=v), ev)
            out[f"dg_{ev}_{v}"] = res.delta_g
    # Kirkwood sphere (config 1): Plain energy with the direct vacuum solve
    sysk = pb.MolecularSystem([pb.Atom((0.0, 0.0, 0.0), 1.0, 2.0)], label="kirkwood")
    kw = KIRKWOOD
    pk = pb.protein_problem(sysk, h=kw["h"], padding=kw["padding"], kappa_bar=kw["kappa_bar"],
                            eps_m=kw["eps_m"], eps_s=kw["eps_s"])
    res = pb.energy_pipeline(pk, MarchConfig(dt=kw["dt"], T=kw["T"], variant="LODIE2"), "Plain")
    out["dg_kirkwood_plain"] = res.delta_g
    out["kirkwood_phi0_plane"] = res.phi_0.data[res.phi_0.data.shape[0] // 2]
    save("vacuum", **out)


def comparison_cases():
    """ADI1 / ADI2 / ExplicitEuler (schemes.py:240-253, 331-363) on the march_variants
    problem: ADI at the splitting step size, Euler at a stable step, plus an Euler run that
    diverges (threshold stop)."""
    atoms = synthetic_atoms(8, 2.5, 21)
    prob = pb.protein_problem(system_of(atoms), h=0.5, padding=3.0, kappa_bar=1.0,
                              eps_m=2.0, eps_s=80.0)
    out = dict(atoms=np.array(atoms), padding=3.0, kappa_bar=1.0, eps_m=2.0, eps_s=80.0,
               **grid_meta(prob.grid))
    for v in ("ADI1", "ADI2"):
        rep = march(prob, MarchConfig(dt=0.3, T=1.5, variant=v))
        out[v] = rep.final.data
        out[v + "_steps"] = rep.steps_taken
    rep = march(prob, MarchConfig(dt=2e-4, T=2e-2, variant="ExplicitEuler"))
    out["Euler"] = rep.final.data
    out["Euler_steps"] = rep.steps_taken
    rep = march(prob, MarchConfig(dt=0.01, T=1.0, variant="ExplicitEuler",
                                  divergence_threshold=1e6))
    out["Euler_div_final"] = rep.final.data
    out["Euler_div_steps"] = rep.steps_taken
    out["Euler_div_step"] = -1 if rep.diverged_step is None else rep.diverged_step
    save("comparison", **out)


CASES = {"assembly": lambda: (assembly_case("a40", 40, 5.0, 11, 0.5, 4.0, 0.0, 1.1283),
                              assembly_case("a60_probe", 60, 6.0, 12, 0.4, 4.0, 1.4, 0.9212)),
         "march": march_cases, "small_api": small_api_cases, "sphere": sphere_case,
         "energy": energy_case, "kirkwood": kirkwood_case, "vacuum": vacuum_case,
         "comparison": comparison_cases}



sys.path.insert(0, HERE)
from make_golden_cases import CLI_CASES  # noqa: E402


def cli_cases():
    """CSV reports of the reference CLI (cli.py) for small ladders -> tests/golden/cli/."""
    from pbsplit.cli import main as ref_main

    d = os.path.join(HERE, "cli")
    sysf = os.path.join(d, "mini.sys")
    for name, argv in CLI_CASES.items():
        argv = [sysf if a == "SYS" else a for a in argv]
        out = os.path.join(d, name + ".csv")
        rc = ref_main(argv + ["--out", out])
        print(name, "rc", rc, os.path.getsize(out))


CASES["cli"] = cli_cases


if __name__ == "__main__":
    for name in (sys.argv[1:] or list(CASES)):
        CASES[name]()
