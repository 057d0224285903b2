"""Device parity at the MEASURED scales against fixtures produced by the real reference.

`tests/golden/make_golden_scale.py` ran `pbsplit.march` / `pbsplit.energy_pipeline`
(schemes.py:399-425, energy.py:109-164) in the build container on the same seeded inputs;
the committed fixtures hold hashes of the assembled maps, mid-planes, a seeded node sample,
field statistics and dG.  Bars (north_star): max|du| <= 1e-9 * max|u_ref| on every committed
node, |dG - dG_ref| <= 1e-8 |dG_ref|; assembly (integer / ordering work) bit-exact.

* config 3: REplusV at 257^3 (four marches: solvent and vacuum LODIE2 at dt 0.5 and 0.25,
  T = 50, i.e. 100 + 200 steps each);
* config 4: 513^3, 10,000 atoms, LODIE2 at dt 0.5, 50 steps (the benched workload);
* config 5: all 64 proteins x {AOSIE1, LODIE2}, 100 steps each.
"""

import hashlib

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from paper_1410_2788_b200 import _native as nat
from paper_1410_2788_b200.configs import (CONFIGS, batch_sizes, cubic_box, kappa_bar,
                                          synthetic_atoms)
from tests.golden.scale_common import field_stats, mask_digest, sample_index
from tests.helpers import golden, system_of

pytestmark = pytest.mark.gpu

POT_TOL = 1e-9
DG_TOL = 1e-8


def device_masks(p, eps_m):
    """The four solute masks (node, half-edge x/y/z in the reference's mesh shapes) from the
    device codes, without materialising the dense float maps."""
    from paper_1410_2788_b200.schemes import device_problem

    g = p.grid
    n0, n1, n2 = g.shape
    dp = device_problem(p)
    pitch = dp.gs.pitch
    c = dp.codes[:n0 * n1 * pitch].view(n0, n1, pitch)[:, :, nat.PBG_OFFSET:nat.PBG_OFFSET + n2]
    c = c.cpu().numpy()
    eps_pal, _ = dp.pal.as_tuple()
    node_pal = p.region._node_pal

    def pick(bits, pal):
        return np.where(bits != 0, pal[1] == eps_m, pal[0] == eps_m)

    node = pick(c & 1, node_pal)
    hx = pick(c[1:] & 2, eps_pal[0])
    hy = pick(c[:, 1:] & 4, eps_pal[1])
    hz = pick(c[:, :, 1:] & 8, eps_pal[2])
    return node, hx, hy, hz


def check_assembly(p, d, eps_m, big=False):
    node, hx, hy, hz = device_masks(p, eps_m)
    for name, mk in (("node", node), ("hx", hx), ("hy", hy), ("hz", hz)):
        assert mask_digest(mk) == str(d["dig_" + name]), name
    assert hashlib.sha256(p.qfrac.data.tobytes()).hexdigest() == str(d["dig_qfrac"])
    assert hashlib.sha256(p.rho.data.tobytes()).hexdigest() == str(d["dig_rho"])
    fs = field_stats(p.boundary.values)
    assert np.allclose(fs, d["faces_stats"], rtol=1e-12, atol=0)


def check_field(u, d, prefix):
    stats = d[prefix + "_stats"]
    scale = float(stats[0])
    got = field_stats(u)
    assert abs(got[0] - scale) <= POT_TOL * scale
    # sums over the whole grid: reassociated fp64 differences only
    assert abs(got[1] - stats[1]) <= POT_TOL * scale * u.size ** 0.5
    assert abs(got[2] - stats[2]) <= 1e-9 * abs(stats[2])
    samp = u.ravel()[sample_index(u.shape)]
    assert np.max(np.abs(samp - d[prefix + "_sample"])) <= POT_TOL * scale
    if prefix + "_plane" in d:
        plane = u[u.shape[0] // 2]
        assert np.max(np.abs(plane - d[prefix + "_plane"])) <= POT_TOL * scale


def cubic_problem(c, atoms):
    from paper_1410_2788_b200.problem import assemble_on_grid

    lo, hi = cubic_box(atoms, c.n, c.h)
    grid = pb.make_grid(lo, hi, c.h)
    return assemble_on_grid(system_of(atoms), grid, kappa_bar(c.ionic_strength), c.eps_m,
                            c.eps_s)


def test_config4_513_lodie2_50_steps_vs_reference():
    d = golden("scale_c4")
    c = CONFIGS["c4"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    p = cubic_problem(c, atoms)
    assert p.grid.shape == tuple(int(v) for v in d["shape"])
    check_assembly(p, d, c.eps_m)
    rep = pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * c.steps, variant=c.variant))
    assert rep.steps_taken == int(d["steps"]) == 50 and not rep.diverged
    check_field(rep.final.data, d, "u")


def test_config3_257_replusv_vs_reference():
    d = golden("scale_c3")
    c = CONFIGS["c3"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    p = cubic_problem(c, atoms)
    check_assembly(p, d, c.eps_m)
    res = pb.energy_pipeline(p, pb.MarchConfig(dt=float(d["dt"]), T=float(d["T"]),
                                               variant=c.variant), "REplusV")
    want = float(d["delta_g"])
    assert not res.diverged
    assert abs(res.delta_g - want) <= DG_TOL * abs(want)
    check_field(res.phi_m.data, d, "phim")
    check_field(res.phi_0.data, d, "phi0")


def test_config5_all_64_proteins_vs_reference():
    from paper_1410_2788_b200.batch import config5_problem, march_many

    d = golden("scale_c5")
    sizes = batch_sizes()
    assert list(d["sizes"]) == sizes
    probs = [config5_problem(i, sizes[i]) for i in range(len(sizes))]
    for i, (c, p) in enumerate(probs):
        node, hx, hy, hz = device_masks(p, c.eps_m)
        for name, mk in (("node", node), ("hx", hx), ("hy", hy), ("hz", hz)):
            assert mask_digest(mk) == str(d["dig_" + name][i]), (i, name)
        assert hashlib.sha256(p.qfrac.data.tobytes()).hexdigest() == str(d["dig_qfrac"][i])
    jobs = [((i, v), p, pb.MarchConfig(dt=c.dt, T=c.dt * c.steps, variant=v))
            for i, (c, p) in enumerate(probs) for v in ("AOSIE1", "LODIE2")]
    reps = march_many(jobs, streams=8)
    for (i, v), rep in sorted(reps.items()):
        assert rep.steps_taken == int(d[v + "_steps"][i]) == 100 and not rep.diverged
        u = rep.final.data
        stats = d[v + "_stats"][i]
        scale = float(stats[0])
        got = field_stats(u)
        assert abs(got[0] - scale) <= POT_TOL * scale, (i, v)
        assert abs(got[2] - stats[2]) <= 1e-9 * abs(stats[2]), (i, v)
        samp = u.ravel()[sample_index(u.shape)]
        assert np.max(np.abs(samp - d[v + "_sample"][i])) <= POT_TOL * scale, (i, v)
