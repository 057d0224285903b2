"""Environment-switch A/B of the march: best-of-3 step time per config and variant, and a
hash of the final field (bitwise equality across switches) -- dev tool."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import ctypes, sys, os, time, json, hashlib
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.configs import CONFIGS, synthetic_atoms, cubic_box, kappa_bar
from paper_1410_2788_b200.problem import assemble_on_grid
key, v = sys.argv[1], sys.argv[2]
c = CONFIGS[key]
atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
lo, hi = cubic_box(atoms, c.n, c.h)
g = pb.make_grid(lo, hi, c.h)
p = assemble_on_grid(pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms]), g,
                     kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 3, variant=v))
best = 1e9
for _ in range(3):
    rep = pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 20, variant=v))
    best = min(best, rep.wall_time / rep.steps_taken)
u = rep.final.data
from paper_1410_2788_b200 import _native as nat
lib = nat.lib()
lib.pbg_set_profiling(1)
pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 20, variant=v))
ms = (ctypes.c_double * 3)(); n = (ctypes.c_int64 * 3)()
lib.pbg_get_profile(ms, n)
lib.pbg_set_profiling(0)
ax = [round(1e3 * ms[q] / max(1, n[q]), 1) for q in range(3)]
print(json.dumps({"us": round(best * 1e6, 1), "axes_us": ax, "sha": hashlib.sha256(u.tobytes()).hexdigest()[:16]}))
'''.replace("ROOT", repr(ROOT))
# usage: fuse_ab.py CONFIGS VARIANTS ENVS_JSON, e.g. c3,c4 LODIE2 '[{}, {"PBG_ROWTMA": "0"}]'
keys = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c4"]
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["LODIE2", "LODIE1"]
envs = json.loads(sys.argv[3]) if len(sys.argv) > 3 else [{}]
for key in keys:
    for v in variants:
        for env in envs:
            e = dict(os.environ, **env)
            out = subprocess.run([sys.executable, "-c", CHILD, key, v], env=e,
                                 capture_output=True, text=True)
            try:
                r = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                r = {"err": out.stderr[-400:]}
            print(key, v, env, r, flush=True)
