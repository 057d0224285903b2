"""Config-5 batched march: per-axis kernel time per step (dev tool)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200 import _native as nat
from paper_1410_2788_b200.batch import BatchMarch, config5_problem
from paper_1410_2788_b200.configs import batch_sizes

count = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sizes = batch_sizes()
probs = [config5_problem(i, sizes[i])[1] for i in range(count)]
bm = BatchMarch(probs)
lib = nat.lib()
for v in ("LODIE2", "AOSIE1"):
    cfg = pb.MarchConfig(dt=0.5, T=0.5 * 20, variant=v)
    bm.march(cfg, keep_fields=False)
    best = min(bm.march(cfg, keep_fields=False)[1] for _ in range(3))
    lib.pbg_set_profiling(1)
    bm.march(cfg, keep_fields=False)
    ms = (ctypes.c_double * 3)(); n = (ctypes.c_int64 * 3)()
    lib.pbg_get_profile(ms, n)
    lib.pbg_set_profiling(0)
    print(v, "us/step", round(best / 20 * 1e6, 1), "axes_us",
          [round(1e3 * ms[q] / max(1, n[q]), 1) for q in range(3)], flush=True)
