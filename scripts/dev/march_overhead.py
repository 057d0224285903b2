"""Dev tool: host overhead of one march() call at config-5 size."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.batch import config5_problem
from paper_1410_2788_b200.configs import batch_sizes
c, p = config5_problem(0, batch_sizes()[0])
for v in ("LODIE2", "AOSIE1"):
    for n in (1, 1, 1, 50, 50):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rep = pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * n, variant=v))
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(v, n, f"wall {dt*1e3:.2f} ms  device loop {rep.wall_time*1e3:.3f} ms")
import cProfile, pstats
cProfile.run("pb.march(p, pb.MarchConfig(dt=c.dt, T=c.dt * 1, variant='LODIE2'))", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("cumtime").print_stats(12)
