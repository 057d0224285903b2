"""Dev tool: config-5 batch throughput vs number of concurrent streams."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.batch import config5_problem, march_many
from paper_1410_2788_b200.configs import batch_sizes
from paper_1410_2788_b200.schemes import device_problem

count = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sizes = batch_sizes()
probs = [config5_problem(i, sizes[i]) for i in range(count)]
for c, p in probs:
    device_problem(p)
torch.cuda.synchronize()
nint = 95 ** 3
for v in ("LODIE2", "AOSIE1"):
    jobs = [((i, v), p, pb.MarchConfig(dt=c.dt, T=c.dt * steps, variant=v)) for i, (c, p) in enumerate(probs)]
    for s in (4, 8, 12, 16, 24, 32):
        march_many(jobs[:s], streams=s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        march_many(jobs, streams=s)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(v, "streams", s, f"{count*steps*nint/dt/1e9:.1f} Gupd/s", f"{dt*1e3:.1f} ms")
