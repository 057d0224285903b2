"""Per-rank cost of the slab-sharded c4 step at N ranks, measured on ONE GPU: the N
partitions run in one process (LocalExchange), and each partition's phase A (all chunks),
and interface + phase B + axis-1/2 sweeps are timed separately with CUDA events; the
exchange bytes per step come from pbg_slab_phase.  Prints one JSON line (dev tool; feeds
DESIGN §6's projection)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1410_2788_b200 as pb
from paper_1410_2788_b200 import slab as S
from paper_1410_2788_b200.configs import CONFIGS, cubic_box, kappa_bar, synthetic_atoms
from paper_1410_2788_b200.problem import assemble_on_grid

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
# "queued": a ~150 us spin kernel runs ahead of every timed region, so the region's launches
# are already queued when it starts (what a rank sees in steady state: the host runs ahead of
# the device); without it every region starts on an idle stream and pays its launch latency.
QUEUED = len(sys.argv) > 2 and sys.argv[2] == "queued"
steps = 10
c = CONFIGS["c4"]
atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
lo, hi = cubic_box(atoms, c.n, c.h)
g = pb.make_grid(lo, hi, c.h)
p = assemble_on_grid(pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms]), g,
                     kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
cfg = pb.MarchConfig(dt=c.dt, T=c.dt * steps, variant=c.variant)
import ctypes
from paper_1410_2788_b200 import _native as nat
E = int(nat.lib().pbg_slab_exchange_elems(ctypes.byref(S._local_gs(g, (c.n - 2) // N + 3))))
recv = torch.empty(N * E, dtype=torch.float64, device="cuda")
parts, nsteps, cn = S.make_slabs(p, cfg, range(N), N, recv=recv)
ex = S.LocalExchange()
ex.gather(parts, *parts[0].phase(S.SETUP, 0))
for q in parts:
    q.setup()
nc = parts[0].nchunks
ev = lambda: torch.cuda.Event(enable_timing=True)
tA = [0.0] * N
tB = [0.0] * N
for s in range(steps):
    for r, q in enumerate(parts):
        e0, e1 = ev(), ev()
        if QUEUED:
            torch.cuda._sleep(300000)
        e0.record()
        for ch in range(nc):
            q.step_a_chunk(ch)
        e1.record()
        torch.cuda.synchronize()
        if s >= 2:
            tA[r] += e0.elapsed_time(e1)
    for ch in range(nc):
        ex.gather(parts, *parts[0].phase(S.STEP, ch))
    for r, q in enumerate(parts):
        e0, e1 = ev(), ev()
        if QUEUED:
            torch.cuda._sleep(300000)
        e0.record()
        q.step_b()
        e1.record()
        torch.cuda.synchronize()
        if s >= 2:
            tB[r] += e0.elapsed_time(e1)
k = steps - 2
step_bytes = sum(parts[0].phase(S.STEP, ch)[1] for ch in range(nc)) * 8
out = {"ranks": N, "chunks": nc, "queued": QUEUED, "p4": os.environ.get("PBG_P4", "1"), "planes_per_rank": [q.stop - q.first for q in parts],
       "phaseA_ms": [round(t / k, 4) for t in tA], "phaseB_ms": [round(t / k, 4) for t in tB],
       "exchange_bytes_per_rank_per_step": step_bytes,
       "allgather_bytes_received_per_rank": step_bytes * (N - 1)}
print(json.dumps(out))
for q in parts:
    q.close()
