"""Benchmark: pseudo-transient LOD step throughput (interior grid-point updates/s, fp64).

Workload (BASELINE.json metric is quoted at 1/2/4/8 B200 on the sharded config): config 4,
a 10,000-atom synthetic protein on a 513^3 grid (h = 0.3 A, eps 2/80, 0.15 M), LODIE2,
dt = 0.5.  One bench "step" = one LODIE2 time step over the whole grid (flow + source +
three implicit line sweeps).  Fields are 1.1 GB each (>> 126 MB L2), so no L2 flush is
needed between steps (`--config c3`: 257^3, 142 MB fields, still larger than L2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c3|c2|c5] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU, NCCL): the grid is split into axis-0 slabs, one per
rank (paper_1410_2788_b200.slab: partitioned axis-0 solve, one all-gather of the chunk end
rows per step) -- strong scaling, `value` = whole-grid updates/s, time = max over ranks.
`--mode replicas` instead marches an independent copy per rank (weak scaling).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_LOD = 48  # algorithmic bytes per interior update per LOD step
BYTES_SWEEP = 16  # one fp64 read + one fp64 write per interior node per sweep launch


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--c5-streams", action="store_true",
                    help="config 5: one march per protein on 8 streams instead of batched")
    ap.add_argument("--mode", default=None, choices=["slab", "replicas"],
                    help="slab-sharded single grid (default for N > 1; with N = 1 it runs "
                         "the slab path as one NCCL rank) or independent replicas")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, f[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_problem(cfg_key):
    import paper_1410_2788_b200 as pb
    from paper_1410_2788_b200.configs import CONFIGS, cubic_box, kappa_bar, synthetic_atoms
    from paper_1410_2788_b200.problem import assemble_on_grid

    c = CONFIGS[cfg_key]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    grid = pb.make_grid(lo, hi, c.h)
    system = pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms], label=c.name)
    t0 = time.perf_counter()
    p = assemble_on_grid(system, grid, kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    import torch

    torch.cuda.synchronize()
    return c, p, time.perf_counter() - t0


def march_desc(p, c, nsteps):
    from paper_1410_2788_b200 import _native as nat
    from paper_1410_2788_b200.schemes import device_problem

    dp = device_problem(p)
    w0, w1 = dp.work_pair()
    d = nat.PbgMarchDesc()
    d.grid = dp.gs
    d.pal = dp.pal
    d.variant = nat.VARIANT_IDS[c.variant]
    d.dt, d.alpha, d.divergence_threshold = c.dt, p.alpha, 1e12
    d.nsteps, d.check_divergence = nsteps, 1
    d.codes, d.rho = dp.codes.data_ptr(), dp.rho.data_ptr()
    d.initial = w0.data_ptr()  # protein default: zero interior, Dirichlet faces
    d.work[0], d.work[1] = w0.data_ptr(), w1.data_ptr()
    return d, dp, (w0, w1)


def run_march(d, nsteps):
    from paper_1410_2788_b200 import _native as nat

    d.nsteps = nsteps
    taken, dstep, slot = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    ms = ctypes.c_float()
    nat.check(nat.lib().pbg_march(ctypes.byref(d), ctypes.byref(taken), ctypes.byref(dstep),
                                  ctypes.byref(slot), ctypes.byref(ms), nat.stream_ptr()))
    if taken.value != nsteps or dstep.value:
        raise RuntimeError(f"march diverged at step {dstep.value}")
    return ms.value


def faces_packed(arr):
    return np.concatenate([arr[0].ravel(), arr[-1].ravel(), arr[:, 0].ravel(),
                           arr[:, -1].ravel(), arr[:, :, 0].ravel(), arr[:, :, -1].ravel()])


def e2e_measure(p, c, dp, nsteps):
    """Same metric through the C ABI with HOST buffers (pbg_march_host): uploads codes,
    sparse source and packed faces from pinned memory, marches, downloads the final field."""
    import torch

    from paper_1410_2788_b200 import _native as nat

    g = p.grid
    codes_h = torch.empty(dp.codes.numel(), dtype=torch.uint8, pin_memory=True)
    codes_h.copy_(dp.codes)
    rho = p.rho._dev
    n0, n1, n2 = g.shape
    pitch = dp.gs.pitch
    rd = rho[:n0 * n1 * pitch].view(n0, n1, pitch)[:, :, nat.PBG_OFFSET:nat.PBG_OFFSET + n2]
    flat = torch.nonzero(rd.reshape(-1)).reshape(-1)
    idx_h = flat.cpu().numpy().astype(np.int64)
    val_h = rd.reshape(-1)[flat].cpu().numpy()
    bnd = dp.bnd[:n0 * n1 * pitch].view(n0, n1, pitch)[:, :, nat.PBG_OFFSET:nat.PBG_OFFSET + n2]
    fc = torch.cat([bnd[0].reshape(-1), bnd[-1].reshape(-1), bnd[:, 0].reshape(-1),
                    bnd[:, -1].reshape(-1), bnd[:, :, 0].reshape(-1), bnd[:, :, -1].reshape(-1)])
    faces_h = torch.empty(fc.numel(), dtype=torch.float64, pin_memory=True)
    faces_h.copy_(fc)
    out_h = torch.empty((n0, n1, n2), dtype=torch.float64, pin_memory=True)
    desc = nat.PbgMarchDesc()
    desc.grid = dp.gs
    desc.pal = dp.pal
    desc.variant = nat.VARIANT_IDS[c.variant]
    desc.dt, desc.alpha, desc.divergence_threshold = c.dt, p.alpha, 1e12
    desc.nsteps, desc.check_divergence = nsteps, 1
    taken, dstep = ctypes.c_int32(), ctypes.c_int32()
    ms = ctypes.c_float()

    def call():
        nat.check(nat.lib().pbg_march_host(
            ctypes.byref(desc), codes_h.data_ptr(), len(idx_h), idx_h.ctypes.data,
            val_h.ctypes.data, faces_h.data_ptr(), None, out_h.data_ptr(), ctypes.byref(taken),
            ctypes.byref(dstep), ctypes.byref(ms), nat.stream_ptr()))

    call()  # warm the allocator pool
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    call()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    h2d = codes_h.numel() + idx_h.nbytes + val_h.nbytes + faces_h.numel() * 8
    d2h = out_h.numel() * 8
    return wall, h2d, d2h, float(np.isfinite(out_h[n0 // 2].numpy()).all())


def host_planes(dp, grid, i0, i1):
    """Planes i0 <= i < i1 of the device problem's codes, source and boundary buffers."""
    from paper_1410_2788_b200 import _native as nat

    n0, n1, n2 = grid.shape
    pitch = dp.gs.pitch
    sl = slice(nat.PBG_OFFSET, nat.PBG_OFFSET + n2)
    nn = n0 * n1 * pitch
    pick = lambda t: t[:nn].view(n0, n1, pitch)[i0:i1, :, sl].cpu().numpy()
    return pick(dp.codes), pick(dp.rho), pick(dp.bnd)


def oracle_slab(p, dp, nplanes, planes=None, i0=0):
    """CPU oracle problem for planes i0 <= i < i0+nplanes of the device problem (test/baseline
    infrastructure): same codes, source and faces; the slab's first and last planes act as
    Dirichlet faces.  `planes` = host_planes(...) of a range starting at plane 0 of the slab
    sample set (reused by the reference arm's workers)."""
    from oracle import pbs_oracle as O

    g = p.grid
    n0, n1, n2 = g.shape
    if planes is None:
        planes = host_planes(dp, g, i0, i0 + nplanes)
        i0 = 0
    codes = planes[0][i0:i0 + nplanes]
    rho = planes[1][i0:i0 + nplanes].copy()
    bv = planes[2][i0:i0 + nplanes].copy()
    rho[-1] = 0.0
    rho[0] = 0.0
    eps = dp.pal.as_tuple()[0]
    k2p = dp.pal.as_tuple()[1]
    pick = lambda bit, pal: np.where((codes & bit) != 0, pal[1], pal[0])
    eh = (pick(2, eps[0])[1:], pick(4, eps[1])[:, 1:], pick(8, eps[2])[:, :, 1:])
    k2 = pick(1, k2p)
    region = O.ORegion(pick(1, (eps[0][0], eps[0][1])), eh, k2)
    og = O.OGrid(g.lo, g.h, (nplanes, n1, n2))
    init = np.zeros(og.shape)
    O.apply_faces(init, bv)
    return O.OProblem(og, region, rho, np.zeros(og.shape), bv, p.alpha, init)


def cpu_oracle_rate(p, dp, c, nplanes=65, steps=1):
    from oracle import pbs_oracle as O

    op = oracle_slab(p, dp, nplanes)
    st = O.OStepper(op, c.variant, c.dt)
    u = op.initial.copy()
    t0 = time.perf_counter()
    for _ in range(steps):
        u = st.step(u)
    wall = time.perf_counter() - t0
    nint = (nplanes - 2) * (p.grid.ny - 2) * (p.grid.nz - 2)
    return nint * steps / wall, nint, wall


def c3_target(args):
    """north_star's single-GPU target, measured in the same run: the full LODIE2 step at
    257^3 (config 3) against the 60% mark of the 48 B/node roofline (8 TB/s nominal and the
    measured copy bandwidth)."""
    import torch

    c, p, _ = build_problem("c3")
    nint = (c.n - 2) ** 3
    d, dp, keep = march_desc(p, c, args.steps)
    run_march(d, max(3, args.warmup))
    torch.cuda.synchronize()
    ms = run_march(d, args.steps) / args.steps
    peak, kind = peaks()
    step_gbs = BYTES_LOD * nint / (ms / 1e3) / 1e9
    return {"c3_257_lodie2": {"ms_per_step": ms, "updates_per_s": nint / (ms / 1e3),
                              "step_GBps_48B": step_gbs, "frac_of_8TBs": step_gbs / 8000.0,
                              "frac_of_measured": step_gbs / peak,
                              "target_ms_60pct_of_8TBs": BYTES_LOD * nint / (0.6 * 8e12) * 1e3,
                              "met": step_gbs / 8000.0 >= 0.6}}


def profiled_kernels(d, nsteps):
    from paper_1410_2788_b200 import _native as nat

    lib = nat.lib()
    lib.pbg_set_profiling(1)
    run_march(d, nsteps)
    ms = (ctypes.c_double * 3)()
    n = (ctypes.c_int64 * 3)()
    lib.pbg_get_profile(ms, n)
    lib.pbg_set_profiling(0)
    return [ms[a] / max(1, n[a]) for a in range(3)], [int(n[a]) for a in range(3)]


def ncu_traffic(config_name, axis):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get(config_name, {}).get(str(axis))
    except Exception:
        return None


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":  # host only: no torch, no package, no libpbg.so
        return reference_arm(args, world, rank)
    import torch

    torch.cuda.set_device(local)
    dist = None
    mode = args.mode or ("slab" if world > 1 else "single")
    if world > 1 or mode == "slab":
        import torch.distributed as dist

        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    if args.config == "c5":
        return c5_main(args, world, rank, local, dist)
    c, p, t_asm = build_problem(args.config)
    nint = (c.n - 2) ** 3
    if dist and mode == "slab":
        return slab_main(args, c, p, t_asm, world, rank, local, dist)
    d, dp, keep = march_desc(p, c, args.steps)
    run_march(d, max(3, args.warmup))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = run_march(d, args.steps)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = nint * args.steps * world / (ms_max / 1e3)

    field_mb = p.grid.nx * p.grid.ny * dp.gs.pitch * 8 / 1e6
    per_ms, launches = profiled_kernels(d, min(args.steps, 20))
    dom = int(np.argmax(per_ms))
    peak, peak_kind = peaks()
    achieved = BYTES_SWEEP * nint / (per_ms[dom] / 1e3) / 1e9
    step_gbs = BYTES_LOD * nint / (ms_max / args.steps / 1e3) / 1e9

    targets = None
    if rank == 0 and world == 1 and args.config == "c4":
        targets = c3_target(args)
    e2e = None
    if not args.no_e2e:
        wall, h2d, d2h, ok = e2e_measure(p, c, dp, args.steps)
        e2e = {"value": nint * args.steps / wall, "unit": "grid-point updates/s",
               "h2d_bytes_per_step": int(h2d / args.steps),
               "d2h_bytes_per_step": int(d2h / args.steps),
               "note": f"pbg_march_host: {args.steps}-step march from pinned host buffers "
                       "(codes, sparse source, packed faces) incl. allocation, H2D, D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, nn, wall = cpu_oracle_rate(p, dp, c)
        cpu = {"value": rate, "unit": "grid-point updates/s", "cores": 1, "kind": "port",
               "sample": f"1 {c.variant} step of {c.name} restricted to planes i<65 "
                         f"({nn} interior nodes, {wall:.1f} s), numpy oracle port of "
                         "pbsplit Stepper"}
    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": "LOD grid-point updates/s (fp64)",
            "value": value,
            "unit": "grid-point updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded generator, configs.py)",
            "config": {"workload": c.name, "grid": [c.n] * 3, "atoms": c.n_atoms, "h": c.h,
                       "variant": c.variant, "dt": c.dt, "interior_nodes": nint,
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": f"field {field_mb:.0f} MB > 126 MB L2 (each sweep streams a whole "
                             "field), no flush", "assembly_s": round(t_asm, 3)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(c.name, dom),
                         "kernel": ["k_sweep_col axis 0 (register-direct column tiles, "
                                    "+ source)",
                                    "k_sweep_col axis 1 (register-direct column tiles)",
                                    ({513: "k_sweep_rowlean axis 2 (TMA in / TMA out, one line per "
                                           "warp, + flow)",
                                      257: "k_sweep_rowlean axis 2 (TMA in / TMA out, two lines per "
                                           "warp, + flow)",
                                      129: "k_sweep_rowwarp axis 2 (two lines per warp, + flow)",
                                      97: "k_sweep_rowwarp axis 2 (four lines per warp, + flow)"}
                                     .get(c.n, "k_sweep_strided axis 2 (row tiles, + flow)"))][dom],
                         "kernel_ms": per_ms, "peak_kind": peak_kind,
                         "step_GBps_48B": step_gbs, "step_frac": step_gbs / peak},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "targets": targets,
            "gpu_launches": 3 * args.steps + 2,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def c5_main(args, world, rank, local, dist):
    """Config 5: 64 independent 97^3 proteins, AOSIE1 and LODIE2, round-robin over ranks
    (replicas, weak in proteins per rank), 8 concurrent streams per GPU."""
    import torch

    import paper_1410_2788_b200 as pb
    from paper_1410_2788_b200.batch import config5_problem, march_many, rank_indices
    from paper_1410_2788_b200.configs import batch_sizes
    from paper_1410_2788_b200.schemes import device_problem

    sizes = batch_sizes()
    mine = rank_indices(len(sizes), rank, world)
    t0 = time.perf_counter()
    probs = {i: config5_problem(i, sizes[i]) for i in mine}
    for i in mine:
        device_problem(probs[i][1])
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t0
    variants = ("AOSIE1", "LODIE2")
    if not args.c5_streams:
        return c5_batched(args, world, rank, local, dist, sizes, mine, probs, t_asm, variants)
    jobs = [((i, v), probs[i][1], pb.MarchConfig(dt=probs[i][0].dt, T=probs[i][0].dt * args.steps,
                                                 variant=v)) for i in mine for v in variants]
    warm = [((k, v), p, pb.MarchConfig(dt=cfg.dt, T=cfg.dt * max(3, args.warmup), variant=v))
            for (k, v), p, cfg in jobs]
    march_many(warm, streams=8)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    from paper_1410_2788_b200.batch import _stream_pool

    pool = _stream_pool(torch, 8)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev0.record(cur)  # device clock: start on the default stream, every march stream
        for s in pool:   # waits on it, and the default stream joins all of them at the end
            s.wait_event(ev0)
        reps = march_many(jobs, streams=8)
        for s in pool:
            cur.wait_stream(s)
        ev1.record(cur)
        torch.cuda.synchronize()
        host_wall = time.perf_counter() - t0
        wall = ev0.elapsed_time(ev1) / 1e3
    bad = [k for k, r in reps.items() if r.diverged or r.steps_taken != args.steps]
    if bad:
        raise RuntimeError(f"config 5 marches diverged: {bad[:4]}")
    t = torch.tensor([wall], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall_max = float(t.item())
    n = probs[mine[0]][0].n
    total = len(sizes) * len(variants) * args.steps * (n - 2) ** 3
    e2e = None
    if not args.no_e2e:  # the public call from host inputs (atoms) to host results (fields)
        from paper_1410_2788_b200.batch import run_config5

        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        items = run_config5(rank, world, count=len(sizes), nsteps=args.steps, streams=8,
                            group=None)
        torch.cuda.synchronize()
        tw = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        bad = [(it.index, it.variant) for it in items if it.diverged]
        if bad:
            raise RuntimeError(f"config 5 e2e marches diverged: {bad[:4]}")
        atoms_bytes = sum(sizes[i] for i in mine) * 5 * 8
        e2e = {"value": total / float(tw.item()), "unit": "grid-point updates/s",
               "h2d_bytes_per_step": int(atoms_bytes / args.steps),
               "d2h_bytes_per_step": int(len(mine) * len(variants) * n ** 3 * 8 / args.steps),
               "note": "batch.run_config5: assembly from host atom lists, plan setup, the "
                       "marches and the final fields downloaded (max over ranks)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import pbs_oracle as O
        from paper_1410_2788_b200.configs import batch_config, cubic_box, kappa_bar, synthetic_atoms

        cb = batch_config(0, sizes[0])
        atoms = synthetic_atoms(cb.n_atoms, cb.ball_radius, cb.seed)
        lo, hi = cubic_box(atoms, cb.n, cb.h)
        op = O.protein_on_grid(O.grid_from_bounds(lo, hi, cb.h), atoms, cb.eps_m, cb.eps_s,
                               kappa_bar(cb.ionic_strength))
        wall = 0.0
        ksteps = 5
        for v in variants:
            st = O.OStepper(op, v, cb.dt)
            u = op.initial.copy()
            t0 = time.perf_counter()
            for _ in range(ksteps):
                u = st.step(u)
                np.max(np.abs(u))
            wall += time.perf_counter() - t0
        cpu = {"value": len(variants) * ksteps * (n - 2) ** 3 / wall,
               "unit": "grid-point updates/s", "cores": 1, "kind": "port",
               "sample": f"protein 0 ({sizes[0]} atoms, {n}^3), {ksteps} AOSIE1 + {ksteps} "
                         "LODIE2 steps, numpy oracle port of pbsplit Stepper, one core"}
    if rank == 0:
        line = {
            "metric": "LOD/AOS grid-point updates/s (fp64), config-5 batch",
            "value": total / wall_max, "unit": "grid-point updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": wall_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, configs.py)",
            "config": {"workload": "c5-batch64-97", "proteins": len(sizes), "grid": [n] * 3,
                       "variants": list(variants), "dt": 0.5,
                       "parallelism": f"proteins round-robin over {world} rank(s), 8 streams "
                                      "per GPU", "assembly_s": round(t_asm, 3),
                       "timing": "CUDA events: start on the default stream, joined from all 8 "
                                 "march streams at the end (per-march setup inside), max over "
                                 "ranks", "host_wall_s": round(host_wall, 4)},
            "roofline": {"bound": "hbm", "achieved": None, "peak": peaks()[0], "unit": "GB/s",
                         "frac": None, "traffic": None,
                         "note": "97^3 fields (7 MB) are L2-resident: no HBM roofline "
                                 "(SURVEY.md §8d caveat); step bytes "
                                 f"{(48 + 64) / 2 * total / wall_max / 1e9:.0f} GB/s "
                                 "equivalent (48 B LOD, 64 B AOS per node)"},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": sum(3 * r.steps_taken + 2 for r in reps.values()) * world,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def c5_batched(args, world, rank, local, dist, sizes, mine, probs, t_asm, variants):
    """Config 5 with batched launches: the rank's proteins stacked into one BatchMarch, one
    launch per sweep for all of them; AOSIE1 then LODIE2, each `steps`
    steps, timed with CUDA events on the launching stream."""
    import torch

    import paper_1410_2788_b200 as pb
    from paper_1410_2788_b200.batch import BatchMarch

    bm = BatchMarch([probs[i][1] for i in mine])
    dt = probs[mine[0]][0].dt
    for v in variants:  # warm-up (plans prepared here, as the reference's Stepper setup)
        bm.march(pb.MarchConfig(dt=dt, T=dt * max(3, args.warmup), variant=v), keep_fields=False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per_variant = {}
    with ClockSampler(local) as clk:
        ev0.record()
        for v in variants:
            reps, secs = bm.march(pb.MarchConfig(dt=dt, T=dt * args.steps, variant=v),
                                  keep_fields=False)
            per_variant[v] = secs
            bad = [i for i, r in zip(mine, reps) if r.diverged or r.steps_taken != args.steps]
            if bad:
                raise RuntimeError(f"config 5 {v} marches diverged: {bad[:4]}")
        ev1.record()
        torch.cuda.synchronize()
    wall = ev0.elapsed_time(ev1) / 1e3
    if dist:
        dist.barrier()
    t = torch.tensor([wall], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall_max = float(t.item())
    n = probs[mine[0]][0].n
    total = len(sizes) * len(variants) * args.steps * (n - 2) ** 3
    mine_nodes = len(mine) * (n - 2) ** 3
    e2e = None
    if not args.no_e2e:  # the public call from host inputs (atoms) to host results (fields)
        from paper_1410_2788_b200.batch import run_config5

        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        items = run_config5(rank, world, count=len(sizes), nsteps=args.steps)
        torch.cuda.synchronize()
        tw = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        if any(it.diverged for it in items):
            raise RuntimeError("config 5 e2e marches diverged")
        atoms_bytes = sum(sizes[i] for i in mine) * 5 * 8
        e2e = {"value": total / float(tw.item()), "unit": "grid-point updates/s",
               "h2d_bytes_per_step": int(atoms_bytes / args.steps),
               "d2h_bytes_per_step": int(len(mine) * len(variants) * n ** 3 * 8 / args.steps),
               "note": "batch.run_config5: assembly from host atom lists, batched plan setup, "
                       "the marches, final fields downloaded (max over ranks)"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = c5_cpu_baseline(sizes, n, variants)
    peak, kind = peaks()
    aos_s, lod_s = per_variant["AOSIE1"], per_variant["LODIE2"]
    lod_gbs = 48 * mine_nodes * args.steps / lod_s / 1e9
    aos_gbs = 64 * mine_nodes * args.steps / aos_s / 1e9
    if rank == 0:
        line = {
            "metric": "LOD/AOS grid-point updates/s (fp64), config-5 batch",
            "value": total / wall_max, "unit": "grid-point updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": wall_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, configs.py)",
            "config": {"workload": "c5-batch64-97", "proteins": len(sizes), "grid": [n] * 3,
                       "variants": list(variants), "dt": 0.5,
                       "parallelism": f"proteins round-robin over {world} rank(s); each "
                                      "rank's proteins in one batched march (one launch per "
                                      "sweep)", "assembly_s": round(t_asm, 3),
                       "per_variant_ms_per_step": {v: per_variant[v] / args.steps * 1e3
                                                   for v in variants},
                       "l2": f"{len(mine)} x 7.3 MB fields, batch {len(mine) * 7.3:.0f} MB "
                             "per field > L2"},
            "roofline": {"bound": "hbm", "achieved": lod_gbs, "peak": peak, "unit": "GB/s",
                         "frac": lod_gbs / peak, "traffic": None, "peak_kind": kind,
                         "kernel": "whole batched LODIE2 step (48 B/node)",
                         "aos_step_GBps_64B": aos_gbs, "aos_frac": aos_gbs / peak},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": (len(variants) * (3 * args.steps + 1 + len(mine))) * world,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def c5_cpu_baseline(sizes, n, variants):
    from oracle import pbs_oracle as O
    from paper_1410_2788_b200.configs import batch_config, cubic_box, kappa_bar, synthetic_atoms

    cb = batch_config(0, sizes[0])
    atoms = synthetic_atoms(cb.n_atoms, cb.ball_radius, cb.seed)
    lo, hi = cubic_box(atoms, cb.n, cb.h)
    op = O.protein_on_grid(O.grid_from_bounds(lo, hi, cb.h), atoms, cb.eps_m, cb.eps_s,
                           kappa_bar(cb.ionic_strength))
    wall = 0.0
    ksteps = 5
    for v in variants:
        st = O.OStepper(op, v, cb.dt)
        u = op.initial.copy()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            u = st.step(u)
            np.max(np.abs(u))
        wall += time.perf_counter() - t0
    return {"value": len(variants) * ksteps * (n - 2) ** 3 / wall,
            "unit": "grid-point updates/s", "cores": 1, "kind": "port",
            "sample": f"protein 0 ({sizes[0]} atoms, {n}^3), {ksteps} AOSIE1 + {ksteps} "
                      "LODIE2 steps, numpy oracle port of pbsplit Stepper, one core"}


def slab_main(args, c, p, t_asm, world, rank, local, dist):
    """N > 1: one axis-0 slab per rank, NCCL all-gather exchange (strong scaling)."""
    import torch

    import paper_1410_2788_b200 as pb
    from paper_1410_2788_b200.schemes import device_problem
    from paper_1410_2788_b200.slab import (GroupExchange, make_slabs, plane_costs, run_slabs,
                                           slab_ranges)

    nint = (c.n - 2) ** 3
    cfg = pb.MarchConfig(dt=c.dt, T=c.dt * args.steps, variant=c.variant)
    (part,), _, cn = make_slabs(p, cfg, [rank], world)
    ex = GroupExchange()
    warm = max(3, args.warmup)
    res = run_slabs([part], ex, warm, cn)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        res = run_slabs([part], ex, args.steps, cn)
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    taken, dstep, final = res[0]
    if dstep is not None:
        raise RuntimeError(f"slab march diverged at step {dstep}")
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = nint * args.steps / (ms_max / 1e3)
    own = part.stop - part.first
    local_nodes = own * (c.n - 2) ** 2

    e2e = None
    if not args.no_e2e:  # host inputs of the rank's slab -> device, march, owned planes -> host
        pin = lambda t: torch.empty(t.numel(), dtype=t.dtype, pin_memory=True).copy_(t)
        host = [pin(part.codes), pin(part.rho), pin(part.work[0])]
        out_h = torch.empty(part.owned(final).numel(), dtype=torch.float64, pin_memory=True)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part.codes.copy_(host[0], non_blocking=True)
        part.rho.copy_(host[1], non_blocking=True)
        part.work[0].copy_(host[2], non_blocking=True)
        part.work[1].copy_(host[2], non_blocking=True)
        part.initial.copy_(host[2], non_blocking=True)
        res = run_slabs([part], ex, args.steps, cn)
        out_h.copy_(part.owned(res[0][2]))
        torch.cuda.synchronize()
        tw = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        h2d = sum(h.numel() * h.element_size() for h in host)
        e2e = {"value": nint * args.steps / float(tw.item()), "unit": "grid-point updates/s",
               "h2d_bytes_per_step": int(h2d / args.steps),
               "d2h_bytes_per_step": int(out_h.numel() * 8 / args.steps),
               "note": "per rank: slab inputs from pinned host buffers, the sharded march, "
                       "owned planes back to the host; max over ranks"}
    clocks = clk.summary()
    if rank == 0:
        rng = slab_ranges(c.n, world, plane_costs(device_problem(p)))
        line = {
            "metric": "LOD grid-point updates/s (fp64)",
            "value": value,
            "unit": "grid-point updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": warm,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded generator, configs.py)",
            "config": {"workload": c.name, "grid": [c.n] * 3, "atoms": c.n_atoms, "h": c.h,
                       "variant": c.variant, "dt": c.dt, "interior_nodes": nint,
                       "parallelism": f"axis-0 slabs x{world} (partitioned solve, NCCL "
                                      "all-gather of chunk end rows)",
                       "slab_planes": [b - a for a, b in rng],
                       "l2": "slabs >> L2, no flush", "assembly_s": round(t_asm, 3)},
            "roofline": {"bound": "hbm", "achieved": BYTES_LOD * local_nodes /
                         (ms_max / args.steps / 1e3) / 1e9, "peak": peaks()[0],
                         "unit": "GB/s", "traffic": None,
                         "note": "rank-0 step bytes (48 B/owned node) / step time"},
            "cpu_baseline": None,
            "e2e": e2e,
            "gpu_launches": (7 if cn else 5) * args.steps,
            "clocks": clocks,
        }
        line["roofline"]["frac"] = line["roofline"]["achieved"] / line["roofline"]["peak"]
        print(json.dumps(line), flush=True)
    part.close()
    dist.destroy_process_group()


def _configs():
    """paper_1410_2788_b200/configs.py loaded by file path: the reference arm must not import
    the package (which loads libpbg.so) -- only the seeded input generator."""
    import importlib.util

    path = os.path.join(ROOT, "paper_1410_2788_b200", "configs.py")
    spec = importlib.util.spec_from_file_location("_pbg_configs", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules.setdefault("_pbg_configs", mod)
    spec.loader.exec_module(mod)
    return mod


def host_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_FACE = {}  # face points of the current BoundarySpec face, inherited by forked workers


def _face_chunk(span):
    from oracle import pbs_oracle as O

    lo, hi = span
    return O.coulomb_values(_FACE["pts"][lo:hi], _FACE["atoms"], _FACE["eps_s"], _FACE["kbar"])


def oracle_problem_cpu(c, cfg_mod, workers):
    """The benched problem built on the host by the oracle restatement of protein_problem's
    assembly on the cubic box (culled classification, np.add.at deposit, screened-Coulomb
    faces).  Face values are computed per point exactly as coulomb_screened_values does
    (problem.py:106-117: a per-point sum over the atoms in order), split over forked workers
    by point ranges, so the values are identical to a serial evaluation."""
    import multiprocessing as mp

    from oracle import pbs_oracle as O

    atoms = cfg_mod.synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    kbar = cfg_mod.kappa_bar(c.ionic_strength)
    lo, hi = cfg_mod.cubic_box(atoms, c.n, c.h)
    g = O.grid_from_bounds(lo, hi, c.h)
    region = O.union_region(g, atoms, c.eps_m, c.eps_s, kbar ** 2)
    qfrac, rho = O.deposit(g, atoms)
    _FACE.update(atoms=atoms, eps_s=c.eps_s, kbar=kbar)
    ctx = mp.get_context("fork")

    def fn(pts):
        _FACE["pts"] = pts
        n = pts.shape[0]
        spans = [(w * n // workers, (w + 1) * n // workers) for w in range(workers)]
        with ctx.Pool(workers) as pool:
            parts = pool.map(_face_chunk, spans, chunksize=1)
        return np.concatenate(parts)

    bvals = O.faces_from_function(g, fn)
    init = np.zeros(g.shape)
    O.apply_faces(init, bvals)
    return O.OProblem(g, region, rho, qfrac, bvals, 1.0, init, c.eps_m, c.eps_s, kbar,
                      list(atoms))


def reference_arm(args, world, rank):
    """CPU reference arm: the reference's own CPU algorithm for the benched workload, i.e.
    the numpy oracle port of pbsplit's Stepper/march (the reference is Python and cannot
    travel to the box; the port is pinned to it and times at 0.8-0.93x of it),
    on the SAME full grid and the same number of steps as our arm: inputs built on the host
    (no torch, no libpbg.so), W untimed warm-up steps, then K steps timed like
    MarchReport.wall_time (schemes.py:413-422: the step loop with its per-step max|u|
    divergence test, setup excluded).  The reference is single-threaded numpy (one core);
    only the untimed setup uses the other cores.  Rank 0 only (N > 1: the others exit)."""
    if rank != 0:
        return
    from oracle import pbs_oracle as O

    cfg_mod = _configs()
    if args.config not in cfg_mod.CONFIGS:
        print(json.dumps({"impl": "reference",
                          "unavailable": f"reference arm covers {sorted(cfg_mod.CONFIGS)}"}))
        return
    c = cfg_mod.CONFIGS[args.config]
    workers = max(1, len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    op = oracle_problem_cpu(c, cfg_mod, workers)
    st = O.OStepper(op, c.variant, c.dt)
    t_setup = time.perf_counter() - t0
    u = op.initial.copy()
    thr = 1e12
    for _ in range(args.warmup):
        u = st.step(u)
        np.max(np.abs(u))
    t0 = time.perf_counter()
    for k in range(args.steps):
        u = st.step(u)
        amax = np.max(np.abs(u))
        if not np.isfinite(amax) or amax > thr:
            raise RuntimeError(f"reference march diverged at step {k + 1}")
    wall = time.perf_counter() - t0
    nint = (c.n - 2) ** 3
    v = nint * args.steps / wall
    sample = (f"full {c.name} grid ({c.n}^3, {nint} interior nodes), {args.steps} timed "
              f"{c.variant} steps after {args.warmup} warm-up steps, numpy oracle port of "
              f"pbsplit Stepper/march, single-threaded; host {host_model()}, nproc {workers}; "
              f"setup {t_setup:.1f} s untimed")
    line = {"metric": "LOD grid-point updates/s (fp64)", "value": v,
            "unit": "grid-point updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, configs.py)",
            "config": {"workload": c.name, "grid": [c.n] * 3, "atoms": c.n_atoms, "h": c.h,
                       "variant": c.variant, "dt": c.dt, "interior_nodes": nint,
                       "parallelism": "one host core"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "grid-point updates/s", "cores": 1,
                             "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "grid-point updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "host": {"model": host_model(), "nproc": workers},
            "final_max_abs": float(np.max(np.abs(u)))}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
