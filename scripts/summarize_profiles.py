"""Dev tool: turn gpurun_out captures into the committed profile summaries.

    python scripts/summarize_profiles.py TAG   (reads gpurun_out/{launches_TAG.csv,
    c4_full_TAG.ncu-rep, [c3_full_TAG.ncu-rep,] bench_*.json}; writes profiles/*_TAG*)
"""
import collections, csv, io, json, os, subprocess, sys

tag = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles")
go = os.path.join(root, "gpurun_out")
NODES = 133432831

# bench lines
lines = []
for name in ("bench_c4.json", "bench_c3.json", "bench_ref.json", "bench_c5.json", "bench_slab1.json"):
    p = os.path.join(go, name)
    if os.path.exists(p):
        lines += [ln for ln in open(p).read().splitlines() if ln.startswith("{")]
open(os.path.join(out, f"bench_{tag}.jsonl"), "w").write("\n".join(lines) + "\n")

# launch list
lpath = os.path.join(go, f"launches_{tag}.csv")
if not os.path.exists(lpath):  # re-run: the list was already moved into profiles/
    lpath = os.path.join(out, f"launches_{tag}.csv")
rows = [r for r in csv.reader(open(lpath)) if len(r) > 5]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows[1:]:
    a = agg.setdefault(r[ki], [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale[r[ui]]
sweeps = {k: v for k, v in agg.items() if "k_sweep" in k}
tot, tsw = sum(a[1] for a in agg.values()), sum(a[1] for a in sweeps.values())
md = [f"# ncu launch list, {tag}", "",
      "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python "
      "bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e` (config c4, 513^3, LODIE2).",
      "Per-launch times are cold-cache and serialised; compare shares with `roofline.kernel_ms` "
      f"in `bench_{tag}.jsonl`.", "",
      "| kernel | launches | total us | mean us | share of all kernel time | share of sweep time |",
      "|---|---|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    sh = f"{t / tsw * 100:.1f}%" if k in sweeps else "-"
    md.append(f"| `{k[:80]}` | {n} | {t:.1f} | {t / n:.1f} | {t / tot * 100:.1f}% | {sh} |")
md += ["", "Setup kernels (`k_coulomb_faces`, `k_classify_*`, `k_build_desc`, `k_seg_factors`) run "
       "once per problem / march, outside the timed step loop."]
open(os.path.join(out, f"launches_{tag}_summary.md"), "w").write("\n".join(md) + "\n")
if lpath != os.path.join(out, f"launches_{tag}.csv"):
    os.replace(lpath, os.path.join(out, f"launches_{tag}.csv"))

# full captures: c4 (always) and c3 (when the c3 capture exists)
def full_capture(rep, cname, nodes, cmd):
    if rep.endswith(".csv"):  # raw page exported on the box
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    g = lambda r, k: r[hdr.index(k)]
    md = [f"## {cname}", "", f"Command: `{cmd}` (LODIE2; one launch per sweep axis; cold-cache "
          "serialised replays).", "",
          "| kernel | duration us | DRAM read GB | DRAM write GB | DRAM busy % | SM busy % | warps "
          "active % | regs | thread-instr / node | fp64 pipe % | top stalls (cycles/issue) |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    for ax, r in enumerate(rows[2:5]):  # the capture holds K0, K1, K2 of one step, in order
        name = g(r, "Kernel Name")
        rd, wr = float(g(r, "dram__bytes_read.sum")), float(g(r, "dram__bytes_write.sum"))
        mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[units[hdr.index("dram__bytes_read.sum")]]
        traffic[str(ax)] = (rd + wr) * mult
        st = sorted([(float(r[i]) if r[i] else 0.0, hdr[i]) for i in stall], reverse=True)[:3]
        sts = ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {v:.1f}" for v, h in st)
        md.append(f"| `{name}` | {float(g(r, 'gpu__time_duration.sum')):.0f} | {rd * mult / 1e9:.3f} | "
                  f"{wr * mult / 1e9:.3f} | {float(g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                  f"{float(g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                  f"{float(g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} | "
                  f"{g(r, 'launch__registers_per_thread')} | "
                  f"{float(g(r, 'smsp__inst_executed.sum')) * 32 / nodes:.1f} | "
                  f"{float(g(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')):.1f} | {sts} |")
    md += ["", f"Algorithmic bytes per sweep launch: 16 B x {nodes:,} interior nodes = "
           f"{16 * nodes / 1e9:.3f} GB.", ""]
    return md, traffic


md = [f"# ncu --set full, {tag}", ""]
tr = json.load(open(os.path.join(out, "ncu_traffic.json")))
for cname, nodes, fname, cfg in (("c4-protein10000-513", NODES, "c4", ""),
                                 ("c3-protein2500-257", 16581375, "c3", " --config c3")):
    rep = os.path.join(go, f"{fname}_full_{tag}.ncu-rep")
    if not os.path.exists(rep):
        rep = os.path.join(go, f"{fname}_full_{tag}_raw.csv")
    if not os.path.exists(rep):
        continue
    cmd = (f"ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 9 -c 3 "
           f"python bench.py{cfg} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e")
    m, traffic = full_capture(rep, cname, nodes, cmd)
    md += m
    tr[cname] = traffic
md += ["Template arguments: `k_sweep_col<S, P, CN, LB>` (axes 0, 1: register-direct column "
       "tiles), `k_sweep_strided<S, P, CN, LB, RT>` (staged tiles) = rows per segment, "
       "segments per line, Crank-Nicolson, lines per tile, row tiles; `k_sweep_rowwarp<S, G>` "
       "(axis 2, one warp per line) = rows per segment, lanes per line."]
open(os.path.join(out, f"ncu_{tag}_summary.md"), "w").write("\n".join(md) + "\n")
tr["_note"] = f"dram read+write bytes per launch by sweep axis, ncu --set full captures {tag}"
json.dump(tr, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
print("\n".join(md))

# slab model lines (scripts/dev/collect_final.sh): add the split's beta and the per-rank totals
sm = os.path.join(go, f"slab_model_{tag}.jsonl")
if os.path.exists(sm):
    with open(os.path.join(out, f"slab_model_{tag}.jsonl"), "w") as f:
        for ln in open(sm):
            r = json.loads(ln)
            sizes = r["planes_per_rank"]
            r["beta"] = 0 if max(sizes) - min(sizes) <= 1 else 6
            r["total_ms"] = [round(a + b, 4) for a, b in zip(r["phaseA_ms"], r["phaseB_ms"])]
            f.write(json.dumps(r) + "\n")
            print(r["ranks"], r["beta"], sizes, "A", min(r["phaseA_ms"]), max(r["phaseA_ms"]), "B",
                  min(r["phaseB_ms"]), max(r["phaseB_ms"]), "slowest", max(r["total_ms"]))
