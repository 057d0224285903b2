"""Attribute ncu SASS-page samples / executed instructions to source lines.

    nvdisasm -g <cubin> > all.txt
    ncu -i rep --page source --csv --print-source sass --kernel-id ::regex:.*:N > sass.csv
    python scripts/sass_lines.py all.txt sass.csv <mangled kernel name> [outer]

`outer` attributes inlined code to the kernel-body line that inlined it.
"""
import csv
import re
import sys
from collections import defaultdict

allf, sassf, fn = sys.argv[1:4]
outer = len(sys.argv) > 4
lines = open(allf).read().split("\n")
start = None
for i, l in enumerate(lines):
    if l.startswith(fn + ":"):
        start = i
        break
off2line = {}
cur = None
pat = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
for l in lines[start + 1:]:
    if l and not l[0].isspace() and not l.startswith(".text") and l.endswith(":") and not l.startswith("."):
        if not l.startswith(fn):
            break
    m = pat.search(l)
    if m:
        f, ln = m.group(1), int(m.group(2))
        if outer and m.group(4):
            # take the last 'inlined at' (outermost)
            allm = re.findall(r'inlined at "([^"]+)", line (\d+)', l)
            f, ln = allm[-1][0], int(allm[-1][1])
        cur = (f.split("/")[-1], ln)
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        off2line[int(m.group(1), 16)] = (cur, m.group(2).strip())
rows = list(csv.reader(open(sassf)))
hdr = rows[1]
ia = hdr.index("Address")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) > iex and r[ia].startswith("0x")]
base = min(int(r[ia], 16) for r in data)
agg = defaultdict(lambda: [0, 0])
tot = [0, 0]
for r in data:
    off = int(r[ia], 16) - base
    key = off2line.get(off, (("?", 0), ""))[0]
    s, e = int(r[isamp] or 0), int(r[iex] or 0)
    agg[key][0] += s
    agg[key][1] += e
    tot[0] += s
    tot[1] += e
print(f"total samples {tot[0]}, warp-instr {tot[1]}")
for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:45]:
    print(f"{k[0]}:{k[1]:5d}  samples {100*s/tot[0]:5.1f}%  instr {100*e/tot[1]:5.1f}%")

# coarse phases of k_sweep_strided (line ranges in sweep.cu; pbg_internal.cuh = flow)
def phase(k):
    f, ln = k
    if f == "pbg_internal.cuh" or (f == "sweep.cu" and 68 <= ln <= 73):
        return "flow"
    if f != "sweep.cu":
        return "other:" + f
    for name, a, b in (("solve", 75, 230), ("stage", 289, 412), ("pro", 413, 449),
                       ("solve", 450, 557), ("store", 558, 640)):
        if a <= ln <= b:
            return name
    return "other"


ph = defaultdict(lambda: [0, 0])
for k, (s, e) in agg.items():
    ph[phase(k)][0] += s
    ph[phase(k)][1] += e
for k, (s, e) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
    print(f"PHASE {k:24s} samples {100*s/tot[0]:5.1f}%  instr {100*e/tot[1]:5.1f}%")
