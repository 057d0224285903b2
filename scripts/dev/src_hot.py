"""Per-CUDA-line instruction and stall-sample shares from an ncu source-page CSV
(--page source --csv --print-source cuda,sass) -- dev tool."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None; per = collections.Counter(); samp = collections.Counter(); src = {}; hdr = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': print(r[1]); continue
    if r[0] == 'Line No':
        hdr = r; iE = hdr.index('Instructions Executed'); iS = hdr.index('Warp Stall Sampling (All Samples)'); continue
    if hdr is None or not r[0].strip(): continue
    key = (cur, int(r[0])); src[key] = r[1]
    try:
        per[key] += int(r[iE]); samp[key] += int(r[iS])
    except ValueError:
        pass
tot = sum(per.values()); ts = sum(samp.values())
print('total warp instr', tot, 'samples', ts)
for k, v in per.most_common(n):
    print(f"{k[0][:14]:14s}:{k[1]:5d} {v:9d} {100*v/tot:5.1f}% samp {100*samp[k]/max(1,ts):5.1f}%  {src[k].strip()[:80]}")
