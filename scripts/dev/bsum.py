"""Summarise bench JSON lines: workload, ms/step, G updates/s, per-axis kernel ms, step frac."""
import json
import sys

for f in sys.argv[1:]:
    for l in open(f):
        l = l.strip()
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        r = d.get("roofline") or {}
        e = d.get("e2e") or {}
        km = r.get("kernel_ms")
        print(d["config"].get("workload"), f"{d['ms_per_step']:.4f} ms", f"{d['value']/1e9:.2f} G/s",
              [round(x * 1000, 1) for x in km] if km else None, "step_frac", r.get("step_frac"),
              "e2e", round(e.get("value", 0) / 1e9, 2) if e else None)
