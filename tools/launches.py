"""Summarise an ncu --metrics gpu__time_duration.sum launch list (median per kernel)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches_tf32.csv")))
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.append((d["Kernel Name"][:60], float(d["Metric Value"])))
seen = {}
for k, v in out:
    seen.setdefault(k, []).append(v)
# one SGD update per step
steps = next((len(v) for k, v in seen.items() if 'sgd_update' in k), max(len(v) for v in seen.values()))
tot = 0.0
for k, v in sorted(seen.items(), key=lambda kv: -sorted(kv[1])[len(kv[1]) // 2] * len(kv[1])):
    m = sorted(v)[len(v) // 2]
    per = m * len(v) / steps
    tot += per
    print(f"{m / 1000:8.2f} us  x{len(v):3d}  {k}")
print(f"sum of medians per step ~ {tot / 1000:.1f} us")
