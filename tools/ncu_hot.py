"""Top warp-stall-sampled SASS instructions of an ncu report (dev tool):
python tools/ncu_hot.py <report.ncu-rep> [n]"""
import csv, subprocess, sys
rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
iS, iA = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_")]
data = []
for idx, r in enumerate(rows[1:]):
    if len(r) != len(h):
        continue
    s = int(r[iA] or 0)
    top = sorted(((int(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:2]
    data.append((s, idx, r[iS].strip(), top))
tot = sum(d[0] for d in data)
print(f"total samples {tot}")
for s, idx, src, top in sorted(data, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}%  #{idx:5d}  {src[:60]:60s} {top}")
