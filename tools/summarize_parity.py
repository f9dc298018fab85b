"""Summarise a parity report (gpurun_out/parity.jsonl, written by the -m gpu
suite with PN_PARITY_LOG set) as markdown: per test, every check with its
worst err/(rtol*S), bitwise mismatch count, norm-wise / relative error, and
the excused near-tie counts with their caps."""
import json
import sys
from collections import OrderedDict

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/parity.jsonl"
rows = [json.loads(l) for l in open(src)]
by = OrderedDict()
for r in rows:
    by.setdefault(r["test"].split("::", 1)[-1], []).append(r)
print("# GPU parity report (every check of the -m gpu suite)\n")
print("Columns: `worst` = max |gpu - oracle| / bound (must be <= 1; element-wise rtol*S, or the net-level")
print("measured-incoming-error bound of tests/netcheck.py); bitwise = mismatching elements (must be 0);")
print("mask / argmax = excused near-ties (each listed in the jsonl) and their cap.\n")
for t, rs in by.items():
    print(f"## {t}\n")
    print("| check | kind | result | n |")
    print("|---|---|---|---:|")
    for r in rs:
        k = r["kind"]
        if k == "elementwise":
            res = f"worst {r['worst_err_over_rtolS']:.3g} (rtol {r['rtol']:g})"
        elif k == "bitwise":
            res = f"{r['mismatches']} mismatches"
        elif k in ("mask", "argmax"):
            res = f"{r['excused']} near-ties excused (cap {r['cap']})"
        elif k == "relative":
            res = f"rel {r['rel_err']:.3g} (bound {r['bound']:g})"
        else:
            res = f"rel {r['rel_err']:.3g}" + (f" (bound {r['bound']:g})" if "bound" in r else "")
        print(f"| {r['check']} | {k} | {res} | {r.get('n', '')} |")
    print()
