"""Summarise an ncu source-page CSV (--print-source sass) by runs of equal
execution count: stall share and dominant stall reasons per run."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
iS, iW, iE = col["Source"], col["Warp Stall Sampling (All Samples)"], col["Instructions Executed"]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[iW] or 0) for r in data)
runs, cur = [], None
for k, r in enumerate(data):
    e = r[iE]
    if not (cur and cur["e"] == e):
        cur = {"e": e, "k": k, "w": 0.0, "n": 0, "ops": collections.Counter(),
               "why": collections.Counter()}
        runs.append(cur)
    cur["w"] += float(r[iW] or 0)
    cur["n"] += 1
    src = r[iS].strip().split()
    if src:
        cur["ops"][src[1] if src[0].startswith("@") and len(src) > 1 else src[0]] += 1
    for h in reasons:
        cur["why"][h[6:]] += float(r[col[h]] or 0)
print(f"total samples {tot:.0f}")
for run in sorted(runs, key=lambda x: -x["w"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    why = ", ".join(f"{k}:{v / max(run['w'], 1) * 100:.0f}%" for k, v in run["why"].most_common(3))
    print(f"line {run['k']:5d} exec {run['e']:>9s} n={run['n']:4d} share {run['w'] / tot * 100:5.1f}%"
          f"  [{why}]  {dict(run['ops'].most_common(5))}")
