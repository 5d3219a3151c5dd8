"""ncu launch list (--metrics gpu__time_duration.sum --csv) -> compact CSV
(launch_id, kernel, ns) and a per-kernel share table for profiles/."""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)             # drop the parameter list
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"at::|cuda::|::detail|_GLOBAL__N__[0-9a-f_]+", "", name)
    return name[:90]


def main(src, out_csv, out_txt, title=""):
    rows = []
    with open(src) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        rows.append((int(r["ID"]), short(r["Kernel Name"]), ns))
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch_id", "kernel", "gpu__time_duration_ns"])
        for row in rows:
            w.writerow([row[0], row[1], int(row[2])])
    agg = defaultdict(lambda: [0, 0.0])
    for _, k, ns in rows:
        agg[k][0] += 1
        agg[k][1] += ns
    tot = sum(v[1] for v in agg.values()) or 1.0
    with open(out_txt, "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        if title:
            f.write(title.rstrip() + "\n")
        f.write("\n")
        for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
            f.write(f"{k[:60]:60s} n={n:5d} total={ns / 1e6:9.3f} ms share={ns / tot * 100:5.1f}%\n")
    print(open(out_txt).read())


if __name__ == "__main__":
    main(*sys.argv[1:])
