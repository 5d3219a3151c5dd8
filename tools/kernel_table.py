"""Per-kernel table from an ncu CSV (--csv --print-units base, metrics
below): device time, DRAM bytes and achieved GB/s against the measured HBM
peak, FP64 / FMA / tensor pipe utilisation.  usage:
  python tools/kernel_table.py gpurun_out/kernels.csv > profiles/r1_kernel_table.txt"""
import csv
import json
import os
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = defaultdict(lambda: defaultdict(float))
    for r in rows[1:]:
        if r[ix["Metric Name"]] not in METRICS:
            continue
        full = r[ix["Kernel Name"]].replace("(anonymous namespace)::", "")
        full = full.replace("<unnamed>::", "").replace("void ", "").replace("vr::", "")
        base = full.split("(")[0]
        # kernel<d> (the first template argument is the dimension), plus the
        # tensor-core flag of the pruned kernel and the ray source
        name = base.split("<")[0].strip()
        if "<" in base:
            targs = base[base.index("<") + 1:].split(",")
            name += "<" + targs[0].strip(" >") + ">"
            if name.startswith("k_raycast_pruned"):
                name += " mma" if targs[-1].strip(" >") == "1" else " ffma2"
            if "SrcMC" in base:
                name += " MC"
        key = (r[ix["ID"]], name)
        try:
            agg[key][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            pass
    per = defaultdict(lambda: defaultdict(float))
    for (_, name), m in agg.items():
        t = m["gpu__time_duration.sum"]
        p = per[name]
        p["n"] += 1
        p["t"] += t
        p["bytes"] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        for k in METRICS[3:]:
            p[k] += m[k] * t
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
    hbm = peaks.get("hbm_gbs", 6454.6)
    tot = sum(p["t"] for p in per.values())
    print(f"ncu {', '.join(METRICS)} (cold-cache, serialised); HBM peak {hbm} GB/s measured")
    print(f"{'kernel':40s} {'n':>4s} {'ms':>9s} {'share':>6s} {'GB/s':>8s} {'%HBM':>5s} "
          f"{'fp64%':>6s} {'fma%':>5s} {'tens%':>6s} {'warps%':>6s}")
    for name, p in sorted(per.items(), key=lambda kv: -kv[1]["t"]):
        t = p["t"]
        gbs = p["bytes"] / t if t else 0.0  # ns -> bytes/ns = GB/s
        w = lambda k: p[k] / t if t else 0.0  # noqa: E731
        print(f"{name[:40]:40s} {int(p['n']):4d} {t / 1e6:9.3f} {100 * t / tot:5.1f}% {gbs:8.1f} "
              f"{100 * gbs / hbm:5.1f} {w(METRICS[3]):6.1f} {w(METRICS[4]):5.1f} "
              f"{w(METRICS[5]):6.1f} {w(METRICS[6]):6.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
