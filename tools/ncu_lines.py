"""Aggregate an ncu `--page source --csv --print-source cuda,sass` dump per
CUDA source line: warp-stall samples and warp instructions executed."""
import csv
import sys
from collections import defaultdict


def _int(v):
    try:
        return int(v)
    except ValueError:
        return 0


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    fname = None
    hdr = None
    agg = defaultdict(lambda: [0, 0, "", defaultdict(int)])
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or r[0] == "" or len(r) < 8:
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        samp = _int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = _int(r[hdr.index("Instructions Executed")])
        a = agg[(fname, ln)]
        a[0] += samp
        a[1] += inst
        a[2] = r[1][:60]
        for ci, name in enumerate(hdr):
            if name.startswith("stall_") and "Not Issued" not in name:
                a[3][name[6:]] += _int(r[ci])
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i:.3e}")
    tot_st = defaultdict(int)
    for v in agg.values():
        for k, c in v[3].items():
            tot_st[k] += c
    print("stalls:", ", ".join(f"{k} {c / tot_s:.1%}" for k, c in
                              sorted(tot_st.items(), key=lambda kv: -kv[1])[:8]))
    for (f, ln), (s, i, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        tops = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        why = " ".join(f"{k}:{c / max(s, 1):.0%}" for k, c in tops)
        print(f"{s / tot_s:6.1%} {i / tot_i:6.1%}  {f}:{ln:<5d} {src:60s} [{why}]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
