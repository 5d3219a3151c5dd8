"""Summarise an ncu report (raw page) into the numbers profiles/ keeps."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_bytes.sum", "L2 traffic"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__inst_executed_pipe_tma.sum", "TMA instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def main(rep):
    hdr, units, data = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    for row in data:
        name = row[col["Kernel Name"]] if "Kernel Name" in col else "?"
        print(f"kernel: {name[:140]}")
        for key, label in KEYS:
            if key in col:
                print(f"  {label:30s} {row[col[key]]:>18s} {units[col[key]]}")
        stalls = [(h[len("smsp__pcsamp_warps_issue_stalled_"):], float(row[col[h]] or 0))
                  for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued")]
        tot = sum(v for _, v in stalls) or 1.0
        top = sorted(stalls, key=lambda kv: -kv[1])[:6]
        print("  stall samples: " + ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
