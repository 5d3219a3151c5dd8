"""Aggregate an ncu source-page CSV of k_raycast_pruned by code region
(function line ranges of raycast_core.cuh): stall samples and instructions."""
import csv
import sys
from collections import defaultdict

import os
import re

# region = [first line of the named function .. first line of the next one)
ANCHORS = [("ray_setup", r"void ray_setup\("), ("set_best", r"void ray_set_best\("),
           ("load_helpers", r"void load_rec\("), ("rare_block", r"void ray_rare_block\("),
           ("ray_power", r"double ray_power\("), ("src_load", r"^struct SrcExplicit"),
           ("philox/mc", r"void philox4x32_10\("), ("store", r"void ray_store\("),
           ("screen_tile(other)", r"^struct WarpCounters"), ("box_test(other)", r"bool ray_needs_box\("),
           ("box_test", r"bool ray_needs_box32_ch_d2\("), ("ray_needs", r"bool ray_needs\("),
           ("seed64", r"void seed_tile\("), ("seed32", r"void seed_tile32\("),
           ("cursor", r"^struct TreeCursor"), ("remap", r"int remap_max\(\)"),
           ("mma_instr", r"void mma_tf32\("), ("mma_store", r"void mma_store_a\("),
           ("mma_load/block", r"void mma_load_a\("), ("spread4", r"uint32_t spread4\("),
           ("screen_nohit", r"void screen_tile_mma\("), ("screen_hit", r"Some pair passed: recompute"),
           ("hsweep", r"k_raycast_hsweep"), ("kernel_main", r"\s+k_raycast_pruned\(Src src"),
           ("coop", r"^constexpr int WIDE = 32")]


def regions():
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2405_10050_b200",
                       "csrc", "raycast_core.cuh")
    lines = open(src).read().splitlines()
    starts = []
    for name, pat in ANCHORS:
        rx = re.compile(pat)
        for n, ln in enumerate(lines, 1):
            if rx.search(ln):
                starts.append((n, name))
                break
    starts.sort()
    out = []
    for k, (n, name) in enumerate(starts):
        end = starts[k + 1][0] - 1 if k + 1 < len(starts) else len(lines)
        out.append((n, end, name))
    return out


REGIONS = regions()


def _int(v):
    try:
        return int(v)
    except ValueError:
        return 0


def main(path, nwarps, top=45):
    rows = list(csv.reader(open(path)))
    fname = None
    hdr = None
    agg = defaultdict(lambda: [0, 0])
    lines = defaultdict(lambda: [0, 0, ''])
    for r in rows:
        if len(r) == 2 and r[0] == 'File Path':
            fname = r[1].rsplit('/', 1)[-1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            si = hdr.index('Warp Stall Sampling (All Samples)')
            ii = hdr.index('Instructions Executed')
            continue
        if hdr is None or not r or r[0] == '':
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        s = _int(r[si])
        i = _int(r[ii])
        reg = fname
        if fname == 'raycast_core.cuh':
            reg = 'core:other'
            for a, b, n in REGIONS:
                if a <= ln <= b:
                    reg = n
        agg[reg][0] += s
        agg[reg][1] += i
        lines[(fname, ln)][0] += s
        lines[(fname, ln)][1] += i
        lines[(fname, ln)][2] = r[1][:70]
    ts = sum(v[0] for v in agg.values())
    ti = sum(v[1] for v in agg.values())
    print('total samples', ts, 'instr', ti, 'per warp', ti / nwarps)
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f'{k:22s} samples {v[0] / ts:6.1%}  instr {v[1] / ti:6.1%}  instr/warp {v[1] / nwarps:8.0f}')
    print()
    for (f, ln), v in sorted(lines.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f'{v[1] / ti:6.1%} {v[0] / ts:6.1%} {f}:{ln} {v[2]}')


if __name__ == '__main__':
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 31250.0)
