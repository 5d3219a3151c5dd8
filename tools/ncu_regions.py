"""Aggregate an ncu source-page CSV of k_raycast_pruned by code region
(function line ranges of raycast_core.cuh): stall samples and instructions."""
import csv
import sys
from collections import defaultdict

REGIONS = [(88, 145, 'ray_setup'), (148, 197, 'set_best'), (200, 242, 'load_helpers'),
           (252, 316, 'rare_block'), (333, 357, 'src_load'), (460, 487, 'store'),
           (891, 916, 'box_test'), (980, 1039, 'seed32'), (1047, 1143, 'cursor'),
           (1251, 1266, 'mma_instr'), (1276, 1313, 'mma_store'), (1319, 1342, 'mma_load/block'),
           (1345, 1349, 'spread4'), (1351, 1371, 'screen_nohit'), (1372, 1418, 'screen_hit'),
           (1530, 1712, 'kernel_main')]


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
