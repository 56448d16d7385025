"""Per-instruction stall attribution from `ncu --page source --csv --print-source sass`."""
import csv
import sys
from collections import Counter


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    I = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[I['Address']].startswith('0x')]
    def n(r, k):
        v = r[I[k]]
        return int(v) if v.isdigit() else 0
    cols = ['stall_mio', 'stall_long_sb', 'stall_short_sb', 'stall_barrier', 'stall_lg', 'stall_wait', 'stall_math', 'stall_selected']
    tot = sum(n(r, 'Warp Stall Sampling (All Samples)') for r in data)
    print('total samples', tot, {c: sum(n(r, c) for r in data) for c in cols})
    byop = Counter()
    for r in data:
        toks = r[I['Source']].split()
        op = toks[1] if toks and toks[0].startswith('@') else (toks[0] if toks else '')
        byop[op.split('.')[0]] += n(r, 'Warp Stall Sampling (All Samples)')
    print('by opcode', byop.most_common(12))
    for r in sorted(data, key=lambda r: -n(r, 'Warp Stall Sampling (All Samples)'))[:top]:
        print(n(r, 'Warp Stall Sampling (All Samples)'), r[I['Address']][-5:], r[I['Source']][:60],
              {c: n(r, c) for c in cols if n(r, c)})


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
