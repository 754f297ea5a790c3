"""Summarise an ncu --page source --print-source sass CSV: samples per instruction region."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    his = [i for i, r in enumerate(rows) if r and 'Source' in r and 'Address' in r]
    h = rows[his[0]]
    data = rows[his[0] + 1:his[1] if len(his) > 1 else None]
    return h, [r for r in data if len(r) == len(h)]


def main(path, top=40, lo=0, hi=None):
    h, data = load(path)
    si = h.index('Warp Stall Sampling (All Samples)')
    ie = h.index('Instructions Executed')
    f = lambda x: float(x) if x not in ('', None) else 0.0
    tot = sum(f(r[si]) for r in data)
    print(f"samples {tot:.0f} instructions {sum(f(r[ie]) for r in data):.0f} sass {len(data)}")
    for a in range(0, len(data), 100):
        b = min(a + 100, len(data))
        s = sum(f(r[si]) for r in data[a:b])
        n = sum(f(r[ie]) for r in data[a:b])
        ex = collections.Counter(r[ie] for r in data[a:b]).most_common(1)[0][0]
        if s > 0:
            print(f"{a:5d}-{b:5d} {s:5.0f} ({100 * s / tot:4.1f}%) instr {n:9.0f} exec~{ex}")
    cols = [h.index(c) for c in ('stall_long_sb', 'stall_wait', 'stall_short_sb', 'stall_selected',
                                 'stall_branch_resolving', 'stall_barrier', 'stall_no_inst', 'stall_mio')]
    print("idx samples exec | long_sb wait short_sb selected branch barrier no_inst mio")
    hi = len(data) if hi is None else hi
    ranked = sorted(range(lo, hi), key=lambda k: -f(data[k][si]))[:top]
    for k in sorted(ranked):
        r = data[k]
        print(f"{k:5d} {f(r[si]):4.0f} {r[ie]:>6s} {r[1][:60]:60s} " + " ".join(f"{f(r[c]):3.0f}" for c in cols))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
