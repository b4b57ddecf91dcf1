#!/usr/bin/env python
"""Summarises an `ncu --page source --csv --print-source sass` export: stall
reasons overall, and the hottest SASS addresses (diagnostic helper)."""
import csv
import sys


def main(path, top=40, lo=None, hi=None):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
    base = int(data[0][ix['Address']], 16)
    tot = {s: 0 for s in stalls}
    recs = []
    for r in data:
        a = int(r[ix['Address']], 16) - base
        st = {s: int(r[ix[s]]) for s in stalls if r[ix[s]].isdigit() and int(r[ix[s]])}
        for s, v in st.items():
            tot[s] += v
        n = int(r[ix['# Samples']]) if r[ix['# Samples']].isdigit() else 0
        ex = int(r[ix['Instructions Executed']]) if r[ix['Instructions Executed']].isdigit() else 0
        recs.append((a, n, ex, r[ix['Source']].strip(), st))
    print("total samples:", sum(tot.values()))
    print(sorted(((k[6:], v) for k, v in tot.items() if v), key=lambda x: -x[1]))
    for a, n, ex, src, st in sorted(recs, key=lambda x: -x[1])[:top]:
        print(f"{n:6d} {a:#7x} exec={ex:8d} {src[:60]:60s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
