"""Aggregate an ncu source-page SASS CSV (tools only): dynamic warp-level
instruction counts and stall samples by opcode class."""
import csv
import collections
import re
import sys


def main(path, n_units=None):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    iexe, thr, samp = h.index("Instructions Executed"), h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ops = collections.Counter()
    tops = collections.Counter()
    st = collections.Counter()
    tot = ttot = stot = 0
    for r in rows[2:]:
        src = r[1].strip()
        m = re.match(r'(?:@!?U?P\w+\s+)?([A-Z0-9_]+)', src)
        if not m:
            continue
        op = m.group(1)
        n = int(r[iexe] or 0)
        t = int(r[thr] or 0)
        s = int(r[samp] or 0)
        ops[op] += n
        tops[op] += t
        st[op] += s
        tot += n
        ttot += t
        stot += s
    print(f"total warp inst {tot:.4g}  thread inst {ttot:.4g}  samples {stot}")
    for op, n in ops.most_common(40):
        per = f"  {n / n_units:.3f}/unit" if n_units else ""
        print(f"{op:10s} {n:12d} {100 * n / tot:5.1f}%  thr/warp {tops[op] / max(n, 1):5.1f}  stall% {100 * st[op] / max(stot, 1):5.1f}{per}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
