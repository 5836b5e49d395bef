"""Group an ncu SASS source-page CSV into contiguous regions of equal
execution count (tools only): where the warp instructions go."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ie = h.index("Instructions Executed")
    lines = [(r[1].strip(), int(r[ie] or 0)) for r in rows[2:]]
    ranges, cur = [], None
    for i, (s, n) in enumerate(lines):
        parts = s.split()
        op = (parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (parts[0] if parts else "")).split(".")[0]
        if cur and cur[0] == n:
            cur[2][op] += 1
            cur[3] = i
        else:
            if cur:
                ranges.append(cur)
            cur = [n, i, collections.Counter({op: 1}), i]
    ranges.append(cur)
    tot = sum(n for _, n in lines)
    ranges.sort(key=lambda r: -r[0] * sum(r[2].values()))
    for n, a, c, b in ranges[:top]:
        w = n * sum(c.values())
        print(f"lines {a}-{b} x{n} = {w / 1e6:.1f}M ({100 * w / tot:.1f}%) {dict(c.most_common(7))}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
