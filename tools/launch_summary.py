"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel time and share (tools only).  Cold-cache serialised per-launch
times: compare SHARES with the live bench, not absolutes."""
import collections
import csv
import sys


def main(path, steps):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    name_i, val_i = h.index("Kernel Name"), h.index("Metric Value")
    t = collections.Counter()
    n = collections.Counter()
    for r in rows[1:]:
        k = r[name_i].split("(")[0][:70]
        t[k] += float(r[val_i]) / 1e6
        n[k] += 1
    # parameter initialisation (init_params before the first step: random
    # init, and the codec encode of the host masters) is not part of any
    # step: listed apart, out of the shares
    setup = {k for k in t if "k_init_normal" in k or "k_encode" in k}
    tot = sum(v for k, v in t.items() if k not in setup)
    for k, v in t.most_common():
        if k not in setup:
            print(f"{v / steps:9.2f} ms/step {100 * v / tot:5.1f}%  n={n[k]:5d}  {k}")
    for k in setup:
        print(f"{t[k]:9.2f} ms total (setup, not a step)  n={n[k]:5d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
