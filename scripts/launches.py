"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        seq.append((r[ki].split("(")[0].replace("void ", "")[:48], v / 1e3))
    return seq


if __name__ == "__main__":
    seq = load(sys.argv[1])
    tot = sum(t for _, t in seq)
    print(f"launches {len(seq)}  total {tot / 1e3:.2f} ms (serialised, cold)")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, t in seq:
        agg[n][0] += 1
        agg[n][1] += t
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
        print(f"{t / 1e3:8.2f} ms {100 * t / tot:5.1f}%  n={n:4d}  {k}")
    if len(sys.argv) > 2:
        a = int(sys.argv[2])
        for i, (n, t) in enumerate(seq[a:a + int(sys.argv[3])]):
            print(a + i, f"{t:8.1f}us", n)
