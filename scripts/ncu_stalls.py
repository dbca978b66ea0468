"""Summarise an `ncu --page source --csv --print-source sass` dump: stall samples by reason and
the hottest SASS instructions with their dominant stall reasons.
python scripts/ncu_stalls.py dump.csv [top_n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {r: 0 for r in reasons}
body = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    st = {k: int(r[ix[k]] or 0) for k in reasons}
    for k in reasons:
        tot[k] += st[k]
    body.append((s, r[ix["Address"]], r[ix["Source"]].strip(), st))
allsum = sum(tot.values())
print("total samples", allsum)
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v:
        print(f"  {k:24s} {v:8d} {100 * v / allsum:5.1f}%")
print()
for i, (s, a, src, st) in enumerate(body):
    body[i] = (s, i, a, src, st)
for s, i, a, src, st in sorted(body, key=lambda x: -x[0])[:top]:
    tops = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{s:7d} {100 * s / allsum:5.1f}%  #{i:5d} {src[:60]:60s} " + " ".join(f"{k[6:]}={v}" for k, v in tops if v))
