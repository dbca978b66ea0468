"""Per-source-line warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r][0]
h = rows[hi]
S = h.index("Warp Stall Sampling (All Samples)")
E = h.index("Instructions Executed")
stalls = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
lines = []
for r in rows[hi + 1:]:
    if len(r) > S and r[0].isdigit() and r[S].isdigit():
        top = sorted(((int(r[i]) if r[i].isdigit() else 0, h[i][6:]) for i in stalls), reverse=True)[:2]
        lines.append((int(r[S]), int(r[E]) if r[E].isdigit() else 0, r[0], r[1].strip()[:80], top))
tot = sum(x[0] for x in lines)
print("samples", tot, "instructions", sum(x[1] for x in lines))
for smp, ins, ln, src, top in sorted(lines, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{smp:6d} {100 * smp / tot:5.1f}% ins={ins:9d} L{ln}: {src}  {top}")
