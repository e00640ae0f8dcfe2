"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return None


rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
si, ei, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
data = [r for r in rows[hi + 1:] if len(r) > si and num(r[si])]
tot = sum(num(r[si]) for r in data)
ninst = sum(num(r[ei]) or 0 for r in rows[hi + 1:] if len(r) > ei)
print(f"samples {tot:.0f}, warp-instructions executed {ninst:.0f}")
for r in sorted(data, key=lambda r: -num(r[si]))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{r[si]:>6} {num(r[si]) / tot * 100:5.1f}%  exec={r[ei]:>8}  {r[src].strip()[:90]}")
