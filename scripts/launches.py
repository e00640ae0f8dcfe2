"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) > h.index("Metric Value")]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
last = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
seq = [(r[ki][:48], float(r[vi].replace(",", "")), r[gi] if gi is not None else "") for r in data]
seq = [s for s in seq if "k1_build" not in s[0]][-last:]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for n, v, g in seq:
    tot[n] += v
    cnt[n] += 1
T = sum(tot.values())
print(f"{len(seq)} launches, {T/1e3:.1f} us total (ncu-serialised)")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v/1e3:9.1f} us {100*v/T:5.1f}%  n={cnt[k]:4d}  {k}")
if len(sys.argv) > 3:
    for n, v, g in sorted(seq, key=lambda s: -s[1])[: int(sys.argv[3])]:
        print(f"{v/1e3:8.1f} {n} {g}")
