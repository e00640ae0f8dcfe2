"""Per-SASS-line stall samples of the first kernel in an ncu source-page CSV,
grouped into execution-count regions (a region = one role's loop body).

    python scripts/src_stalls.py src.csv [min_samples]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mins = int(sys.argv[2]) if len(sys.argv) > 2 else 5
start = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[start]
ci = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[start + 1:]:
    if len(r) < 3 or r[0] in ("Kernel Name", "Address"):
        break
    data.append(r)
S = ci["Warp Stall Sampling (All Samples)"]
reasons = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
tot = sum(int(r[S] or 0) for r in data)
print("instructions", len(data), "samples", tot)
for i, r in enumerate(data):
    n = int(r[S] or 0)
    if n < mins:
        continue
    rs = {h[6:]: int(r[ci[h]]) for h in reasons if int(r[ci[h]] or 0)}
    print(f"{i:5d} {n:5d} {r[ci['Instructions Executed']]:>8s} {r[ci['Source']].strip()[:70]:70s} {rs}")
