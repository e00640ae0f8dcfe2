"""Median window-issue period (kind 11 events) and tile period of the first
launch in SYNO_TC_TRACE files, in SM cycles.

    python scripts/trace_period.py trace_*.txt
"""
import statistics
import sys

for path in sys.argv[1:]:
    evs, cur = [], None
    for line in open(path):
        if line.startswith("launch"):
            if cur is not None:
                break
            cur = line.strip()
        elif cur is not None:
            evs.append(tuple(map(int, line.split())))
    by = {}
    for t, k, tile, w, cta in evs:
        by.setdefault(cta, []).append((t, k, tile, w))
    gaps, tiles = [], []
    for cta, es in by.items():
        es.sort()
        win = [e for e in es if e[1] == 11]
        gaps += [b[0] - a[0] for a, b in zip(win, win[1:]) if b[2] == a[2]]
        done = [e[0] for e in es if e[1] == 6]
        tiles += [b - a for a, b in zip(done, done[1:])]
    print(f"{path}: window period {statistics.median(gaps):.0f} cyc, tile period {statistics.median(tiles):.0f} cyc"
          if gaps and tiles else f"{path}: no events")
