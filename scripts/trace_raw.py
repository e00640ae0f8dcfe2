"""Raw per-CTA event list (MMA-warp kinds) of one launch of a SYNO_TC_TRACE file."""
import sys
sys.path.insert(0, "scripts")
from trace_view import launches  # noqa: E402

NAMES = {0: "start", 1: "A-issue", 2: "B-issue", 3: "A-ready", 4: "B-ready", 5: "acc-free", 6: "issued",
         7: "epi-full", 8: "epi-done", 9: "decoded", 10: "committed", 11: "win-issued"}
path, sel = sys.argv[1], int(sys.argv[2])
kinds = set(map(int, sys.argv[3].split(","))) if len(sys.argv) > 3 else None
tmax = int(sys.argv[4]) if len(sys.argv) > 4 else 3
head, evs = list(launches(path))[sel]
t0 = min(e[0] for e in evs)
ctas = sorted({e[4] for e in evs})
print(head)
for e in sorted(evs):
    if (kinds is None or e[1] in kinds) and e[2] < tmax:
        print(f"{(e[0]-t0)/1965.0:7.3f}  cta{ctas.index(e[4])} t{e[2]} {NAMES[e[1]]:10s} w{e[3]}")
