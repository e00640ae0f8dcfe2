"""Render the SM-0 event log written by SYNO_TC_TRACE=<file> (tc_gemm).

    python scripts/trace_view.py trace.txt [launch_index|-1] [mode]
Event kinds: 0 start, 1 prod A issue, 2 prod B issue, 3 mma A ready, 4 mma B
ready, 5 mma acc free, 6 mma tile issued, 7 epi acc full, 8 epi drained.
"""
import collections
import sys

NAMES = {0: "start", 1: "A-issue", 2: "B-issue", 3: "A-ready", 4: "B-ready", 5: "acc-free", 6: "issued",
         7: "epi-full", 8: "epi-done", 9: "decoded", 10: "committed", 11: "win-issued"}


def launches(path):
    cur = None
    for line in open(path):
        if line.startswith("launch"):
            cur = [line.strip(), []]
            yield cur
        elif cur is not None:
            t, k, tile, w, cta = map(int, line.split())
            cur[1].append((t, k, tile, w, cta))


def main():
    path = sys.argv[1]
    sel = int(sys.argv[2]) if len(sys.argv) > 2 else -1
    mode = sys.argv[3] if len(sys.argv) > 3 else None
    ls = [l for l in launches(path) if mode is None or f"mode={mode}" in l[0]]
    head, evs = ls[sel]
    print(head, f"({len(evs)} events)")
    t0 = min(e[0] for e in evs)
    by = collections.defaultdict(list)
    for e in sorted(evs):
        by[e[4]].append(e)
    for cta, es in by.items():
        print(f"-- CTA {cta}")
        tiles = collections.defaultdict(dict)
        for t, k, tile, w, _ in es:
            d = tiles[tile]
            us = (t - t0) / 1965.0
            if k in (2, 4):
                d.setdefault(NAMES[k], []).append(us)
            else:
                d.setdefault(NAMES[k], us)
        for tile in sorted(tiles):
            d = tiles[tile]
            br = d.get("B-ready", [])
            gaps = [b - a for a, b in zip(br, br[1:])]
            print(f"  t{tile}: A-issue {d.get('A-issue', -1):6.2f} A-ready {d.get('A-ready', -1):6.2f} "
                  f"acc-free {d.get('acc-free', -1):6.2f} B-ready {br[0] if br else -1:6.2f}..{br[-1] if br else -1:6.2f} "
                  f"(n={len(br)}, med gap {sorted(gaps)[len(gaps)//2] if gaps else 0:.3f}) issued {d.get('issued', -1):6.2f} "
                  f"epi {d.get('epi-full', -1):6.2f}-{d.get('epi-done', -1):6.2f}")


if __name__ == "__main__":
    main()
