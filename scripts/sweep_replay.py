"""Replay the candidate sweep's schedule on measured per-candidate device
times: N ranks claim candidates one at a time from the shared LPT order
(bench.py --workload sweep, sweep.StoreClaim), each rank's load is the sum of
its candidates' times; prints max/mean load and the implied 1 -> N speed-up
(device time only: no launch or host overhead is modelled).  Also the static
LPT plan (sweep.lpt_shard on predicted costs) for comparison.

    python scripts/sweep_replay.py gpurun_out/.../sweep_w1.log [ranks...]
"""
import heapq
import re
import sys

sys.path.insert(0, ".")


def load(path):
    t = {}
    for line in open(path):
        m = re.match(r"diag id=(\d+) device_us=([\d.]+)", line)
        if m:
            t[int(m.group(1))] = float(m.group(2)) * 1e-6
    return t


def dynamic(order, times, n):
    """Greedy list scheduling: the next claim goes to the rank that frees up first."""
    heap = [(0.0, r) for r in range(n)]
    loads = [0.0] * n
    for i in order:
        t, r = heapq.heappop(heap)
        loads[r] = t + times.get(i, 0.0)
        heapq.heappush(heap, (loads[r], r))
    return loads


def main():
    from bench import sweep_setup
    from paper_2410_23745_b200.sweep import lpt_order, lpt_shard
    times = load(sys.argv[1])
    ranks = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
    graphs, costs, _, _ = sweep_setup()
    order = lpt_order(costs)
    total = sum(times.values())
    print(f"{len(times)} candidates, {total:.3f} s device time")
    for n in ranks:
        d = dynamic(order, times, n)
        s = [sum(times.get(i, 0.0) for i in shard) for shard in lpt_shard(costs, n)]
        print(f"N={n}: dynamic LPT claims max/mean {max(d) / (total / n):.3f} (speed-up {total / max(d):.2f}x), "
              f"static LPT plan max/mean {max(s) / (total / n):.3f} (speed-up {total / max(s):.2f}x)")


if __name__ == "__main__":
    main()
