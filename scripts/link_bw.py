"""Host<->device copy bandwidth of this box (pinned memory, CUDA events):
H2D alone, D2H alone, and both directions at once on two streams -- the
ceiling of bench.py's e2e number (ResNet-18 moves ~328 MB up and ~346 MB
down per step).

    python scripts/link_bw.py [MB]
"""
import json
import sys

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = mb * (1 << 20)
h_up = torch.empty(n, dtype=torch.uint8).pin_memory()
h_dn = torch.empty(n, dtype=torch.uint8).pin_memory()
d_up = torch.empty(n, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def up():
    d_up.copy_(h_up, non_blocking=True)


def down():
    h_dn.copy_(d_dn, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        up()
    with torch.cuda.stream(s2):
        down()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_up, t_dn, t_both = timed(up), timed(down), timed(both)
print(json.dumps({"bytes": n, "h2d_gbs": n / t_up / 1e9, "d2h_gbs": n / t_dn / 1e9,
                  "bidirectional_gbs_each": n / t_both / 1e9}))
