"""Shape-distance throughput: native solver vs the reference (cold memo), on the
golden random problems.  Runs in this container (needs /root/reference)."""
import json, sys, time
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ".")
from opsmith import shapedist as R
from opsmith.symexpr import Variable, parse_size
from paper_2410_23745_b200 import shapedist as S

gold = json.load(open("tests/golden/shapedist.json"))
vs = tuple(Variable(n) for n in ("C_out", "C_in", "H", "W")) + tuple(Variable(n, primary=False) for n in ("K", "s"))
vm = {v.name: v for v in vs}
probs = [([R.DimDesc(parse_size(s, vm), p, st) for s, p, st in q["current"]], [parse_size(t, vm) for t in q["inputs"]])
         for q in gold["problems"]]
mine = [([S.DimDesc(d.size, d.reduce_pure, d.strided) for d in c], t) for c, t in probs]
for name, mod, data in (("reference", R, probs), ("native", S, mine)):
    mod.clear_cache()
    t0 = time.perf_counter()
    for c, t in data:
        mod.shape_distance(c, t, True)
    dt = time.perf_counter() - t0
    print(f"{name}: {len(data)} problems cold in {dt*1e3:.1f} ms ({len(data)/dt:.0f}/s)")
