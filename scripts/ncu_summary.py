"""Summarise an `ncu --set full` raw CSV of one workload's dominant-kernel
launches into profiles/<name>.txt and its entry of profiles/traffic.json
(mean DRAM bytes per launch, keyed by bench workload and kernel class).

    python scripts/ncu_summary.py raw.csv profiles/r02_ncu_tc_gemm_resnet18.txt resnet18 tc_gemm "first step"
"""
import csv
import json
import os
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def main(src, dst, workload="resnet18", kclass="tc_gemm", what="first step"):
    rows = list(csv.reader(open(src)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name, scale_to=1):
        i = col[name]
        return float(r[i].replace(",", "")) * UNIT.get(units[i], 1) / scale_to

    out = []
    for r in data:
        out.append(dict(name=r[col["Kernel Name"]], us=val(r, "gpu__time_duration.sum"),
                        tensor=val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                        sm=val(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                        dram=val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")))
    n = len(out)
    mean = lambda k: sum(o[k] for o in out) / n
    lines = [f"ncu --set full of {n} {kclass} launches of the {workload} bench ({what}; cold L2 per replay)",
             f"launches {n}; mean duration {mean('us'):.1f} us; mean tensor-pipe active {mean('tensor'):.1f} %; "
             f"mean SM throughput {mean('sm'):.1f} %; mean DRAM bytes/launch {mean('dram') / 1e6:.2f} MB", "",
             f"{'us':>8} {'tensor%':>8} {'sm%':>6} {'DRAM MB':>8}  kernel"]
    for o in out:
        lines.append(f"{o['us']:8.1f} {o['tensor']:8.1f} {o['sm']:6.1f} {o['dram'] / 1e6:8.2f}  {o['name'][:60]}")
    open(dst, "w").write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(dst), "traffic.json")
    table = json.load(open(tj)) if os.path.exists(tj) else {}
    if "tc_gemm" in table and "dram_bytes_per_launch" in table["tc_gemm"]:
        table = {}  # round-1 flat format
    table.setdefault(workload, {})[kclass] = {
        "dram_bytes_per_launch": mean("dram"), "launches_captured": n, "tensor_active_pct": mean("tensor"),
        "note": f"ncu --set full (cache control on: cold L2 per replay), {workload} {what}, {n} {kclass} launches; "
                "mean dram__bytes_read.sum+dram__bytes_write.sum per launch"}
    json.dump(table, open(tj, "w"), indent=1, sort_keys=True)
    print("\n".join(lines[:2]))


if __name__ == "__main__":
    main(*sys.argv[1:])
