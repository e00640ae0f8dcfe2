"""Benchmark: synthesized-operator fwd+bwd on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload resnet18|resnet34|cfg1|qkv|sweep]
                    [--impl syno|reference]

Default workload = BASELINE configs[1]: the 20 conv layers of ResNet-18
(CIFAR, 32x32) each replaced by a synthesized operator, forward + backward
(grad-input and grad-weight) in bf16 at batch 128 per GPU.  A step runs
every layer's forward and backward once on synthetic inputs resident in HBM.
Multi-GPU (torchrun): every rank runs its own batch (weak scaling, no
data-path collective: the layers' units are independent images).

--impl reference times the reference's CPU implementation of the same
path (the pinned numpy restatement in oracle/, since the reference is pure
Python and has no compiled artifact) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        p["source"] = "measured"
        return p
    p = dict(FALLBACK_PEAKS)
    p["source"] = "fallback"
    return p


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, n in enumerate(names):
                if r[4 + k].lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------

def layer_work(h, n_weights, esize=2):
    """Algorithmic FLOPs and compulsory bytes of one fwd+bwd of a layer.

    FLOPs: forward = codegen.flops(staged=True) (2 per MAC, batch included);
    grad-input and grad-weight are one contraction each of the same volume.
    Bytes: fwd reads x, w and writes y; bwd reads x, w, dy and writes dx, dw."""
    f = h.flops_staged
    nx = math.prod(h.x_shape)
    ny = math.prod(h.y_shape)
    nw = sum(math.prod(s) for s in h.w_shapes)
    return {"fwd_flops": f, "bwd_flops": 2 * f,
            "fwd_bytes": esize * (nx + nw + ny), "bwd_bytes": esize * (nx + nw + ny + nx + nw)}


def build_layers(name, batch):
    from paper_2410_23745_b200 import workloads as WL
    if name == "resnet18":
        return WL.resnet18_cifar(batch or 128)
    if name == "resnet34":
        return WL.resnet34_imagenet(batch or 256)
    if name == "cfg1":
        return [WL.cfg1_conv(batch or 8)]
    if name == "qkv":
        return [WL.qkv(batch or 16)]
    raise ValueError(name)


def run_layers(args, rank, world, device, peaks):
    import numpy as np
    import torch

    from paper_2410_23745_b200 import _lib, ops
    from paper_2410_23745_b200 import pgraph as P

    dtype = torch.float32 if args.workload == "cfg1" else torch.bfloat16
    esize = 4 if dtype == torch.float32 else 2
    fwd_only = args.workload == "cfg1"
    layers = build_layers(args.workload, args.batch)
    gen = torch.Generator(device="cpu").manual_seed(1234 + rank)
    state = []
    for L in layers:
        h = P.handle_for(L.graph)
        x = torch.randn(h.x_shape, generator=gen).to(device=device, dtype=dtype)
        ws = [(torch.randn(s, generator=gen) / math.sqrt(max(1, math.prod(s[1:])))).to(device=device, dtype=dtype)
              for s in h.w_shapes]
        dy = torch.randn(h.y_shape, generator=gen).to(device=device, dtype=dtype)
        y = torch.empty(h.y_shape, device=device, dtype=dtype)
        dx = torch.empty(h.x_shape, device=device, dtype=dtype)
        dws = [torch.empty(s, device=device, dtype=dtype) for s in h.w_shapes]
        state.append(dict(L=L, h=h, x=x, ws=ws, dy=dy, y=y, dx=dx, dws=dws,
                          work=layer_work(h, len(ws), esize)))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)  # > 126 MB L2
    # a dedicated stream: CUDA-graph capture needs a non-default stream, and the
    # library keeps one workspace per (device, stream)
    stream = torch.cuda.Stream(device)
    import ctypes
    sp = ctypes.c_void_p(stream.cuda_stream)
    code = ops._DT[dtype]

    def call_fwd(s):
        warr = (ctypes.c_void_p * max(1, len(s["ws"])))(*[w.data_ptr() for w in s["ws"]])
        rc = _lib.lib.syno_forward(s["h"].ptr, code, ctypes.c_void_p(s["x"].data_ptr()), warr, len(s["ws"]),
                                   ctypes.c_void_p(s["y"].data_ptr()), sp)
        assert rc == 0, _lib.last_error()

    def call_bwd(s):
        warr = (ctypes.c_void_p * max(1, len(s["ws"])))(*[w.data_ptr() for w in s["ws"]])
        dwarr = (ctypes.c_void_p * max(1, len(s["ws"])))(*[g.data_ptr() for g in s["dws"]])
        rc = _lib.lib.syno_backward(s["h"].ptr, code, ctypes.c_void_p(s["x"].data_ptr()), warr, len(s["ws"]),
                                    ctypes.c_void_p(s["dy"].data_ptr()), ctypes.c_void_p(s["dx"].data_ptr()),
                                    dwarr, sp)
        assert rc == 0, _lib.last_error()

    phases = [("fwd", call_fwd)] + ([] if fwd_only else [("bwd", call_bwd)])
    nev = len(state) * len(phases)
    times = {(i, p): [] for i in range(len(state)) for p, _ in phases}

    def one_step(record):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(nev + 1)] if record else None
        if record:
            evs[0].record(stream)
        k = 0
        for i, s in enumerate(state):
            for p, fn in phases:
                fn(s)
                if record:
                    evs[k + 1].record(stream)
                k += 1
        return evs

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            one_step(False)
    torch.cuda.synchronize(device)

    # The step is captured once as a CUDA graph (kernel launches only: the
    # library allocates nothing and never synchronises in steady state).
    graph = None
    launches_per_step = None
    if args.graph:
        c0 = _lib.lib.syno_launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            one_step(False)
        launches_per_step = _lib.lib.syno_launch_count() - c0
        with torch.cuda.stream(stream):
            graph.replay()
        torch.cuda.synchronize(device)

    sampler = ClockSampler(torch.cuda.current_device() if device.index is None else device.index)
    if rank == 0:
        sampler.start()
    barrier(world)
    torch.cuda.synchronize(device)
    launches0 = _lib.lib.syno_launch_count()
    step_ms = []
    evs = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between timed steps, outside the step's events
        with torch.cuda.stream(stream):
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                one_step(False)
            e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize(device)
    barrier(world)
    launches = _lib.lib.syno_launch_count() - launches0
    if graph is not None:
        launches = launches_per_step * args.steps
    if rank == 0:
        sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]

    # per-(layer, phase) breakdown: a separate eager pass with events between calls
    for _ in range(2):
        with torch.cuda.stream(stream):
            flush.zero_()
            all_evs = one_step(True)
        torch.cuda.synchronize(device)
        k = 0
        for i in range(len(state)):
            for p, _ in phases:
                times[(i, p)].append(all_evs[k].elapsed_time(all_evs[k + 1]))
                k += 1
    ms = statistics.mean(step_ms)
    ms_max = allreduce_max(ms, world, device)
    batch_units = state[0]["h"].x_shape[0] if state[0]["h"].batch_rank else 1
    value = world * batch_units / (ms_max / 1e3)

    # dominant (layer, phase) call and its roofline
    avg = {k: statistics.mean(v) for k, v in times.items()}
    (di, dp), dms = max(avg.items(), key=lambda kv: kv[1])
    w = state[di]["work"]
    F = w[f"{dp}_flops"]
    B = w[f"{dp}_bytes"]
    tflops_peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    t_tensor = F / (tflops_peak * 1e12)
    t_hbm = B / (peaks["hbm_gbs"] * 1e9)
    if t_tensor >= t_hbm:
        achieved = F / (dms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tflops_peak, "unit": "TFLOP/s",
                "frac": achieved / tflops_peak}
    else:
        achieved = B / (dms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"]}
    roof.update({"traffic": load_traffic(state[di]["L"].name, dp),
                 "kernel": f"{state[di]['L'].name}:{dp} (one library call: pack + fold + tcgen05 GEMMs)",
                 "kernel_ms": dms, "share_of_step": dms / ms, "peak_source": peaks["source"]})
    # whole-step roofline: sum of per-call roofline times over the measured step time
    t_roof = 0.0
    for s in state:
        for p, _ in phases:
            t_roof += max(s["work"][f"{p}_flops"] / (tflops_peak * 1e12), s["work"][f"{p}_bytes"] / (peaks["hbm_gbs"] * 1e9))
    step_flops = sum(s["work"]["fwd_flops"] + (0 if fwd_only else s["work"]["bwd_flops"]) for s in state)

    with torch.cuda.stream(stream):
        e2e = measure_e2e(state, phases, args, device, dtype, world)
    breakdown = {f"{state[i]['L'].name}:{p}": round(avg[(i, p)], 4) for (i, p) in avg}
    return {
        "value": value, "ms_per_step": ms_max, "roofline": roof,
        "step_roofline_frac": (t_roof * 1e3) / ms_max, "step_tflops": step_flops / (ms_max / 1e3) / 1e12,
        "gpu_launches": int(launches), "clocks": sampler.summary() if rank == 0 else None,
        "e2e": e2e, "breakdown_ms": breakdown, "dtype": "bf16" if dtype == torch.bfloat16 else "f32",
        "batch": batch_units, "n_layers": len(state), "state": state,
    }


def measure_e2e(state, phases, args, device, dtype, world):
    """Same step through the public API with HOST buffers: pinned host -> device
    copies of every layer's x (and dy), compute, device -> host copies of y
    (and dx, dW), all inside the timed region."""
    import torch

    from paper_2410_23745_b200 import ops
    host = []
    h2d = d2h = 0
    fwd_only = len(phases) == 1
    for s in state:
        hx = s["x"].cpu().pin_memory()
        hdy = s["dy"].cpu().pin_memory()
        hy = torch.empty(s["y"].shape, dtype=dtype).pin_memory()
        hdx = torch.empty(s["x"].shape, dtype=dtype).pin_memory()
        hdw = [torch.empty(g.shape, dtype=dtype).pin_memory() for g in s["dws"]]
        host.append((hx, hdy, hy, hdx, hdw))
        esz = s["x"].element_size()
        h2d += hx.numel() * esz + (0 if fwd_only else hdy.numel() * esz)
        d2h += hy.numel() * esz + (0 if fwd_only else (hdx.numel() + sum(g.numel() for g in hdw)) * esz)
    stream = torch.cuda.current_stream(device)

    def step():
        for s, (hx, hdy, hy, hdx, hdw) in zip(state, host):
            s["x"].copy_(hx, non_blocking=True)
            if not fwd_only:
                s["dy"].copy_(hdy, non_blocking=True)
            ops.forward(s["h"], s["x"], s["ws"], out=s["y"])
            hy.copy_(s["y"], non_blocking=True)
            if not fwd_only:
                dx, dws = ops.backward(s["h"], s["x"], s["ws"], s["dy"])
                hdx.copy_(dx, non_blocking=True)
                for a, b in zip(hdw, dws):
                    a.copy_(b, non_blocking=True)

    for _ in range(max(1, min(args.warmup, 3))):
        step()
    torch.cuda.synchronize(device)
    n = max(1, min(args.steps, 10))
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(n):
        step()
    t1.record(stream)
    torch.cuda.synchronize(device)
    ms = t0.elapsed_time(t1) / n
    ms = allreduce_max(ms, world, device)
    units = state[0]["h"].x_shape[0]
    return {"value": world * units / (ms / 1e3), "unit": "images/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}


def load_traffic(layer, phase):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        t = json.load(f)
    return t.get(f"{layer}:{phase}")


# ---------------------------------------------------------------------------
# CPU baseline: the pinned oracle restatement of the reference path
# ---------------------------------------------------------------------------

def _oracle_layer_job(args):
    """One image of one layer, fwd + grad-input + grad-weight, with the oracle."""
    import numpy as np

    from oracle import nest_oracle as O
    text, env, xshape, wshapes, yshape, fwd_only, seed = args
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(xshape)
    ws = [rng.standard_normal(s) for s in wshapes]
    up = rng.standard_normal(yshape)
    t0 = time.perf_counter()
    O.interpret(text, env, x, ws)
    if fwd_only:
        return time.perf_counter() - t0
    O.input_gradient(text, env, x, up, ws)
    if ws:
        O.weight_gradient(text, env, x, up, ws)
    return time.perf_counter() - t0


def cpu_sample_spec(args):
    """The bounded CPU sample: one image through one representative layer,
    extrapolated to the whole step by the layers' FLOP share."""
    from paper_2410_23745_b200 import codegen as C
    from paper_2410_23745_b200 import pgraph as P
    layers = build_layers(args.workload, args.batch)
    pick = {"resnet18": "l1b0c2", "resnet34": "l2b1c2", "cfg1": "cfg1_conv3x3", "qkv": "qkv"}[args.workload]
    L = next(l for l in layers if l.name == pick)
    one = dict(L.assignment)
    bkey = "N" if "N" in one else "B"
    batch = one[bkey]
    if args.workload == "qkv":
        one["T"] = 128  # the reference's full-grid interpreter needs ~58 GB per T=1024 element
    one[bkey] = 1
    text = C.emit_loop_nest(L.graph, one)
    h1 = P.handle_for(L.graph, one)
    spec = (text, one, h1.x_shape[1:], [tuple(s) for s in h1.w_shapes], h1.y_shape[1:], args.workload == "cfg1")
    flops_one = 3 * h1.flops_staged
    total_flops_per_image = sum(3 * P.handle_for(l.graph).flops_staged for l in layers) / batch
    if args.workload == "cfg1":
        flops_one = h1.flops_staged
        total_flops_per_image = P.handle_for(L.graph).flops_staged / batch
    desc = (f"1 image of layer {L.name} ({L.op}) "
            + ("forward" if args.workload == "cfg1" else "fwd+grad-input+grad-weight")
            + (" at T=128" if args.workload == "qkv" else "")
            + "; images/s extrapolated by FLOP share of the full step")
    return spec, flops_one, total_flops_per_image, desc


def cpu_baseline(args, processes=1):
    import multiprocessing as mp
    spec, flops_one, per_image, desc = cpu_sample_spec(args)
    jobs = [spec + (k,) for k in range(processes)]
    t0 = time.perf_counter()
    if processes == 1:
        _oracle_layer_job(jobs[0])
    else:
        with mp.get_context("fork").Pool(processes) as pool:
            pool.map(_oracle_layer_job, jobs)
    dt = time.perf_counter() - t0
    flops_rate = processes * flops_one / dt
    return {"value": flops_rate / per_image, "unit": "images/s", "cores": processes, "kind": "port",
            "sample": desc + f" ({processes} process(es), {dt:.1f} s)", "seconds": dt}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(cores, 64))
    for _ in range(args.warmup):
        pass  # the oracle has no warm state worth warming beyond imports
    vals, secs = [], []
    for _ in range(max(1, args.steps)):
        r = cpu_baseline(args, procs)
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": procs, "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

METRIC = "synthesized-operator fwd+bwd throughput (operator fwd+bwd latency & % roofline)"


def workload_config(args):
    from paper_2410_23745_b200 import workloads as WL  # noqa: F401
    desc = {
        "resnet18": ("cfg2: ResNet-18 CIFAR conv layers (20) as synthesized operators "
                     "(sep_shared / conv3x3 / conv3x3_s2 / 1x1-s2 shortcut), fwd+bwd"),
        "resnet34": "cfg3: ResNet-34 ImageNet-shape layers as synthesized operators, fwd+bwd",
        "cfg1": "cfg1: conv3x3 in Syno primitives, N=8 C=64 H=W=32, forward",
        "qkv": "cfg4: GPT-2 small QKV projection as a synthesized operator, fwd+bwd",
    }[args.workload]
    batch = args.batch or {"resnet18": 128, "resnet34": 256, "cfg1": 8, "qkv": 16}[args.workload]
    return {"workload": desc, "batch_per_gpu": batch, "l2": "flushed between timed steps (256 MB write)",
            "inputs": "synthetic N(0,1), resident in HBM"}


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(v, world, device):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="resnet18", choices=["resnet18", "resnet34", "cfg1", "qkv"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--impl", default="syno", choices=["syno", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="eager launches instead of a CUDA graph")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
    peaks = load_peaks()
    r = run_layers(args, rank, world, device, peaks)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(args, 1)
            cpu.pop("seconds", None)
        line = {
            "metric": METRIC, "value": r["value"], "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": r["dtype"], "data": "synthetic", "config": workload_config(args),
            "roofline": r["roofline"], "step_roofline_frac": r["step_roofline_frac"],
            "step_tflops": r["step_tflops"], "cpu_baseline": cpu, "e2e": r["e2e"], "gpu_launches": r["gpu_launches"],
            "clocks": r["clocks"], "breakdown_ms": r["breakdown_ms"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
