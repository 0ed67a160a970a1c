#!/usr/bin/env python
"""Benchmark of the nb200 hot path (BASELINE.json metric: "CIFAR ResNet-34
transformed-net inference ms; Fisher candidates/sec").

Workload (configs[1]): the 33-conv ResNet-34 CIFAR chain at batch 128,
synthetic data (make_batch, seed 1) and init_weights (seed 42); a step is one
Fisher Potential evaluation (forward + activation gradients + per-channel
A*g reduction, I/nnet.hpp:321) of one candidate network from a per-layer
neural search.  Candidates are sharded across ranks by LPT on estimated
FLOPs (weak scaling: a fixed candidate count per GPU), with no collective on
the data path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nb200|reference]

Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CIFAR ResNet-34 transformed-net inference ms; Fisher candidates/sec"
UNIT = "candidates/s"
N_BATCH = 128
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="nb200", choices=["nb200", "reference"])
    p.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "simt"])
    p.add_argument("--candidates-per-gpu", type=int, default=16)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-layers", type=int, default=2)
    return p.parse_args()


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      "--query-gpu=" + self.Q, "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 6:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref: the unmodified nestopt compiled in place)

def reference_sample(layers: int, threads: int):
    """Times the reference's fisher_potential on a bounded slice of the R34
    chain (its first `layers` convs, one image) on `threads` host threads at
    once (one candidate per thread, like evaluate_all's jobs), and scales it
    to candidates/s of the full chain at N=128 by the Fisher-MAC ratio (the
    reference's cost is linear in MACs and examples, I/nnet.hpp:184,206)."""
    from oracle.oracle import Reference
    from paper_2102_06599_b200.api import Network
    from paper_2102_06599_b200.workloads import resnet34_chain

    full = resnet34_chain()
    sl = Network(full.layers[:layers], num_classes=10, seed=42)
    R = Reference()

    def fisher_macs(net, n):
        from paper_2102_06599_b200.api import count_macs
        m = [count_macs(l.spec) for l in net.layers]
        return n * (sum(m) + sum(m[1:]))

    errs = []

    def one():
        try:
            R.fisher(sl, 1, 1)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    t0 = time.perf_counter()
    ts = [threading.Thread(target=one) for _ in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    if errs:
        raise errs[0]
    scale = fisher_macs(full, N_BATCH) / fisher_macs(sl, 1)
    cand_per_s = threads / (dt * scale)
    return cand_per_s, dt, (f"reference fisher_potential (oracle/_ref) on R34 layers 0-{layers - 1}"
                            f" at N=1, {threads} concurrent on {threads} host threads, "
                            f"{dt:.2f} s wall, scaled x{scale:.0f} by Fisher MACs to the full "
                            f"chain at N={N_BATCH} (extrapolated)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # CPU code has no warm-up effects beyond the first call; keep the whole
    # arm within a few minutes (each step is a ~10 s sample).
    warm, steps = min(args.warmup, 1), min(args.steps, 8)
    for _ in range(warm):
        reference_sample(args.cpu_sample_layers, threads)
    vals, walls = [], []
    for _ in range(steps):
        v, dt, sample = reference_sample(args.cpu_sample_layers, threads)
        vals.append(v)
        walls.append(dt)
    v = statistics.mean(vals)
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": steps, "warmup": warm,
            "ms_per_step": 1e3 * statistics.mean(walls), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "resnet34_chain_fisher", "global_batch": N_BATCH,
                       "network": "ResNet-34 CIFAR 33-conv chain (SURVEY App. B)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# nb200 arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2102_06599_b200 as nb
    from paper_2102_06599_b200 import Precision
    from paper_2102_06599_b200.workloads import (fixture_path, load_candidates,
                                                 per_layer_candidates, resnet34_chain)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prec = {"fp32": Precision.FP32, "tf32": Precision.TF32, "simt": Precision.SIMT}[args.precision]

    origin = resnet34_chain()
    fx = fixture_path("r34_candidates.json")
    pool_n = args.candidates_per_gpu * world
    if os.path.exists(fx):
        pool = load_candidates(fx, origin)
        pool = [pool[i % len(pool)] for i in range(pool_n)]
        cand_src = "tests/golden/r34_candidates.json (reference draw_candidates + host gates)"
    else:
        pool = per_layer_candidates(origin, pool_n)
        cand_src = "workloads.per_layer_candidates (programmatic per-layer neural rewrites)"
    costs = [nb.fisher_flops(n, N_BATCH) for n in pool]
    assign = nb.schedule_lpt(costs, world)
    mine = [n for n, a in zip(pool, assign) if a == rank]
    my_flops = sum(c for c, a in zip(costs, assign) if a == rank)

    ctx = nb.Context(local)
    batch = nb.make_batch(origin, N_BATCH, 1)
    sess = nb.Session(origin, batch, ctx=ctx)
    stream = torch.cuda.ExternalStream(ctx.stream())

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(fn, k):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(k):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    step = lambda i: sess.fisher(mine[i % len(mine)], prec)
    for i in range(args.warmup):
        step(i)
    ctx.reset_stats()
    ctx.set_profiling(True)
    l0 = ctx.launch_count()
    with Clocks(local) as clk:
        ms = timed(step, args.steps)
    launches = ctx.launch_count() - l0
    ctx.set_profiling(False)
    kstats = ctx.kernel_stats()
    total_units = args.steps * world
    value = total_units / (ms / 1e3)

    # steps per rank cover (steps/len(mine)) of its queue; FLOP-weighted per step
    step_flops = sum(nb.fisher_flops(mine[i % len(mine)], N_BATCH) for i in range(args.steps))

    # ---- e2e: public API with host (pinned) batch each step
    xin = torch.from_numpy(batch.inputs).pin_memory()
    lab = torch.from_numpy(batch.labels).pin_memory()
    hbatch = nb.Batch(xin.numpy(), lab.numpy(), batch.seed)
    e2e_step = lambda i: nb.fisher_potential(mine[i % len(mine)], hbatch, prec, ctx=ctx)
    for i in range(min(2, args.warmup)):
        e2e_step(i)
    e2e_ms = timed(e2e_step, args.steps)
    e2e_val = total_units / (e2e_ms / 1e3)
    h2d = batch.inputs.nbytes + batch.labels.nbytes
    d2h = 8 * (sum(l.spec.co_eff() for l in origin.layers) + len(origin.layers) +
               N_BATCH * origin.num_classes)

    # ---- transformed-net inference (forward of the best-ranked candidate shape)
    best = min(mine, key=lambda n: nb.network_macs(n))
    inf_ms = timed(lambda i: sess.forward(best, prec), args.steps) / args.steps
    inf_origin_ms = timed(lambda i: sess.forward(origin, prec), args.steps) / args.steps

    # ---- roofline of the dominant kernel family
    pk, pk_kind = peaks()
    dom_name, dom = max(kstats.items(), key=lambda kv: kv[1]["ms"]) if kstats else ("", None)
    roof = None
    if dom:
        avg_ms = dom["ms"] / dom["launches"]
        if dom["flops"] > 0:
            ach = dom["flops"] / dom["launches"] / (avg_ms / 1e3) / 1e12
            peak = pk["bf16_tflops"]
            roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                    "frac": ach / peak, "traffic": None, "kernel": dom_name,
                    "peak_source": f"{pk_kind} bf16 dense (MEASURED_PEAKS.json)",
                    "launch_ms": avg_ms, "share_of_step": dom["ms"] / ms if ms else None}
        else:
            ach = dom["bytes"] / dom["launches"] / (avg_ms / 1e3) / 1e9
            peak = pk["hbm_gbs"]
            roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                    "frac": ach / peak, "traffic": None, "kernel": dom_name,
                    "peak_source": f"{pk_kind} HBM copy (MEASURED_PEAKS.json)",
                    "launch_ms": avg_ms, "share_of_step": dom["ms"] / ms if ms else None}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, dt, sample = reference_sample(args.cpu_sample_layers, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision != "tf32" else "tf32", "data": "synthetic",
            "config": {"workload": "resnet34_chain_fisher_search", "global_batch": N_BATCH,
                       "network": "ResNet-34 CIFAR 33-conv chain (SURVEY App. B)",
                       "candidates": cand_src, "candidates_per_gpu": args.candidates_per_gpu,
                       "precision": args.precision, "parallelism": f"candidate-sharded x{world}",
                       "l2": "inputs larger than L2 (~0.5 GB activations per evaluation)"},
            "inference_ms": inf_ms, "inference_origin_ms": inf_origin_ms,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "achieved_tflops_step": step_flops / (ms / 1e3) / 1e12 * 1,
            "roofline": roof,
            "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3)}
                        for k, v in kstats.items()},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
