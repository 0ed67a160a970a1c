#!/usr/bin/env python
"""Benchmark of the nb200 hot path (BASELINE.json metric: "CIFAR ResNet-34
transformed-net inference ms; Fisher candidates/sec").

Workload (configs[1]): the 33-conv ResNet-34 CIFAR chain at batch 128,
synthetic data (make_batch, seed 1) and init_weights (seed 42).  The
candidate pool is the reference's own per-layer neural search
(tests/golden/r34_candidates.json: draw_candidates + evaluate_candidate's host
gates over 12 masked layers, 726 distinct networks).  A step is one Fisher
Potential evaluation (forward + activation gradients + per-channel A*g
reduction, I/nnet.hpp:321) of one candidate; every rank scores its LPT share
of the pool through the product's scheduler (nb_evaluate: --streams
concurrent sessions per GPU), weak scaling, no collective on the data path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nb200|reference]
                  [--single-process]   (one process driving all N GPUs through
                                        nb_evaluate instead of torchrun ranks)

Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import gc
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

# Precision tiers (the values live in
# paper_2102_06599_b200/api.py TOLERANCE): what each mode computes in and
# the stated tolerance of its Fisher scores against the fp64 reference.
# The FP32 tier's tensor-core split (paper_2102_06599_b200.fp32_split():
# "3xf16" by default, NB_TC_SPLIT=tf32 / bf16 for the alternatives).
def _split() -> str:
    e = os.environ.get("NB_TC_SPLIT")
    return {"tf32": "3xtf32", "bf16": "3xbf16"}.get(e, "3xf16")


SPLIT = _split()
MODE_KEY = {"fp32": "fp32_" + SPLIT, "tf32": "tf32", "simt": "simt"}
DTYPE = {"fp32_" + SPLIT: SPLIT, "tf32": "tf32", "simt": "f32"}
_SPLIT_DESC = {
    "3xf16": "3xF16 tcgen05 kind::f16 implicit GEMM (fp16 hi/lo halves of per-image / per-layer "
             "power-of-two scaled fp32 operands, hi*hi + hi*lo + lo*hi, fp32 accumulate)",
    "3xbf16": "3xBF16 tcgen05 kind::f16 implicit GEMM (bf16 hi/lo halves, hi*hi + hi*lo + lo*hi, "
              "fp32 accumulate)",
    "3xtf32": "3xTF32 tcgen05 implicit GEMM (hi*hi + hi*lo + lo*hi, fp32 accumulate)"}
ARITH = {"fp32": _SPLIT_DESC[SPLIT] + " for tensor-core-shaped ranges, fp32 FFMA for the rest; "
                 "head/softmax/Fisher fp64",
         "tf32": "1xTF32 tcgen05 (throughput tier); head/softmax/Fisher fp64",
         "simt": "fp32 FFMA everywhere (true fp32); head/softmax/Fisher fp64"}
TOL_NOTE = {"fp32_" + SPLIT: "Fisher totals <= 5e-4, per layer <= 5e-3 relative (chains of <= 10 "
                             "layers); 1.5e-3 / 5e-3 on the 33-layer R34 chain",
            "tf32": "Fisher totals <= 5e-2, per layer <= 2e-1 relative",
            "simt": "Fisher totals <= 1e-5, per layer <= 1e-4 relative (chains of <= 10 layers); "
                    "3e-4 / 1.5e-3 on the R34 chain"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--single-process", action="store_true",
                   help="drive all --gpus GPUs from this one process through the scheduler "
                        "(nb_evaluate's per-GPU workers) instead of one rank per GPU")
    p.add_argument("--steps", type=int, default=64)
    p.add_argument("--warmup", type=int, default=8)
    p.add_argument("--impl", default="nb200", choices=["nb200", "reference"])
    p.add_argument("--precision", default="fp32", choices=["fp32", "tf32", "simt"])
    p.add_argument("--streams", type=int, default=4, help="concurrent sessions per GPU")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-peaks", action="store_true", help="skip the peak microbenchmarks")
    p.add_argument("--no-modes", action="store_true",
                   help="skip the other precision tiers' figures")
    p.add_argument("--no-inference", action="store_true",
                   help="skip the whole-pool search behind the inference figure (profiling runs)")
    p.add_argument("--no-kernel-events", action="store_true",
                   help="skip the per-launch CUDA events (no roofline; overhead check)")
    return p.parse_args()


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


def measured_peaks():
    """The peaks of the arithmetic nb200 issues, measured on this GPU now
    (scripts/peaks/peaks.cu): dense tcgen05 kind::tf32 and kind::f16 (bf16)
    issue rates on every SM, fp32 FFMA, plus cuBLAS TF32 (torch.matmul
    8192^3 fp32 with TF32 allowed) as a library cross-check."""
    import ctypes as C
    import torch
    out = {}
    so = os.path.join(ROOT, "scripts", "peaks", "libnb200_peaks.so")
    if os.path.exists(so):
        lib = C.CDLL(so)
        lib.nbp_tc_tflops.restype = C.c_double
        lib.nbp_tc_tflops.argtypes = [C.c_int]
        lib.nbp_ffma_tflops.restype = C.c_double
        out["tcgen05_tf32_tflops"] = lib.nbp_tc_tflops(0)
        out["tcgen05_bf16_tflops"] = lib.nbp_tc_tflops(1)
        out["ffma_fp32_tflops"] = lib.nbp_ffma_tflops()
    try:
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn(8192, 8192, device="cuda")
        b = torch.randn(8192, 8192, device="cuda")
        for _ in range(3):
            a @ b
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out["cublas_tf32_tflops"] = 2 * 8192 ** 3 / (best / 1e3) / 1e12
        torch.backends.cuda.matmul.allow_tf32 = prev
        del a, b
    except Exception as e:  # pragma: no cover
        out["cublas_tf32_error"] = str(e)
    out["how"] = ("scripts/peaks/peaks.cu: one launch of 148 CTAs, M=128 N=256 tcgen05.mma "
                  "back to back from shared-memory operands, CUDA events; FFMA 8 chains/thread")
    return out


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

    def _run_nvml(self):
        """NVML directly: a sample every ~5 ms (the timed region can be ~0.1 s)."""
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
                ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4)]
        while not self._stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active"
                                                       for _, b in bits])
            self._stop.wait(0.005)

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            pass
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
            self._stop.wait(0.1)

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
# the candidate pool (plain JSON: the reference arm never loads the product)

def _out(l):
    """(co_eff, out_h, out_w) of a layer JSON (ConvSpec, I/ir.hpp:40-50)."""
    p, s = l.get("pad", 0), l.get("stride", 1)
    oh = ((l["h"] + 2 * p - l.get("kh", 1)) // s + 1) // l.get("spatial_div_h", 1)
    ow = ((l["w"] + 2 * p - l.get("kw", 1)) // s + 1) // l.get("spatial_div_w", 1)
    return l["co"] // l.get("bottleneck", 1), oh, ow


def timed_pool(steps, warmup, world):
    """The candidate networks both arms use, as network JSON: the
    reference's R34 per-layer pool (tests/golden/r34_candidates.json: each
    candidate is the origin with one layer replaced, shapes repaired as
    repair_network does, I/nnet.hpp:372-380) in a fixed shuffled order; the
    first max(1, W) warm up, the next K x world are timed, the rest spare."""
    import numpy as np
    with open(os.path.join(ROOT, "tests", "golden", "r34_candidates.json")) as f:
        data = json.load(f)
    origin = data["origin"]
    pool = []
    for c in data["candidates"]:
        layers = [dict(l) for l in origin["layers"]]
        layers[c["diff"][0]] = dict(c["diff"][1])
        for l in range(1, len(layers)):
            layers[l]["ci"], layers[l]["h"], layers[l]["w"] = _out(layers[l - 1])
        pool.append(dict(origin, layers=layers))
    order = np.random.default_rng(0).permutation(len(pool))
    pool = [pool[i] for i in order]
    warm = pool[:max(1, warmup)]
    timed = pool[len(warm):]
    need = steps * world
    if need > len(timed):
        raise SystemExit(f"--steps x gpus = {need} exceeds the {len(timed)} distinct candidates")
    return origin, warm, timed[:need], timed[need:]


def _macs(l):
    """count_macs of a layer JSON (I/interp.hpp:190-202)."""
    co, oh, ow = _out(l)
    ranges = l.get("channel_splits") or [{"begin": 0, "end": co, "groups": l.get("groups", 1)}]
    return sum((r["end"] - r["begin"]) * oh * ow * (l["ci"] // r.get("groups", 1))
               * l.get("kh", 1) * l.get("kw", 1) for r in ranges)


def config_block(steps, streams, world):
    """`config` of both arms (identical, so the driver compares like with like)."""
    return {"workload": "resnet34_chain_fisher_search", "global_batch": N_BATCH,
            "network": "ResNet-34 CIFAR 33-conv chain (SURVEY App. B)",
            "candidates": "tests/golden/r34_candidates.json (reference draw_candidates + "
                          "host gates, 12 masked layers)",
            "candidates_per_gpu": steps, "streams_per_gpu": streams,
            "parallelism": f"candidate-sharded x{world} (LPT, no collective)",
            "l2": "inputs larger than L2 (~0.5 GB of activations per evaluation)"}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref: the unmodified nestopt compiled in place)

def cpu_info():
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Thread(s) per core", "Core(s) per socket",
                             "Socket(s)", "CPU max MHz"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    return info


def cpu_baseline_sample(timed, threads):
    """cpu_baseline of the nb200 arm: a bounded (~10-30 s) sample of the
    reference on the box's host cores.  One timed-pool candidate is cut into
    `threads` contiguous layer slices, each scored at N=1 by the reference's
    fisher_potential on its own thread (evaluate_all's pool); every layer
    runs in its own shape, the overlap layers' extra forwards are timed and
    subtracted (oracle/refbench.py).  The candidate's N=1 thread-seconds,
    x128 by the reference's exact linearity in N (I/nnet.hpp:184, 206), give
    candidates/s on `threads` cores (extrapolated)."""
    from oracle.refbench import RefArm, candidate_seconds_by_slices, fisher_macs
    # the timed-pool candidate of median Fisher MACs (candidate 0 can be an
    # early crop whose whole network runs at 2x2: 50x cheaper than most)
    order = sorted(range(len(timed)), key=lambda i: fisher_macs(timed[i], 1))
    pick = order[len(order) // 2]
    net = timed[pick]
    sec, wall, parts = candidate_seconds_by_slices(RefArm(), net, threads)
    v = threads / (sec * N_BATCH)
    return v, (f"reference fisher_potential (oracle/_ref) on timed-pool candidate {pick} "
               f"(median Fisher MACs of the pool, {fisher_macs(net, 1) / 1e9:.2f} GMAC per "
               f"example) at N=1, "
               f"cut into {parts} layer slices run concurrently on {threads} host threads "
               f"({wall:.1f} s wall); {sec:.1f} thread-s per N=1 evaluation x{N_BATCH} "
               f"examples (exact linearity in N), {threads} candidates in flight (extrapolated)")


def run_reference(args):
    """--impl reference: the reference's own CPU path on this box's host
    cores, through oracle/refbench.py only (the product is never imported).
    A whole candidate at N=1 costs the reference ~50-200 thread-seconds
    (55-100 ns/MAC), so each step is a bounded sample: step k is
    one MAC-balanced layer slice of timed candidate k (each candidate cut into
    `threads` slices, slices() in oracle/refbench.py; slice k mod the count),
    so the K steps sample the nb200 arm's K timed candidates once each,
    scored at N=1 by the reference's fisher_potential,
    the K steps self-scheduled on every host thread as evaluate_all does
    (I/search.hpp:315-334).  Every slice but a candidate's first starts one
    layer early so that its first layer's dgrad runs; that layer's extra
    forward is timed (layer_forward) and subtracted.  value = threads x
    (candidates the K slices cover) / (128 x their thread-seconds): a
    candidate at N=128 is 128 such evaluations (I/nnet.hpp:184, 206),
    labelled extrapolated."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.refbench import RefArm, slices
    threads = os.cpu_count() or 1
    world = int(os.environ.get("WORLD_SIZE", "1"))
    _, warm, timed, spare = timed_pool(args.steps, args.warmup, world)
    arm = RefArm()

    def cut(net):
        out = []
        sl = slices(net, threads)
        for k, (a, b) in enumerate(sl):
            lo = a - 1 if k > 0 else a
            out.append(({"schema_version": 1, "seed": net.get("seed", 42),
                         "num_classes": net.get("num_classes", 10),
                         "layers": [dict(l) for l in net["layers"][lo:b + 1]]},
                        net["layers"][a - 1] if k > 0 else None, 1.0 / len(sl)))
        return out

    # step k: one slice of timed candidate k (slice k mod its slice count), so
    # the K steps sample every timed candidate of the nb200 arm once
    steps = []
    for k in range(args.steps):
        parts = cut(timed[k % len(timed)])
        steps.append(parts[k % len(parts)])
    ci = min(args.steps, len(timed))
    # warm-up: W untimed slices of the cheapest spare candidate (the CPU path
    # has no caches to fill; this only pages the code in)
    cheap = min(spare or warm, key=lambda n: sum(_macs(l) for l in n["layers"]))
    wsteps = cut(cheap)[:max(1, args.warmup)]
    arm.fisher_jobs([x[0] for x in wsteps], 1, threads)
    totals, secs, wall = arm.fisher_jobs([x[0] for x in steps], 1, threads)
    fwd = {}
    extra = 0.0
    for _, ov, _ in steps:
        if ov is not None:
            key = json.dumps(ov, sort_keys=True)
            if key not in fwd:
                fwd[key] = arm.layer_forward_seconds(ov)
            extra += fwd[key]
    thread_s = sum(secs) - extra
    cands = sum(x[2] for x in steps)
    v = threads * cands / (N_BATCH * thread_s)
    sample = (f"reference fisher_potential (oracle/_ref, evaluate_all's thread pool) on "
              f"{len(steps)} MAC-balanced layer slices, one of each of the {ci} timed "
              f"candidates ({cands:.2f} candidates' worth), each at N=1 (example 0 of the batch), on "
              f"{threads} host threads: {wall:.1f} s wall, {thread_s:.1f} thread-s after the "
              f"overlap layers' forwards; {thread_s / cands:.1f} thread-s per candidate at N=1, "
              f"x{N_BATCH} examples (exact linearity in N, extrapolated)")
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": len(steps), "warmup": len(wsteps),
            "ms_per_step": 1e3 * wall / len(steps), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args.steps, args.streams, world),
            "precision": "fp64 (the reference's double arithmetic)",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample},
            "cpu": cpu_info(),
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
    from paper_2102_06599_b200.workloads import shard_lpt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prec = {"fp32": Precision.FP32, "tf32": Precision.TF32, "simt": Precision.SIMT}[args.precision]

    # warm-up networks and the timed pool are disjoint; the timed pool is
    # K per rank, LPT-sharded over the ranks by estimated FLOPs
    # single-process multi-GPU: one rank drives every GPU (sessions on each)
    devs = list(range(args.gpus)) if (args.single_process and world == 1) else [local]
    ngpu = world * len(devs)
    origin_j, warm_j, timed_j, spare_j = timed_pool(args.steps, args.warmup, ngpu)
    origin = nb.Network.from_json(origin_j)
    warm_pool = [nb.Network.from_json(n) for n in warm_j]
    timed = [nb.Network.from_json(n) for n in timed_j]
    costs = [nb.fisher_flops(n, N_BATCH) for n in timed]
    # (a single process driving several GPUs takes them all: nb_evaluate's
    # dynamic queue balances them over its per-GPU workers)
    assign = shard_lpt(costs, world, args.steps * len(devs))
    mine = [n for n, a in zip(timed, assign) if a == rank]

    batch = nb.make_batch(origin, N_BATCH, 1)
    ctxs = [nb.Context(d) for d in devs for _ in range(args.streams)]
    sessions = [nb.Session(origin, batch, ctx=c) for c in ctxs]
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    def timed_region(fn):
        # (Python's cyclic GC is collected before and held off inside, as
        # timeit does: a gen-2 pass over torch's heap costs ~40 ms of host
        # time that is not the product's)
        gc.collect()
        gc.disable()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        gc.enable()
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    # warm-up (W steps on networks outside the timed pool): packed weights of
    # the origin's layers, z-streams and arenas on every context
    nb.evaluate(sessions, warm_pool, prec)
    for s in sessions:
        s.fisher(origin, prec)
    origin_rep = sessions[0].fisher(origin, prec)

    for c in ctxs:
        c.reset_stats()
        # events on every 8th evaluation: the dominant kernel's duration is
        # sampled inside the timed region without paying per-launch event
        # records on every launch
        c.set_profiling(not args.no_kernel_events, every=8)
    l0 = sum(c.launch_count() for c in ctxs)
    with Clocks(local) as clk:
        ms, (reps, st) = timed_region(lambda: nb.evaluate(sessions, mine, prec))
    launches = sum(c.launch_count() for c in ctxs) - l0
    kstats = {}
    for c in ctxs:
        c.set_profiling(False)
        for k, v in c.kernel_stats().items():
            a = kstats.setdefault(k, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
            for f in a:
                a[f] += v[f]
    total_units = args.steps * ngpu
    value = total_units / (ms / 1e3)

    # ---- e2e: the reference-facing call with HOST buffers: sessions built
    # from the pinned host batch (H2D), evaluate_all over the K candidates,
    # reports back on the host (D2H), all inside the timed region
    xin = torch.from_numpy(batch.inputs).pin_memory()
    lab = torch.from_numpy(batch.labels).pin_memory()
    hbatch = nb.Batch(xin.numpy(), lab.numpy(), batch.seed)

    # the e2e run gets the timed run's starting state on its own contexts:
    # fresh caches warmed by the same warm-up pool and origin evaluation (a
    # cache cleared in place does not return to that state: its device
    # z-streams and slab refill differently), then new sessions from the
    # host batch inside the timed region
    ectxs = [nb.Context(d) for d in devs for _ in range(args.streams)]

    def e2e(pool=mine):
        ss = [nb.Session(origin, hbatch, ctx=c) for c in ectxs]
        r = nb.evaluate(ss, pool, prec)
        for s in ss:
            s.close()
        return r

    wsess = [nb.Session(origin, batch, ctx=c) for c in ectxs]
    nb.evaluate(wsess, warm_pool, prec)
    for s in wsess:
        s.fisher(origin, prec)
        s.close()
    e2e_ms, _ = timed_region(e2e)
    e2e_val = total_units / (e2e_ms / 1e3)
    h2d = (batch.inputs.nbytes + batch.labels.nbytes) * len(ctxs) / args.steps
    d2h = sum(8 * (sum(l.spec.co_eff() for l in n.layers) + len(n.layers) + 2 +
                   N_BATCH * n.num_classes) for n in mine) / args.steps

    # ---- transformed-net inference: forward of the search's choice, i.e.
    # survivors_ranked.front() over the whole pool (every candidate of the
    # reference's per-layer search scored by the scheduler, outside the
    # timed regions; fisher_accepts >= the origin, rank_survivors: macs
    # ascending, fisher descending, I/search.hpp:338-349, 381)
    full = [] if args.no_inference else [nb.Network.from_json(n) for n in warm_j + timed_j + spare_j]
    full_reps, _ = nb.evaluate(sessions, full, prec) if full else ([], None)
    surv = [(nb.network_macs(n), -r.total, i) for i, (n, r) in enumerate(zip(full, full_reps))
            if r.total >= origin_rep.total]
    bi = min(surv)[2] if surv else -1
    best = full[bi] if surv else origin
    best_info = {"pool": len(full), "survivors": len(surv),
                 "macs": nb.network_macs(best), "origin_macs": nb.network_macs(origin),
                 "fisher_total": full_reps[bi].total if surv else origin_rep.total,
                 "origin_fisher_total": origin_rep.total,
                 "changed_layer": next((l for l, (a, b) in enumerate(zip(best.layers, origin.layers))
                                        if a.spec != b.spec), None)}
    for _ in range(3):
        sessions[0].forward(best, prec)
    inf_ms, _ = timed_region(lambda: [sessions[0].forward(best, prec) for _ in range(10)])
    inf_o_ms, _ = timed_region(lambda: [sessions[0].forward(origin, prec) for _ in range(10)])

    # ---- roofline of the dominant kernel family: CUDA events around every
    # launch, on the launching stream, in a single-stream replay of this
    # rank's timed pool (in the concurrent timed region a launch's event time
    # also covers other streams' kernels sharing the SMs; both are reported)
    pk, pk_kind = peaks()
    pk_meas = measured_peaks() if not args.no_peaks else {}

    def roofline(stats, note):
        kern = {k: v for k, v in stats.items() if not k.startswith("host_")}
        if not kern:
            return None
        name, dom = max(kern.items(), key=lambda kv: kv[1]["ms"])
        avg_ms = dom["ms"] / dom["launches"]
        total_ms = sum(v["ms"] for v in kern.values())
        if dom["flops"] > 0:
            ach = dom["flops"] / dom["launches"] / (avg_ms / 1e3) / 1e12
            r = {"bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops"],
                 "unit": "TFLOP/s", "frac": ach / pk["bf16_tflops"],
                 "peak_source": f"{pk_kind} bf16 dense burst (MEASURED_PEAKS.json); "
                                "kernel_ceiling = the measured peak of the arithmetic issued"}
            # the arithmetic the precision mode issues, against its MEASURED
            # peak: the FP32 split = 3 MMAs per fp32 product (kind::f16 for
            # 3xF16 / 3xBF16, kind::tf32 for 3xTF32), TF32 = 1 kind::tf32
            f16 = args.precision == "fp32" and SPLIT != "3xtf32"
            mp = pk_meas.get("tcgen05_bf16_tflops" if f16 else "tcgen05_tf32_tflops")
            div = {"fp32": 3.0, "tf32": 1.0}.get(args.precision)
            if div and mp and mp > 0:
                r["kernel_ceiling"] = {
                    "value": mp / div, "unit": "TFLOP/s", "frac": ach / (mp / div),
                    "mode": args.precision,
                    "source": "measured tcgen05 kind::%s peak / %g" % ("f16" if f16 else "tf32", div)}
        else:
            ach = dom["bytes"] / dom["launches"] / (avg_ms / 1e3) / 1e9
            r = {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                 "frac": ach / pk["hbm_gbs"],
                 "peak_source": f"{pk_kind} HBM copy (MEASURED_PEAKS.json)"}
        r.update({"traffic": None, "kernel": name, "launches": dom["launches"],
                  "launch_ms": avg_ms, "share_of_kernel_time": dom["ms"] / total_ms,
                  "measured": note})
        return r

    roof_conc = roofline(kstats, f"concurrent timed region ({args.streams} streams, events on "
                                 "every 8th evaluation)")
    c1 = ctxs[0]
    c1.reset_stats()
    c1.set_profiling(True)
    nb.evaluate(sessions[:1], mine, prec)
    c1.set_profiling(False)
    roof = roofline(c1.kernel_stats(), "single-stream replay of the timed pool, events on every "
                                       "launch")
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if roof and os.path.exists(tf):
        t = json.load(open(tf)).get(roof["kernel"])
        if t:
            roof["traffic"] = t["dram_bytes_per_launch"]
            roof["traffic_note"] = t["note"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, sample = cpu_baseline_sample(timed_j, threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
               "sample": sample}

    # ---- the other precision tiers on the same timed pool (device-timed,
    # same sessions): SIMT = true fp32 FFMA everywhere, TF32 = 1xTF32
    modes = {}
    if not args.no_modes:
        for name, pm in (("simt", Precision.SIMT), ("tf32", Precision.TF32),
                         ("fp32_" + SPLIT, Precision.FP32)):
            if pm == prec:
                continue
            nb.evaluate(sessions, warm_pool, pm)
            mms, _ = timed_region(lambda: nb.evaluate(sessions, mine, pm))
            modes[name] = {"value": total_units / (mms / 1e3), "unit": UNIT,
                           "dtype": DTYPE[name], "tolerance": TOL_NOTE[name]}

    if rank == 0:
        cfg = config_block(args.steps, args.streams, ngpu)
        if len(devs) > 1:
            cfg["parallelism"] += ", one process driving every GPU"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ngpu,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": DTYPE[MODE_KEY[args.precision]], "data": "synthetic",
            "config": cfg,
            "precision": {"mode": args.precision,
                          "arithmetic": ARITH[args.precision],
                          "tolerance": TOL_NOTE[MODE_KEY[args.precision]]},
            "other_precisions": modes,
            "inference_ms": inf_ms / 10, "inference_origin_ms": inf_o_ms / 10,
            "inference_net_macs": nb.network_macs(best),
            "inference_network": best_info,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            # all ranks' algorithmic FLOPs over the max-over-ranks time
            "achieved_tflops_step": sum(costs) / (ms / 1e3) / 1e12,
            # LPT shard balance: the largest rank's estimated FLOPs over the mean
            "lpt_max_over_mean": (max(sum(c for c, a in zip(costs, assign) if a == r)
                                      for r in range(world)) / (sum(costs) / world)),
            "scheduler": {"evaluated": st.evaluated, "deduplicated": st.deduplicated,
                          "busy_ms": [round(b, 2) for b in st.busy_ms]},
            "roofline": roof,
            "roofline_concurrent": roof_conc,
            "peaks_measured": pk_meas,
            "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3)}
                        for k, v in kstats.items()},
            "cpu_baseline": cpu,
            "cpu": cpu_info() if rank == 0 else None,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
