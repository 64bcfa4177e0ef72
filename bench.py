#!/usr/bin/env python
"""bench.py — timesteps/s and neuron-updates/s of the B200 executor on the
headline workload (BASELINE.json config 4: 2048 ensembles x 512 LIF = 1,048,576
neurons, 8-D, 8 decoded out-connections each, 256 white-noise inputs,
minibatch 256) against the measured HBM roofline, beside the reference CPU
executor (EngineCore<float> built from the reference sources).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  A "step" is one simulation timestep of the whole
minibatch.  `value` is device-timed (CUDA events on the launching stream, all
feeds resident in HBM, one persistent launch for the K timed steps); `e2e` is
the same metric through the C ABI entry neng_gpu_run with host f64 feeds and
host f64 probe outputs (H2D/D2H inside the timed region).  Multi-GPU: one
process per GPU.  Default (`--shard batch --scaling strong`): the north
star's minibatch sharding — the global minibatch of 256 rows is split into
256/N rows per GPU, each rank simulates its rows of the same network with no
collective on the data path (batch rows are independent, test_exec.cpp:246-267).
`--scaling weak` keeps 256 rows per GPU (N replicas).  `--shard ensemble`
splits the ensembles instead, with a per-step NCCL all-gather of the decoded
outputs.  Time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "timesteps/sec and neuron-updates/sec (×minibatch) vs HBM roofline, 1/2/4/8 GPU"
UNIT = "neuron-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="--shard batch: 'strong' splits the global minibatch (--batch) into batch/N rows per GPU; "
                         "'weak' runs --batch rows on every GPU")
    ap.add_argument("--shard", choices=["batch", "ensemble"], default="batch",
                    help="multi-GPU mode: 'batch' = one minibatch replica per GPU (weak scaling, no collective); "
                         "'ensemble' = the ensembles split across GPUs with a per-step NCCL all-gather of the "
                         "decoded outputs (strong scaling of one network)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def rows_per_rank(args, world):
    """Minibatch rows this rank simulates."""
    if args.shard == "batch" and args.scaling == "strong":
        if args.batch % world:
            raise SystemExit(f"--batch {args.batch} does not split over {world} GPUs")
        return args.batch // world
    return args.batch


def build_workload(args, rank, rows):
    from paper_1805_11144_b200 import networks, passes
    w = networks.random_network(args.seed, 2048, 512, 8, 8, 256, rows, 1, name="config4_random_2048x512")
    t0 = time.time()
    pm = passes.run_passes(w.model)
    plan_s = time.time() - t0
    return w, pm, plan_s


def feeds_for(w, steps, rank, seed):
    rng = np.random.default_rng(seed * 1000 + rank)
    return {node: rng.standard_normal((w.batch, steps, w.model.feed_slots[i].dim))
            for i, node in enumerate(sorted(w.feeds))}


def cpu_baseline(pm, neurons, sample_steps=20):
    """The reference EngineCore<float> (oracle/_ref) on the box's host cores:
    one single-row engine per thread (batch rows are independent), reference
    protocol: warm-up, reset, timed run."""
    from oracle import refapi
    threads = os.cpu_count() or 1
    secs = refapi.time_engines(pm, threads, 1, 1, sample_steps)
    rows = threads
    return {"value": rows * sample_steps * neurons / secs, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{threads} batch rows x {sample_steps} timesteps of the config-4 network "
                      f"({threads} single-row EngineCore<float>, one per host thread)",
            "seconds": secs}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1805_11144_b200 import networks
    w, pm, _ = build_workload(args, rank, args.batch)
    neurons = networks.neuron_count(w.model)
    from oracle import refapi
    threads = os.cpu_count() or 1
    rp = refapi.planned_from_python(pm)
    steps = max(args.steps // 100, 2)  # bounded sample: a few timesteps of `threads` rows
    secs = refapi.time_engines(rp, threads, 1, max(args.warmup // 5, 1), steps)
    value = threads * steps * neurons / secs
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": max(args.warmup // 5, 1), "ms_per_step": 1e3 * secs / steps * (args.batch / threads),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "config4_random_2048x512", "neurons": neurons, "batch": args.batch,
                       "sample_rows": threads, "engine": "EngineCore<float> (oracle/_ref, unmodified sources)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{threads} rows x {steps} timesteps, one single-row engine per thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    rank, world, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1805_11144_b200 import networks
    from paper_1805_11144_b200.engine import GpuEngine

    w, pm, plan_s = build_workload(args, rank, rows_per_rank(args, world))
    B = w.batch
    split = args.shard == "batch" and args.scaling == "strong"
    neurons = networks.neuron_count(w.model)
    bytes_step = networks.algorithmic_bytes_per_step(w.model, B)
    sharded = args.shard == "ensemble"
    eng = GpuEngine(pm, B, device=local, shard=(rank, world) if sharded else None)
    gather = None
    if sharded:
        from paper_1805_11144_b200.shard import TorchGather, attach_xhat_buffer, run_stepped
        xbuf, rank_floats = attach_xhat_buffer(eng, torch.device("cuda", local))
        gather = TorchGather(xbuf, rank_floats, rank, world) if world > 1 else (lambda parity: None)

    def advance(n, fptr, pptr):
        if sharded:
            return run_stepped(eng, n, fptr, pptr, gather, stream.cuda_stream)
        eng.run_device(n, fptr, pptr, stream.cuda_stream)
        return eng.last_launch_count()
    K, W = args.steps, max(args.warmup, 1)

    # device-resident feeds [slot][step][dim][B] f32 (white noise, generated on the device)
    slots = w.model.feed_slots
    dev = torch.device("cuda", local)
    # one explicit stream for everything (feeds, kernels, collectives, events); the
    # legacy default stream would not order against the engine's own stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    gen = torch.Generator(device=dev)
    gen.manual_seed(args.seed * 1000 + rank)

    def stage(steps):
        per = [steps * fs.dim * B for fs in slots]
        flat = torch.randn(max(sum(per), 1), generator=gen, device=dev, dtype=torch.float32)
        ptrs, at = [], 0
        for n in per:
            ptrs.append(flat.data_ptr() + 4 * at)
            at += n
        return flat, ptrs

    def probes(steps):
        dims = [w.model.signals[p.signal].size() for p in w.model.probes]
        ring = torch.empty(max(sum(dims) * steps * B, 1), dtype=torch.float32, device=dev)
        ptrs, at = [], 0
        for d in dims:
            ptrs.append(ring.data_ptr() + 4 * at)
            at += d * steps * B
        return ring, ptrs

    wf, wptr = stage(W)
    wr, wrp = probes(W)
    advance(W, wptr, wrp)
    torch.cuda.synchronize(dev)
    tf, tptr = stage(K)
    tr, trp = probes(K)

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = advance(K, tptr, trp)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    clocks = sampler.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    steps_per_s = K / (ms / 1e3)
    # batch sharding: every rank advances its own B rows; ensemble sharding: one minibatch in total
    global_b = B if sharded else B * world
    value = steps_per_s * neurons * global_b

    # end to end through the C ABI with host buffers (f64 feeds in, f64 probes out)
    e2e = None
    if not args.no_e2e and not sharded:
        Ke = min(K, 200)
        hfeeds = feeds_for(w, Ke, rank, args.seed)
        eng.reset()
        eng.run(Ke, hfeeds)  # warm-up call of the same size: staging buffers are allocated once per engine
        eng.reset()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        eng.run(Ke, hfeeds)
        sec = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([sec], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            sec = float(t.item())
        h2d = sum(fs.dim for fs in slots) * B * 4
        d2h = sum(w.model.signals[p.signal].size() for p in w.model.probes) * B * 4
        e2e = {"value": Ke / sec * neurons * global_b, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": Ke,
               "note": "neng_gpu_run: host f64 feeds -> f32 staging -> H2D -> fused kernel -> probe D2H -> f64"}

    if rank != 0:
        return
    peak, peak_src = peaks()
    launch_s = (ms / 1e3) / max(launches, 1)
    bytes_rank = bytes_step / world if sharded else bytes_step  # a shard moves its ensembles' share
    achieved = bytes_rank * (K / max(launches, 1)) / launch_s / 1e9
    traffic = None
    try:
        if sharded:
            raise FileNotFoundError("the committed capture is of the unsharded kernel")
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            prof = json.load(f)
        traffic = prof["dram_bytes_per_step"] * (K / max(launches, 1))
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if (sharded or split) else "weak",
        "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": "config4_random_2048x512", "neurons": neurons, "batch_per_gpu": B,
                   "global_batch": global_b,
                   "parallelism": (f"ensemble shards x{world} (per-step NCCL all-gather of xhat)" if sharded
                                   else f"minibatch split x{world} ({B} rows per GPU, no collective)" if split
                                   else f"minibatch replicas x{world}"),
                   "ensembles": 2048, "neurons_per_ensemble": 512, "dims": 8, "out_connections": 8,
                   "inputs": 256, "operators": len(pm.model.operators), "groups_per_step": len(pm.plan),
                   "plan_seconds": round(plan_s, 2), "mode": "fused" if eng.mode() == 2 else "generic",
                   "l2": "no flush: per-step working set (v, r = 2.1 GB) exceeds the 126 MB L2"},
        "timesteps_per_sec": steps_per_s,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_step": bytes_step},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import refapi
            line["cpu_baseline"] = cpu_baseline(refapi.planned_from_python(pm), neurons)
        except Exception as ex:  # the oracle travels prebuilt; report rather than die
            line["cpu_baseline"] = {"error": str(ex)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
