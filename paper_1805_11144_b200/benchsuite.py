"""The reference's benchmark suite and CSV schema on the B200 engine
(SURVEY §8(f)4): proj/src/bench.cpp:207-278 (run_bench, ablation_suite,
bench_csv_header / bench_csv_row) and the CLI of proj/tools/nengine_main.cpp.

The three benchmark networks follow bench.cpp's builders (integrator: one
recurrent memory per dimension; cconv: circular convolution through 4 product
ensembles per spectral bin of the unitary DFT; pes: a learned decoded
connection) with this package's NetBuilder lowering and least-squares
decoders (NetBuilder.solve_decoders, the frontend's solve without Eigen).
The lowering is the unfolded one (decoders, then transforms), so operator
counts differ from the reference frontend's folded lowering of the same
network.  Run time follows run_bench's protocol: warm-up run, reset, timed
run (bench.cpp:221-225) — here GpuEngine.run with host f64 feeds and probes.

    python -m paper_1805_11144_b200.benchsuite --benchmark cconv --dims 8 --ablation [--output f.csv]

`correctness_max_err` needs a reference executor, which the product does not
ship: the CLI prints nan unless a checker is passed to run_bench (the tests
pass the reference's run_reference, tests/test_benchsuite.py)."""
from __future__ import annotations

import argparse
import math
import time
from dataclasses import dataclass, field, replace
from typing import Callable, Dict, List, Optional

import numpy as np

from . import ir, networks, passes
from .engine import GpuEngine
from .ir import BuildError

CSV_HEADER = ("benchmark,dims,batch,planner,tree_depth,unroll,merge,sort,simplify,"
              "operator_count,groups_per_step,contiguous_read_fraction,build_time_s,"
              "run_time_s,steps,correctness_max_err")


@dataclass
class BenchmarkSpec:  # bench.hpp:17-26
    name: str = "integrator"  # integrator | cconv | pes
    dims: int = 4
    neurons_per_dim: int = 50
    steps: int = 1000
    dt: float = 0.001
    seed: int = 1
    batch: int = 1
    unroll: int = 1


@dataclass
class BenchmarkSetup:
    model: ir.BuiltModel
    feeds: Dict[int, np.ndarray]
    outputs: List[int] = field(default_factory=list)


@dataclass
class BenchResult:
    spec: BenchmarkSpec
    config: ir.PipelineConfig
    operator_count: int = 0
    stats: ir.ContiguityStats = field(default_factory=ir.ContiguityStats)
    build_time_s: float = 0.0
    run_time_s: float = 0.0
    correctness_max_err: float = float("nan")


def _validate(spec: BenchmarkSpec):  # bench.cpp:17-23
    if spec.dims < 1:
        raise BuildError("benchmark dims must be at least 1")
    if spec.steps < 1:
        raise BuildError("benchmark steps must be at least 1")
    if spec.batch < 1:
        raise BuildError("benchmark batch must be at least 1")
    if spec.neurons_per_dim < 1:
        raise BuildError("benchmark neurons-per-dim must be at least 1")


def constant_feed(batch: int, steps: int, row, vary_batch: bool) -> np.ndarray:
    """[batch][steps][dim], row scaled by 1 / (1 + 0.25 b) when vary_batch (bench.cpp:26-39)."""
    row = np.asarray(row, dtype=np.float64)
    f = 1.0 / (1.0 + 0.25 * np.arange(batch)) if vary_batch else np.ones(batch)
    return np.broadcast_to(f[:, None, None] * row[None, None, :], (batch, steps, row.size)).copy()


def build_integrator(spec: BenchmarkSpec) -> BenchmarkSetup:
    tau = 0.1
    nb = networks.NetBuilder(spec.seed, spec.dt)
    node, u = nb.feedable_node(spec.dims, np.zeros(spec.dims))
    outs = []
    for k in range(spec.dims):
        e = nb.ensemble(spec.neurons_per_dim, 1, radius=1.2)
        xhat = nb.decoded(e, nb.solve_decoders(e, radius=1.2))
        sel = np.zeros((1, spec.dims))
        sel[0, k] = tau
        nb.connect(u, e.in_, sel, synapse=tau)
        nb.connect(xhat, e.in_, None, synapse=tau)
        outs.append(nb.probe(xhat, f"x{k}"))
    drive = [1.0 - 0.5 * k / max(1, spec.dims - 1) for k in range(spec.dims)]
    return BenchmarkSetup(nb.m, {node: constant_feed(spec.batch, spec.steps, drive, True)}, outs)


def build_cconv(spec: BenchmarkSpec) -> BenchmarkSetup:
    d = spec.dims
    s = 0.7 * math.sqrt(d)
    root_d = math.sqrt(d)
    jk = (np.arange(d)[:, None] * np.arange(d)[None, :]) % d
    U = np.cos(2 * math.pi * jk / d) / root_d
    V = -np.sin(2 * math.pi * jk / d) / root_d
    nb = networks.NetBuilder(spec.seed, spec.dt)
    node_a, a = nb.feedable_node(d, np.zeros(d))
    node_b, b = nb.feedable_node(d, np.zeros(d))
    c = nb.passthrough_node(d)
    out_gain = root_d / (s * s)
    for j in range(d):
        for typ, (ra, rb) in enumerate(((U[j], U[j]), (V[j], V[j]), (U[j], V[j]), (V[j], U[j]))):
            e = nb.ensemble(2 * spec.neurons_per_dim, 2, radius=math.sqrt(2.0))
            xhat = nb.decoded(e, nb.solve_decoders(e, lambda p: p[:, :1] * p[:, 1:2], 1, radius=math.sqrt(2.0)))
            nb.connect(a, e.in_, np.vstack([s * ra, np.zeros(d)]), synapse=0.0)
            nb.connect(b, e.in_, np.vstack([np.zeros(d), s * rb]), synapse=0.0)
            sign = -1.0 if typ == 1 else 1.0
            basis = U if typ < 2 else V
            nb.connect(xhat, c, (sign * out_gain * basis[:, j])[:, None], synapse=0.01)
    outs = [nb.probe(c, "c")]
    fa, fb = np.zeros(d), np.zeros(d)
    fa[0] = 1.0
    fb[1 % d] += 0.7
    fb[min(3, d - 1)] += 0.5
    fb *= 0.86 / np.linalg.norm(fb)
    feeds = {node_a: constant_feed(spec.batch, spec.steps, fa, True),
             node_b: constant_feed(spec.batch, spec.steps, fb, True)}
    return BenchmarkSetup(nb.m, feeds, outs)


def build_pes(spec: BenchmarkSpec) -> BenchmarkSetup:
    d = spec.dims
    level = 0.5 / math.sqrt(d)
    nb = networks.NetBuilder(spec.seed, spec.dt)
    node_u, u = nb.feedable_node(d, np.full(d, level))
    node_t, target = nb.feedable_node(d, np.full(d, level))
    e = nb.ensemble(spec.neurons_per_dim * d, d)
    out = nb.passthrough_node(d)
    err = nb.passthrough_node(d)
    nb.connect(u, e.in_, None, synapse=0.005)
    # the learned connection starts at the zero function's decoders
    nb.connect(e.out, out, np.zeros((d, e.n)), synapse=0.005, learned_rate=1e-4, error=err)
    nb.connect(out, err, scalar=1.0, synapse=0.0)
    nb.connect(target, err, scalar=-1.0, synapse=0.0)
    outs = [nb.probe(out, "out"), nb.probe(err, "err")]
    feeds = {node_u: constant_feed(spec.batch, spec.steps, np.full(d, level), False),
             node_t: constant_feed(spec.batch, spec.steps, np.full(d, level), True)}
    return BenchmarkSetup(nb.m, feeds, outs)


def build_benchmark(spec: BenchmarkSpec) -> BenchmarkSetup:
    _validate(spec)
    builders = {"integrator": build_integrator, "cconv": build_cconv, "pes": build_pes}
    if spec.name not in builders:
        raise BuildError(f"unknown benchmark '{spec.name}'")
    return builders[spec.name](spec)


Checker = Callable[[ir.PlannedModel, ir.BuiltModel, int, dict, int, dict], float]


def run_bench(spec: BenchmarkSpec, config: ir.PipelineConfig, checker: Optional[Checker] = None,
              device: int = 0) -> BenchResult:
    """bench.cpp:207-232 on the GPU engine; checker(planned, model, steps, feeds, batch, probes) -> max abs error."""
    r = BenchResult(spec, config)
    t0 = time.perf_counter()
    setup = build_benchmark(spec)
    pm = passes.run_passes(setup.model, config)
    r.operator_count = len(pm.model.operators)
    r.stats = pm.stats
    eng = GpuEngine(pm, spec.batch, spec.unroll, device=device)
    r.build_time_s = time.perf_counter() - t0
    eng.run(spec.steps, setup.feeds)  # warm-up, excluded from timing
    eng.reset()
    t1 = time.perf_counter()
    out = eng.run(spec.steps, setup.feeds)
    r.run_time_s = time.perf_counter() - t1
    if checker is not None:
        r.correctness_max_err = checker(pm, setup.model, spec.steps, setup.feeds, spec.batch, out)
    return r


def ablation_suite(base: BenchmarkSpec, checker: Optional[Checker] = None, tree_depth: int = 3,
                   device: int = 0) -> List[BenchResult]:
    """The cumulative optimisation ladder (bench.cpp:234-260)."""
    unrolled = base.unroll if base.unroll > 1 else 10
    cfg = ir.PipelineConfig(merge=True, simplify=False, planner=ir.Planner.Greedy, tree_depth=1, sort=False)
    rows = []
    spec = replace(base, unroll=1)
    rows.append(run_bench(spec, replace(cfg), checker, device))  # merge only, greedy
    spec = replace(base, unroll=unrolled)
    rows.append(run_bench(spec, replace(cfg), checker, device))  # + unroll
    cfg = replace(cfg, planner=ir.Planner.Tree, tree_depth=tree_depth)
    rows.append(run_bench(spec, replace(cfg), checker, device))  # + tree planner
    cfg = replace(cfg, sort=True)
    rows.append(run_bench(spec, replace(cfg), checker, device))  # + sort
    cfg = replace(cfg, simplify=True)
    rows.append(run_bench(spec, replace(cfg), checker, device))  # + simplify
    return rows


def csv_row(r: BenchResult) -> str:  # bench.cpp:268-278 (printf formats)
    c, s = r.config, r.spec
    return "%s,%d,%d,%s,%d,%d,%d,%d,%d,%d,%d,%.17g,%.6f,%.6f,%d,%.17g" % (
        s.name, s.dims, s.batch, "greedy" if c.planner == ir.Planner.Greedy else "tree", c.tree_depth, s.unroll,
        int(c.merge), int(c.sort), int(c.simplify), r.operator_count, r.stats.groups_per_step,
        r.stats.contiguous_read_fraction, r.build_time_s, r.run_time_s, s.steps, r.correctness_max_err)


def main(argv=None):  # tools/nengine_main.cpp:10-76
    ap = argparse.ArgumentParser(description="B200 engine: the reference benchmark suite, CSV output")
    ap.add_argument("--benchmark", choices=["integrator", "cconv", "pes"], default="integrator")
    ap.add_argument("--dims", type=int, default=4)
    ap.add_argument("--neurons-per-dim", type=int, default=50)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--dt", type=float, default=0.001)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--unroll", type=int, default=1)
    ap.add_argument("--planner", choices=["greedy", "tree"], default="tree")
    ap.add_argument("--tree-depth", type=int, default=3)
    ap.add_argument("--no-merge", action="store_true")
    ap.add_argument("--no-sort", action="store_true")
    ap.add_argument("--no-simplify", action="store_true")
    ap.add_argument("--ablation", action="store_true")
    ap.add_argument("--output", default="")
    a = ap.parse_args(argv)
    for k in ("dims", "neurons_per_dim", "steps", "batch", "unroll", "tree_depth"):
        if getattr(a, k) < 1:
            ap.error(f"--{k.replace('_', '-')} must be positive")
    spec = BenchmarkSpec(a.benchmark, a.dims, a.neurons_per_dim, a.steps, a.dt, a.seed, a.batch, a.unroll)
    cfg = ir.PipelineConfig(merge=not a.no_merge, simplify=not a.no_simplify,
                            planner=ir.Planner.Greedy if a.planner == "greedy" else ir.Planner.Tree,
                            tree_depth=a.tree_depth, sort=not a.no_sort)
    rows = ablation_suite(spec, None, a.tree_depth) if a.ablation else [run_bench(spec, cfg)]
    csv = CSV_HEADER + "\n" + "".join(csv_row(r) + "\n" for r in rows)
    print(csv, end="")
    if a.output:
        with open(a.output, "w") as f:
            f.write(csv)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
