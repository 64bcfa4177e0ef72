"""The reference's benchmark suite / CSV schema / ablation ladder on the GPU
engine (paper_1805_11144_b200/benchsuite.py, bench.cpp:207-278,
tools/nengine_main.cpp).  The GPU rows' probes are checked bit-for-bit against
the reference EngineCore<float> on the same plan, and correctness_max_err is
the reference's own column: max |engine - run_reference| (the f64 interpreter,
compare(out, ref, 0, 0).max_abs_err)."""
import os

import numpy as np
import pytest

from oracle import refapi
from paper_1805_11144_b200 import benchsuite as bs
from paper_1805_11144_b200 import ir

REF_HEADER = ("benchmark,dims,batch,planner,tree_depth,unroll,merge,sort,simplify,operator_count,"
              "groups_per_step,contiguous_read_fraction,build_time_s,run_time_s,steps,correctness_max_err")


def test_csv_header_and_row_format_match_the_reference():
    assert bs.CSV_HEADER == REF_HEADER
    r = bs.BenchResult(bs.BenchmarkSpec("cconv", 8, 50, 100, 0.001, 1, 2, 10),
                       ir.PipelineConfig(True, True, ir.Planner.Tree, 3, True), 258,
                       ir.ContiguityStats(0.875, 12, 24), 1.25, 0.5, 1e-6)
    assert bs.csv_row(r) == "cconv,8,2,tree,3,10,1,1,1,258,24,0.875,1.250000,0.500000,100,9.9999999999999995e-07"


def test_spec_validation_messages():
    for kw, msg in (({"dims": 0}, "dims"), ({"steps": 0}, "steps"), ({"batch": 0}, "batch"),
                    ({"neurons_per_dim": 0}, "neurons-per-dim")):
        with pytest.raises(ir.BuildError, match=msg):
            bs.build_benchmark(bs.BenchmarkSpec(**kw))
    with pytest.raises(ir.BuildError, match="unknown benchmark"):
        bs.build_benchmark(bs.BenchmarkSpec("nope"))


def _checker(pm, model, steps, feeds, batch, out):
    ref32 = refapi.RefEngine(pm, batch).run(steps, feeds)
    for k in ref32:
        assert np.array_equal(out[k].view(np.uint64), ref32[k].view(np.uint64)), f"probe {k}"
    ref = refapi.run_reference(model, steps, feeds, batch)
    return max(float(np.abs(out[k] - ref[k]).max()) for k in ref)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["integrator", "cconv", "pes"])
def test_ablation_ladder_on_the_gpu(name):
    spec = bs.BenchmarkSpec(name, dims=4, neurons_per_dim=50, steps=200, batch=2)
    rows = bs.ablation_suite(spec, _checker)
    assert [(r.config.planner, r.config.sort, r.config.simplify, r.spec.unroll) for r in rows] == [
        (ir.Planner.Greedy, False, False, 1), (ir.Planner.Greedy, False, False, 10), (ir.Planner.Tree, False, False, 10),
        (ir.Planner.Tree, True, False, 10), (ir.Planner.Tree, True, True, 10)]
    csv = bs.CSV_HEADER + "\n" + "".join(bs.csv_row(r) + "\n" for r in rows)
    print("\n" + csv)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/ablation_{name}.csv", "w") as f:
        f.write(csv)
    for r in rows:
        # fp32 against the f64 interpreter: the reference's own engines differ by this much too
        assert r.correctness_max_err < 0.05, (name, r.correctness_max_err)
