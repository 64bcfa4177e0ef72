"""CPU-only: the product's planner (csrc/host/passes.cpp, exported through
neng_run_passes) against the reference's run_passes (oracle/_ref): plans,
member order, buffer assignment, layout order and contiguity stats must be
identical (acceptance.cpp:178-188 pattern), together with dependency edges,
toposort and validation errors (ir.cpp)."""
import time

import numpy as np
import pytest

from oracle import refapi
from paper_1805_11144_b200 import ir, networks, passes
from paper_1805_11144_b200.ir import Operator, SignalRef
from tests.support.models import chain_model, learning_model, make_signal, pipeline_variants
from tests.support.random_models import random_model


def same_plan(a: ir.PlannedModel, b: ir.PlannedModel):
    assert a.plan == b.plan
    assert a.buffers.buffer_of == b.buffers.buffer_of
    assert a.buffers.row_offset == b.buffers.row_offset
    assert [(x.rows, x.order, x.trailing, x.minibatched, x.trainable) for x in a.buffers.buffers] == \
        [(x.rows, x.order, x.trailing, x.minibatched, x.trainable) for x in b.buffers.buffers]
    assert a.stats.contiguous_read_fraction == b.stats.contiguous_read_fraction
    assert a.stats.gather_row_count == b.stats.gather_row_count
    assert a.stats.groups_per_step == b.stats.groups_per_step
    assert [(o.id, o.kind) for o in a.model.operators] == [(o.id, o.kind) for o in b.model.operators]


@pytest.mark.parametrize("seed", range(1, 31))
def test_random_models_plan_identical(seed):
    model = random_model(seed, 45)
    assert passes.dependency_edges(model) == refapi.dependency_edges(model)
    assert passes.toposort(model) == refapi.toposort(model)
    for cfg in pipeline_variants() + [ir.PipelineConfig(tree_depth=2), ir.PipelineConfig(tree_depth=4)]:
        same_plan(passes.run_passes(model, cfg), refapi.run_passes(model, cfg).to_python())


def test_built_networks_plan_identical():
    for model in (chain_model()[0], learning_model()[0],
                  networks.random_network(2, 16, 64, 4, 3, 4, 2, 1).model, networks.config0(steps=1).model):
        for cfg in pipeline_variants():
            same_plan(passes.run_passes(model, cfg), refapi.run_passes(model, cfg).to_python())


def test_planner_errors_match_reference():
    m = random_model(4, 20)
    with pytest.raises(ir.BuildError, match="transitive closure"):
        passes.run_passes(m, ir.PipelineConfig(planner=ir.Planner.TransitiveClosure))
    with pytest.raises(ir.BuildError, match="depth must be at least 1"):
        passes.run_passes(m, ir.PipelineConfig(tree_depth=0))
    # structural and ordering errors raise the reference's exception types (ir.cpp:228-463)
    bad = ir.BuiltModel()
    bad.signals = [make_signal(0, "c", [2], constant=True, initial=[1, 2]), make_signal(1, "t", [3])]
    bad.operators = [Operator.copy(0, SignalRef.full(bad.signals[0]), SignalRef.full(bad.signals[1]), False)]
    for fn in (passes.validate, refapi.validate):
        with pytest.raises(ir.StructuralError, match="src/dst shapes do not agree"):
            fn(bad)
    conflict = ir.BuiltModel()
    conflict.signals = [make_signal(0, "x", [1])]
    f = SignalRef.full(conflict.signals[0])
    conflict.operators = [Operator.reset(0, f, [1.0]), Operator.reset(1, f, [2.0])]
    for fn in (passes.validate, refapi.validate):
        with pytest.raises(ir.BuildError, match="write conflict on signal 'x'"):
            fn(conflict)


def test_config4_graph_plans_in_seconds():
    """The reference planner needs ~7 min and ~0.8 GB (O(n^2) merge matrix) on
    this 78,849-operator graph; ours indexes writes per signature."""
    w = networks.random_network(1, 2048, 512, 8, 8, 256, 1, 1)
    t0 = time.time()
    pm = passes.run_passes(w.model)
    dt = time.time() - t0
    assert len(pm.model.operators) == 78849
    assert 30 <= len(pm.plan) <= 60
    assert dt < 60, f"planning took {dt:.1f} s"
    # every group is single-kind and the plan is valid for the reference's own checker
    kinds = {o.id: o.kind for o in pm.model.operators}
    assert all(len({kinds[i] for i in g}) == 1 for g in pm.plan)


def test_config4_plan_identical_to_the_reference_planners():
    """Plan identity at config-4 scale: the repo planner's plan of the 78,849-
    operator graph equals the plan the reference's own run_passes produced
    (cached by oracle/make_ref_plan.py — the reference needs ~7 min for it)."""
    from oracle import make_ref_plan
    w = networks.random_network(1, 2048, 512, 8, 8, 256, 1, 1, name="config4_random_2048x512")
    ref, _ = make_ref_plan.load(w.model)  # raises if the cache was planned for another model
    same_plan(passes.run_passes(w.model), ref)
