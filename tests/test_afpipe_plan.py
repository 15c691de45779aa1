"""AF-Pipe issue order: the runtime's planner reproduces the reference simulator's
per-lane order and start times (tests/golden/afpipe_orders.json, generated from
/root/reference sim.simulate / taskgraph._build_afpipe by make_golden.py)."""

import json
from pathlib import Path

import pytest

from paper_2605_11005_b200.afpipe import (
    COMPUTE,
    StageDurations,
    exposed_comm_global,
    exposed_comm_per_rank,
    plan_afpipe,
)

GOLD = json.loads((Path(__file__).parent / "golden" / "afpipe_orders.json").read_text())


def _plan(case):
    d = case["durations_ns"]
    return plan_afpipe(case["layers"], case["depth"], case["microbatches"],
                       StageDurations(attn_fwd=d["attn_fwd"], ffn_fwd=d["ffn_fwd"], m2n=d["m2n"]))


@pytest.mark.parametrize("name", sorted(GOLD))
def test_lane_orders_match_reference(name):
    case = GOLD[name]
    plan = _plan(case)
    assert len(plan.tasks) == case["num_tasks"]
    assert plan.credits == case["credits"]
    assert plan.iteration_ns == case["iteration_ns"]
    for key, expected in case["lanes"].items():
        owner, lane = key.split("|")
        got = [[t.id, t.start_ns, t.end_ns] for t in plan.order(owner, lane)]
        assert got == expected, key


@pytest.mark.parametrize("name", sorted(GOLD))
def test_exposed_comm_matches_reference_definition(name):
    case = GOLD[name]
    plan = _plan(case)
    events = [(t.start_ns, t.end_ns, t.lane == COMPUTE) for t in plan.tasks]
    assert exposed_comm_global(events) == case["exposed_comm_ns"]


def test_single_layer_graph_shape():
    plan = plan_afpipe(1, 1, 1, StageDurations(1000, 1000, 100))
    kinds = [t.kind for t in plan.tasks]
    assert kinds.count("FwdCompute") == 2 and kinds.count("BwdCompute") == 2
    assert kinds.count("M2NSend") == 2 and kinds.count("M2NRecv") == 2


def test_twins_share_start():
    plan = plan_afpipe(2, 1, 3, StageDurations(700, 900, 150))
    for t in plan.tasks:
        if t.twin is not None:
            assert plan.tasks[t.twin].start_ns == t.start_ns


def test_per_rank_exposed_is_at_least_global():
    plan = plan_afpipe(1, 1, 4, StageDurations(300, 500, 600))
    ev = [(t.start_ns, t.end_ns, t.lane == COMPUTE) for t in plan.tasks]
    by_rank = {}
    for t in plan.tasks:
        by_rank.setdefault(t.owner, []).append((t.start_ns, t.end_ns, t.lane == COMPUTE))
    per = exposed_comm_per_rank(by_rank)
    assert max(per.values()) >= exposed_comm_global(ev)
