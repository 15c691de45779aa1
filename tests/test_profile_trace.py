"""Measured-profile hook for the reference allocator's Phase 3 and trace export in the
reference trace-event schema (CPU tests; the reference is imported from /root/reference
when present — it is in the build container, not on the GPU box)."""

import json
import sys
from pathlib import Path

import pytest

from paper_2605_11005_b200.config import load_experiment
from paper_2605_11005_b200.profile import MeasuredStages, export_trace, measured_profile, predict_iteration

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/pkg/src")
STAGES = ROOT / "profiles" / "r01" / "stage_times_mixtral.json"


def _stages():
    if STAGES.exists():
        return MeasuredStages.from_json(STAGES.read_text())
    # shape of the Mixtral layer with representative per-micro-batch seconds
    return MeasuredStages(T=4096, H=4096, E=8, k=2, De=14336, a_fwd=7e-5, a_turn=7e-5, a_bwd=1e-4,
                          f_fwd=2.2e-3, f_bwd=2.3e-3, f_w=2.1e-3, link_gbs=700.0)


def test_prediction_monotone_in_ffn_share():
    ms = _stages()
    t_11 = predict_iteration(ms, 1, 1, 4)
    t_13 = predict_iteration(ms, 1, 3, 4)
    t_31 = predict_iteration(ms, 3, 1, 4)
    assert t_13 < t_11 < t_31          # more F ranks -> less F work per rank
    # A:F 2:2 processes twice the tokens of 1:1 in about the same time
    assert predict_iteration(ms, 2, 2, 4) == pytest.approx(t_11, rel=0.15)


def test_profile_is_deterministic_and_memoised():
    exp = load_experiment(str(ROOT / "configs" / "mixtral_layer.yaml"))
    prof = measured_profile(exp, _stages())

    class Alloc:
        attn_gpus, ffn_gpus = 2, 6

    assert prof(Alloc) == prof(Alloc) > 0


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_reference_phase3_refine_accepts_measured_profile():
    sys.path.insert(0, str(REF))
    from afpipe.allocator import AllocatorParams, canonical_allocation, phase3_refine

    exp = load_experiment(str(ROOT / "configs" / "mixtral_layer.yaml"))
    prof = measured_profile(exp, _stages())
    seed = canonical_allocation(4, 4, 8, 8, 8)
    best, t, improvements, trace = phase3_refine(seed, AllocatorParams(trials=40, radius=3, rng_seed=0), prof,
                                                 8, 8, 8)
    assert t <= prof(seed)
    assert len(trace) == 41
    # with no attention on the A side, the measured profile prefers more FFN GPUs
    assert best.ffn_gpus >= seed.ffn_gpus


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_trace_export_validates_against_reference_schema():
    jsonschema = pytest.importorskip("jsonschema")
    schema = json.loads((REF / "afpipe" / "schemas" / "trace_event.schema.json").read_text())
    ranks = [
        {"rank": 0, "role": "A", "ivs": [("A_f", 0, "compute", 0.0, 0.1, 0), ("M2N", 0, "comm.send", 0.1, 0.2, 1 << 20),
                                         ("A_t", 0, "compute", 2.0, 2.1, 0)]},
        {"rank": 1, "role": "F", "ivs": [("F_f", 0, "compute", 0.2, 1.9, 0), ("N2M", 0, "comm.send", 1.9, 2.0, 1 << 20),
                                         ("W", -1, "compute", 5.0, 6.0, 0)]},
    ]
    events = export_trace(ranks)
    jsonschema.validate(events, schema)
    sys.path.insert(0, str(REF))
    from afpipe.trace_io import parse_trace_events

    triples = parse_trace_events(json.dumps(events))
    assert len(triples) == 6 and triples[0] == (0, 100000, "A0")


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_reference_memory_estimate_restatement_matches_reference():
    sys.path.insert(0, str(REF))
    from afpipe.allocator import canonical_allocation
    from afpipe.config import load_experiment as ref_load
    from afpipe.placement import assign_layers, memory_estimate

    from paper_2605_11005_b200.profile import reference_memory_estimate

    for cfg in ("tiny.yaml", "mixtral_layer.yaml", "dsv3_layer.yaml"):
        path = str(ROOT / "configs" / cfg)
        ours, ref = load_experiment(path), ref_load(path)
        for n_attn, n_ffn in ((1, 1), (2, 6), (4, 4)):
            alloc = canonical_allocation(n_attn, n_ffn, n_attn + n_ffn, n_attn + n_ffn, n_attn + n_ffn)
            for comp in ("A", "F"):
                plan = assign_layers(ref.model.layers, ref.pipeline_depth, comp)
                want = memory_estimate(plan, ref.model, ref.workload, alloc).total
                assert reference_memory_estimate(ours, comp, n_attn, n_ffn) == pytest.approx(want, rel=1e-12)


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_reference_roofline_restatements_match_reference():
    sys.path.insert(0, str(REF))
    from afpipe import costs
    from afpipe.config import load_experiment as ref_load

    from paper_2605_11005_b200.profile import reference_intensities, reference_turning_points, roofline_attainable

    for cfg in ("tiny.yaml", "mixtral_layer.yaml", "dsv3_layer.yaml"):
        path = str(ROOT / "configs" / cfg)
        ours, ref = load_experiment(path), ref_load(path)
        ia, if_ = costs.arithmetic_intensities(ref.model, ref.workload)
        assert reference_intensities(ours) == pytest.approx((float(ia), float(if_)), rel=1e-15)
        for m, n in ((1, 1), (2, 6), (4, 4)):
            assert reference_turning_points(ref.cluster.gpu_peak, ref.cluster.ib_bw, m, n) == pytest.approx(
                costs.turning_points(ref.cluster, m, n), rel=1e-15)
        assert roofline_attainable(float(if_), 1.683e15, 9e11) == costs.roofline_attainable(if_, 1.683e15, 9e11)
