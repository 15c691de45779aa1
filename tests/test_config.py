"""Config drop-in parity: the reference's own config cases (pkg/tests/test_config.py)
re-run against paper_2605_11005_b200.config, plus every outcome pinned by the
reference itself in tests/golden/config_cases.json (make_golden.py)."""

import json

import pytest

from paper_2605_11005_b200.config import (
    ConfigError,
    InvalidValue,
    MissingField,
    ScheduleKind,
    SchemaViolation,
    load_experiment,
    parse_experiment,
    serialize_experiment,
    validate,
)

CASES = json.loads((__import__("pathlib").Path(__file__).parent / "golden" / "config_cases.json").read_text())
DEEPSEEK_DOC = CASES["deepseek"]["doc"]


@pytest.mark.parametrize("name", sorted(CASES))
def test_outcome_matches_reference(name):
    case = CASES[name]
    if case["ok"]:
        exp = parse_experiment(case["doc"])
        assert serialize_experiment(exp) == case["canonical"]
    else:
        with pytest.raises(ConfigError) as exc:
            parse_experiment(case["doc"])
        assert type(exc.value).__name__ == case["error"]
        assert getattr(exc.value, "name", None) == case["name"]
        assert str(exc.value) == case["message"]


def test_parse_deepseek_card():
    exp = parse_experiment(DEEPSEEK_DOC)
    assert (exp.model.layers, exp.model.hidden, exp.model.experts, exp.model.topk, exp.model.moe_hidden) == (
        28, 2048, 64, 4, 1408)
    assert exp.schedule_kind is ScheduleKind.AFPIPE
    assert exp.pipeline_depth == 2 and exp.virtual_stages == 14
    assert validate(exp) == []


def test_defaults_applied():
    exp = parse_experiment(DEEPSEEK_DOC)
    assert exp.model.bytes_per_element == 2 and exp.model.gqa_group == 1 and exp.cluster.nvlink_bw == 0.0


def test_topk_exceeding_experts_is_invalid():
    doc = DEEPSEEK_DOC.replace("topk: 4", "topk: 8").replace("experts: 64", "experts: 4")
    with pytest.raises(InvalidValue) as exc:
        parse_experiment(doc)
    assert exc.value.name == "topk" and "exceeds" in exc.value.reason


def test_missing_required_field():
    with pytest.raises(MissingField) as exc:
        parse_experiment(DEEPSEEK_DOC.replace("  seq_len: 4096\n", ""))
    assert exc.value.name == "workload.seq_len"


def test_unknown_key_and_section():
    with pytest.raises(SchemaViolation):
        parse_experiment(DEEPSEEK_DOC.replace("model:\n", "model:\n  vocab: 32000\n"))
    with pytest.raises(SchemaViolation):
        parse_experiment(DEEPSEEK_DOC + "\nextras:\n  foo: 1\n")


def test_round_trip_identity():
    exp = parse_experiment(DEEPSEEK_DOC)
    text = serialize_experiment(exp)
    assert parse_experiment(text) == exp and serialize_experiment(parse_experiment(text)) == text


def test_validate_returns_all_violations():
    exp = parse_experiment(DEEPSEEK_DOC)
    object.__setattr__(exp.model, "layers", 0)
    v = validate(exp)
    assert any(s.startswith("layers:") for s in v) and any(s.startswith("pipeline_depth:") for s in v)


@pytest.mark.parametrize("name", ["tiny.yaml", "mixtral_layer.yaml", "dsv3_layer.yaml"])
def test_repo_configs_parse(name):
    from pathlib import Path

    exp = load_experiment(str(Path(__file__).resolve().parents[1] / "configs" / name))
    assert exp.schedule_kind is ScheduleKind.AFPIPE
    assert exp.model.bytes_per_element == 2


def test_reference_deepseek_experiment_is_a_valid_hot_path_shape():
    """The layer of the reference's own shipped experiment (pkg/configs/deepseek_moe.yaml:
    hidden 2048, 64 experts top-4, moe_hidden 1408) maps to a hot-path shape the kernels
    accept (128-wide GEMM tails; GPU parity in test_gpu_parity.py
    deepseek_moe_yaml_De1408 / deepseek_moe_yaml_layer)."""
    from paper_2605_11005_b200.moe import MoEShape

    shape = MoEShape.from_experiment(parse_experiment(DEEPSEEK_DOC))
    assert (shape.H, shape.E, shape.k, shape.De) == (2048, 64, 4, 1408)
    shape.validate()
    with pytest.raises(ValueError):
        MoEShape(T=8, H=2048, E=64, k=4, De=1400).validate()
