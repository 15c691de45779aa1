"""Measure per-stage times of the fused layer on one B200 and compare the
planner's predictions against measured AF-Pipe iterations (sweep JSONL).

    python scripts/measure_stages.py --out profiles/r01/stage_times_mixtral.json
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11005_b200.config import load_experiment  # noqa: E402
from paper_2605_11005_b200.moe import MoEShape  # noqa: E402
from paper_2605_11005_b200.profile import MeasuredStages, measure_stages, predict_iteration  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="configs/mixtral_layer.yaml")
ap.add_argument("--out", default=None)
ap.add_argument("--stages", default=None, help="reuse a stage-time JSON instead of measuring")
ap.add_argument("--sweep", default=None, help="sweep JSONL to compare predictions against")
a = ap.parse_args()
if a.stages:
    ms = MeasuredStages.from_json(Path(a.stages).read_text())
else:
    ms = measure_stages(MoEShape.from_experiment(load_experiment(a.config)))
    print(ms.to_json())
    if a.out:
        Path(a.out).write_text(ms.to_json())
if a.sweep:
    for line in open(a.sweep):
        r = json.loads(line)
        pred = predict_iteration(ms, r["A"], r["F"], r["mb"]) * 1e3
        print(f"{r['A']}:{r['F']} mb={r['mb']}: measured {r['ms_per_step']:.2f} ms, predicted {pred:.2f} ms "
              f"({pred / r['ms_per_step'] - 1:+.1%})")
