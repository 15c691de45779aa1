"""Generate the committed golden fixtures under tests/golden/.

Runs in the build container only (it imports the reference from
/root/reference, which does not exist on the GPU box):

    python tests/golden/make_golden.py

Produces
  afpipe_orders.json   reference build_task_graph + simulate (taskgraph.py:262-356,
                       sim.py:101-216) per-(owner, lane) task order and start times
                       for several AF-Pipe DAGs, plus the reference exposed_comm.
  config_cases.json    reference parse_experiment outcome (canonical document or
                       exception type / name) for valid and invalid documents.
  moe_kat_*.npz        oracle known-answer vectors for small shapes (the reference
                       has no MoE arithmetic, so these are this repo's own KATs:
                       "parity unpinned" — see DESIGN.md §3).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src")

AFPIPE_CASES = [
    # name, layers, depth, microbatches, t_attn, t_ffn, t_m2n (seconds)
    ("single_layer_4mb", 1, 1, 4, 1e-3, 1e-3, 0.25e-3),
    ("tiny_L2_2mb", 2, 1, 2, 1e-3, 1e-3, 0.25e-3),
    ("mixtral_like_4mb", 1, 1, 4, 0.4e-3, 2.2e-3, 0.08e-3),
    ("comm_heavy_8mb", 1, 1, 8, 0.3e-3, 0.5e-3, 0.6e-3),
    ("depth2_L4_4mb", 4, 2, 4, 0.7e-3, 1.3e-3, 0.2e-3),
    ("depth2_L6_3mb", 6, 2, 3, 1.1e-3, 0.9e-3, 0.35e-3),
    ("depth3_L3_5mb", 3, 3, 5, 0.5e-3, 0.8e-3, 0.1e-3),
]

BASE_DOC = """
model:
  layers: 28
  hidden: 2048
  experts: 64
  topk: 4
  moe_hidden: 1408
workload:
  seq_len: 4096
  micro_batch: 1
  num_microbatches: 8
cluster:
  total_gpus: 16
  gpus_per_node: 8
  total_nics: 16
  gpu_peak: 9.89e14
  ib_bw: 1.0e11
schedule:
  schedule_kind: afpipe
  pipeline_depth: 2
  virtual_stages: 14
  ep_size: 16
"""

CONFIG_CASES = {
    "deepseek": BASE_DOC,
    "default_vstages": BASE_DOC.replace("  virtual_stages: 14\n", ""),
    "topk_exceeds": BASE_DOC.replace("topk: 4", "topk: 8").replace("experts: 64", "experts: 4"),
    "missing_seq": BASE_DOC.replace("  seq_len: 4096\n", ""),
    "unknown_key": BASE_DOC.replace("model:\n", "model:\n  vocab: 32000\n"),
    "unknown_section": BASE_DOC + "\nextras:\n  foo: 1\n",
    "non_int": BASE_DOC.replace("layers: 28", "layers: twenty"),
    "depth_bound": BASE_DOC.replace("virtual_stages: 14", "virtual_stages: 16"),
    "one_gpu": BASE_DOC.replace("total_gpus: 16", "total_gpus: 1"),
    "bad_kind": BASE_DOC.replace("schedule_kind: afpipe", "schedule_kind: pipedream"),
    "bool_int": BASE_DOC.replace("topk: 4", "topk: true"),
    "float_str": BASE_DOC.replace("ib_bw: 1.0e11", "ib_bw: '1e11'"),
    "bad_float": BASE_DOC.replace("ib_bw: 1.0e11", "ib_bw: fast"),
    "empty": "",
    "list_top": "- 1\n- 2\n",
    "null_section": BASE_DOC.replace("schedule:\n  schedule_kind: afpipe\n  pipeline_depth: 2\n  virtual_stages: 14\n  ep_size: 16\n", "schedule:\n"),
    "scalar_section": BASE_DOC.replace("workload:\n  seq_len: 4096\n  micro_batch: 1\n  num_microbatches: 8\n", "workload: 3\n"),
    "bytes4": BASE_DOC.replace("moe_hidden: 1408", "moe_hidden: 1408\n  bytes_per_element: 4"),
    "bytes3": BASE_DOC.replace("moe_hidden: 1408", "moe_hidden: 1408\n  bytes_per_element: 3"),
    "gpn9": BASE_DOC.replace("gpus_per_node: 8", "gpus_per_node: 9"),
    "zero_peak": BASE_DOC.replace("gpu_peak: 9.89e14", "gpu_peak: 0"),
    "malformed": "model: [1, 2\n",
}

KAT_CASES = [
    # name, T, H, E, k, De, seed, extra kwargs for make_inputs
    ("tiny", 64, 256, 8, 2, 256, 0, {}),
    ("ties", 48, 256, 8, 2, 256, 3, {"tie_rows": [(1, 5), (2, 6)]}),
    ("skew", 64, 256, 8, 2, 256, 4, {"skew": 2.0}),
    ("topk4", 40, 512, 16, 4, 256, 5, {}),
]


def _ref():
    sys.path.insert(0, str(REF_SRC))
    import afpipe  # noqa: F401  (the reference package)
    return afpipe


def afpipe_orders():
    _ref()
    from afpipe.allocator import canonical_allocation
    from afpipe.config import ClusterConfig, Experiment, ModelConfig, ScheduleKind, Workload
    from afpipe.costs import StageTimes
    from afpipe.placement import ATTN, FFN, assign_layers
    from afpipe.sim import exposed_comm, simulate
    from afpipe.taskgraph import build_task_graph

    out = {}
    for name, L, p, mb, ta, tf, tm in AFPIPE_CASES:
        exp = Experiment(
            model=ModelConfig(layers=L, hidden=64, experts=8, topk=2, moe_hidden=64),
            workload=Workload(seq_len=64, micro_batch=1, num_microbatches=mb),
            cluster=ClusterConfig(total_gpus=2, gpus_per_node=2, total_nics=2, gpu_peak=1e12, ib_bw=1e10),
            schedule_kind=ScheduleKind.AFPIPE, pipeline_depth=p, virtual_stages=L // p, ep_size=1)
        alloc = canonical_allocation(1, 1, 2, 2, 2)
        graph = build_task_graph(exp, alloc, assign_layers(L, p, ATTN), assign_layers(L, p, FFN),
                                 times=StageTimes(t_attn=ta, t_ffn=tf, t_a2a=0.0, t_m2n=tm, t_p2p=0.0))
        trace, res = simulate(graph)
        lanes: dict[str, list] = {}
        for ev in sorted(trace.events, key=lambda e: (e.owner, e.lane, e.start_ns, e.task_id)):
            lanes.setdefault(f"{ev.owner}|{ev.lane}", []).append([ev.task_id, ev.start_ns, ev.end_ns])
        out[name] = {
            "layers": L, "depth": p, "microbatches": mb,
            "durations_ns": {"attn_fwd": round(ta * 1e9), "ffn_fwd": round(tf * 1e9), "m2n": round(tm * 1e9)},
            "num_tasks": len(graph), "credits": graph.credits,
            "iteration_ns": trace.iteration_ns, "exposed_comm_ns": round(exposed_comm(trace) * 1e9),
            "lanes": lanes,
        }
    (HERE / "afpipe_orders.json").write_text(json.dumps(out, indent=1, sort_keys=True))


def config_cases():
    _ref()
    from afpipe.config import parse_experiment, serialize_experiment

    out = {}
    for name, doc in CONFIG_CASES.items():
        try:
            exp = parse_experiment(doc)
            out[name] = {"doc": doc, "ok": True, "canonical": serialize_experiment(exp)}
        except Exception as exc:  # noqa: BLE001
            out[name] = {"doc": doc, "ok": False, "error": type(exc).__name__,
                         "name": getattr(exc, "name", None), "message": str(exc)}
    (HERE / "config_cases.json").write_text(json.dumps(out, indent=1, sort_keys=True))


def moe_kats():
    sys.path.insert(0, str(ROOT))
    from oracle import oracle as O

    for name, T, H, E, k, De, seed, kw in KAT_CASES:
        x, wg, w1, w3, w2, dy = O.make_inputs(T, H, E, k, De, seed=seed, **kw)
        f = O.moe_forward(x, wg, w1, w3, w2, k)
        b = O.moe_backward(f, x, wg, w1, w3, w2, dy)
        np.savez_compressed(
            HERE / f"moe_kat_{name}.npz",
            shape=np.array([T, H, E, k, De, seed]),
            x_bits_sum=np.array([int(x.astype(np.int64).sum())]),
            logits=f.logits, idx=f.idx, w=f.w, counts=f.counts, pad_off=f.pad_off, row_map=f.row_map,
            y=f.y.astype(np.float32), dx=b.dx.astype(np.float32), dwg=b.dwg.astype(np.float32),
            dlogit=b.dlogit.astype(np.float32),
            dw1_rowsum=b.dw1.sum(axis=2).astype(np.float32), dw1_colsum=b.dw1.sum(axis=1).astype(np.float32),
            dw3_rowsum=b.dw3.sum(axis=2).astype(np.float32), dw3_colsum=b.dw3.sum(axis=1).astype(np.float32),
            dw2_rowsum=b.dw2.sum(axis=2).astype(np.float32), dw2_colsum=b.dw2.sum(axis=1).astype(np.float32),
        )
    meta = {n: {"T": T, "H": H, "E": E, "k": k, "De": De, "seed": s, "kwargs": kw}
            for n, T, H, E, k, De, s, kw in KAT_CASES}
    (HERE / "moe_kats.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


if __name__ == "__main__":
    afpipe_orders()
    config_cases()
    moe_kats()
    print("golden fixtures written to", HERE)
