"""Measured stage times -> the reference allocator's Profile(M, M_a) and the
reference trace-event schema.

1. Algorithm 1's Phase 3 refines an allocation with "Profile(M, M_a)" — measured
   per-step times (reference allocator.phase3_refine,
   /root/reference/pkg/src/afpipe/allocator.py:205-237, whose default `profile`
   is the simulator, allocator.py:240-261). `measured_profile(exp, stages)`
   returns a drop-in `profile(alloc) -> seconds` built from stage times measured
   on this B200 path (`measure_stages`) and the runtime's own issue-order planner
   (afpipe.plan_layer), so the reference's phase3_refine can search A:F splits
   against real kernel times instead of the analytic cost model.
2. `export_trace(...)` writes measured runtime intervals in the reference's
   Chrome/Perfetto trace-event schema (trace_io.py:33-67,
   schemas/trace_event.schema.json), so simulated and measured AF-Pipe timelines
   diff in the same viewer.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

from .afpipe import LayerDurations, plan_layer


@dataclass(frozen=True)
class MeasuredStages:
    """Seconds per micro-batch of T tokens measured on one B200 (fused path).

    A stages are per A rank and micro-batch; F stages are for the *full* expert
    set (an F rank owning a share s of the experts takes s times as long);
    f_w is the deferred weight-gradient pass per micro-batch; link_gbs the
    measured per-direction P2P bandwidth."""

    T: int
    H: int
    E: int
    k: int
    De: int
    a_fwd: float
    a_turn: float
    a_bwd: float
    f_fwd: float
    f_bwd: float
    f_w: float
    link_gbs: float = 700.0

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=1)

    @classmethod
    def from_json(cls, text: str) -> "MeasuredStages":
        return cls(**json.loads(text))


def _ns(s: float) -> int:
    return max(1, int(round(s * 1e9)))


def predict_iteration(ms: MeasuredStages, attn_gpus: int, ffn_gpus: int, microbatches: int) -> float:
    """Seconds for one runtime iteration: every A rank runs `microbatches`
    micro-batches of T tokens (DP); F ranks own balanced contiguous expert blocks
    (reference taskgraph._balanced_blocks), so the slowest F rank holds
    ceil(E / N) experts and sees the union of all A ranks' rows for them."""
    share = math.ceil(ms.E / ffn_gpus) / ms.E
    f_scale = attn_gpus * share
    # one exchange: the busiest endpoint moves its slices of e*T*k*H bytes per A rank
    per_a = 2 * ms.T * ms.k * ms.H
    per_f = attn_gpus * per_a * share
    m2n = max(per_a, per_f) / (ms.link_gbs * 1e9)
    d = LayerDurations(a_fwd=_ns(ms.a_fwd), a_turn=_ns(ms.a_turn), a_bwd=_ns(ms.a_bwd),
                       f_fwd=_ns(ms.f_fwd * f_scale), f_bwd=_ns(ms.f_bwd * f_scale), m2n=_ns(m2n))
    it = plan_layer(microbatches, d).iteration_ns / 1e9
    return it + ms.f_w * microbatches * f_scale


def measured_profile(exp, ms: MeasuredStages):
    """profile(alloc) -> seconds to process one iteration's worth of exp's tokens
    (num_microbatches x seq_len x micro_batch) with alloc.attn_gpus A ranks and
    alloc.ffn_gpus F ranks. Deterministic and memoised on (M, N) — the contract of
    the reference's profile callable (allocator.py:249-259)."""
    tokens = exp.workload.num_microbatches * exp.workload.seq_len * exp.workload.micro_batch
    per_mb = ms.T
    cache: dict[tuple[int, int], float] = {}

    def profile(alloc) -> float:
        key = (alloc.attn_gpus, alloc.ffn_gpus)
        if key not in cache:
            m, n = key
            # each A rank takes ceil(total micro-batches / M) of the iteration's micro-batches
            mbs = max(1, math.ceil(tokens / per_mb / m))
            cache[key] = predict_iteration(ms, m, n, mbs) * tokens / (m * mbs * per_mb)
        return cache[key]

    return profile


def measure_stages(shape, device="cuda", iters: int = 5, link_gbs: float = 700.0) -> MeasuredStages:
    """Time each stage of the fused layer with CUDA events (GPU only)."""
    import torch

    from .moe import MoELayer, a_combine, a_combine_bwd, a_dispatch, a_dispatch_bwd, f_backward, f_forward

    layer = MoELayer.random(shape, device=device, seed=3, num_buffers=2)
    for b in layer.buffers:
        b.x.normal_()
        b.dy.normal_()
    buf = layer.buffers[0]

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / iters / 1e3

    a_fwd = timed(lambda: a_dispatch(buf, layer.router))
    f_fwd = timed(lambda: f_forward(buf, layer.experts))
    a_turn = timed(lambda: (a_combine(buf), a_combine_bwd(buf)))
    f_bwd = timed(lambda: f_backward(buf, layer.experts, False, defer_wgrad=True))
    a_bwd = timed(lambda: a_dispatch_bwd(buf, layer.router, False))
    layer.forward_backward(layer.buffers[1], defer_wgrad=True)
    f_w = timed(lambda: layer.wgrad(2)) / 2
    s = shape
    return MeasuredStages(T=s.T, H=s.H, E=s.E, k=s.k, De=s.De, a_fwd=a_fwd, a_turn=a_turn, a_bwd=a_bwd,
                          f_fwd=f_fwd, f_bwd=f_bwd, f_w=f_w, link_gbs=link_gbs)


# --------------------------------------------------------------------- traces
_KIND = {
    "A_f": ("FwdCompute", "forward", "fwd"), "F_f": ("FwdCompute", "forward", "fwd"),
    "A_t": ("BwdCompute", "backward", "bwd"), "F_b": ("BwdCompute", "backward", "bwd"),
    "A_b": ("BwdCompute", "backward", "bwd"), "W": ("BwdCompute", "backward", "bwd"),
    "M2N": ("M2NSend", "comm", "fwd"), "N2M": ("M2NSend", "comm", "fwd"),
    "M2N_b": ("M2NSend", "comm", "bwd"), "N2M_b": ("M2NSend", "comm", "bwd"),
}
_LANE_TID = {"compute": 0, "comm.send": 1, "comm.recv": 2}


def export_trace(ranks: list[dict]) -> list[dict]:
    """ranks: [{"rank": r, "role": "A"|"F", "ivs": runtime.trace_intervals(...)}, ...]
    -> complete ('X') events: pid = rank, tid = lane, microsecond timestamps
    (reference trace_io.export_trace field set)."""
    events = []
    task = 0
    t0 = min((s for g in ranks for (_, _, _, s, _, _) in g["ivs"]), default=0.0)
    for g in sorted(ranks, key=lambda g: g["rank"]):
        owner = f"{g['role']}{g['rank']}"
        for name, mb, lane, s, e, _nbytes in g["ivs"]:
            kind, stream, direction = _KIND.get(name, ("FwdCompute", "forward", "fwd"))
            events.append({
                "name": f"{kind} mb{max(mb, 0)} {name}", "ph": "X", "ts": (s - t0) * 1e3,
                "dur": max(0.0, (e - s) * 1e3), "pid": int(g["rank"]), "tid": _LANE_TID[lane],
                "args": {"owner": owner, "stream": stream, "lane": lane, "kind": kind,
                         "microbatch": max(mb, 0), "layer": 0, "virtual_index": 0,
                         "direction": direction, "task": task},
            })
            task += 1
    events.sort(key=lambda ev: (ev["ts"], ev["pid"], ev["tid"], ev["args"]["task"]))
    return events


def reference_memory_estimate(exp, component: str, n_attn: int, n_ffn: int) -> float:
    """Per-GPU bytes of the reference's memory model for pipeline_depth p and the
    largest group (restated from `placement.memory_estimate`, placement.py:78-120):
    bf16 parameters + 8 B/param optimizer state + one hidden-state tensor per
    assigned layer per in-flight micro-batch. Attention parameters (QKV + output,
    H²(2 + 2/g) + H² per layer) are replicated across the A group; expert
    parameters (E·2·H·D_e per layer) are sharded over the F group's GPUs. Used to
    compare the model with the runtime's measured peak memory."""
    from fractions import Fraction

    m, w = exp.model, exp.workload
    p = max(1, exp.pipeline_depth)
    layers = -(-m.layers // p)                       # virtual stages of the largest group
    h, g = m.hidden, m.gqa_group
    if component == "A":
        per_layer = Fraction(2 * (g + 1), g) * h * h + h * h
        params = float(layers * per_layer)
        first_visit = 0
    else:
        per_gpu_group = n_ffn / p
        params = layers * m.experts * 2 * h * m.moe_hidden / per_gpu_group
        first_visit = 1
    param_bytes = params * 2
    optimizer_bytes = params * 8.0
    hidden = m.bytes_per_element * w.micro_batch * w.seq_len * h
    in_flight = min(w.num_microbatches, max(1, 2 * p * layers - first_visit))
    return param_bytes + optimizer_bytes + float(layers * hidden * in_flight)


def reference_intensities(exp) -> tuple[float, float]:
    """(I_attn, I_ffn) FLOPs per exchanged byte of the reference cost model
    (restated from `costs.arithmetic_intensities`, costs.py:117-122): I_attn =
    ((2(g+1)/g)·H + 4s) / (2k), I_ffn = 2·D_e."""
    from fractions import Fraction

    m, w = exp.model, exp.workload
    g = m.gqa_group
    i_attn = Fraction(Fraction(2 * (g + 1), g) * m.hidden + 4 * w.seq_len, 2 * m.topk)
    return float(i_attn), float(2 * m.moe_hidden)


def reference_turning_points(peak_flops: float, bandwidth: float, attn_nodes: int, ffn_nodes: int):
    """(I_hat, I_attn_eff, I_ffn_eff) of `costs.turning_points` (costs.py:125-139):
    the system turning point P/B split by node share, 2m/(m+n)·I_hat and its complement."""
    i_hat = peak_flops / bandwidth
    i_attn = 2.0 * attn_nodes / (attn_nodes + ffn_nodes) * i_hat
    return i_hat, i_attn, 2.0 * i_hat - i_attn


def roofline_attainable(intensity: float, peak_flops: float, bandwidth: float) -> float:
    """min(P, I·B) (`costs.roofline_attainable`, costs.py:142-144)."""
    return min(float(peak_flops), float(intensity) * float(bandwidth))
