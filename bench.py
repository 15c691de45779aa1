#!/usr/bin/env python
"""Benchmark: MoE layer fwd+bwd tokens/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config configs/mixtral_layer.yaml]
                    [--impl ours|reference]

A step = one iteration of the layer over `num_microbatches` micro-batches of
T = seq_len * micro_batch synthetic tokens (fwd + bwd each, weight gradients
accumulated across micro-batches, fp32). N=1 runs the fused single-device path
(A and F stages on one GPU) on BASELINE configs[1] (Mixtral-8x7B layer).
N>1 runs the AF-Pipe runtime split into attention:FFN groups when it is
available, otherwise independent replicas (weak scaling), as stated in the
JSON line's config.parallelism.

`--impl reference` times the CPU oracle port (oracle/, the reference has no
MoE arithmetic to run — DESIGN.md §3) on the host cores on a bounded token
sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE fwd+bwd tokens/s at 1/2/4/8 B200; exposed A2F comm %; roofline %"
UNIT = "tokens/s"


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu   # nvidia-smi --id: ordinal or "GPU-<uuid>"
        self.proc = None
        self.lines: list[str] = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, which: str) -> None:
        setattr(self, "t_" + which, time.time())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0 = getattr(self, "t_start", 0.0) - 0.05
        t1 = getattr(self, "t_end", float("inf")) + 0.15   # nvidia-smi output lags its sample
        window = [ln for t, ln in self.lines if t0 <= t <= t1]
        if not window:  # very short timed region: fall back to the samples nearest to it
            window = [ln for _, ln in self.lines[-3:]]
        for ln in window:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 10:
                continue
            try:
                sm.append(float(f[2]))
                smax.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "window_s": round(t1 - t0 - 0.2, 3)}


_WEIGHTS = {}


def _oracle_weights(H, E, De):
    """Random-init layer weights for the CPU arms, generated once per shape (generating a
    Mixtral layer's 1.4 G fp32 values takes longer than timing it)."""
    import numpy as np

    key = (H, E, De)
    if key not in _WEIGHTS:
        rng = np.random.default_rng(11)
        _WEIGHTS[key] = ((rng.standard_normal((E, H), dtype=np.float32) * 0.02),
                         (rng.standard_normal((E, De, H), dtype=np.float32) * 0.02),
                         (rng.standard_normal((E, De, H), dtype=np.float32) * 0.02),
                         (rng.standard_normal((E, H, De), dtype=np.float32) * 0.02))
    return _WEIGHTS[key]


CPU_SAMPLE_TOKENS = 1024


def cpu_baseline(shape, tokens: int | None = None, layer=None, layers: int = 1, seed: int = 7):
    """Time the oracle port (numpy fp32 BLAS, all host threads) on a sample of `tokens`
    tokens (default min(T, 1024)) of one micro-batch: the full fwd + bwd of every one of
    `layers` identical-shape layers, measured once — no extrapolation. The oracle reuses
    the fp32 weights in place (no per-call copies), so a 1024-token sample is dominated by
    the GEMMs, not by fixed per-call costs."""
    import numpy as np

    from oracle import oracle as O

    threads = O.cpu_threads()
    H, E, k, De = shape.H, shape.E, shape.k, shape.De
    rng = np.random.default_rng(seed)
    if layer is not None:
        from paper_2605_11005_b200.moe import split_w13

        w1t, w3t = split_w13(layer.experts.w13)
        w1 = w1t.float().cpu().numpy()
        w3 = w3t.float().cpu().numpy()
        w2 = layer.experts.w2.float().cpu().numpy()
        wg = (layer.router.wg if hasattr(layer, "router") else layer.wg).float().cpu().numpy()
    else:
        wg, w1, w3, w2 = _oracle_weights(H, E, De)
    T = min(shape.T, tokens or CPU_SAMPLE_TOKENS)
    x = O.f32_to_bf16_bits(rng.standard_normal((T, H), dtype=np.float32))
    dy = O.round_bf16(rng.standard_normal((T, H), dtype=np.float32))
    # every host thread for BLAS, whatever OMP_NUM_THREADS says (torchrun sets it to 1)
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        for _ in range(layers):
            f = O.moe_forward(x, wg, w1, w3, w2, k, dtype=np.float32)
            O.moe_backward(f, x, wg, w1, w3, w2, dy, dtype=np.float32)
        dt = time.perf_counter() - t0
    return {"value": T / dt, "unit": UNIT, "cores": threads, "kind": "port", "tokens": T, "seconds": round(dt, 3),
            "sample": f"{T} of the {shape.T} tokens of one micro-batch, full fwd+bwd of {layers} layer(s) "
                      f"(H={H}, E={E}, k={k}, D_e={De}), numpy fp32 BLAS oracle on {threads} threads, "
                      f"measured {dt:.2f} s (no extrapolation)"}


def run_reference(args, shape, exp):
    """The reference arm: the reference has no MoE arithmetic, so this times
    the oracle port (oracle/oracle.py) on the host cores. One step = one sample of
    min(T, 1024) tokens through every layer's fwd + bwd; value = tokens / measured time
    of that sample, ms_per_step = that measured time (the timed work IS the step)."""
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    steps, warm = args.steps, args.warmup
    samples = []
    t_run = time.perf_counter()
    for i in range(warm + steps):
        r = cpu_baseline(shape, layers=exp.model.layers, seed=7 + i)
        if i >= warm:
            samples.append(r)
    t_run = time.perf_counter() - t_run
    secs = [s["seconds"] for s in samples]
    tokens = samples[-1]["tokens"]
    ms = statistics.median(secs) * 1e3
    value = tokens / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": round(ms, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": Path(args.config).stem, "T": shape.T, "H": shape.H, "E": shape.E,
                   "k": shape.k, "D_e": shape.De, "layers": exp.model.layers,
                   "microbatches": exp.workload.num_microbatches, "tokens_per_step": tokens},
        "cpu_baseline": {**{kk: v for kk, v in samples[-1].items() if kk != "seconds"}, "value": round(value, 3)},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "consistency": {"timed_s": round(sum(secs), 4), "run_s": round(t_run, 4)},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, shape, exp):
    import torch
    import torch.distributed as dist

    from paper_2605_11005_b200 import _lib
    from paper_2605_11005_b200 import kernels as K
    from paper_2605_11005_b200.moe import MoELayer, MoEStack

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 under torchrun, or without "
                         f"WORLD_SIZE set so that bench.py starts the {args.gpus} ranks itself")
    if args.attention and exp.model.bytes_per_element == 4:
        raise SystemExit("--attention runs bf16 attention blocks; fp32 mode (bytes_per_element 4) is MoE-only")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    if world > 1 and not args.replicas:
        return run_afpipe(args, shape, exp, world, rank, local, dev)
    mb = exp.workload.num_microbatches
    L = exp.model.layers
    fp32 = exp.model.bytes_per_element == 4
    if exp.model.bytes_per_element not in (2, 4):
        raise SystemExit(f"bytes_per_element {exp.model.bytes_per_element}: only bf16 (2) and fp32 (4) modes exist")
    if fp32:
        from paper_2605_11005_b200.moe_f32 import MoELayerF32 as LayerCls
    else:
        LayerCls = MoELayer
    # L > 1: the stack of residual MoE blocks (configs[0]: 2 layers); L = 1: the plain layer;
    # --attention: each layer = A-side attention block + residual MoE block
    attn = None
    if args.attention:
        from paper_2605_11005_b200.attention import AttentionBlock

        attn = [AttentionBlock(shape.H, exp.model.gqa_group, dev, seed=77 + l) for l in range(L)]
    stack = MoEStack([LayerCls.random(shape, device=dev, seed=1234 + rank + 1000 * l, num_buffers=mb,
                                      residual=L > 1 or attn is not None) for l in range(L)],
                     attention=attn, seq_len=exp.workload.seq_len)
    layer = stack.layers[0]
    stream = torch.cuda.current_stream(dev)
    for i in range(mb):
        stack.input(i).normal_()
        stack.output_grad(i).normal_()

    # per-stage CUDA events: GEMM (F) time and HBM-kernel (A) time inside the timed region
    class Ev:
        def __init__(self):
            self.pairs = {"gemm": [], "dispatch": [], "combine_fwd": [], "combine_bwd": [], "permute_bwd": [],
                          "router_wgrad": [], "attention": []}

        def mark(self, name, fn):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            e.record(stream)
            self.pairs[name].append((s, e))

        def total_ms(self, name):
            return sum(s.elapsed_time(e) for s, e in self.pairs[name])

    batched = stack.batched_supported(mb)

    def step(ev=None):
        if ev is None:
            stack.iteration(mb)
            return
        if batched:   # the order MoEStack.iteration runs: layer-major, one GEMM launch per stage
            for l, ly in enumerate(stack.layers):
                for i in range(mb):
                    if attn is not None:
                        x_in = stack.inp[i] if l == 0 else stack.layers[l - 1].buffers[i].y
                        ev.mark("attention", lambda: attn[l].forward(i, x_in, ly.buffers[i].x, stack.seq_len))
                for i in range(mb):
                    ev.mark("dispatch", lambda: ly.stage_dispatch(ly.buffers[i]))
                ev.mark("gemm", lambda: ly.f_forward_all(mb))
                for i in range(mb):
                    ev.mark("combine_fwd", lambda: ly.stage_combine(ly.buffers[i]))
            for l in reversed(range(L)):
                ly = stack.layers[l]
                for i in range(mb):
                    ev.mark("combine_bwd", lambda: ly.stage_combine_bwd(ly.buffers[i]))
                ev.mark("gemm", lambda: ly.f_backward_all(mb))
                for i in range(mb):
                    ev.mark("permute_bwd", lambda: ly.stage_permute_bwd(ly.buffers[i]))
                    ev.mark("router_wgrad", lambda: ly.stage_router_wgrad(ly.buffers[i], i > 0))
                if attn is not None:
                    for i in range(mb):
                        dst = stack.dinp[i] if l == 0 else stack.layers[l - 1].buffers[i].dy
                        ev.mark("attention", lambda: attn[l].backward(i, ly.buffers[i].dx, dst, i > 0))
            for ly in stack.layers:
                ev.mark("gemm", lambda: ly.wgrad(mb))
            return
        for i in range(mb):
            acc = i > 0
            for l, ly in enumerate(stack.layers):
                buf = ly.buffers[i]
                if attn is not None:
                    x_in = stack.inp[i] if l == 0 else stack.layers[l - 1].buffers[i].y
                    ev.mark("attention", lambda: attn[l].forward(i, x_in, buf.x, stack.seq_len))
                ev.mark("dispatch", lambda: ly.stage_dispatch(buf))
                ev.mark("gemm", lambda: ly.stage_f_forward(buf))
                ev.mark("combine_fwd", lambda: ly.stage_combine(buf))
            for l in reversed(range(L)):
                ly = stack.layers[l]
                buf = ly.buffers[i]
                ev.mark("combine_bwd", lambda: ly.stage_combine_bwd(buf))
                ev.mark("gemm", lambda: ly.stage_f_backward(buf, acc))
                ev.mark("permute_bwd", lambda: ly.stage_permute_bwd(buf))
                ev.mark("router_wgrad", lambda: ly.stage_router_wgrad(buf, acc))
                if attn is not None:
                    dst = stack.dinp[i] if l == 0 else stack.layers[l - 1].buffers[i].dy
                    ev.mark("attention", lambda: attn[l].backward(i, buf.dx, dst, acc))
        for ly in stack.layers:
            ev.mark("gemm", lambda: ly.wgrad(mb))

    # the iteration as CUDA graphs (one per micro-batch + the W pass): same kernels,
    # n+1 host launches per step instead of ~13 per layer and micro-batch
    graphs = None
    if not args.eager:
        try:
            graphs = stack.capture(mb)
        except RuntimeError as ex:   # e.g. a library attention backend that cannot be captured
            print(f"[bench] CUDA-graph capture failed ({str(ex)[:160]}); timing eager launches", file=sys.stderr)
            graphs = None

    def run():
        if graphs is not None:
            graphs.replay()
        else:
            step()

    sampler = ClockSampler(_clock_target(dev)) if rank == 0 else None
    if sampler:
        sampler.start()
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if sampler:
        sampler.mark("start")
    launches0 = _lib.launch_count()
    t_s = torch.cuda.Event(enable_timing=True)
    t_e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_s.record(stream)
    for _ in range(args.steps):
        run()
    t_e.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.mark("end")
    launches = (graphs.launches_per_iteration * args.steps if graphs is not None
                else _lib.launch_count() - launches0)
    ms = t_s.elapsed_time(t_e)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
        dist.barrier()
    clocks = sampler.stop() if sampler else None

    # per-stage breakdown: a separate eager pass with CUDA events around every stage
    ev = Ev()
    for _ in range(args.steps):
        step(ev)
    torch.cuda.synchronize()

    # ---- e2e: public API with pinned host buffers, copies inside the timed region
    e2e = run_e2e(args, stack, shape, mb, dev, world, graphs)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    peaks, peak_kind = _peaks()
    tokens = args.steps * mb * shape.T * world
    value = tokens / (ms / 1e3)
    gemm_ms = ev.total_ms("gemm")
    gemm_flops = args.steps * mb * L * (shape.gemm_flops_fwd() + shape.gemm_flops_bwd())
    achieved_tf = gemm_flops / (gemm_ms / 1e3) / 1e12
    peak_tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    # which roofline binds the GEMMs: tensor FLOPs or the HBM bytes they must move
    # (weights streamed per micro-batch fwd + dgrad, fp32 dW, activations)
    gemm_bytes = args.steps * L * shape.gemm_hbm_bytes(mb, 4 if fp32 else 2, batched=batched)
    ideal_tensor_ms = gemm_flops / (peak_tf * 1e12) * 1e3
    ideal_hbm_ms = gemm_bytes / (peaks["hbm_gbs"] * 1e9) * 1e3
    hbm_bound = ideal_hbm_ms > ideal_tensor_ms
    achieved_gbs = gemm_bytes / (gemm_ms / 1e3) / 1e9
    esz = 4 if fp32 else 2
    hb = shape.hbm_bytes(esz)
    hbm = {}
    hb["router_wgrad"] = shape.T * shape.H * esz + shape.T * shape.k * 8
    for name in ("dispatch", "combine_fwd", "combine_bwd", "permute_bwd", "router_wgrad"):
        t = ev.total_ms(name) / (args.steps * mb * L)
        gbs = hb[name] / (t / 1e3) / 1e9
        hbm[name] = {"ms": round(t, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peaks["hbm_gbs"], 3)}
    # A-side kernels in isolation: CUDA-graph replays of [L2 flush, stage] minus [L2 flush]
    # (flush = 160 MB memset > 126 MB L2), i.e. cold-L2 kernel time at the live clocks,
    # without the per-stage event overhead of the in-step numbers above
    iso = {}
    if world == 1 and not args.no_isolated:
        b0, ly0 = stack.layers[0].buffers[0], stack.layers[0]
        fns = {"dispatch": lambda: ly0.stage_dispatch(b0), "combine_fwd": lambda: ly0.stage_combine(b0),
               "combine_bwd": lambda: ly0.stage_combine_bwd(b0), "permute_bwd": lambda: ly0.stage_permute_bwd(b0),
               "router_wgrad": lambda: ly0.stage_router_wgrad(b0, False)}
        iso = isolated_stage_ms(fns, dev)
        for name, t in iso.items():
            gbs = hb[name] / (t / 1e3) / 1e9
            hbm[name]["isolated_ms"] = round(t, 4)
            hbm[name]["isolated_frac"] = round(gbs / peaks["hbm_gbs"], 3)
    # measured DRAM bytes of one iteration's GEMM launches (ncu; scripts/gemm_traffic.py),
    # per step like `achieved`, when a capture for this workload is committed
    traffic, traffic_info = None, None
    for tfile in sorted((ROOT / "profiles").glob(f"*/gemm_traffic_{Path(args.config).stem}.json")):
        try:
            tj = json.loads(tfile.read_text())
            traffic = tj.get("bytes_per_iteration")
            n_l = len(tj.get("launches", [])) or None
            traffic_info = {"unit": "DRAM bytes per step (all GEMM launches of one iteration, ncu)",
                            "launches_per_step": n_l,
                            "per_launch_avg": round(traffic / n_l) if traffic and n_l else None,
                            "algorithmic_bytes_per_step": tj.get("algorithmic_bytes_per_iteration"),
                            "ratio_to_algorithmic": tj.get("ratio"), "source": str(tfile.relative_to(ROOT))}
        except (ValueError, OSError):
            traffic, traffic_info = None, None
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if fp32 else "bf16", "data": "synthetic",
        "config": {
            "workload": Path(args.config).stem, "T": shape.T, "H": shape.H, "E": shape.E, "k": shape.k,
            "D_e": shape.De, "layers": L,
            "precision": ("fp32 mode: fp32 activations/weights, split-3 bf16 tensor-core GEMMs (3x MMA work)"
                          if fp32 else "bf16 operands, fp32 accumulation and weight gradients"),
            "microbatches": mb, "tokens_per_step": mb * shape.T * world,
            "parallelism": "fused single-device (A+F on one GPU)" if world == 1 else f"replicas x{world}",
            "weights": "random-init", "l2": "inputs+weights (2.8 GB) larger than L2 (126 MB)",
            "wgrad": "fp32, deferred: one grouped GEMM per iteration over all micro-batches (K = mb*T*k rows)",
            "launch": "eager" if graphs is None else ("CUDA graphs (all micro-batches' fwd + bwd, then the W pass)"
                                                       if batched else "CUDA graphs (per micro-batch + W pass)"),
            "f_side": ("batched: each expert GEMM stage is one launch over all micro-batches, expert-major groups "
                       "(weights streamed once per iteration)" if batched else "per micro-batch"),
            "stage_breakdown": "separate eager pass with CUDA events per stage (not the timed region)",
        },
        "roofline": ({
            "bound": "hbm", "kernel": "grouped expert GEMMs (K4/K5/K8: 4 launches per micro-batch + 2 deferred wgrad launches per step)",
            "achieved": round(achieved_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved_gbs / peaks["hbm_gbs"], 4), "traffic": traffic, "traffic_detail": traffic_info,
            "peak_kind": f"{peak_kind} HBM copy bandwidth (MEASURED_PEAKS.json)",
            "algorithmic_bytes_per_step": gemm_bytes // args.steps,
            "tensor_achieved_tflops": round(achieved_tf, 1), "tensor_frac": round(achieved_tf / peak_tf, 4),
            "why": f"ideal HBM time {ideal_hbm_ms / args.steps:.2f} ms/step > ideal tensor time "
                   f"{ideal_tensor_ms / args.steps:.2f} ms/step (weights streamed per micro-batch)",
            "gemm_ms_per_microbatch_layer": round(gemm_ms / (args.steps * mb * L), 4),
        } if hbm_bound else {
            "bound": "tensor", "kernel": "grouped expert GEMMs (K4/K5/K8: 4 launches per micro-batch + 2 deferred wgrad launches per step)",
            "achieved": round(achieved_tf, 1), "peak": peak_tf, "unit": "TFLOP/s",
            "frac": round(achieved_tf / peak_tf, 4), "traffic": traffic, "traffic_detail": traffic_info,
            "peak_kind": f"{peak_kind} sustained bf16 (MEASURED_PEAKS.json)",
            "gemm_ms_per_microbatch_layer": round(gemm_ms / (args.steps * mb * L), 4),
            "frac_of_burst": round(achieved_tf / peaks["bf16_tflops"], 4),
            "hbm_achieved_gbs": round(achieved_gbs, 1),
        }),
        "roofline_hbm": {"peak_GB/s": peaks["hbm_gbs"], **hbm,
                         "note": "ms/frac: in-step CUDA events around each stage; isolated_*: graph replay, "
                                 "median of 31 replays of graph [160 MB L2 flush, stage] minus median of [flush]"},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
    }
    if attn is not None:
        a_ms = ev.total_ms("attention") / (args.steps * mb * L)
        fa, fb = attn[0].flops(exp.workload.seq_len, exp.workload.micro_batch)
        line["attention"] = {
            "ms_per_microbatch_layer": round(a_ms, 4), "TFLOP/s": round((fa + fb) / (a_ms / 1e3) / 1e12, 1),
            "impl": _attention_impl_label(attn[0].last_path),
            "gqa_group": exp.model.gqa_group, "seq_len": exp.workload.seq_len}
        line["config"]["layer"] = "attention + residual MoE block"
        line["config"]["launch"] = "CUDA graphs" if graphs is not None else "eager"
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(shape, layer=layer, layers=L)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _union(iv):
    out = []
    for s, e in sorted(iv):
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return out


def _uncovered(a, b):
    """Length of union(a) not covered by union(b) (the reference's exposed_comm, sim.py:273-299)."""
    a, b = _union(a), _union(b)
    tot, j = 0.0, 0
    for s, e in a:
        cur = s
        while cur < e:
            while j < len(b) and b[j][1] <= cur:
                j += 1
            if j == len(b) or b[j][0] >= e:
                tot += e - cur
                break
            if b[j][0] > cur:
                tot += b[j][0] - cur
            cur = min(b[j][1], e)
    return tot


def _attention_impl_label(path) -> str:
    """Which attention path actually ran (AttentionBlock.last_path), for the bench line."""
    if path == "own":
        return ("own sm_100a kernels only: flash-attention fwd/bwd (dm_attention_fwd/_bwd), projections and "
                "their gradients on the grouped tcgen05 GEMM (dm_grouped_w2_fwd / w13_dgrad / wgrad)")
    return "library: cuBLAS projections + torch SDPA (cuDNN/flash), autograd"


def _clock_target(dev) -> str:
    """nvidia-smi --id for a torch device: its UUID (robust to CUDA_VISIBLE_DEVICES remaps)."""
    import torch

    try:
        return f"GPU-{torch.cuda.get_device_properties(dev).uuid}"
    except Exception:  # noqa: BLE001 - older torch: fall back to the ordinal
        return str(dev.index)


def _merge_clocks(per_rank: list[dict], roles: list[str]) -> dict:
    """Bench-line clocks for N>1: the F ranks (where the expert GEMMs run) — the lowest
    median SM clock among them and the union of their throttle reasons — plus every rank's
    own record."""
    f = [c for c, r in zip(per_rank, roles) if r == "F" and c and c.get("sm_mhz")] or \
        [c for c in per_rank if c and c.get("sm_mhz")]
    out = {"sm_mhz": min(c["sm_mhz"] for c in f) if f else None,
           "sm_max_mhz": max(c["sm_max_mhz"] for c in f) if f else None,
           "reasons": sorted({x for c in f for x in c.get("reasons", [])}),
           "source": "F ranks (expert GEMMs): min of per-rank medians, union of reasons"}
    out["per_rank"] = [{"rank": i, "role": r, **(c or {})} for i, (c, r) in enumerate(zip(per_rank, roles))]
    return out


def run_afpipe(args, shape, exp, world, rank, local, dev):
    """N>1: A:F-split AF-Pipe runtime (one process per GPU, NCCL over NVLink)."""
    import torch
    import torch.distributed as dist

    from paper_2605_11005_b200 import _lib
    from paper_2605_11005_b200.profile import reference_memory_estimate
    from paper_2605_11005_b200.runtime import AFPipeRank, Topology, trace_intervals

    if exp.model.bytes_per_element != 2:
        raise SystemExit("AF-Pipe runtime exchanges bf16 micro-batches; fp32 mode (bytes_per_element 4) runs on "
                         "the fused single-device path (N=1, or --replicas)")
    mb = exp.workload.num_microbatches
    topo = Topology.default(world, shape.E, args.n_attn, args.depth or exp.pipeline_depth)
    L = exp.model.layers
    r = AFPipeRank(shape, topo, rank, mb, dev, seed=1234, layers=L, attention=args.attention,
                   seq_len=exp.workload.seq_len, gqa_group=exp.model.gqa_group)
    r.init_groups()
    if r.role == "A":
        for i in range(mb):
            if r.has_input:
                r.input(i).normal_()
            if r.has_output:
                r.out_bufs[i].dy.normal_()
    # 1A:1F per pipeline group (fixed-size exchange, no host sync): the whole iteration —
    # kernels, NCCL P2P on the send/recv streams, W pass — replays as one CUDA graph per rank
    graph = r.capture() if (r.capturable and not args.eager) else None
    step = graph.replay if graph is not None else r.run_iteration
    sampler = ClockSampler(_clock_target(dev))   # every rank samples its own GPU
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    if sampler:
        sampler.mark("start")
    n0 = _lib.launch_count()
    t_s, t_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    t_s.record()
    for _ in range(args.steps):
        step()
    t_e.record()
    torch.cuda.synchronize()
    if sampler:
        sampler.mark("end")
    launches = _lib.launch_count() - n0 + (r.graph_launches * args.steps if graph is not None else 0)
    ms = t_s.elapsed_time(t_e)
    tt = torch.tensor([ms, float(launches)], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = tt[0].item()
    lsum = torch.tensor([float(launches)], device=dev)
    dist.all_reduce(lsum)
    clk_all = [None] * world
    dist.all_gather_object(clk_all, sampler.stop())
    roles = [topo.role(q)[0] for q in range(world)]
    clocks = _merge_clocks(clk_all, roles)

    # measured peak device memory per rank vs the reference's memory model
    mem_all = [None] * world
    dist.all_gather_object(mem_all, {"rank": rank, "role": r.role,
                                     "peak_GB": round(torch.cuda.max_memory_allocated(dev) / 1e9, 3)})

    # one instrumented iteration: per-task CUDA-event intervals on every rank
    r.record_events = True
    torch.cuda.synchronize()
    dist.barrier()
    r.run_iteration()
    torch.cuda.synchronize()
    ivs = trace_intervals(r)
    r.record_events = False
    gathered = [None] * world if rank == 0 else None
    dist.gather_object({"rank": rank, "role": r.role, "ivs": ivs}, gathered, dst=0)
    if rank == 0 and args.trace:
        from paper_2605_11005_b200.profile import export_trace

        Path(args.trace).write_text(json.dumps(export_trace(gathered), indent=1))

    # e2e: A ranks feed x/dy from pinned host memory and read y/dx back every micro-batch
    T, H = shape.T, shape.H
    if r.role == "A":
        mk = lambda: torch.empty(T, H, dtype=torch.bfloat16).pin_memory()  # noqa: E731
        xs = [torch.randn(T, H).to(torch.bfloat16).pin_memory() for _ in range(mb)]
        dys = [torch.randn(T, H).to(torch.bfloat16).pin_memory() for _ in range(mb)]
        r.set_host_io(xs, dys, [mk() for _ in range(mb)], [mk() for _ in range(mb)])
    r.run_iteration()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        r.run_iteration()
    e1.record()
    torch.cuda.synchronize()
    ems = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ems, op=dist.ReduceOp.MAX)
    ems = ems.item()

    if rank == 0:
        peaks, peak_kind = _peaks()
        tokens = args.steps * mb * shape.T * topo.streams
        value = tokens / (ms / 1e3)
        comp_all, comm_all, per_rank, it_end = [], [], {}, 0.0
        gemm_ms, link = 0.0, []
        for g in gathered:
            comp = [(s, e) for n, i, lane, s, e, b in g["ivs"] if lane == "compute"]
            comm = [(s, e) for n, i, lane, s, e, b in g["ivs"] if lane != "compute"]
            comp_all += comp
            comm_all += comm
            it_end = max([it_end] + [e for _, e in comp + comm])
            per_rank[g["rank"]] = _uncovered(comm, comp)
            if g["role"] == "F":
                gemm_ms += sum(e - s for n, i, lane, s, e, b in g["ivs"] if lane == "compute")
            link += [b / ((e - s) / 1e3) / 1e9 for n, i, lane, s, e, b in g["ivs"]
                     if lane != "compute" and e > s and b > 0]
        exposed = _uncovered(comm_all, comp_all)
        f_flops = mb * L * (shape.gemm_flops_fwd() + shape.gemm_flops_bwd()) * topo.streams
        achieved = f_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
        peak_tf = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        # HBM-bound when streaming each F rank's weights per micro-batch dominates (fine-grained MoE)
        import dataclasses

        f_bytes = L * dataclasses.replace(shape, T=shape.T * topo.streams).gemm_hbm_bytes(mb)
        hbm_bound = f_bytes / (peaks["hbm_gbs"] * 1e9) > f_flops / (peak_tf * 1e12)
        achieved_gbs = f_bytes / (gemm_ms / 1e3) / 1e9 if gemm_ms > 0 else None
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {
                "workload": Path(args.config).stem, "T": shape.T, "H": shape.H, "E": shape.E, "k": shape.k,
                "D_e": shape.De, "layers": L, "microbatches": mb, "tokens_per_step": mb * shape.T * topo.streams,
                "pipeline_depth": topo.depth,
                "parallelism": f"AF-Pipe {topo.n_attn}A:{topo.n_ffn}F" + (f" x {topo.depth} pipeline groups"
                                                                           if topo.depth > 1 else "") + " (A: DP "
                               + ("attention + " if args.attention else "") + "routing/combine, F: EP experts)",
                "layer": "attention + residual MoE block (attention: own kernels)" if args.attention
                         else "MoE block",
                "transport": "NCCL send/recv (torch.distributed P2P) over NVLink",
                "launch": ("one CUDA graph per rank per iteration (kernels + NCCL P2P + W pass)" if graph is not None
                           else "eager (data-dependent message sizes: host reads the counts headers)"),
                "weights": "random-init", "l2": "inputs+weights larger than L2",
                "wgrad": "fp32, deferred per iteration on F ranks",
            },
            "roofline": {
                "bound": "hbm", "kernel": "grouped expert GEMMs on F ranks (F_f + F_b + W tasks)",
                "achieved": round(achieved_gbs, 1) if achieved_gbs else None, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved_gbs / peaks["hbm_gbs"], 4) if achieved_gbs else None,
                "traffic": None, "tensor_frac": round(achieved / peak_tf, 4) if achieved else None,
                "peak_kind": f"{peak_kind} HBM, per F GPU (algorithmic GEMM bytes / sum of F compute time)",
            } if hbm_bound else {
                "bound": "tensor", "kernel": "grouped expert GEMMs on F ranks (F_f + F_b + W tasks)",
                "achieved": round(achieved, 1) if achieved else None, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": round(achieved / peak_tf, 4) if achieved else None, "traffic": None,
                "peak_kind": f"{peak_kind} sustained bf16, per F GPU (sum of F compute time over F ranks)",
            },
            "exposed_comm": {
                "global_ms": round(exposed, 4), "global_pct": round(100 * exposed / it_end, 3) if it_end else None,
                "per_rank_max_pct": round(100 * max(per_rank.values()) / it_end, 3) if it_end else None,
                "iteration_ms_instrumented": round(it_end, 3),
                "definition": "reference sim.exposed_comm: comm running while every compute engine idles; "
                              "per-rank: comm not covered by that rank's own compute; send-side intervals",
            },
            "link": {"mean_GB/s": round(statistics.mean(link), 1) if link else None,
                     "max_GB/s": round(max(link), 1) if link else None,
                     "peak_GB/s": 900.0, "note": "bytes / (data ready -> send complete), per transfer group"},
            "reference_model": _reference_model(exp, topo, shape, mb, L, f_flops, link, peaks, achieved),
            "schedule_model": _schedule_model(gathered, mb, L, topo.depth, it_end),
            "gpu_launches": int(lsum.item()),
            "clocks": clocks,
            "memory": {
                "measured_peak_GB": {f"{m['role']}{m['rank']}": m["peak_GB"] for m in mem_all},
                "reference_model_GB": {c: round(reference_memory_estimate(exp, c, topo.n_attn, topo.n_ffn) / 1e9, 3)
                                       for c in ("A", "F")},
                "note": "reference placement.memory_estimate: bf16 params + 8 B/param optimizer + in-flight hidden "
                        "states; measured: weights + fp32 grads (no optimizer) + every micro-batch's activations "
                        "resident for the deferred W pass (+ attention graphs with --attention)",
            },
            "e2e": {"value": round(tokens / (ems / 1e3), 1), "unit": UNIT,
                    "h2d_bytes_per_step": 2 * T * H * 2 * mb * topo.streams,
                    "d2h_bytes_per_step": 2 * T * H * 2 * mb * topo.streams,
                    "ms_per_step": round(ems / args.steps, 3),
                    "path": "AFPipeRank.run_iteration with pinned host x/dy in, y/dx out per micro-batch"},
        }
        print(json.dumps(line), flush=True)
    del graph, step   # before the process group goes (a live graph holding NCCL work hangs teardown)
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()
    return 0


def isolated_stage_ms(fns: dict, dev, reps: int = 31) -> dict:
    """ms per launch of each stage with a cold L2: the median over `reps` single replays of a
    CUDA graph [160 MB write (> the 126 MB L2), stage] minus the median of [write] alone.
    Medians of individually timed replays: one timing of a 10-flush graph (the earlier
    method) left several us of flush-to-flush noise on 20-40 us stages."""
    import torch

    flush = torch.empty(160 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)

    def median_replay(g):
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    g0 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g0, stream=s):
        flush.zero_()
    g0.replay()
    base = median_replay(g0)
    out = {}
    for name, fn in fns.items():
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            flush.zero_()
            fn()
        g.replay()
        out[name] = max(median_replay(g) - base, 1e-6)
    return out


def _schedule_model(gathered, mb, L, depth, measured_ms):
    """The reference's schedule (afpipe.plan_layer: the same DAG, credits and list-scheduling
    priority as the reference build_task_graph + simulate, pinned by tests/golden) fed THIS
    run's measured task durations (medians over ranks and micro-batches of the instrumented
    iteration), next to the measured iteration: how far the runtime is from the schedule the
    reference model predicts for the same stage times (SURVEY §8(d) CPU-A)."""
    import statistics

    from paper_2605_11005_b200.afpipe import LayerDurations, plan_layer

    dur: dict = {}
    for g in gathered:
        for n, i, lane, s, e, b in g["ivs"]:
            dur.setdefault(n, []).append(e - s)
    med = lambda k: statistics.median(dur[k]) if dur.get(k) else 0.0  # noqa: E731
    comm = [x for k in ("M2N", "N2M", "M2N_b", "N2M_b") for x in dur.get(k, [])]
    ns = lambda ms_: max(1, int(ms_ * 1e6))  # noqa: E731
    d = LayerDurations(a_fwd=ns(med("A_f")), a_turn=ns(med("A_t")), a_bwd=ns(med("A_b")), f_fwd=ns(med("F_f")),
                       f_bwd=ns(med("F_b")), m2n=ns(statistics.median(comm) if comm else 0.0))
    try:
        plan = plan_layer(mb, d, layers=L, depth=depth)
    except Exception as ex:  # noqa: BLE001 - a model failure must not fail the bench line
        return {"error": str(ex)[:200]}
    w_ms = max(dur.get("W", [0.0]))
    pred = plan.iteration_ns / 1e6 + w_ms
    return {"predicted_iteration_ms": round(pred, 3), "measured_iteration_ms": round(measured_ms, 3),
            "measured_over_predicted": round(measured_ms / pred, 3) if pred > 0 else None,
            "durations_ms": {"A_f": round(med("A_f"), 4), "A_t": round(med("A_t"), 4), "A_b": round(med("A_b"), 4),
                             "F_f": round(med("F_f"), 4), "F_b": round(med("F_b"), 4),
                             "exchange": round(statistics.median(comm), 4) if comm else None, "W": round(w_ms, 4)},
            "note": "afpipe.plan_layer (the reference schedule restated) on this run's median task times; "
                    "measured = the instrumented iteration"}


def _reference_model(exp, topo, shape, mb, L, f_flops, link, peaks, achieved_tf):
    """The reference's analytic roofline (costs.py:117-144) next to the measured figures:
    intensities, the NVLink turning points for this A:F split, the attainable FFN
    throughput at the measured link bandwidth, and this run's FFN FLOPs per exchanged byte."""
    from paper_2605_11005_b200.profile import reference_intensities, reference_turning_points, roofline_attainable

    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * 1e12
    link_bw = (statistics.mean(link) if link else 900.0) * 1e9
    i_attn, i_ffn = reference_intensities(exp)
    i_hat, i_attn_eff, i_ffn_eff = reference_turning_points(peak, link_bw, topo.n_attn, topo.n_ffn)
    moved = 4 * shape.T * shape.k * shape.H * exp.model.bytes_per_element * mb * L * topo.streams
    return {
        "I_attn": round(i_attn, 1), "I_ffn": round(i_ffn, 1),
        "turning_point_system": round(i_hat, 1), "turning_point_ffn_effective": round(i_ffn_eff, 1),
        "ffn_attainable_TFLOPs_at_measured_link": round(roofline_attainable(i_ffn, peak, link_bw) / 1e12, 1),
        "ffn_flops_per_exchanged_byte_measured_run": round(f_flops / moved, 1),
        "ffn_achieved_TFLOPs_per_gpu": round(achieved_tf, 1) if achieved_tf else None,
        "note": "reference costs.arithmetic_intensities / turning_points / roofline_attainable with P = measured "
                "sustained bf16 and B = this run's mean link GB/s; I_ffn >> turning point means the F side is "
                "compute-bound, the exchange hides behind it",
    }


def run_e2e(args, stack, shape, mb, dev, world, graphs=None):
    """Same metric through the public API with host buffers: per micro-batch H2D of
    x and dy from pinned memory and D2H of y and dx, overlapped on a copy stream."""
    import torch
    import torch.distributed as dist

    T, H = shape.T, shape.H
    dt = stack.layers[0].dtype
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    hx = [torch.randn(T, H).to(dt).pin_memory() for _ in range(mb)]
    hdy = [torch.randn(T, H).to(dt).pin_memory() for _ in range(mb)]
    hy = [torch.empty(T, H, dtype=dt).pin_memory() for _ in range(mb)]
    hdx = [torch.empty(T, H, dtype=dt).pin_memory() for _ in range(mb)]

    batched = graphs is not None and graphs.batched
    state = {"free": None}   # batched: event after the previous backward (x / dy buffers free)

    def step_batched():
        # x and dy of every micro-batch land while the previous step's W pass runs; y leaves
        # during the backward, dx during this step's W pass
        g_fwd, g_bwd = graphs.microbatch
        with torch.cuda.stream(copy):
            if state["free"] is not None:
                copy.wait_event(state["free"])
            else:
                copy.wait_stream(comp)
            for i in range(mb):
                stack.input(i).copy_(hx[i], non_blocking=True)
            x_in = torch.cuda.Event()
            x_in.record(copy)
            for i in range(mb):
                stack.output_grad(i).copy_(hdy[i], non_blocking=True)
            dy_in = torch.cuda.Event()
            dy_in.record(copy)
        comp.wait_event(x_in)
        g_fwd.replay()
        fwd_done = torch.cuda.Event()
        fwd_done.record(comp)
        comp.wait_event(dy_in)
        g_bwd.replay()
        bwd_done = torch.cuda.Event()
        bwd_done.record(comp)
        state["free"] = bwd_done
        with torch.cuda.stream(copy):
            copy.wait_event(fwd_done)
            for i in range(mb):
                hy[i].copy_(stack.output(i), non_blocking=True)
            copy.wait_event(bwd_done)
            for i in range(mb):
                hdx[i].copy_(stack.input_grad(i), non_blocking=True)
        graphs.wgrad.replay()
        comp.wait_stream(copy)

    def step():
        # micro-batch i's next-step x / dy are loaded as soon as its fwd + bwd is done (its y
        # and dx copied out first), so the loads overlap the rest of the step and the W pass
        if batched:
            return step_batched()
        loaded = state.get("loaded")
        if loaded is None:
            loaded = [torch.cuda.Event() for _ in range(mb)]
            copy.wait_stream(comp)
            with torch.cuda.stream(copy):
                for i in range(mb):
                    stack.input(i).copy_(hx[i], non_blocking=True)
                    stack.output_grad(i).copy_(hdy[i], non_blocking=True)
                    loaded[i].record(copy)
        nxt = [torch.cuda.Event() for _ in range(mb)]
        for i in range(mb):
            comp.wait_event(loaded[i])
            if graphs is not None:
                graphs.microbatch[i].replay()
            else:
                stack.forward_backward(i, accumulate=i > 0, defer_wgrad=True)
            done = torch.cuda.Event()
            done.record(comp)
            with torch.cuda.stream(copy):
                copy.wait_event(done)
                hy[i].copy_(stack.output(i), non_blocking=True)
                hdx[i].copy_(stack.input_grad(i), non_blocking=True)
                stack.input(i).copy_(hx[i], non_blocking=True)
                stack.output_grad(i).copy_(hdy[i], non_blocking=True)
                nxt[i].record(copy)
        state["loaded"] = nxt
        if graphs is not None:
            graphs.wgrad.replay()
        else:
            for ly in stack.layers:
                ly.wgrad(mb)

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(comp)
    for _ in range(args.steps):
        step()
    comp.wait_stream(copy)   # every step's y / dx are on the host
    t1.record(comp)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
    per = T * H * hx[0].element_size()
    return {"value": round(args.steps * mb * T * world / (ms / 1e3), 1), "unit": UNIT,
            "h2d_bytes_per_step": 2 * per * mb, "d2h_bytes_per_step": 2 * per * mb,
            "ms_per_step": round(ms / args.steps, 3),
            "path": ("MoEStack.capture graphs (iteration + W pass)" if graphs is not None else
                     "MoEStack.forward_backward") + " with pinned host x/dy in, y/dx out (copy stream overlapped)"}


def _self_launch(n: int, argv: list) -> int:
    """`python bench.py --gpus N` without torchrun: start the N ranks the way the driver
    does (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1) and pass
    rank 0's JSON line through."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]
    return subprocess.run(cmd).returncode


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=str(ROOT / "configs" / "mixtral_layer.yaml"))
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--n-attn", type=int, default=None, help="A ranks for N>1 (default N/2)")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent fused replicas instead of AF-Pipe")
    ap.add_argument("--seq-len", type=int, default=None, help="override workload.seq_len (sweeps)")
    ap.add_argument("--trace", default=None, help="N>1: write the instrumented iteration as reference-schema trace JSON")
    ap.add_argument("--microbatches", type=int, default=None, help="override workload.num_microbatches")
    ap.add_argument("--layers", type=int, default=None, help="override model.layers")
    ap.add_argument("--depth", type=int, default=None,
                    help="N>1: pipeline depth p (layers alternate over p A+F groups); default schedule.pipeline_depth")
    ap.add_argument("--eager", action="store_true", help="N=1: launch kernels eagerly instead of CUDA graphs")
    ap.add_argument("--no-isolated", action="store_true", help="skip the isolated A-side kernel timing")
    ap.add_argument("--attention", action="store_true",
                    help="add the A-side causal attention block to every layer (own kernels where the shape allows; sweeps)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    from paper_2605_11005_b200.config import load_experiment
    from paper_2605_11005_b200.moe import MoEShape

    exp = load_experiment(args.config)
    if args.seq_len or args.microbatches or args.layers:
        import dataclasses

        wl = dataclasses.replace(exp.workload, seq_len=args.seq_len or exp.workload.seq_len,
                                 num_microbatches=args.microbatches or exp.workload.num_microbatches)
        md = dataclasses.replace(exp.model, layers=args.layers or exp.model.layers)
        exp = dataclasses.replace(exp, workload=wl, model=md,
                                  virtual_stages=md.layers if args.layers else exp.virtual_stages)
    shape = MoEShape.from_experiment(exp)
    if args.impl == "reference":   # CPU arm: rank 0 only, no GPU ranks to start
        return run_reference(args, shape, exp)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args.gpus, argv if argv is not None else sys.argv[1:])
    return run_ours(args, shape, exp)


if __name__ == "__main__":
    sys.exit(main())
