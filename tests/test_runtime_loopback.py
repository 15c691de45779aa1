"""The multi-rank AF-Pipe runtime in ONE process on ONE device through the loopback
transport (transport.LoopbackWorld: ranks are host threads with their own CUDA streams;
every M2N / N2M send meets its receive in a hub that issues the device copy on a
per-direction lane stream). This is the same AFPipeRank code the NCCL runs execute —
issue order, counts headers, data-dependent slices, (A rank, expert) grouping on the F
side, deferred wgrad over absolute segments, host I/O streams, the A-group all-reduce —
so the driver's single-GPU box verifies it with the real sm_100a kernels (`-m gpu`), and
the CPU suite verifies it with the CPU stage restatement.

Reference semantics: send/recv twins (pkg/src/afpipe/taskgraph.py:204-242), the
A -> F -> A chain (taskgraph.py:328-340), full-duplex lanes (sim.py:3-7)."""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests"))

import test_runtime_gloo as G  # noqa: E402
from test_runtime_gloo import DE, E, H, K, MB, T, check_against_oracle, collect  # noqa: E402


def _bf(a):
    from oracle import oracle as O

    return torch.from_numpy(O.f32_to_bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16)


def run_loopback(world, n_attn, layers, depth, device, skew=0.0, host_io=False, iterations=2):
    """Build and run `world` ranks on `device`; returns the per-rank collected outputs."""
    from paper_2605_11005_b200.moe import MoEShape, interleave_w13
    from paper_2605_11005_b200.runtime import AFPipeRank, Topology
    from paper_2605_11005_b200.transport import LoopbackWorld

    G.SKEW = skew
    dev = torch.device(device)
    cuda = dev.type == "cuda"
    weights = []
    for l in range(layers):
        wg, w1, w3, w2 = G._weights(l)
        weights.append({"wg": torch.from_numpy(wg), "w13": interleave_w13(_bf(w1), _bf(w3)), "w2": _bf(w2)})
    topo = Topology(world, n_attn, E, depth)

    def build(r, tx):
        stages = None
        if not cuda:
            from af_cpu_stages import CpuStages

            stages = CpuStages()
        rk = AFPipeRank(MoEShape(T, H, E, K, DE), topo, r, MB, dev, stages=stages, weights=weights,
                        layers=layers, transport=tx, record_events=cuda)
        rk.init_groups()
        return rk

    def go(r, tx):
        rk = ranks[r]
        if host_io:
            G.run_host_io(rk, _bf, pin=(lambda t: t.contiguous().pin_memory()) if cuda else (lambda t: t.contiguous()))
        else:
            if rk.role == "A":
                for i in range(MB):
                    x, dy = G._inputs(rk.member, i)
                    if rk.has_input:
                        rk.input(i).copy_(torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16))
                    if rk.has_output:
                        rk.out_bufs[i].dy.copy_(_bf(dy))
            for _ in range(iterations):   # later iterations re-use every buffer (stream-ordering check)
                rk.run_iteration()
        if cuda:
            torch.cuda.synchronize(dev)
        return collect(rk, lambda t: t.cpu().numpy())

    with LoopbackWorld(world, dev, timeout_s=120.0) as lw:
        ranks = lw.run(build)
        outs = lw.run(go)
        moved = lw.hub.bytes_moved
    assert moved > 0
    return outs


def _check(outs, n_attn, depth, layers, skew=0.0):
    G.SKEW = skew
    try:
        check_against_oracle(outs, n_attn // depth, layers)
    finally:
        G.SKEW = 0.0


# ------------------------------------------------------------------ CPU (not gpu)
@pytest.mark.parametrize("world,n_attn,layers,depth", [(2, 1, 1, 1), (3, 1, 1, 1), (3, 2, 1, 1), (4, 2, 2, 2),
                                                       (2, 1, 2, 1)])
def test_loopback_runtime_cpu_matches_oracle(world, n_attn, layers, depth):
    outs = run_loopback(world, n_attn, layers, depth, "cpu", iterations=1)
    _check(outs, n_attn, depth, layers)


def test_loopback_runtime_cpu_skew_and_host_io():
    outs = run_loopback(3, 1, 1, 1, "cpu", skew=40.0, iterations=1)
    _check(outs, 1, 1, 1, skew=40.0)
    outs = run_loopback(2, 1, 2, 1, "cpu", host_io=True)
    _check(outs, 1, 1, 2)


def test_loopback_transport_mismatch_times_out():
    """A receive with no matching send fails loudly (NCCL would hang)."""
    from paper_2605_11005_b200.transport import LoopbackTimeout, LoopbackWorld

    with LoopbackWorld(2, "cpu", timeout_s=0.5) as lw:
        def fn(r, tx):
            if r == 1:
                for w in tx.exchange([("recv", torch.zeros(4), 0)]):
                    w.wait()
        with pytest.raises(LoopbackTimeout):
            lw.run(fn)


def test_loopback_transport_fifo_and_all_reduce():
    from paper_2605_11005_b200.transport import LoopbackWorld

    with LoopbackWorld(3, "cpu") as lw:
        def fn(r, tx):
            out = [torch.zeros(3), torch.zeros(3)]
            if r == 0:
                ws = tx.exchange([("send", torch.full((3,), 1.0), 1), ("send", torch.full((3,), 2.0), 1)])
            elif r == 1:
                ws = tx.exchange([("recv", out[0], 0), ("recv", out[1], 0)])
            else:
                ws = []
            for w in ws:
                w.wait()
            t = torch.full((2,), float(r + 1))
            tx.all_reduce(t, tx.new_group([0, 1, 2]))
            return out, t
        res = lw.run(fn)
    assert torch.equal(res[1][0][0], torch.full((3,), 1.0)) and torch.equal(res[1][0][1], torch.full((3,), 2.0))
    for _, t in res:
        assert torch.equal(t, torch.full((2,), 6.0))


# ------------------------------------------------------------------ GPU (1 B200)
@pytest.mark.gpu
@pytest.mark.parametrize("world,n_attn,layers,depth", [(2, 1, 1, 1), (2, 1, 2, 1), (3, 1, 1, 1), (3, 2, 1, 1),
                                                       (4, 2, 1, 1), (4, 1, 1, 1), (4, 2, 2, 2), (4, 2, 4, 2)])
def test_loopback_runtime_gpu_matches_oracle(cuda, world, n_attn, layers, depth):
    """The AF-Pipe runtime with the sm_100a kernels, A:F = 1:1 (fixed-size exchange),
    1:2 / 1:3 (data-dependent slices), 2:1 / 2:2 (A-group all-reduce), depth 2 with 2 and
    4 layers, all on one GPU: outputs and gradients match the oracle."""
    outs = run_loopback(world, n_attn, layers, depth, cuda)
    _check(outs, n_attn, depth, layers)


@pytest.mark.gpu
def test_loopback_runtime_gpu_skewed_routing_empty_f_rank(cuda):
    """All tokens routed to experts 0..1: the F rank owning experts 2..3 gets empty slices
    and returns zero gradients."""
    outs = run_loopback(3, 1, 1, 1, cuda, skew=40.0)
    _check(outs, 1, 1, 1, skew=40.0)
    f_hi = next(o for o in outs if o["role"] == "F" and o["lo"] == 2)
    assert np.abs(f_hi["dw2"][0]).max() == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("world,n_attn,layers,depth", [(2, 1, 2, 1), (3, 1, 1, 1), (4, 2, 2, 2)])
def test_loopback_runtime_gpu_host_io(cuda, world, n_attn, layers, depth):
    """The e2e path bench.py times (pinned host x/dy in, y/dx out on the h2d/d2h
    streams) is correct and bit-reproducible across iterations."""
    outs = run_loopback(world, n_attn, layers, depth, cuda, host_io=True)
    _check(outs, n_attn, depth, layers)


@pytest.mark.gpu
@pytest.mark.parametrize("world,n_attn,depth", [(2, 1, 1), (4, 2, 2)])
def test_loopback_attention_gpu_matches_fused_stack(cuda, world, n_attn, depth):
    """A-side attention inside AF-Pipe (2 layers) == the fused single-GPU stack."""
    from oracle import oracle as O
    from paper_2605_11005_b200.attention import AttentionBlock
    from paper_2605_11005_b200.moe import MoELayer, MoEShape, MoEStack
    from paper_2605_11005_b200.runtime import AFPipeRank, Topology
    from paper_2605_11005_b200.transport import LoopbackWorld

    layers = 2
    ws = G._attn_weights(layers)
    topo = Topology(world, n_attn, E, depth)

    def build(r, tx):
        rk = AFPipeRank(MoEShape(T, H, E, K, DE), topo, r, MB, cuda, weights=ws, layers=layers, attention=True,
                        seq_len=T, transport=tx)
        rk.init_groups()
        return rk

    def go(r, tx):
        rk = ranks[r]
        if rk.role == "A":
            for i in range(MB):
                x, dy = G._attn_inputs(rk.member, i)
                if rk.has_input:
                    rk.input(i).copy_(x)
                if rk.has_output:
                    rk.out_bufs[i].dy.copy_(dy)
        rk.run_iteration()
        torch.cuda.synchronize(cuda)
        out = {"role": rk.role, "member": rk.member, "layers": rk.my_layers}
        if rk.role == "A":
            if rk.has_output:
                out["y"] = [b.y.float().cpu() for b in rk.out_bufs]
            if rk.has_input:
                out["dx"] = [rk.input_grad(i).float().cpu() for i in range(MB)]
            out["dqkv"] = {l: rk.attn[l].dw_qkv.cpu() for l in rk.my_layers}
            out["dwg"] = {l: rk.routers[l].dwg.cpu() for l in rk.my_layers}
        return out

    with LoopbackWorld(world, cuda, timeout_s=120.0) as lw:
        ranks = lw.run(build)
        outs = lw.run(go)
    a_outs = [o for o in outs if o["role"] == "A" and o["member"] == 0]
    y_got = next(o["y"] for o in a_outs if "y" in o)
    dx_got = next(o["dx"] for o in a_outs if "dx" in o)
    dqkv = {l: v for o in a_outs for l, v in o["dqkv"].items()}
    dwg = {l: v for o in a_outs for l, v in o["dwg"].items()}
    shape = MoEShape(T, H, E, K, DE)
    stack = MoEStack([MoELayer(shape, w["wg"], w["w13"], w["w2"], cuda, num_buffers=MB, residual=True) for w in ws],
                     attention=[AttentionBlock(H, 1, cuda, seed=77 + l) for l in range(layers)], seq_len=T)
    for i in range(MB):
        x, dy = G._attn_inputs(0, i)
        stack.input(i).copy_(x)
        stack.output_grad(i).copy_(dy)
    stack.iteration()
    torch.cuda.synchronize()
    for i in range(MB):
        assert O.normwise_rel_err(y_got[i].numpy(), stack.output(i).float().cpu().numpy()) < 1e-2
        assert O.normwise_rel_err(dx_got[i].numpy(), stack.input_grad(i).float().cpu().numpy()) < 1e-2
    for l in range(layers):
        assert O.normwise_rel_err(dqkv[l].numpy(), stack.attn[l].dw_qkv.cpu().numpy()) < 1e-2
        assert O.normwise_rel_err(dwg[l].numpy(), stack.layers[l].router.dwg.cpu().numpy()) < 1e-2
