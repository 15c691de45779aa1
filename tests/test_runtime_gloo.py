"""Multi-process AF-Pipe runtime on CPU (gloo, world_size 2-3): the protocol —
counts headers, data-dependent slices, planned issue order, F-side grouping over
(A rank, expert), deferred wgrad over absolute segments, the A-group dW_g
all-reduce — must reproduce the single-process oracle's gradients."""

import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]

T, H, E, K, DE, MB = 48, 256, 4, 2, 256, 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


SKEW = 0.0   # > 0: routing biased onto experts 0..K-1 (oracle.make_inputs), so some F ranks get no rows


def _weights(layer: int = 0):
    from oracle import oracle as O

    _, wg, w1, w3, w2, _ = O.make_inputs(T, H, E, K, DE, seed=7 + 31 * layer, skew=SKEW)
    return wg, w1, w3, w2


def _inputs(a: int, i: int):
    from oracle import oracle as O

    x, _, _, _, _, dy = O.make_inputs(T, H, E, K, DE, seed=100 + 10 * a + i, skew=SKEW)
    return x, dy


def collect(r, to_np=lambda t: t.numpy()):
    """Per-rank results keyed by layer (a rank holds only its pipeline group's layers)."""
    out = {"role": r.role, "group": r.group, "member": r.member, "layers": r.my_layers}
    bits = lambda t: to_np(t.contiguous().view(torch.int16)).view(np.uint16)  # noqa: E731
    if r.role == "A":
        if r.has_input:
            out["dx"] = [to_np(r.input_grad(i).float()) for i in range(MB)]
        if r.has_output:
            out["y"] = [to_np(b.y.float()) for b in r.out_bufs]
        out["xin"] = {l: [bits(r.lbufs[l][i].x) for i in range(MB)] for l in r.my_layers if l > 0}
        out["dwg"] = {l: to_np(rt.dwg) for l, rt in r.routers.items()}
    else:
        out["lo"], out["hi"] = r.lo, r.hi
        out["dw13"] = {l: to_np(ex.dw13) for l, ex in r.expert_layers.items()}
        out["dw2"] = {l: to_np(ex.dw2) for l, ex in r.expert_layers.items()}
    return out


def run_host_io(r, bf, pin=lambda t: t.contiguous()):
    """e2e mode (set_host_io): host inputs copied in and y / dx copied out by the runtime,
    three back-to-back iterations (real, other, real inputs); the two real iterations must
    give identical host outputs equal to the device buffers. Shared with the NCCL test
    (pinned buffers there, so the copies overlap the previous iteration's tail)."""
    empty = lambda: [pin(torch.empty(T, H, dtype=torch.bfloat16)) for _ in range(MB)]  # noqa: E731
    real, other = ([], []), ([], [])
    g = torch.Generator().manual_seed(5)
    for i in range(MB):
        x, dy = _inputs(r.member, i)
        real[0].append(pin(torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16)))
        real[1].append(pin(bf(dy)))
        other[0].append(pin(torch.randn(T, H, generator=g).to(torch.bfloat16)))
        other[1].append(pin(torch.randn(T, H, generator=g).to(torch.bfloat16)))
    outs = []
    for xs, dys in (real, other, real):
        ys, dxs = empty(), empty()
        if r.role == "A":
            r.set_host_io(xs, dys, ys, dxs)
        r.run_iteration()
        outs.append((ys, dxs))
    if r.device.type == "cuda":
        torch.cuda.synchronize()
    if r.role == "A":
        for i in range(MB):
            if r.has_output:
                assert torch.equal(outs[0][0][i], outs[2][0][i])
                assert torch.equal(outs[2][0][i], r.out_bufs[i].y.cpu())
            if r.has_input:
                assert torch.equal(outs[0][1][i], outs[2][1][i])
                assert torch.equal(outs[2][1][i], r.input_grad(i).cpu())


def _worker(rank, world, n_attn, port, outdir, layers=1, depth=1, skew=0.0, host_io=False):
    global SKEW
    SKEW = skew
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from af_cpu_stages import CpuStages
    from oracle import oracle as O
    from paper_2605_11005_b200.moe import MoEShape, interleave_w13
    from paper_2605_11005_b200.runtime import AFPipeRank, Topology

    bf = lambda a: torch.from_numpy(O.f32_to_bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16)  # noqa: E731
    weights = []
    for l in range(layers):
        wg, w1, w3, w2 = _weights(l)
        weights.append({"wg": torch.from_numpy(wg), "w13": interleave_w13(bf(w1), bf(w3)), "w2": bf(w2)})
    topo = Topology(world, n_attn, E, depth)
    r = AFPipeRank(MoEShape(T, H, E, K, DE), topo, rank, MB, torch.device("cpu"), stages=CpuStages(),
                   weights=weights, layers=layers)
    r.init_groups()
    if host_io:
        run_host_io(r, bf)
    else:
        if r.role == "A":
            for i in range(MB):
                x, dy = _inputs(r.member, i)
                if r.has_input:
                    r.input(i).copy_(torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16))
                if r.has_output:
                    r.out_bufs[i].dy.copy_(bf(dy))
        r.run_iteration()
    torch.save(collect(r), os.path.join(outdir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def check_against_oracle(outs, n_streams, layers, tol=1e-2):
    """Compare gathered rank outputs with the oracle residual stack (layers == 1: the
    plain MoE layer), summing parameter gradients over streams and micro-batches.
    Stream j's layer-0 input/gradient, its layer inputs and its output may live on
    different ranks (pipeline groups): they are joined by (member, layer)."""
    from oracle import oracle as O

    ws = [_weights(l) for l in range(layers)]
    acc = [{k: 0 for k in ("dwg", "dw1", "dw3", "dw2")} for _ in range(layers)]
    a_outs = [o for o in outs if o["role"] == "A"]
    for j in range(n_streams):
        mine = [o for o in a_outs if o["member"] == j]
        dx_got = next(o["dx"] for o in mine if "dx" in o)
        y_got = next(o["y"] for o in mine if "y" in o)
        xin = {l: v for o in mine for l, v in o["xin"].items()}
        for i in range(MB):
            x, dy = _inputs(j, i)
            if layers == 1:
                f = O.moe_forward(x, *ws[0], K)
                b = O.moe_backward(f, x, *ws[0], dy)
                y, dx, bs = f.y, b.dx, [b]
            else:
                inputs = [xin[l][i] for l in range(1, layers)]
                y, dx, _, bs, xs = O.moe_stack(x, ws, K, dy, inputs=inputs)
                for a_got, a_ref in zip(inputs, xs[1:]):
                    assert O.normwise_rel_err(O.bf16_bits_to_f32(a_got), O.bf16_bits_to_f32(a_ref)) < tol
            assert O.normwise_rel_err(y_got[i], y) < tol
            assert O.normwise_rel_err(dx_got[i], dx) < tol
            for l in range(layers):
                for k in acc[l]:
                    acc[l][k] = acc[l][k] + getattr(bs[l], k)
    for o in outs:
        for l in o["layers"]:
            if o["role"] == "A":
                assert O.normwise_rel_err(o["dwg"][l], acc[l]["dwg"]) < tol  # all-reduced over the A group
            else:
                lo, hi = o["lo"], o["hi"]
                G = 64   # DM_GLU_BLOCK
                v = o["dw13"][l].reshape(hi - lo, DE // G, 2, G, H)
                g1 = v[:, :, 0].reshape(hi - lo, DE, H)
                g3 = v[:, :, 1].reshape(hi - lo, DE, H)
                assert O.normwise_rel_err(g1, acc[l]["dw1"][lo:hi]) < tol
                assert O.normwise_rel_err(g3, acc[l]["dw3"][lo:hi]) < tol
                assert O.normwise_rel_err(o["dw2"][l], acc[l]["dw2"][lo:hi]) < tol


@pytest.mark.parametrize("world,n_attn,layers,depth", [
    (2, 1, 1, 1), (3, 1, 1, 1), (3, 2, 1, 1), (4, 2, 1, 1), (2, 1, 2, 1), (3, 1, 3, 1),
    (4, 2, 2, 2), (4, 2, 4, 2),   # pipeline_depth 2: layers alternate between two A+F groups
    (8, 4, 1, 1), (8, 4, 2, 2),   # the 8-GPU 4A:4F split of BASELINE configs[1] (protocol on CPU)
])
def test_afpipe_runtime_matches_oracle(world, n_attn, layers, depth):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, n_attn, _free_port(), d, layers, depth), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt"), weights_only=False) for r in range(world)]
    check_against_oracle(outs, n_attn // depth, layers)


@pytest.mark.parametrize("world,n_attn,layers,depth", [(2, 1, 2, 1), (4, 2, 2, 2)])
def test_afpipe_runtime_host_io(world, n_attn, layers, depth):
    """The e2e host-I/O path bench.py times (set_host_io), on CPU."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, n_attn, _free_port(), d, layers, depth, 0.0, True), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt"), weights_only=False) for r in range(world)]
    check_against_oracle(outs, n_attn // depth, layers)


def test_afpipe_runtime_skewed_routing_empty_f_ranks():
    """Routing biased onto experts 0..K-1: the F rank owning experts 2..3 receives no rows
    (empty slices are skipped symmetrically on both ends) and still returns zero grads."""
    global SKEW
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(3, 1, _free_port(), d, 1, 1, 40.0), nprocs=3, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt"), weights_only=False) for r in range(3)]
    SKEW = 40.0
    try:
        check_against_oracle(outs, 1, 1)
    finally:
        SKEW = 0.0
    f_hi = next(o for o in outs if o["role"] == "F" and o["lo"] == 2)
    assert np.abs(f_hi["dw2"][0]).max() == 0.0


def test_topology_blocks_match_reference_balanced_blocks():
    from paper_2605_11005_b200.runtime import Topology, balanced_blocks

    assert balanced_blocks(256, 6) == [43, 43, 43, 43, 42, 42]
    t = Topology(8, 2, 256)
    assert [t.expert_block(f) for f in range(6)][0] == (0, 43)
    assert t.expert_block(5) == (214, 256)
    assert Topology.default(8, 8) == Topology(8, 4, 8)
    with pytest.raises(ValueError):
        Topology(4, 0, 8)
    with pytest.raises(ValueError):
        Topology(10, 1, 8)


def _attn_worker(rank, world, n_attn, port, outdir, layers, depth=1):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from af_cpu_stages import CpuStages
    from paper_2605_11005_b200.moe import MoEShape
    from paper_2605_11005_b200.runtime import AFPipeRank, Topology

    weights = _attn_weights(layers)
    r = AFPipeRank(MoEShape(T, H, E, K, DE), Topology(world, n_attn, E, depth), rank, MB, torch.device("cpu"),
                   stages=CpuStages(), weights=weights, layers=layers, attention=True, seq_len=T)
    r.init_groups()
    out = {"role": r.role, "member": r.member, "layers": r.my_layers}
    if r.role == "A":
        for i in range(MB):
            x, dy = _attn_inputs(r.member, i)
            if r.has_input:
                r.input(i).copy_(x)
            if r.has_output:
                r.out_bufs[i].dy.copy_(dy)
    r.run_iteration()
    if r.role == "A":
        if r.has_output:
            out["y"] = [b.y.float() for b in r.out_bufs]
        if r.has_input:
            out["dx"] = [r.input_grad(i).float() for i in range(MB)]
        out["dwg"] = {l: rt.dwg.clone() for l, rt in r.routers.items()}
        out["dqkv"] = {l: a.dw_qkv.clone() for l, a in r.attn.items()}
    torch.save(out, os.path.join(outdir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _attn_weights(layers):
    from oracle import oracle as O
    from paper_2605_11005_b200.moe import interleave_w13

    bf = lambda a: torch.from_numpy(O.f32_to_bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16)  # noqa: E731
    out = []
    for l in range(layers):
        wg, w1, w3, w2 = _weights(l)
        out.append({"wg": torch.from_numpy(wg), "w13": interleave_w13(bf(w1), bf(w3)), "w2": bf(w2)})
    return out


def _attn_inputs(a, i):
    g = torch.Generator().manual_seed(500 + 10 * a + i)
    return (torch.randn(T, H, generator=g).to(torch.bfloat16), torch.randn(T, H, generator=g).to(torch.bfloat16))


def _sequential_reference(n_attn, layers):
    """Single process, same CPU stage arithmetic and attention blocks, full expert set,
    micro-batches run one after another: what the distributed schedule must reproduce."""
    sys.path.insert(0, str(ROOT / "tests"))
    from af_cpu_stages import CpuStages
    from paper_2605_11005_b200.attention import AttentionBlock
    from paper_2605_11005_b200.moe import ActivationSlab, ExpertParams, MicroBatchBuffers, MoEShape, RouterParams

    st = CpuStages()
    shape = MoEShape(T, H, E, K, DE)
    ws = _attn_weights(layers)
    res = {}
    for a in range(n_attn):
        blocks = [AttentionBlock(H, 1, "cpu", seed=77 + l) for l in range(layers)]
        routers = [RouterParams(w["wg"].float()) for w in ws]
        experts = [ExpertParams(w["w13"], w["w2"]) for w in ws]
        slabs = [ActivationSlab(shape, MB, "cpu") for _ in range(layers)]
        bufs = [[MicroBatchBuffers(shape, "cpu", slabs[l], i, residual=True) for i in range(MB)] for l in range(layers)]
        ys, dxs = [], []
        for i in range(MB):
            x, dy = _attn_inputs(a, i)
            dx = torch.empty(T, H, dtype=torch.bfloat16)
            x_in = x
            for l in range(layers):
                b = bufs[l][i]
                blocks[l].forward(i, x_in, b.x, T)
                st.a_dispatch(b, routers[l])
                st.f_forward(b, experts[l], b.pad_off)
                st.a_combine(b)
                x_in = b.y
            ys.append(bufs[-1][i].y.float())
            bufs[-1][i].dy.copy_(dy)
            for l in reversed(range(layers)):
                b = bufs[l][i]
                st.a_combine_bwd(b)
                st.f_backward(b, experts[l], b.pad_off)
                st.a_backward(b, routers[l], i > 0)
                dst = dx if l == 0 else bufs[l - 1][i].dy
                blocks[l].backward(i, b.dx, dst, i > 0)
            dxs.append(dx.float())
        res[a] = {"y": ys, "dx": dxs, "dwg": [r.dwg for r in routers], "dqkv": [b.dw_qkv for b in blocks]}
    return res


@pytest.mark.parametrize("world,n_attn,layers,depth", [(2, 1, 2, 1), (3, 2, 1, 1), (4, 2, 2, 2)])
def test_afpipe_runtime_with_attention_matches_sequential(world, n_attn, layers, depth):
    """A-side attention inside the AF-Pipe schedule (attention.py): the distributed run
    reproduces a single-process sequential execution of the same blocks; attention and
    router gradients are all-reduced over the A group."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_attn_worker, args=(world, n_attn, _free_port(), d, layers, depth), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt"), weights_only=False) for r in range(world)]
    ref = _sequential_reference(n_attn // depth, layers)
    from oracle import oracle as O

    tot_dwg = [sum(ref[a]["dwg"][l] for a in ref) for l in range(layers)]
    tot_qkv = [sum(ref[a]["dqkv"][l] for a in ref) for l in range(layers)]
    for o in outs:
        if o["role"] != "A":
            continue
        r = ref[o["member"]]
        for i in range(MB):
            if "y" in o:
                assert O.normwise_rel_err(o["y"][i].numpy(), r["y"][i].numpy()) < 1e-2
            if "dx" in o:
                assert O.normwise_rel_err(o["dx"][i].numpy(), r["dx"][i].numpy()) < 1e-2
        for l in o["layers"]:
            assert O.normwise_rel_err(o["dwg"][l].numpy(), tot_dwg[l].numpy()) < 1e-2
            assert O.normwise_rel_err(o["dqkv"][l].numpy(), tot_qkv[l].numpy()) < 1e-2
