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


def _weights(layer: int = 0):
    from oracle import oracle as O

    _, wg, w1, w3, w2, _ = O.make_inputs(T, H, E, K, DE, seed=7 + 31 * layer)
    return wg, w1, w3, w2


def _inputs(a: int, i: int):
    from oracle import oracle as O

    x, _, _, _, _, dy = O.make_inputs(T, H, E, K, DE, seed=100 + 10 * a + i)
    return x, dy


def _worker(rank, world, n_attn, port, outdir, layers=1):
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
    topo = Topology(world, n_attn, E)
    r = AFPipeRank(MoEShape(T, H, E, K, DE), topo, rank, MB, torch.device("cpu"), stages=CpuStages(),
                   weights=weights, layers=layers)
    r.init_groups()
    if r.role == "A":
        for i, (b, ob) in enumerate(zip(r.bufs, r.out_bufs)):
            x, dy = _inputs(r.idx, i)
            b.x.copy_(torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16))
            ob.dy.copy_(bf(dy))
    r.run_iteration()
    out = {"role": r.role, "idx": r.idx}
    if r.role == "A":
        out["dx"] = [b.dx.float().numpy() for b in r.bufs]
        out["xs"] = [[r.lbufs[l][i].x.view(torch.int16).numpy().view(np.uint16) for l in range(1, layers)]
                     for i in range(MB)]
        out["y"] = [b.y.float().numpy() for b in r.out_bufs]
        out["dwg"] = [rt.dwg.numpy() for rt in r.routers]
    else:
        out["lo"], out["hi"] = r.lo, r.hi
        out["dw13"] = [ex.dw13.numpy() for ex in r.expert_layers]
        out["dw2"] = [ex.dw2.numpy() for ex in r.expert_layers]
    torch.save(out, os.path.join(outdir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def check_against_oracle(outs, n_attn, layers, tol=1e-2):
    """Compare gathered rank outputs with the oracle residual stack (layers == 1: the
    plain MoE layer), summing parameter gradients over A ranks and micro-batches."""
    from oracle import oracle as O

    ws = [_weights(l) for l in range(layers)]
    acc = [{k: 0 for k in ("dwg", "dw1", "dw3", "dw2")} for _ in range(layers)]
    for a in range(n_attn):
        got = next(o for o in outs if o["role"] == "A" and o["idx"] == a)
        for i in range(MB):
            x, dy = _inputs(a, i)
            if layers == 1:
                f = O.moe_forward(x, *ws[0], K)
                b = O.moe_backward(f, x, *ws[0], dy)
                y, dx, bs = f.y, b.dx, [b]
            else:
                y, dx, _, bs, xs = O.moe_stack(x, ws, K, dy, inputs=got["xs"][i])
                for a_got, a_ref in zip(got["xs"][i], xs[1:]):
                    assert O.normwise_rel_err(O.bf16_bits_to_f32(a_got), O.bf16_bits_to_f32(a_ref)) < tol
            assert O.normwise_rel_err(got["y"][i], y) < tol
            assert O.normwise_rel_err(got["dx"][i], dx) < tol
            for l in range(layers):
                for k in acc[l]:
                    acc[l][k] = acc[l][k] + getattr(bs[l], k)
    for o in outs:
        for l in range(layers):
            if o["role"] == "A":
                assert O.normwise_rel_err(o["dwg"][l], acc[l]["dwg"]) < tol  # all-reduced over the A group
            else:
                lo, hi = o["lo"], o["hi"]
                v = o["dw13"][l].reshape(hi - lo, DE // 128, 2, 128, H)
                g1 = v[:, :, 0].reshape(hi - lo, DE, H)
                g3 = v[:, :, 1].reshape(hi - lo, DE, H)
                assert O.normwise_rel_err(g1, acc[l]["dw1"][lo:hi]) < tol
                assert O.normwise_rel_err(g3, acc[l]["dw3"][lo:hi]) < tol
                assert O.normwise_rel_err(o["dw2"][l], acc[l]["dw2"][lo:hi]) < tol


@pytest.mark.parametrize("world,n_attn,layers", [(2, 1, 1), (3, 1, 1), (3, 2, 1), (4, 2, 1), (2, 1, 2), (3, 1, 3)])
def test_afpipe_runtime_matches_oracle(world, n_attn, layers):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, n_attn, _free_port(), d, layers), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt"), weights_only=False) for r in range(world)]
    check_against_oracle(outs, n_attn, layers)


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
