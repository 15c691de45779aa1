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


def _weights():
    from oracle import oracle as O

    _, wg, w1, w3, w2, _ = O.make_inputs(T, H, E, K, DE, seed=7)
    return wg, w1, w3, w2


def _inputs(a: int, i: int):
    from oracle import oracle as O

    x, _, _, _, _, dy = O.make_inputs(T, H, E, K, DE, seed=100 + 10 * a + i)
    return x, dy


def _worker(rank, world, n_attn, port, outdir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from af_cpu_stages import CpuStages
    from oracle import oracle as O
    from paper_2605_11005_b200.moe import MoEShape, interleave_w13
    from paper_2605_11005_b200.runtime import AFPipeRank, Topology

    wg, w1, w3, w2 = _weights()
    bf = lambda a: torch.from_numpy(O.f32_to_bf16_bits(a).view(np.int16).copy()).view(torch.bfloat16)  # noqa: E731
    weights = {"wg": torch.from_numpy(wg), "w13": interleave_w13(bf(w1), bf(w3)), "w2": bf(w2)}
    topo = Topology(world, n_attn, E)
    r = AFPipeRank(MoEShape(T, H, E, K, DE), topo, rank, MB, torch.device("cpu"), stages=CpuStages(),
                   weights=weights)
    r.init_groups()
    if r.role == "A":
        for i, b in enumerate(r.bufs):
            x, dy = _inputs(r.idx, i)
            b.x.copy_(torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16))
            b.dy.copy_(bf(dy))
    r.run_iteration()
    out = {"role": r.role, "idx": r.idx}
    if r.role == "A":
        out["dx"] = [b.dx.float().numpy() for b in r.bufs]
        out["y"] = [b.y.float().numpy() for b in r.bufs]
        out["dwg"] = r.router.dwg.numpy()
    else:
        out["lo"], out["hi"] = r.lo, r.hi
        out["dw13"] = r.experts.dw13.numpy()
        out["dw2"] = r.experts.dw2.numpy()
    torch.save(out, os.path.join(outdir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_attn", [(2, 1), (3, 1), (3, 2), (4, 2)])
def test_afpipe_runtime_matches_oracle(world, n_attn):
    from oracle import oracle as O

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, n_attn, _free_port(), d), nprocs=world, join=True)
        outs = [torch.load(os.path.join(d, f"rank{r}.pt"), weights_only=False) for r in range(world)]
    wg, w1, w3, w2 = _weights()
    dwg = np.zeros_like(wg, dtype=np.float64)
    dw1 = np.zeros_like(w1, dtype=np.float64)
    dw3 = np.zeros_like(w3, dtype=np.float64)
    dw2 = np.zeros_like(w2, dtype=np.float64)
    for a in range(n_attn):
        got = next(o for o in outs if o["role"] == "A" and o["idx"] == a)
        for i in range(MB):
            x, dy = _inputs(a, i)
            f = O.moe_forward(x, wg, w1, w3, w2, K)
            b = O.moe_backward(f, x, wg, w1, w3, w2, dy)
            assert O.normwise_rel_err(got["y"][i], f.y) < 1e-2
            assert O.normwise_rel_err(got["dx"][i], b.dx) < 1e-2
            dwg += b.dwg
            dw1 += b.dw1
            dw3 += b.dw3
            dw2 += b.dw2
    for o in outs:
        if o["role"] == "A":
            assert O.normwise_rel_err(o["dwg"], dwg) < 1e-2  # all-reduced over the A group
        else:
            lo, hi = o["lo"], o["hi"]
            v = o["dw13"].reshape(hi - lo, DE // 128, 2, 128, H)
            g1 = v[:, :, 0].reshape(hi - lo, DE, H)
            g3 = v[:, :, 1].reshape(hi - lo, DE, H)
            assert O.normwise_rel_err(g1, dw1[lo:hi]) < 1e-2
            assert O.normwise_rel_err(g3, dw3[lo:hi]) < 1e-2
            assert O.normwise_rel_err(o["dw2"], dw2[lo:hi]) < 1e-2


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
