"""GPU parity of the sm_100a hot path against the CPU oracle (oracle/), through the C ABI.

Bars: routing — logits, expert ids, counts, padded offsets,
row_map, src_token, x_perm — bit-exact; activations and gradients within a
normwise relative error (max|got-ref| / max|ref|) of 1e-2 in bf16.
"""

import json

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL_BF16 = 1e-2


def to_dev_bf16_bits(bits: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).to(dev)


def to_dev_bf16(vals: np.ndarray, dev) -> torch.Tensor:
    return to_dev_bf16_bits(O.f32_to_bf16_bits(vals), dev)


def f32(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def run_layer(dev, x, wg, w1, w3, w2, dy, k):
    from paper_2605_11005_b200.moe import MoELayer, MoEShape, interleave_w13

    T, H = x.shape
    E, De, _ = w1.shape
    shape = MoEShape(T=T, H=H, E=E, k=k, De=De)
    w13 = interleave_w13(to_dev_bf16(w1, dev), to_dev_bf16(w3, dev))
    layer = MoELayer(shape, torch.from_numpy(wg), w13, to_dev_bf16(w2, dev), dev)
    buf = layer.buffers[0]
    buf.x.copy_(to_dev_bf16_bits(x, dev))
    buf.dy.copy_(to_dev_bf16(dy, dev))
    buf.x_perm.fill_(float("nan"))   # padding rows must be overwritten with zeros
    buf.dy_perm.fill_(float("nan"))
    layer.forward_backward(buf, accumulate=False)
    torch.cuda.synchronize()
    return layer, buf


def check_routing(f, buf, x, k):
    T = x.shape[0]
    assert np.array_equal(buf.idx.cpu().numpy(), f.idx), "expert ids differ"
    assert np.array_equal(buf.counts.cpu().numpy(), f.counts), "per-expert counts differ"
    assert np.array_equal(buf.pad_off.cpu().numpy(), f.pad_off), "padded offsets differ"
    assert np.array_equal(buf.row_map.cpu().numpy(), f.row_map), "permutation indices differ"
    src = buf.src.cpu().numpy()
    end = f.pad_off[-1]
    assert np.array_equal(src[:end], f.src[:end]), "src_token differs"
    xp = buf.x_perm.view(torch.int16).cpu().numpy().view(np.uint16)
    occupied = f.src[:end] >= 0
    assert np.array_equal(xp[:end][occupied], x[f.src[:end][occupied]]), "x_perm not a bit-exact copy"
    assert (xp[:end][~occupied] == 0).all(), "padding rows not zeroed"


def check_values(layer, buf, f, b):
    from paper_2605_11005_b200.moe import split_w13

    errs = {
        "w": O.normwise_rel_err(f32(buf.w), f.w),
        "y": O.normwise_rel_err(f32(buf.y), f.y),
        "dx": O.normwise_rel_err(f32(buf.dx), b.dx),
        "dlogit": O.normwise_rel_err(f32(buf.dlogit), b.dlogit),
        "dwg": O.normwise_rel_err(f32(layer.router.dwg), b.dwg),
        "dw2": O.normwise_rel_err(f32(layer.experts.dw2), b.dw2),
    }
    g1, g3 = split_w13(layer.experts.dw13)
    errs["dw1"] = O.normwise_rel_err(f32(g1), b.dw1)
    errs["dw3"] = O.normwise_rel_err(f32(g3), b.dw3)
    bad = {k_: v for k_, v in errs.items() if not v <= TOL_BF16}
    assert not bad, f"rel errors above {TOL_BF16}: {bad} (all: {errs})"
    return errs


CASES = [
    # T, H, E, k, De, seed, kwargs
    pytest.param(512, 256, 8, 2, 256, 0, {}, id="config1_tiny_T512"),
    pytest.param(1000, 512, 8, 2, 256, 1, {}, id="T_not_multiple_of_chunk"),
    pytest.param(1, 256, 4, 1, 256, 2, {}, id="single_token"),
    pytest.param(200, 256, 8, 2, 256, 3, {"tie_rows": [(0, 3), (1, 6)]}, id="exact_ties"),
    pytest.param(300, 256, 8, 2, 256, 4, {"skew": 40.0}, id="skewed_empty_experts"),
    pytest.param(96, 512, 16, 4, 512, 5, {}, id="topk4_E16"),
    pytest.param(64, 1024, 64, 8, 256, 6, {}, id="fine_grained_E64_k8"),
    pytest.param(130, 768, 3, 3, 256, 7, {}, id="k_equals_E"),
    # 128-wide GEMM tails: the layer of pkg/configs/deepseek_moe.yaml (hidden 2048, 64
    # experts top-4, moe_hidden 1408 = 11 x 128: D_e tail in the SwiGLU' dgrad and dW2),
    # and H = 384 / D_e = 384 (H tail in the W2 fwd, W13 dgrad, dW13 and the dW2 rows)
    pytest.param(256, 2048, 64, 4, 1408, 8, {}, id="deepseek_moe_yaml_De1408"),
    pytest.param(300, 384, 8, 2, 384, 9, {}, id="H384_De384_tails"),
    pytest.param(200, 640, 4, 2, 128, 10, {"skew": 3.0}, id="H640_De128"),
]


@pytest.mark.parametrize("T,H,E,k,De,seed,kw", CASES)
def test_layer_parity_vs_oracle(cuda, T, H, E, k, De, seed, kw):
    x, wg, w1, w3, w2, dy = O.make_inputs(T, H, E, k, De, seed=seed, **kw)
    f = O.moe_forward(x, wg, w1, w3, w2, k)
    b = O.moe_backward(f, x, wg, w1, w3, w2, dy)
    layer, buf = run_layer(cuda, x, wg, w1, w3, w2, dy, k)
    lg = torch.empty(T, E, device=cuda)
    from paper_2605_11005_b200 import kernels as K

    K.router_logits(buf.x, layer.router.wg, lg)
    assert np.array_equal(lg.cpu().numpy().view(np.uint32), f.logits.view(np.uint32)), "logits not bit-exact"
    check_routing(f, buf, x, k)
    check_values(layer, buf, f, b)
    if kw.get("skew"):
        assert (f.counts == 0).any(), "skew case should leave some expert empty"


@pytest.mark.parametrize("name", ["tiny", "ties", "skew", "topk4"])
def test_layer_matches_committed_kats(cuda, golden_dir, name):
    meta = json.loads((golden_dir / "moe_kats.json").read_text())[name]
    kw = {kk: [tuple(p) for p in v] if kk == "tie_rows" else v for kk, v in meta["kwargs"].items()}
    x, wg, w1, w3, w2, dy = O.make_inputs(meta["T"], meta["H"], meta["E"], meta["k"], meta["De"],
                                          seed=meta["seed"], **kw)
    ref = np.load(golden_dir / f"moe_kat_{name}.npz")
    layer, buf = run_layer(cuda, x, wg, w1, w3, w2, dy, meta["k"])
    assert np.array_equal(buf.idx.cpu().numpy(), ref["idx"])
    assert np.array_equal(buf.row_map.cpu().numpy(), ref["row_map"])
    assert np.array_equal(buf.counts.cpu().numpy(), ref["counts"])
    assert O.normwise_rel_err(f32(buf.y), ref["y"]) < TOL_BF16
    assert O.normwise_rel_err(f32(buf.dx), ref["dx"]) < TOL_BF16
    assert O.normwise_rel_err(f32(layer.router.dwg), ref["dwg"]) < TOL_BF16
    assert O.normwise_rel_err(f32(layer.experts.dw2).sum(2), ref["dw2_rowsum"]) < TOL_BF16


@pytest.mark.parametrize("T,H,E,k,De", [
    pytest.param(4096, 4096, 8, 2, 14336, id="config2_mixtral_full"),
    pytest.param(4096, 7168, 256, 8, 2048, id="config3_dsv3_full"),
    pytest.param(32768, 4096, 8, 2, 14336, id="config4_mixtral_T32768"),
    pytest.param(8192, 2048, 64, 4, 1408, id="deepseek_moe_yaml_layer"),
])
def test_full_size_layer_gradients(cuda, T, H, E, k, De):
    """BASELINE sizes (configs #2, #3, the longest config #4 sequence, and the layer of
    the reference's own pkg/configs/deepseek_moe.yaml): routing bit-exact against the C
    oracle over all tokens; y and EVERY gradient (dx incl. the router term, dW_g, dW1,
    dW3, dW2) against an fp32 torch recomputation of the whole layer on the device
    (tests/torch_ref.py; TF32 off), normwise 1e-2."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from torch_ref import layer_errors

    from paper_2605_11005_b200.moe import MoELayer, MoEShape

    rng = np.random.default_rng(123)
    x = O.f32_to_bf16_bits(rng.standard_normal((T, H), dtype=np.float32))
    wg = (rng.standard_normal((E, H), dtype=np.float32) * 0.02).astype(np.float32)
    shape = MoEShape(T=T, H=H, E=E, k=k, De=De)
    layer = MoELayer.random(shape, device=cuda, seed=5)
    layer.router.wg.copy_(torch.from_numpy(wg))
    buf = layer.buffers[0]
    buf.x.copy_(to_dev_bf16_bits(x, cuda))
    buf.dy.normal_()
    layer.forward_backward(buf)
    torch.cuda.synchronize()
    logits, idx, w = O.router(x, wg, k)
    counts, pad_off, row_map, src = O.dispatch(idx, E)
    assert np.array_equal(buf.idx.cpu().numpy(), idx)
    assert np.array_equal(buf.counts.cpu().numpy(), counts)
    assert np.array_equal(buf.pad_off.cpu().numpy(), pad_off)
    assert np.array_equal(buf.row_map.cpu().numpy(), row_map)
    assert np.array_equal(buf.src.cpu().numpy()[: pad_off[-1]], src[: pad_off[-1]])
    assert O.normwise_rel_err(f32(buf.w), w) < 1e-5
    ex = layer.experts
    errs = layer_errors(buf.x, layer.router.wg, ex.w13, ex.w2, buf.idx, buf.dy, buf.y, buf.dx,
                        layer.router.dwg, ex.dw13, ex.dw2)
    bad = {n: v for n, v in errs.items() if not v <= TOL_BF16}
    assert not bad, f"rel errors above {TOL_BF16}: {bad} (all: {errs})"


def test_grad_accumulation_across_microbatches(cuda):
    from paper_2605_11005_b200.moe import MoELayer, MoEShape

    shape = MoEShape(T=256, H=256, E=8, k=2, De=256)
    layer = MoELayer.random(shape, device=cuda, seed=1, num_buffers=2)
    for i, buf in enumerate(layer.buffers):
        buf.x.normal_()
        buf.dy.normal_()
    layer.forward_backward(layer.buffers[0], accumulate=False)
    g0 = (layer.experts.dw13.clone(), layer.experts.dw2.clone(), layer.router.dwg.clone())
    layer.forward_backward(layer.buffers[1], accumulate=False)
    g1 = (layer.experts.dw13.clone(), layer.experts.dw2.clone(), layer.router.dwg.clone())
    layer.forward_backward(layer.buffers[0], accumulate=False)
    layer.forward_backward(layer.buffers[1], accumulate=True)
    torch.cuda.synchronize()
    for a, b_, s in zip(g0, g1, (layer.experts.dw13, layer.experts.dw2, layer.router.dwg)):
        assert torch.allclose(s, a + b_, rtol=1e-5, atol=1e-6)


def test_autograd_function_matches_oracle(cuda):
    from paper_2605_11005_b200.moe import interleave_w13, moe, split_w13

    T, H, E, k, De = 160, 256, 8, 2, 256
    x, wg, w1, w3, w2, dy = O.make_inputs(T, H, E, k, De, seed=21)
    f = O.moe_forward(x, wg, w1, w3, w2, k)
    b = O.moe_backward(f, x, wg, w1, w3, w2, dy)
    xt = to_dev_bf16_bits(x, cuda).requires_grad_(True)
    wgt = torch.from_numpy(wg).to(cuda).requires_grad_(True)
    w13 = interleave_w13(to_dev_bf16(w1, cuda), to_dev_bf16(w3, cuda)).requires_grad_(True)
    w2t = to_dev_bf16(w2, cuda).requires_grad_(True)
    y = moe(xt, wgt, w13, w2t, k)
    y.backward(to_dev_bf16(dy, cuda))
    assert O.normwise_rel_err(f32(y), f.y) < TOL_BF16
    assert O.normwise_rel_err(f32(xt.grad), b.dx) < TOL_BF16
    assert O.normwise_rel_err(f32(wgt.grad), b.dwg) < TOL_BF16
    g1, g3 = split_w13(w13.grad)
    assert O.normwise_rel_err(f32(g1), b.dw1) < TOL_BF16
    assert O.normwise_rel_err(f32(w2t.grad), b.dw2) < TOL_BF16


def test_launch_counter_moves(cuda):
    from paper_2605_11005_b200 import _lib
    from paper_2605_11005_b200.moe import MoELayer, MoEShape

    layer = MoELayer.random(MoEShape(T=64, H=256, E=4, k=2, De=256), device=cuda)
    before = _lib.launch_count()
    layer.forward_backward(layer.buffers[0])
    torch.cuda.synchronize()
    assert _lib.launch_count() - before == layer.launches_per_microbatch()
    before = _lib.launch_count()
    layer.iteration()
    torch.cuda.synchronize()
    assert _lib.launch_count() - before == layer.launches_per_microbatch(True) + MoELayer.launches_per_wgrad_pass


def test_deferred_wgrad_equals_inline_accumulation(cuda):
    """One W pass over a 3-micro-batch slab == per-micro-batch wgrad with beta=1."""
    from paper_2605_11005_b200.moe import MoELayer, MoEShape

    shape = MoEShape(T=300, H=512, E=8, k=2, De=256)
    layer = MoELayer.random(shape, device=cuda, seed=3, num_buffers=3)
    for b in layer.buffers:
        b.x.normal_()
        b.dy.normal_()
    for i, b in enumerate(layer.buffers):
        layer.forward_backward(b, accumulate=i > 0)
    inline = (layer.experts.dw13.clone(), layer.experts.dw2.clone(), layer.router.dwg.clone())
    layer.zero_grad()
    layer.iteration()
    torch.cuda.synchronize()
    for a, b_ in zip(inline, (layer.experts.dw13, layer.experts.dw2, layer.router.dwg)):
        assert O.normwise_rel_err(f32(b_), f32(a)) < 1e-5


def test_iteration_matches_oracle_sum_over_microbatches(cuda):
    from paper_2605_11005_b200.moe import MoELayer, MoEShape, interleave_w13, split_w13

    T, H, E, k, De = 128, 256, 8, 2, 256
    ins = [O.make_inputs(T, H, E, k, De, seed=40 + i) for i in range(2)]
    x0, wg, w1, w3, w2, _ = ins[0]
    layer = MoELayer(MoEShape(T, H, E, k, De), torch.from_numpy(wg),
                     interleave_w13(to_dev_bf16(w1, cuda), to_dev_bf16(w3, cuda)), to_dev_bf16(w2, cuda),
                     cuda, num_buffers=2)
    dw1 = dw2 = 0
    for i, (x, _, _, _, _, dy) in enumerate(ins):
        layer.buffers[i].x.copy_(to_dev_bf16_bits(x, cuda))
        layer.buffers[i].dy.copy_(to_dev_bf16(dy, cuda))
        f = O.moe_forward(x, wg, w1, w3, w2, k)
        b = O.moe_backward(f, x, wg, w1, w3, w2, dy)
        dw1, dw2 = dw1 + b.dw1, dw2 + b.dw2
    layer.iteration()
    torch.cuda.synchronize()
    g1, _ = split_w13(layer.experts.dw13)
    assert O.normwise_rel_err(f32(g1), dw1) < TOL_BF16
    assert O.normwise_rel_err(f32(layer.experts.dw2), dw2) < TOL_BF16


@pytest.mark.parametrize("E,k", [(64, 6), (8, 2)])
def test_router_wgrad_sorted_matches_token_blocked(cuda, E, k):
    """The two router-gradient paths agree (the layer uses the expert-sorted one for E > 16,
    the token-blocked one with its in-kernel ticket reduction for E <= 16); the layer's is
    bit-deterministic across runs and accumulates with beta=1."""
    from paper_2605_11005_b200 import kernels as K
    from paper_2605_11005_b200.moe import MoELayer, MoEShape, a_router_wgrad

    shape = MoEShape(T=1000, H=1024, E=E, k=k, De=256)
    layer = MoELayer.random(shape, device=cuda, seed=9)
    buf = layer.buffers[0]
    buf.x.normal_()
    buf.dy.normal_()
    layer.forward_backward(buf, accumulate=False)
    torch.cuda.synchronize()
    assert buf.dl_perm is not None
    # dl_perm is dlogit scattered to the permuted rows
    rm = buf.row_map.long().flatten()
    assert torch.equal(buf.dl_perm[rm], buf.dlogit.flatten())
    sorted_dwg = layer.router.dwg.clone()   # the layer's own path
    ref = torch.empty_like(sorted_dwg)
    if E > 16:
        K.router_wgrad(buf.x, buf.idx, buf.dlogit, buf.wgrad_ws, ref, 0.0)
    else:
        K.router_wgrad_sorted(buf.x, buf.src, buf.dl_perm, buf.counts, buf.pad_off, ref, 0.0,
                              partial_ws=buf.wgrad_ws)
    torch.cuda.synchronize()
    assert O.normwise_rel_err(f32(sorted_dwg), f32(ref)) < 1e-5
    a_router_wgrad(buf, layer.router, False)
    torch.cuda.synchronize()
    assert torch.equal(layer.router.dwg, sorted_dwg)
    a_router_wgrad(buf, layer.router, True)
    torch.cuda.synchronize()
    assert torch.equal(layer.router.dwg, 2 * sorted_dwg)


@pytest.mark.parametrize("E,k", [(8, 2), (32, 4)])
def test_residual_stack_matches_oracle(cuda, E, k):
    """Fused single-device 2-layer residual stack (x_{l+1} = x_l + MoE_l(x_l)): the
    residual adds fused into combine_fwd / permute_bwd and the in-place layer chaining
    reproduce the oracle stack; all four micro-batch gradients accumulate."""
    from paper_2605_11005_b200.moe import MoELayer, MoEShape, MoEStack, interleave_w13, split_w13

    T, H, De, L = 200, 256, 256, 2
    ws = []
    for l in range(L):
        _, wg, w1, w3, w2, _ = O.make_inputs(T, H, E, k, De, seed=300 + l)
        ws.append((wg, w1, w3, w2))
    shape = MoEShape(T=T, H=H, E=E, k=k, De=De)
    layers = [MoELayer(shape, torch.from_numpy(wg), interleave_w13(to_dev_bf16(w1, cuda), to_dev_bf16(w3, cuda)),
                       to_dev_bf16(w2, cuda), cuda, num_buffers=2, residual=True) for wg, w1, w3, w2 in ws]
    stack = MoEStack(layers)
    ins = [O.make_inputs(T, H, E, k, De, seed=400 + i) for i in range(2)]
    for i, (x, *_, dy) in enumerate(ins):
        stack.buffers[i].x.copy_(to_dev_bf16_bits(x, cuda))
        stack.out_buffers[i].dy.copy_(to_dev_bf16(dy, cuda))
    stack.iteration()
    torch.cuda.synchronize()
    acc = [{n: 0 for n in ("dwg", "dw1", "dw2")} for _ in range(L)]
    for i, (x, *_, dy) in enumerate(ins):
        x1 = layers[1].buffers[i].x.view(torch.int16).cpu().numpy().view(np.uint16)
        y, dx, fs, bs, xs = O.moe_stack(x, ws, k, dy, inputs=[x1])
        assert O.normwise_rel_err(O.bf16_bits_to_f32(x1), O.bf16_bits_to_f32(xs[1])) < TOL_BF16
        assert np.array_equal(layers[1].buffers[i].idx.cpu().numpy(), fs[1].idx), "layer-1 routing differs"
        assert O.normwise_rel_err(f32(stack.out_buffers[i].y), y) < TOL_BF16
        assert O.normwise_rel_err(f32(stack.buffers[i].dx), dx) < TOL_BF16
        for l in range(L):
            for n in acc[l]:
                acc[l][n] = acc[l][n] + getattr(bs[l], n)
    for l in range(L):
        assert O.normwise_rel_err(f32(layers[l].router.dwg), acc[l]["dwg"]) < TOL_BF16
        g1, _ = split_w13(layers[l].experts.dw13)
        assert O.normwise_rel_err(f32(g1), acc[l]["dw1"]) < TOL_BF16
        assert O.normwise_rel_err(f32(layers[l].experts.dw2), acc[l]["dw2"]) < TOL_BF16


def test_stack_graph_replay_matches_eager(cuda):
    """MoEStack.capture(): CUDA-graph replays give bit-identical outputs and gradients
    to eager launches, including after new inputs are written in place."""
    from paper_2605_11005_b200.moe import MoEShape, MoEStack

    shape = MoEShape(T=300, H=256, E=8, k=2, De=256)
    stack = MoEStack.random(shape, 2, device=cuda, seed=5, num_buffers=2)
    graphs = stack.capture()
    assert graphs.launches_per_iteration > 0

    def snap():
        torch.cuda.synchronize()
        out = [b.y.clone() for b in stack.out_buffers] + [b.dx.clone() for b in stack.buffers]
        for ly in stack.layers:
            out += [ly.router.dwg.clone(), ly.experts.dw13.clone(), ly.experts.dw2.clone()]
        return out

    for trial in range(2):
        for b, ob in zip(stack.buffers, stack.out_buffers):
            b.x.normal_()
            ob.dy.normal_()
        stack.iteration()
        eager = snap()
        graphs.replay()
        replay = snap()
        for a, b_ in zip(eager, replay):
            assert torch.equal(a, b_)


TOL_FP32 = 1e-4


@pytest.mark.parametrize("T,H,E,k,De", [
    pytest.param(256, 256, 8, 2, 256, id="f32_tiny"),
    pytest.param(200, 512, 16, 4, 256, id="f32_E16_k4"),
    pytest.param(100, 256, 64, 8, 512, id="f32_E64_k8"),
])
def test_fp32_mode_matches_oracle(cuda, T, H, E, k, De):
    """fp32 mode (bytes_per_element 4): routing bit-exact on fp32 activations; outputs and
    all gradients within 1e-4 normwise of the fp64 oracle (split-3 tensor-core GEMMs)."""
    from paper_2605_11005_b200.moe import MoEShape, interleave_w13, split_w13
    from paper_2605_11005_b200.moe_f32 import MoELayerF32

    rng = np.random.default_rng(11)
    x = rng.standard_normal((T, H), dtype=np.float32)
    wg = (rng.standard_normal((E, H), dtype=np.float32) * 0.02).astype(np.float32)
    w1 = (rng.standard_normal((E, De, H), dtype=np.float32) * 0.02).astype(np.float32)
    w3 = (rng.standard_normal((E, De, H), dtype=np.float32) * 0.02).astype(np.float32)
    w2 = (rng.standard_normal((E, H, De), dtype=np.float32) * 0.02).astype(np.float32)
    dy = rng.standard_normal((T, H), dtype=np.float32)
    f = O.moe_forward(x, wg, w1, w3, w2, k)
    b = O.moe_backward(f, x, wg, w1, w3, w2, dy)
    t = lambda a: torch.from_numpy(a).to(cuda)  # noqa: E731
    layer = MoELayerF32(MoEShape(T=T, H=H, E=E, k=k, De=De), torch.from_numpy(wg),
                        interleave_w13(t(w1), t(w3)), t(w2), cuda)
    buf = layer.buffers[0]
    buf.x.copy_(t(x))
    buf.dy.copy_(t(dy))
    layer.forward_backward(buf)
    torch.cuda.synchronize()
    assert np.array_equal(buf.idx.cpu().numpy(), f.idx), "expert ids differ"
    assert np.array_equal(buf.row_map.cpu().numpy(), f.row_map), "permutation differs"
    assert np.array_equal(buf.pad_off.cpu().numpy(), f.pad_off)
    errs = {
        "y": O.normwise_rel_err(f32(buf.y), f.y),
        "dx": O.normwise_rel_err(f32(buf.dx), b.dx),
        "dwg": O.normwise_rel_err(f32(layer.dwg), b.dwg),
        "dw2": O.normwise_rel_err(f32(layer.experts.dw2), b.dw2),
    }
    g1, g3 = split_w13(layer.experts.dw13)
    errs["dw1"] = O.normwise_rel_err(f32(g1), b.dw1)
    errs["dw3"] = O.normwise_rel_err(f32(g3), b.dw3)
    assert max(errs.values()) < TOL_FP32, errs


def test_fp32_autograd_and_iteration(cuda):
    """moe() on fp32 tensors runs fp32 mode; the deferred W pass over a 2-micro-batch
    slab equals the per-micro-batch inline wgrad (split-3 strided wgrad path)."""
    from paper_2605_11005_b200.moe import MoEShape, moe, split_w13
    from paper_2605_11005_b200.moe_f32 import MoELayerF32

    T, H, E, k, De = 128, 256, 8, 2, 256
    rng = np.random.default_rng(3)
    x = rng.standard_normal((T, H), dtype=np.float32)
    wg = (rng.standard_normal((E, H), dtype=np.float32) * 0.02).astype(np.float32)
    w1 = (rng.standard_normal((E, De, H), dtype=np.float32) * 0.02).astype(np.float32)
    w3 = (rng.standard_normal((E, De, H), dtype=np.float32) * 0.02).astype(np.float32)
    w2 = (rng.standard_normal((E, H, De), dtype=np.float32) * 0.02).astype(np.float32)
    dy = rng.standard_normal((T, H), dtype=np.float32)
    f = O.moe_forward(x, wg, w1, w3, w2, k)
    b = O.moe_backward(f, x, wg, w1, w3, w2, dy)
    from paper_2605_11005_b200.moe import interleave_w13

    t = lambda a: torch.from_numpy(a).to(cuda)  # noqa: E731
    xt = t(x).requires_grad_(True)
    wgt = t(wg).requires_grad_(True)
    w13 = interleave_w13(t(w1), t(w3)).requires_grad_(True)
    w2t = t(w2).requires_grad_(True)
    y = moe(xt, wgt, w13, w2t, k)
    y.backward(t(dy))
    assert y.dtype == torch.float32
    assert O.normwise_rel_err(f32(y), f.y) < TOL_FP32
    assert O.normwise_rel_err(f32(xt.grad), b.dx) < TOL_FP32
    assert O.normwise_rel_err(f32(wgt.grad), b.dwg) < TOL_FP32
    g1, _ = split_w13(w13.grad)
    assert O.normwise_rel_err(f32(g1), b.dw1) < TOL_FP32
    assert O.normwise_rel_err(f32(w2t.grad), b.dw2) < TOL_FP32

    layer = MoELayerF32.random(MoEShape(T=300, H=256, E=8, k=2, De=256), cuda, seed=2, num_buffers=2)
    for bb in layer.buffers:
        bb.x.normal_()
        bb.dy.normal_()
    for i, bb in enumerate(layer.buffers):
        layer.forward_backward(bb, accumulate=i > 0)
    inline = (layer.experts.dw13.clone(), layer.experts.dw2.clone(), layer.dwg.clone())
    layer.zero_grad()
    layer.iteration()
    torch.cuda.synchronize()
    for a, b_ in zip(inline, (layer.experts.dw13, layer.experts.dw2, layer.dwg)):
        assert O.normwise_rel_err(f32(b_), f32(a)) < 1e-5


@pytest.mark.parametrize("T,H,E,k,De,n,L,skew", [(512, 256, 8, 2, 256, 4, 1, 0.0), (384, 512, 64, 4, 384, 3, 1, 0.0),
                                                (256, 256, 8, 2, 256, 2, 2, 0.0), (1024, 256, 2, 1, 256, 3, 1, 0.0),
                                                (512, 256, 32, 2, 256, 4, 1, 1.0)])
def test_batched_iteration_equals_per_microbatch(cuda, T, H, E, k, De, n, L, skew, monkeypatch):
    """The batched iteration (every micro-batch's expert GEMMs as one launch per stage: groups
    expert-major with shared pair tiles for fine-grained experts, micro-batch-major for coarse
    ones — the last case) is bit-identical to micro-batch-by-micro-batch execution: outputs,
    input gradients and every weight gradient; its CUDA-graph replay too."""
    from paper_2605_11005_b200.moe import MoELayer, MoEShape, MoEStack

    monkeypatch.setenv("DM_BATCHED", "1")   # the coarse-expert case is batched only on request
    shape = MoEShape(T, H, E, k, De)
    res = []
    for mode in ("per_mb", "batched", "graph"):
        stack = MoEStack([MoELayer.random(shape, cuda, seed=40 + l, num_buffers=n, residual=L > 1)
                          for l in range(L)])
        if skew:   # about half the tokens pick experts 0 and 1: ragged and empty (expert, mb) ranges
            for ly in stack.layers:
                ly.router.wg[:2] += skew
        g = torch.Generator(device="cpu").manual_seed(5)
        for i in range(n):
            stack.input(i).copy_(torch.randn(T, H, generator=g).to(torch.bfloat16))
            stack.output_grad(i).copy_(torch.randn(T, H, generator=g).to(torch.bfloat16))
        assert stack.batched_supported(n)
        if mode == "per_mb":
            for i in range(n):
                stack.forward_backward(i, accumulate=i > 0, defer_wgrad=True)
            for ly in stack.layers:
                ly.wgrad(n)
        elif mode == "batched":
            stack.iteration(n)
        else:
            gr = stack.capture(n)
            assert gr.batched and len(gr.microbatch) == 2
            gr.replay()
        torch.cuda.synchronize()
        out = [stack.output(i).clone() for i in range(n)] + [stack.input_grad(i).clone() for i in range(n)]
        for ly in stack.layers:
            out += [ly.router.dwg.clone(), ly.experts.dw13.clone(), ly.experts.dw2.clone()]
        res.append(out)
    for mode_out in res[1:]:
        for a, b in zip(res[0], mode_out):
            assert torch.equal(a, b)
