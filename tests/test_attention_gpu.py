"""Own sm_100a causal GQA flash-attention forward (dm_attention_fwd)
against an fp32 PyTorch reference of the same op: output within the bf16-P tolerance,
log-sum-exp to 2e-3 absolute, and agreement with torch's SDPA (cuDNN) on the same inputs."""

import math
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

D = 128


def _reference(qkv, b, s, nh, nkv):
    x = qkv.float().view(b, s, nh + 2 * nkv, D)
    q, k, v = x[:, :, :nh], x[:, :, nh:nh + nkv], x[:, :, nh + nkv:]
    g = nh // nkv
    k = k.repeat_interleave(g, dim=2)
    v = v.repeat_interleave(g, dim=2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))            # [b, nh, s, D]
    sc = q @ k.transpose(-1, -2) / math.sqrt(D)
    mask = torch.triu(torch.ones(s, s, dtype=torch.bool, device=qkv.device), 1)
    sc = sc.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(sc, dim=-1)
    o = torch.softmax(sc, dim=-1) @ v
    return o.transpose(1, 2).reshape(b * s, nh * D), lse


@pytest.mark.parametrize("b,s,nh,nkv", [(1, 256, 2, 1), (2, 256, 4, 2), (3, 512, 2, 2), (1, 1024, 8, 8), (1, 2048, 4, 1), (2, 384, 8, 2), (2, 512, 6, 2)])
def test_attention_fwd_matches_fp32_reference(b, s, nh, nkv):
    from paper_2605_11005_b200 import kernels as K

    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(b * 1000 + s + nh)
    qkv = torch.randn(b * s, (nh + 2 * nkv) * D, generator=g).to(torch.bfloat16).to(dev)
    out = torch.empty(b * s, nh * D, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(b, nh, s, dtype=torch.float32, device=dev)
    K.attention_fwd(qkv, s, nh, nkv, out, lse)
    torch.cuda.synchronize()
    o_ref, lse_ref = _reference(qkv, b, s, nh, nkv)
    err = (out.float() - o_ref).abs().max().item() / o_ref.abs().max().item()
    assert err < 1e-2, err
    assert (lse - lse_ref).abs().max().item() < 2e-3
    # the library path on the same inputs
    x = qkv.view(b, s, nh + 2 * nkv, D).transpose(1, 2)
    o_lib = torch.nn.functional.scaled_dot_product_attention(
        x[:, :nh], x[:, nh:nh + nkv], x[:, nh + nkv:], is_causal=True, enable_gqa=nh != nkv)
    o_lib = o_lib.transpose(1, 2).reshape(b * s, nh * D).float()
    assert (out.float() - o_lib).abs().max().item() / o_lib.abs().max().item() < 1e-2


def test_attention_fwd_rejects_bad_shapes():
    from paper_2605_11005_b200 import _lib
    from paper_2605_11005_b200 import kernels as K

    dev = torch.device("cuda", 0)
    qkv = torch.zeros(200, 4 * D, dtype=torch.bfloat16, device=dev)
    out = torch.empty(200, 2 * D, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(1, 2, 200, dtype=torch.float32, device=dev)
    with pytest.raises(_lib.DMError):
        K.attention_fwd(qkv, 200, 2, 1, out, lse)   # seq_len not a multiple of 128


@pytest.mark.parametrize("s,b,g", [(256, 2, 1), (512, 1, 4)])
def test_attention_block_own_forward_matches_library(s, b, g):
    """AttentionBlock on own kernels only (grouped tcgen05 GEMM projections, dm_attention_fwd /
    _bwd, ragged-K wgrad) equals the all-library block (torch projections + cuDNN SDPA under
    autograd): output, input gradient and both weight gradients, first call and accumulated."""
    from paper_2605_11005_b200.attention import AttentionBlock

    dev = torch.device("cuda", 0)
    H = 512
    gen = torch.Generator(device="cpu").manual_seed(s + g)
    x = torch.randn(b * s, H, generator=gen).to(torch.bfloat16).to(dev)
    dh = torch.randn(b * s, H, generator=gen).to(torch.bfloat16).to(dev)
    res = []
    for own in (True, False):
        blk = AttentionBlock(H, g, dev, seed=3, own_kernel=own)
        out = torch.empty_like(x)
        dx = torch.empty_like(x)
        blk.forward(0, x, out, s)
        assert blk.last_path == ("own" if own else "library")
        blk.backward(0, dh, dx, accumulate=False)
        blk.forward(1, x, out, s)
        blk.backward(1, dh, dx, accumulate=True)   # weight grads: 2x
        torch.cuda.synchronize()
        res.append((out.float(), dx.float(), blk.dw_qkv.clone(), blk.dw_o.clone()))
    for a, r in zip(res[0], res[1]):
        assert (a - r).abs().max().item() / r.abs().max().item() < 1e-2


@pytest.mark.parametrize("b,s,nh,nkv", [(1, 256, 2, 1), (2, 256, 4, 2), (1, 512, 2, 2), (1, 1024, 8, 8), (2, 384, 8, 2), (1, 768, 6, 2)])
def test_attention_bwd_matches_fp32_autograd(b, s, nh, nkv):
    """Own tcgen05 backward (dm_attention_bwd) fed the own forward's (O, LSE): dQ, dK, dV
    against fp32 autograd of the reference attention, normwise 2e-2 per block (bf16 P and
    dS into the MMAs), and against cuDNN's SDPA backward on the same inputs."""
    from paper_2605_11005_b200 import kernels as K

    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(7 * b + s + nh)
    qkv = torch.randn(b * s, (nh + 2 * nkv) * D, generator=g).to(torch.bfloat16).to(dev)
    dout = torch.randn(b * s, nh * D, generator=g).to(torch.bfloat16).to(dev)
    out = torch.empty(b * s, nh * D, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(b, nh, s, dtype=torch.float32, device=dev)
    K.attention_fwd(qkv, s, nh, nkv, out, lse)
    dqkv = torch.empty_like(qkv)
    K.attention_bwd(qkv, out, dout, lse, s, nh, nkv, dqkv)
    torch.cuda.synchronize()
    x = qkv.float().requires_grad_(True)
    o_ref, _ = _reference(x, b, s, nh, nkv)
    (o_ref * dout.float()).sum().backward()
    ref = x.grad
    for lo, hi, name in ((0, nh, "dq"), (nh, nh + nkv, "dk"), (nh + nkv, nh + 2 * nkv, "dv")):
        got_b = dqkv[:, lo * D:hi * D].float()
        ref_b = ref[:, lo * D:hi * D]
        err = (got_b - ref_b).abs().max().item() / ref_b.abs().max().item()
        assert err < 2e-2, (name, err)
    # bit-determinism of the own backward
    dqkv2 = torch.empty_like(qkv)
    K.attention_bwd(qkv, out, dout, lse, s, nh, nkv, dqkv2)
    torch.cuda.synchronize()
    assert torch.equal(dqkv, dqkv2)
