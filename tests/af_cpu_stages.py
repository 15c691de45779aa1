"""TEST-ONLY CPU restatement of the runtime's stage arithmetic, used to drive
paper_2605_11005_b200.runtime under gloo (world_size > 1 on CPU). It mirrors the
GPU buffer layouts (128-aligned expert blocks, interleaved h13, absolute wgrad
segments) with fp32 math and bf16 storage; routing comes from the oracle."""

from __future__ import annotations

import numpy as np
import torch

from oracle import oracle as O

BF16 = torch.bfloat16


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def _silu(g):
    return g / (1 + torch.exp(-g))


B = 64   # DM_GLU_BLOCK: gate/up column interleave of h13 / dh13


def _split(h: torch.Tensor):
    R, two = h.shape
    v = h.view(R, two // (2 * B), 2, B)
    return v[:, :, 0].reshape(R, two // 2), v[:, :, 1].reshape(R, two // 2)


def _join(g: torch.Tensor, u: torch.Tensor) -> torch.Tensor:
    R, De = g.shape
    out = torch.empty(R, 2 * De, dtype=g.dtype)
    v = out.view(R, De // B, 2, B)
    v[:, :, 0] = g.view(R, De // B, B)
    v[:, :, 1] = u.view(R, De // B, B)
    return out


class CpuStages:
    def a_dispatch(self, buf, router):
        s = buf.shape
        logits, idx, w = O.router(_bits(buf.x), router.wg.numpy(), s.k)
        counts, pad_off, row_map, src = O.dispatch(idx, s.E, cap=buf.cap)
        buf.idx.copy_(torch.from_numpy(idx))
        buf.w.copy_(torch.from_numpy(w))
        buf.counts.copy_(torch.from_numpy(counts))
        buf.pad_off.copy_(torch.from_numpy(pad_off))
        buf.row_map.copy_(torch.from_numpy(row_map))
        buf.src.copy_(torch.from_numpy(src))
        buf.x_perm.zero_()
        occ = torch.from_numpy(src >= 0)
        buf.x_perm[occ] = buf.x[torch.from_numpy(src[src >= 0]).long()]

    def a_combine(self, buf):
        rm = buf.row_map.long()
        yp = buf.y_perm.float()[rm]                       # [T, k, H]
        y = (yp * buf.w.unsqueeze(-1)).sum(1)
        if buf.residual:
            y = y + buf.x.float()
        buf.y.copy_(y.to(BF16))

    def a_combine_bwd(self, buf):
        rm = buf.row_map.long()
        yp = buf.y_perm.float()[rm]
        w = buf.w
        dy = buf.dy.float()
        dw = (yp * dy.unsqueeze(1)).sum(-1)
        buf.dw.copy_(dw)
        buf.dlogit.copy_(w * (dw - (w * dw).sum(1, keepdim=True)))
        buf.dy_perm.zero_()
        buf.dy_perm[rm.reshape(-1)] = (w.unsqueeze(-1) * dy.unsqueeze(1)).reshape(-1, dy.shape[1]).to(BF16)

    def a_backward(self, buf, router, accumulate):
        rm = buf.row_map.long()
        idx = buf.idx.long()
        dx = buf.dx_perm.float()[rm].sum(1) + torch.einsum("tk,tkh->th", buf.dlogit, router.wg[idx])
        if buf.residual:
            dx = dx + buf.dy.float()
        buf.dx.copy_(dx.to(BF16))
        g = torch.zeros_like(router.dwg)
        g.index_add_(0, idx.reshape(-1), (buf.dlogit.unsqueeze(-1) * buf.x.float().unsqueeze(1)).reshape(-1, g.shape[1]))
        if accumulate:
            router.dwg += g
        else:
            router.dwg.copy_(g)

    def _groups(self, group_off, E):
        go = group_off.tolist()
        return [(g % E, go[g], go[g + 1]) for g in range(len(go) - 1) if go[g + 1] > go[g]]

    def f_forward(self, fb, experts, group_off, ranges=None):
        E = experts.w13.shape[0]
        for e, a, b in self._groups(group_off, E):
            h = fb.x_perm[a:b].float() @ experts.w13[e].float().t()
            fb.h13[a:b] = h.to(BF16)
            g, u = _split(h)
            act = (_silu(g) * u)
            fb.act[a:b] = act.to(BF16)
            fb.y_perm[a:b] = (fb.act[a:b].float() @ experts.w2[e].float().t()).to(BF16)

    def f_backward(self, fb, experts, group_off, ranges=None):
        E = experts.w13.shape[0]
        for e, a, b in self._groups(group_off, E):
            d_act = fb.dy_perm[a:b].float() @ experts.w2[e].float()
            g, u = _split(fb.h13[a:b].float())
            sg = torch.sigmoid(g)
            dg = d_act * u * sg * (1 + g * (1 - sg))
            du = d_act * g * sg
            fb.dh13[a:b] = _join(dg, du).to(BF16)
            fb.dx_perm[a:b] = (fb.dh13[a:b].float() @ experts.w13[e].float()).to(BF16)

    def f_wgrad(self, slab, experts, seg_off, accumulate, seg_stride_rows=0):
        if not accumulate:
            experts.dw13.zero_()
            experts.dw2.zero_()
        so = seg_off.tolist()
        for i, row in enumerate(so):
            base = i * seg_stride_rows
            for e in range(len(row) - 1):
                a, b = base + row[e], base + row[e + 1]
                if b > a:
                    experts.dw2[e] += slab.dy_perm[a:b].float().t() @ slab.act[a:b].float()
                    experts.dw13[e] += slab.dh13[a:b].float().t() @ slab.x_perm[a:b].float()
