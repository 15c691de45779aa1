"""TEST-ONLY fp32 torch reference of one MoE layer fwd + bwd on the device, for the
BASELINE-size parity checks where the numpy fp64 oracle (oracle/oracle.py) would take
minutes. Routing is taken as given (`idx`, checked bit-exact against the C oracle
separately); everything downstream of it — gate softmax over the selected logits,
SwiGLU experts, weighted combine and every gradient (dx incl. the router term, dW_g,
dW1/dW3, dW2) — is recomputed in fp32 from the bf16 inputs and weights with TF32 off,
expert by expert, and compared with the kernels' results on the fly (normwise relative
error max|got - ref| / max|ref| over the whole tensor), so no full fp32 copy of the
weights or weight gradients is ever materialised (DeepSeek-V3: 45 GB each)."""

from __future__ import annotations

import torch

GLU_BLOCK = 64   # DM_GLU_BLOCK: gate/up row interleave of W13 / dW13


def _split13(w13e: torch.Tensor):
    two_de, h = w13e.shape
    v = w13e.view(two_de // (2 * GLU_BLOCK), 2, GLU_BLOCK, h)
    return v[:, 0].reshape(two_de // 2, h), v[:, 1].reshape(two_de // 2, h)


class _Err:
    def __init__(self):
        self.diff, self.ref = 0.0, 0.0

    def add(self, got: torch.Tensor, ref: torch.Tensor):
        self.diff = max(self.diff, (got.float() - ref).abs().max().item() if ref.numel() else 0.0)
        self.ref = max(self.ref, ref.abs().max().item() if ref.numel() else 0.0)

    @property
    def value(self) -> float:
        return self.diff / self.ref if self.ref > 0 else self.diff


@torch.no_grad()
def layer_errors(x, wg, w13, w2, idx, dy, y, dx, dwg, dw13, dw2) -> dict[str, float]:
    """x, dy, y, dx: [T, H] bf16 (device); wg / dwg fp32 [E, H]; w13 / dw13 [E, 2De, H]
    (bf16 / fp32, DM_GLU_BLOCK-interleaved); w2 / dw2 [E, H, De]; idx int32 [T, k]."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        T, H = x.shape
        E = wg.shape[0]
        xf = x.float()
        dyf = dy.float()
        logits = xf @ wg.t()                                   # [T, E]
        sel = logits.gather(1, idx.long())                     # [T, k]
        gate = torch.softmax(sel, dim=1)                       # [T, k]
        yref = torch.zeros(T, H, device=x.device)
        dxref = torch.zeros(T, H, device=x.device)
        dgate = torch.zeros_like(gate)                         # d loss / d gate[t, j] = <dy[t], o_tj>
        errs = {n: _Err() for n in ("dw1", "dw3", "dw2")}
        flat = idx.long().view(-1)
        order = torch.argsort(flat, stable=True)
        counts = torch.bincount(flat, minlength=E).tolist()
        start = 0
        for e in range(E):
            n = counts[e]
            slots = order[start:start + n]
            start += n
            w1e, w3e = (m.float() for m in _split13(w13[e]))
            w2e = w2[e].float()
            g1e, g3e = _split13(dw13[e])
            if n == 0:
                errs["dw1"].add(g1e, torch.zeros_like(g1e, dtype=torch.float32))
                errs["dw3"].add(g3e, torch.zeros_like(g3e, dtype=torch.float32))
                errs["dw2"].add(dw2[e], torch.zeros_like(dw2[e], dtype=torch.float32))
                continue
            t = slots // idx.shape[1]
            j = slots % idx.shape[1]
            xe = xf[t]
            g = xe @ w1e.t()
            u = xe @ w3e.t()
            sg = torch.sigmoid(g)
            a = g * sg * u
            o = a @ w2e.t()                                    # expert outputs [n, H]
            ge = gate[t, j].unsqueeze(1)
            yref.index_add_(0, t, ge * o)
            dgate[t, j] = (dyf[t] * o).sum(1)
            do = ge * dyf[t]
            errs["dw2"].add(dw2[e], do.t() @ a)
            da = do @ w2e
            dgg = da * u * sg * (1 + g * (1 - sg))
            du = da * g * sg
            errs["dw1"].add(g1e, dgg.t() @ xe)
            errs["dw3"].add(g3e, du.t() @ xe)
            dxref.index_add_(0, t, dgg @ w1e + du @ w3e)
        # softmax over the selected logits: dsel = gate * (dgate - <gate, dgate>)
        dsel = gate * (dgate - (gate * dgate).sum(1, keepdim=True))
        dlogits = torch.zeros(T, E, device=x.device).scatter_(1, idx.long(), dsel)
        dxref += dlogits @ wg
        dwgref = dlogits.t() @ xf
        out = {k: v.value for k, v in errs.items()}
        for name, got, ref in (("y", y, yref), ("dx", dx, dxref), ("dwg", dwg, dwgref)):
            e = _Err()
            e.add(got, ref)
            out[name] = e.value
        return out
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
