"""Test-only torch restatement of the oracle's block step (oracle/swarm_oracle.py
block_step, itself pinned to model.py:314-380) for shapes too large for numpy.

It takes the int8 codes/scales read back from the span (whose bit-exactness is
checked separately against the oracle on smaller shapes) and runs the same
arithmetic in float64 on the GPU.
"""

from __future__ import annotations

import math

import torch


def layer_norm(x):
    mu = x.mean(-1, keepdim=True)
    var = x.var(-1, keepdim=True, unbiased=False)
    return (x - mu) / torch.sqrt(var + 1e-5)


def gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def alibi(H, device):
    return torch.tensor([2.0 ** (-8.0 * h / H) for h in range(1, H + 1)], dtype=torch.float64, device=device)


class RefBlock:
    """Dequantized int8 block (gammas 1, betas/biases 0 as in gen_checkpoint)."""

    def __init__(self, span, j, device="cuda"):
        self.w = []
        for m in range(4):
            codes, scales = span.read_codes(j, m)  # [out, in], [in]
            c = torch.from_numpy(codes).to(device=device, dtype=torch.float64)
            s = torch.from_numpy(scales).to(device=device, dtype=torch.float64)
            self.w.append((c * s[None, :]).T.contiguous())  # [in, out]
        self.H = span.config.n_heads
        self.d = span.config.hidden

    def step(self, x, kv, start, kv_fp16=False):
        """x [t, d] f64; kv = [k [T, H, dh], v] f64 lists (mutated). kv_fp16:
        round the cached K/V to fp16 as the span's paged cache stores them
        (isolates the kernels' arithmetic from the storage format)."""
        t, d = x.shape
        H, dh = self.H, d // self.H
        qkv = layer_norm(x) @ self.w[0]
        q = qkv[:, :d].reshape(t, H, dh)
        kn = qkv[:, d:2 * d].reshape(t, H, dh)
        vn = qkv[:, 2 * d:].reshape(t, H, dh)
        if kv_fp16:
            kn, vn = kn.half().double(), vn.half().double()
        kv[0] = torch.cat([kv[0], kn]) if kv[0] is not None else kn
        kv[1] = torch.cat([kv[1], vn]) if kv[1] is not None else vn
        K, V = kv
        T = K.shape[0]
        s = torch.einsum("ihd,jhd->hij", q, K) / math.sqrt(dh)
        qp = torch.arange(start, start + t, dtype=torch.float64, device=x.device)
        kp = torch.arange(T, dtype=torch.float64, device=x.device)
        rel = kp[None, :] - qp[:, None]
        s = s + alibi(H, x.device)[:, None, None] * rel[None]
        s = torch.where(rel[None] > 0, torch.tensor(float("-inf"), dtype=torch.float64, device=x.device), s)
        p = torch.softmax(s, dim=-1)
        ctx = torch.einsum("hij,jhd->ihd", p, V).reshape(t, d)
        mid = x + ctx @ self.w[1]
        act = gelu(layer_norm(mid) @ self.w[2])
        return mid + act @ self.w[3]
