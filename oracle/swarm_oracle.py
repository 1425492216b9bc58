"""CPU oracle for the block-span server hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference's (swarmlm) arithmetic for
the path this repository accelerates. It exists so that `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs have a checker that travels to the GPU box (where /root/reference does not
exist). The product (`paper_2209_01188_b200`) never imports it.

Pinning: every function here is checked in `tests/test_oracle.py` against
golden vectors produced by the reference itself (`tests/golden/make_golden.py`
imports /root/reference/pkg/src and writes `tests/golden/*.npz`), plus the
reference's own known-answer tests (SplitMix64 / FNV-1a words, frozen embed
weights, codec examples). Parity is therefore pinned to the reference, not to
this restatement.

Citations are to /root/reference/pkg/src/swarmlm/<file>:<line>.
"""

from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15  # model.py:21
MIX_A = 0xBF58476D1E4B21D5  # model.py:22
MIX_B = 0x94D049BB133111EB  # model.py:23
FNV_OFFSET = 0xCBF29CE484222325  # model.py:48
FNV_PRIME = 0x100000001B3  # model.py:50
EPS_LN = 1e-5  # model.py:19
OUTLIER_THRESHOLD = 6.0  # quant.py:14
WIRE_BLOCK = 64  # quant.py:13


# ---------------------------------------------------------------- weight streams


def fnv1a_64(data: bytes) -> int:
    """FNV-1a over bytes (model.py:47-51)."""
    acc = FNV_OFFSET
    for byte in data:
        acc = ((acc ^ byte) * FNV_PRIME) & MASK64
    return acc


def splitmix_words(key: int, count: int, first: int = 1) -> np.ndarray:
    """Counter-form SplitMix64: word i (i = first..first+count-1) of the stream
    keyed by `key` is mix(key + i*gamma) (model.py:36-44)."""
    ctr = np.arange(first, first + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s = np.uint64(key & MASK64) + ctr * np.uint64(GOLDEN_GAMMA)
        s = (s ^ (s >> np.uint64(30))) * np.uint64(MIX_A)
        s = (s ^ (s >> np.uint64(27))) * np.uint64(MIX_B)
        return s ^ (s >> np.uint64(31))


def words_to_weights(words: np.ndarray) -> np.ndarray:
    """u64 -> f32 in [-0.05, 0.05): top 53 bits as an f64 fraction, centred and
    scaled in f64, then rounded once to f32 (model.py:54-57)."""
    frac = (words >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return ((frac - 0.5) * 0.1).astype(np.float32)


def stream_key(seed: int, path: str) -> int:
    return (seed ^ fnv1a_64(path.encode())) & MASK64


def named_tensor(seed: int, path: str, count: int, first: int = 0) -> np.ndarray:
    """Elements [first, first+count) of the named tensor's stream (model.py:60-62)."""
    return words_to_weights(splitmix_words(stream_key(seed, path), count, first + 1))


def block_matrix(seed: int, block: int, name: str, rows: int, cols: int) -> np.ndarray:
    """Row-major [rows, cols] matrix `blocks.{block}.{name}` (model.py:180-181,191-199)."""
    return named_tensor(seed, f"blocks.{block}.{name}", rows * cols).reshape(rows, cols)


class Shape:
    """ModelConfig restatement (model.py:65-84)."""

    def __init__(self, n_layers, hidden, n_heads, vocab, max_seq, mlp_ratio=4):
        assert hidden % n_heads == 0
        self.n_layers, self.hidden, self.n_heads = n_layers, hidden, n_heads
        self.vocab, self.max_seq, self.mlp_ratio = vocab, max_seq, mlp_ratio

    @property
    def head_dim(self):
        return self.hidden // self.n_heads


class Block:
    """One block's f32 tensors in the reference layout (model.py:87-100):
    matrices are [in, out]; gammas 1, betas and biases 0 (model.py:188-201)."""

    def __init__(self, wqkv, wo, wmlp_in, wmlp_out, d, r):
        self.ln1_g = np.ones(d, np.float32)
        self.ln1_b = np.zeros(d, np.float32)
        self.ln2_g = np.ones(d, np.float32)
        self.ln2_b = np.zeros(d, np.float32)
        self.wqkv, self.wo, self.wmlp_in, self.wmlp_out = wqkv, wo, wmlp_in, wmlp_out
        self.bqkv = np.zeros(3 * d, np.float32)
        self.bo = np.zeros(d, np.float32)
        self.bmlp_in = np.zeros(r * d, np.float32)
        self.bmlp_out = np.zeros(d, np.float32)


def make_block(seed: int, shape: Shape, i: int) -> Block:
    d, r = shape.hidden, shape.mlp_ratio
    return Block(
        block_matrix(seed, i, "wqkv", d, 3 * d),
        block_matrix(seed, i, "wo", d, d),
        block_matrix(seed, i, "wmlp_in", d, r * d),
        block_matrix(seed, i, "wmlp_out", r * d, d),
        d,
        r,
    )


def make_embed(seed: int, shape: Shape) -> np.ndarray:
    return named_tensor(seed, "embed", shape.vocab * shape.hidden).reshape(shape.vocab, shape.hidden)


# ------------------------------------------------------------------- int8 codecs


def round_away(v: np.ndarray) -> np.ndarray:
    """Round half away from zero (quant.py:29-30)."""
    return np.copysign(np.floor(np.abs(v) + 0.5), v)


def wire_quantize(x: np.ndarray, block: int = WIRE_BLOCK):
    """Blockwise absmax int8 of the flattened tensor (quant.py:33-54).

    scale_b = f32(absmax_b / 127) (f32 division); code = clip(round_away(
    f64(x) / f64(scale_b)), -127, 127); all-zero blocks keep scale 0, codes 0.
    Vectorised over blocks (the reference loops), same arithmetic."""
    flat = np.asarray(x, np.float32).reshape(-1)
    n = flat.size
    if n == 0:
        return np.zeros(0, np.float32), np.zeros(0, np.int8)
    nb = -(-n // block)
    padded = np.zeros(nb * block, np.float32)
    padded[:n] = flat
    tiles = padded.reshape(nb, block)
    amax = np.abs(tiles).max(axis=1)
    scales = (amax / np.float32(127.0)).astype(np.float32)
    safe = np.where(scales > 0, scales, np.float32(1.0)).astype(np.float64)
    q = round_away(tiles.astype(np.float64) / safe[:, None])
    q = np.clip(q, -127, 127)
    # absmax > 0 whose f32 scale underflowed to 0: the reference divides by
    # 0.0, so x != 0 -> +-inf -> clip +-127 and 0/0 -> NaN -> int8 0
    # (quant.py:48-53). All-zero blocks are skipped (codes 0).
    under = (scales == 0) & (amax > 0)
    q[scales == 0] = 0
    q[under] = np.sign(tiles[under]) * 127
    return scales, q.astype(np.int8).reshape(-1)[:n]


def wire_dequantize(scales: np.ndarray, codes: np.ndarray, block: int = WIRE_BLOCK) -> np.ndarray:
    """code * scale in f32 (quant.py:57-66)."""
    n = codes.size
    per = np.repeat(np.asarray(scales, np.float32), block)[:n]
    return (codes.astype(np.float32) * per).astype(np.float32)


class Int8Matrix:
    """Per-input-feature int8 restatement of quantize_weights_int8(W.T)
    (quant.py:81-108 applied as in quant.py:142-149).

    W is the reference's [in, out] matrix. Feature k (row k of W) is an outlier
    iff max_o |W[k, o]| > threshold; outlier features keep f32 rows.
    codes: [out, in] int8 (zero on outlier features); scales: [in] f32."""

    def __init__(self, w: np.ndarray, threshold: float = OUTLIER_THRESHOLD):
        w = np.asarray(w, np.float32)
        amax = np.abs(w).max(axis=1) if w.size else np.zeros(w.shape[0], np.float32)
        self.outlier = amax > np.float32(threshold)
        self.scales = np.where(self.outlier, np.float32(0.0), amax / np.float32(127.0)).astype(np.float32)
        safe = np.where(self.scales > 0, self.scales, np.float32(1.0)).astype(np.float64)
        q = np.clip(round_away(w.astype(np.float64) / safe[:, None]), -127, 127)
        q[self.scales == 0, :] = 0
        self.codes = np.ascontiguousarray(q.astype(np.int8).T)  # [out, in]
        self.outlier_idx = np.flatnonzero(self.outlier)
        self.outlier_rows = w[self.outlier_idx, :].copy()  # [n_outl, out]
        self.shape_in_out = w.shape

    def dense(self) -> np.ndarray:
        """The [in, out] f32 matrix the int8 path multiplies by: codes x scales,
        outlier features' rows exact."""
        w = (self.codes.astype(np.float32) * self.scales[None, :]).T.copy()
        if self.outlier_idx.size:
            w[self.outlier_idx, :] = self.outlier_rows
        return w.astype(np.float32)

    def apply(self, x: np.ndarray) -> np.ndarray:
        """x [t, in] -> x @ W via dequantised regular part + f32 outlier rows
        (quant.py:117-129; model.py:305-311)."""
        x = np.asarray(x, np.float32)
        deq = self.codes.astype(np.float32) * self.scales[None, :]  # [out, in]
        y = (deq @ x.T).T
        if self.outlier_idx.size:
            y = y + x[:, self.outlier_idx] @ self.outlier_rows
        return y.astype(np.float32)


class QuantBlock:
    def __init__(self, blk: Block, threshold: float = OUTLIER_THRESHOLD):
        self.wqkv = Int8Matrix(blk.wqkv, threshold)
        self.wo = Int8Matrix(blk.wo, threshold)
        self.wmlp_in = Int8Matrix(blk.wmlp_in, threshold)
        self.wmlp_out = Int8Matrix(blk.wmlp_out, threshold)


# ---------------------------------------------------------------- block forward


def layer_norm(x, g, b):
    """Population-variance LayerNorm, eps 1e-5 (model.py:271-276)."""
    mu = x.mean(-1, keepdims=True)
    var = x.var(-1, keepdims=True)
    return (g * ((x - mu) * (1.0 / np.sqrt(var + EPS_LN))) + b).astype(np.float32)


def gelu_tanh(x):
    """tanh-form GELU (model.py:286-292)."""
    c = math.sqrt(2.0 / math.pi)
    return (0.5 * x * (1.0 + np.tanh(c * (x + 0.044715 * x ** 3)))).astype(np.float32)


def alibi(n_heads: int) -> np.ndarray:
    """slope_h = 2^(-8h/H), h = 1..H, for any H (model.py:301-302)."""
    return np.array([2.0 ** (-8.0 * h / n_heads) for h in range(1, n_heads + 1)], np.float32)


class KV:
    """Growing f32 cache [T, H, dh] (model.py:137-151)."""

    def __init__(self, shape: Shape):
        z = np.zeros((0, shape.n_heads, shape.head_dim), np.float32)
        self.k, self.v = z, z.copy()

    @property
    def length(self):
        return self.k.shape[0]


def block_step(blk: Block, x: np.ndarray, kv: KV, start: int, shape: Shape, qblk: QuantBlock | None = None,
               kv_round=None) -> np.ndarray:
    """One pre-LN ALiBi block over t new positions; mutates `kv`
    (model.py:314-380). `qblk` routes the four matmuls through the int8 path
    (model.py:341,362,366,368). `kv_round` (optional callable) models a
    reduced-precision cache for margin studies; None = reference f32."""
    t, d = x.shape
    assert d == shape.hidden and start == kv.length and start + t <= shape.max_seq
    H, dh = shape.n_heads, shape.head_dim
    x = x.astype(np.float32)

    def mm(a, w, qw):
        return qw.apply(a) if qw is not None else a @ w

    h1 = layer_norm(x, blk.ln1_g, blk.ln1_b)
    qkv = mm(h1, blk.wqkv, qblk and qblk.wqkv) + blk.bqkv
    q = qkv[:, :d].reshape(t, H, dh)
    kn = qkv[:, d:2 * d].reshape(t, H, dh)
    vn = qkv[:, 2 * d:].reshape(t, H, dh)
    if kv_round is not None:
        kn, vn = kv_round(kn), kv_round(vn)
    kv.k = np.concatenate([kv.k, kn], 0)
    kv.v = np.concatenate([kv.v, vn], 0)
    T = kv.length
    s = np.einsum("ihd,jhd->hij", q, kv.k).astype(np.float32) / np.float32(math.sqrt(dh))
    qpos = np.arange(start, start + t, dtype=np.float32)
    kpos = np.arange(T, dtype=np.float32)
    rel = kpos[None, :] - qpos[:, None]
    s = s + alibi(H)[:, None, None] * rel[None]
    s = np.where(rel[None] > 0, np.float32(-np.inf), s)
    s = s - s.max(-1, keepdims=True)
    e = np.exp(s, dtype=np.float32)
    p = e / e.sum(-1, keepdims=True)
    ctx = np.einsum("hij,jhd->ihd", p, kv.v).astype(np.float32).reshape(t, d)
    mid = x + (mm(ctx, blk.wo, qblk and qblk.wo) + blk.bo)
    h2 = layer_norm(mid, blk.ln2_g, blk.ln2_b)
    act = gelu_tanh(mm(h2, blk.wmlp_in, qblk and qblk.wmlp_in) + blk.bmlp_in)
    return (mid + mm(act, blk.wmlp_out, qblk and qblk.wmlp_out) + blk.bmlp_out).astype(np.float32)


def final_logits(embed: np.ndarray, h: np.ndarray) -> np.ndarray:
    """Final LN (gamma 1, beta 0) then tied head h @ embed^T (model.py:428-433)."""
    d = h.shape[-1]
    hn = layer_norm(h, np.ones(d, np.float32), np.zeros(d, np.float32))
    return (hn @ embed.T).astype(np.float32)


def greedy(row: np.ndarray) -> int:
    """argmax with lowest-index tie-break (model.py:445-446)."""
    return int(np.argmax(row))


def generate(seed: int, shape: Shape, prompt, n_new: int, quantized: bool, blocks=None, embed=None,
             kv_round=None, return_margins: bool = False):
    """Single-process incremental greedy generation (model.py:472-489); with
    quantized=True every block uses the int8 path (the reference's
    quantize='weights' server semantics, server.py:108-112,383-385)."""
    blocks = blocks if blocks is not None else [make_block(seed, shape, i) for i in range(shape.n_layers)]
    qblocks = [QuantBlock(b) for b in blocks] if quantized else [None] * len(blocks)
    embed = embed if embed is not None else make_embed(seed, shape)
    caches = [KV(shape) for _ in blocks]
    pending, pos, out, margins = list(prompt), 0, [], []
    for _ in range(n_new):
        h = embed[np.asarray(pending)].astype(np.float32)
        for i, blk in enumerate(blocks):
            h = block_step(blk, h, caches[i], pos, shape, qblocks[i], kv_round)
        logits = final_logits(embed, h)[-1]
        nxt = greedy(logits)
        srt = np.sort(logits)
        margins.append(float((srt[-1] - srt[-2]) / max(np.abs(logits).max(), 1e-30)))
        pos += len(pending)
        pending = [nxt]
        out.append(nxt)
    return (out, margins) if return_margins else out


def forward_span(blocks, x: np.ndarray, shape: Shape, quantized: bool) -> np.ndarray:
    """One-shot cache-less forward over consecutive blocks (model.py:464-469)."""
    for blk in blocks:
        x = block_step(blk, x, KV(shape), 0, shape, QuantBlock(blk) if quantized else None)
    return x


# ------------------------------------------------------------------- training (FORWARD tape / BACKWARD)


def gelu_grad(x):
    """model.py:295-298."""
    c = np.float32(math.sqrt(2.0 / math.pi))
    a = np.float32(0.044715)
    t = np.tanh(c * (x + a * x ** 3))
    return (0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * c * (1.0 + 3.0 * a * x ** 2)).astype(np.float32)


def layer_norm_backward(dy, xhat, inv_std, g):
    """model.py:279-283."""
    dxhat = dy * g
    m1 = dxhat.mean(-1, keepdims=True)
    m2 = (dxhat * xhat).mean(-1, keepdims=True)
    return ((dxhat - m1 - xhat * m2) * inv_std).astype(np.float32)


def block_backward(blk: Block, x: np.ndarray, grad_out: np.ndarray, shape: Shape) -> np.ndarray:
    """Gradient of block_forward at empty cache / start 0 (the FORWARD row
    semantics, server.py:418-425) w.r.t. its input: the forward is recomputed
    from x (the tape) and model.py:383-418 is applied. f32 numpy like the
    reference."""
    t, d = x.shape
    H, dh = shape.n_heads, shape.head_dim
    x = x.astype(np.float32)

    def ln(v, g, b):
        mu = v.mean(-1, keepdims=True)
        var = v.var(-1, keepdims=True)
        inv = (1.0 / np.sqrt(var + EPS_LN)).astype(np.float32)
        xh = ((v - mu) * inv).astype(np.float32)
        return (g * xh + b).astype(np.float32), xh, inv

    h1, xh1, inv1 = ln(x, blk.ln1_g, blk.ln1_b)
    qkv = h1 @ blk.wqkv + blk.bqkv
    q = qkv[:, :d].reshape(t, H, dh)
    k = qkv[:, d:2 * d].reshape(t, H, dh)
    v = qkv[:, 2 * d:].reshape(t, H, dh)
    sc = np.einsum("ihd,jhd->hij", q, k).astype(np.float32) / np.float32(math.sqrt(dh))
    pos = np.arange(t, dtype=np.float32)
    rel = pos[None, :] - pos[:, None]
    sc = sc + alibi(H)[:, None, None] * rel[None]
    sc = np.where(rel[None] > 0, np.float32(-np.inf), sc)
    sc = sc - sc.max(-1, keepdims=True)
    e = np.exp(sc, dtype=np.float32)
    p = e / e.sum(-1, keepdims=True)
    ctx = np.einsum("hij,jhd->ihd", p, v).astype(np.float32).reshape(t, d)
    mid = x + (ctx @ blk.wo + blk.bo)
    h2, xh2, inv2 = ln(mid, blk.ln2_g, blk.ln2_b)
    pre = h2 @ blk.wmlp_in + blk.bmlp_in
    g = grad_out.astype(np.float32)
    dact = g @ blk.wmlp_out.T
    dpre = dact * gelu_grad(pre)
    dh2 = dpre @ blk.wmlp_in.T
    dmid = g + layer_norm_backward(dh2, xh2, inv2, blk.ln2_g)
    dctx = (dmid @ blk.wo.T).reshape(t, H, dh)
    dprobs = np.einsum("ihd,jhd->hij", dctx, v).astype(np.float32)
    dv = np.einsum("hij,ihd->jhd", p, dctx).astype(np.float32)
    row = (dprobs * p).sum(-1, keepdims=True)
    dsc = p * (dprobs - row)
    inv_sq = np.float32(1.0 / math.sqrt(dh))
    dq = np.einsum("hij,jhd->ihd", dsc, k).astype(np.float32) * inv_sq
    dk = np.einsum("hij,ihd->jhd", dsc, q).astype(np.float32) * inv_sq
    dqkv = np.concatenate([dq.reshape(t, d), dk.reshape(t, d), dv.reshape(t, d)], axis=1)
    dx = dmid + layer_norm_backward(dqkv @ blk.wqkv.T, xh1, inv1, blk.ln1_g)
    return dx.astype(np.float32)


def dequantized_block(blk: Block) -> Block:
    """The block a span with int8 weights computes with: codes x feature scales,
    outlier features kept exact (quant.py:117-129)."""
    out = Block(*(Int8Matrix(w).dense() for w in (blk.wqkv, blk.wo, blk.wmlp_in, blk.wmlp_out)),
                blk.wo.shape[0], blk.wmlp_in.shape[1] // blk.wmlp_in.shape[0])
    return out
