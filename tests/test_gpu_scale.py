"""Parity at BASELINE's shapes (VERDICT r1 "parity at scale").

* Weight quantizer at the 7B1 / 176B shapes: for 64 sampled input features of
  every matrix, the codes, scales and outlier set generated on the device are
  bit-identical to the oracle's quantize_weights_int8 restatement
  (quant.py:81-108) applied to the same SplitMix64 rows
  (model.py:60-62 `tensor_stream` at offset k*out) -- with and without
  injected outlier features.
* tcgen05 prefill with outlier features (t >= 128) against the oracle.
* A 3-block 176B span: 240-token prefill (tcgen05) + 16 decode steps (GEMV)
  against a float64 restatement built from the span's codes.
* C3: 8 batched 7B1 sessions over two spans (f32 hop), against float64.
* The float64 restatement (tests/torch_ref.py) is itself pinned to the
  reference's mid-shape goldens.

Tolerance: hidden states max-abs error / max |reference| <= 1e-3 (north_star
allows 1e-2); codes / scales / outlier indices bit-exact.
"""

import numpy as np
import pytest

import swarm_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-3
NAMES = ("wqkv", "wo", "wmlp_in", "wmlp_out")


def _rel(a, b):
    return float((a - b).abs().max() / b.abs().max())


def _shape(cfg):
    return [(cfg.hidden, 3 * cfg.hidden), (cfg.hidden, cfg.hidden), (cfg.hidden, cfg.mlp_ratio * cfg.hidden),
            (cfg.mlp_ratio * cfg.hidden, cfg.hidden)]


@pytest.mark.parametrize("shape_name", ["bloom-7b1", "bloom-176b"])
@pytest.mark.parametrize("boost", [0.0, 200.0])
def test_large_shape_codes_sampled_bit_exact(shape_name, boost):
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[shape_name]
    block, every = 5, 97  # global block 5; with boost every 97th input feature is scaled (outlier)
    span = BlockSpan(cfg, block, block + 1, int8=True, page_tokens=64, max_tokens=64, n_pages=4)
    span.generate_weights(42, outlier_boost=boost, boost_every=every if boost else 0)
    rng = np.random.default_rng(17)
    for m, (K, M) in enumerate(_shape(cfg)):
        codes, scales = span.read_codes(0, m)  # [out, in], [in]
        feats = np.unique(np.concatenate([rng.choice(K, 56, replace=False), np.arange(0, K, every)[:8]]))
        rows = np.stack([O.named_tensor(42, f"blocks.{block}.{NAMES[m]}", M, first=int(k) * M) for k in feats])
        if boost:
            boosted = (feats % every) == 0
            rows[boosted] = (rows[boosted] * np.float32(boost)).astype(np.float32)
        want = O.Int8Matrix(rows)  # features = the sampled input features
        assert np.array_equal(scales[feats].view(np.uint32), want.scales.view(np.uint32)), (m, "scales")
        assert np.array_equal(codes[:, feats], want.codes), (m, "codes")
        outl = span.outliers(0, m)
        if boost:
            assert np.array_equal(np.intersect1d(outl, feats), feats[want.outlier]), (m, "outliers")
            assert np.array_equal(outl, np.arange(0, K, every)), (m, "all boosted features, and only those")
        else:
            assert outl.size == 0
    span.close()
    torch.cuda.empty_cache()


def test_tcgen05_prefill_with_outliers_matches_oracle():
    """Outlier features (x200, kept f32) on the tcgen05 path at t=200 (> the
    64-token threshold): the f32 outlier contribution is added in the GEMM
    epilogue. Oracle int8 path with the same fp16 K/V rounding."""
    import torch

    from paper_2209_01188_b200.model import ModelConfig
    from paper_2209_01188_b200.span import BlockSpan

    shape = O.Shape(3, 256, 4, 512, 256)
    rng = np.random.default_rng(8)
    blocks = [O.make_block(42, shape, i) for i in range(3)]
    for b in blocks:
        for w in (b.wqkv, b.wo, b.wmlp_in, b.wmlp_out):
            w[rng.choice(w.shape[0], 3, replace=False), :] *= np.float32(200.0)
    span = BlockSpan(ModelConfig(3, 256, 4, 512, 256), 0, 3, int8=True, page_tokens=16, max_tokens=256,
                     tc_min_tokens=64)
    span.load_weights(blocks)
    x = (rng.normal(size=(200, 256)) * 0.5).astype(np.float32)
    f16 = lambda a: a.astype(np.float16).astype(np.float32)  # noqa: E731
    want = x
    for b in blocks:
        want = O.block_step(b, want, O.KV(shape), 0, shape, O.QuantBlock(b), kv_round=f16)
    got = span.forward(torch.from_numpy(x).cuda()[None])[0].cpu().numpy()
    err = float(np.abs(got - want).max() / np.abs(want).max())
    assert err <= TOL, err
    span.close()


def test_torch_ref_pinned_to_reference_goldens(golden):
    """tests/torch_ref.py (the f64 checker for large shapes) reproduces the
    reference's own int8-weight forward of the mid shape (blocks.npz
    mid_fwd_qw, produced by swarmlm's block_forward(qw))."""
    import torch

    from paper_2209_01188_b200.model import ModelConfig
    from paper_2209_01188_b200.span import BlockSpan
    from torch_ref import RefBlock

    g = golden("blocks")
    shape = O.Shape(3, 256, 4, 512, 256)
    span = BlockSpan(ModelConfig(3, 256, 4, 512, 256), 0, 3, int8=True, page_tokens=16)
    span.generate_weights(42)
    x = torch.from_numpy(O.make_embed(42, shape)[g["mid_tokens"]]).cuda().double()
    for j in range(3):
        x = RefBlock(span, j).step(x, [None, None], 0)
    want = torch.from_numpy(g["mid_fwd_qw"]).cuda().double()
    assert _rel(x, want) <= 1e-5
    span.close()


def test_bloom176b_three_block_span_prefill_and_decode_vs_f64():
    """Three 176B-shape blocks: a 240-token prefill (three 80-token tcgen05
    tiles per matrix, the bench's prefill chunk) then 16 decode steps (IMMA
    GEMV + decode attention), every output against float64."""
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan
    from torch_ref import RefBlock

    cfg = SHAPES["bloom-176b"]
    span = BlockSpan(cfg, 0, 3, int8=True, page_tokens=64, max_tokens=240, n_pages=8)
    span.generate_weights(42)
    refs = [RefBlock(span, j) for j in range(3)]
    gen = torch.Generator(device="cuda").manual_seed(12)
    x = torch.randn(256, cfg.hidden, device="cuda", generator=gen) * 0.05
    seq = span.new_sequence()
    kvs = [[None, None] for _ in range(3)]
    kvs16 = [[None, None] for _ in range(3)]
    chunks = [(0, 240)] + [(240 + i, 241 + i) for i in range(16)]
    worst = worst16 = 0.0
    for a, b in chunks:
        got = span.step([(seq, x[a:b])])[0].double()
        want = want16 = x[a:b].double()
        for r, kv, kv16 in zip(refs, kvs, kvs16):
            want = r.step(want, kv, a)
            want16 = r.step(want16, kv16, a, kv_fp16=True)
        worst = max(worst, _rel(got, want))
        worst16 = max(worst16, _rel(got, want16))
        # kernels vs f64 with the cache's fp16 K/V: 1e-3; vs exact f64 (fp16 KV
        # rounding compounds over blocks): north_star's 1e-2
        assert worst16 <= TOL and worst <= 1e-2, (a, worst16, worst)
    del refs, kvs
    span.close()
    torch.cuda.empty_cache()


def test_c3_bloom7b1_eight_sessions_two_spans_vs_f64():
    """C3 in miniature: 8 sessions of the 7B1 shape with different prompt
    lengths, batched into one step per span, over two spans [0,2) + [2,4)
    with the f32 hidden handed over in HBM; prefill then 8 batched decode
    steps, every session's output against float64. A second pair of spans
    with the int8 wire hop equals the codec projection of the f32 hop
    exactly (quantize -> dequantize of span A's output fed to span B)."""
    import torch

    from paper_2209_01188_b200 import codec
    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan
    from torch_ref import RefBlock

    cfg = SHAPES["bloom-7b1"]
    spans = [BlockSpan(cfg, lo, hi, int8=True, page_tokens=64, max_tokens=256, max_seqs=8, n_pages=64)
             for lo, hi in ((0, 2), (2, 4))]
    for s in spans:
        s.generate_weights(42)
    refs = [RefBlock(s, j) for s in spans for j in range(2)]
    gen = torch.Generator(device="cuda").manual_seed(21)
    lens = [5, 9, 17, 3, 12, 30, 1, 8]
    prompts = [torch.randn(t, cfg.hidden, device="cuda", generator=gen) * 0.05 for t in lens]
    seqs = [[s.new_sequence() for _ in lens] for s in spans]
    kvs = [[[None, None] for _ in refs] for _ in lens]
    pos = [0] * len(lens)
    inputs = prompts
    for step in range(9):
        h = spans[0].step(list(zip(seqs[0], inputs)))
        h = spans[1].step(list(zip(seqs[1], h)))
        for i, (inp, got) in enumerate(zip(inputs, h)):
            want = inp.double()
            for r, kv in zip(refs, kvs[i]):
                want = r.step(want, kv, pos[i])
            assert _rel(got.double(), want) <= TOL, (step, i)
            pos[i] += inp.shape[0]
        inputs = [torch.randn(1, cfg.hidden, device="cuda", generator=gen) * 0.05 for _ in lens]
    # int8 hop == codec projection of the f32 hop, bit for bit
    a, b = spans
    sa, sb = a.new_sequence(), b.new_sequence()
    sa2, sb2 = a.new_sequence(), b.new_sequence()
    x = torch.randn(7, cfg.hidden, device="cuda", generator=gen) * 0.05
    n = x.numel()
    c8 = torch.empty(n, dtype=torch.int8, device="cuda")
    s8 = torch.empty(-(-n // 64), device="cuda")
    y_a = torch.empty_like(x)
    a.step_codes([sa], [7], in_f32=x, out_codes=c8, out_scales=s8, out_f32=y_a)
    hop = torch.empty_like(x)
    b.step_codes([sb], [7], in_codes=c8, in_scales=s8, out_f32=hop)
    ya2 = a.step([(sa2, x)])[0]
    proj = codec.dequantize_blockwise(codec.quantize_blockwise(ya2))
    ref = b.step([(sb2, proj.reshape(7, cfg.hidden))])[0]
    assert torch.equal(y_a, ya2)
    assert torch.equal(hop, ref)
    for s in spans:
        s.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shape_name,B", [("bloom-176b", 32), ("bloom-7b1", 16), ("bloom-7b1", 11)])
def test_batched_decode_tcgen05_stream_k_vs_f64(shape_name, B):
    """Batched decode through the stream-K tcgen05 kernel (k_gemm_tc_sk: one
    16- or 32-token tile, split row groups merged as exact s32 partials): B
    sessions with different contexts, prefill then 3 batched decode steps,
    every session against float64 (fp16-rounded K/V as the cache stores
    them)."""
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan
    from torch_ref import RefBlock

    cfg = SHAPES[shape_name]
    span = BlockSpan(cfg, 0, 2, int8=True, page_tokens=64, max_tokens=64, max_seqs=32, n_pages=2 * B + 4,
                     tc_min_tokens=8)
    span.generate_weights(42)
    refs = [RefBlock(span, j) for j in range(2)]
    gen = torch.Generator(device="cuda").manual_seed(31)
    lens = [1 + (i * 7) % 5 for i in range(B)]
    seqs = [span.new_sequence() for _ in range(B)]
    kvs = [[[None, None], [None, None]] for _ in range(B)]
    pos = [0] * B
    inputs = [torch.randn(t, cfg.hidden, device="cuda", generator=gen) * 0.05 for t in lens]
    for step in range(4):
        span.profile(True)
        outs = span.step(list(zip(seqs, inputs)))
        sk = span.profile_read(span.PROF_TC_DECODE)[1]
        span.profile(False)
        if step > 0:
            assert sk == 8, sk  # 4 matmuls x 2 blocks on the stream-K kernel
        for i in range(B):
            want = inputs[i].double()
            for r, kv in zip(refs, kvs[i]):
                want = r.step(want, kv, pos[i], kv_fp16=True)
            assert _rel(outs[i].double(), want) <= TOL, (step, i)
            pos[i] += inputs[i].shape[0]
        inputs = [torch.randn(1, cfg.hidden, device="cuda", generator=gen) * 0.05 for _ in range(B)]
    del refs
    span.close()
    torch.cuda.empty_cache()
