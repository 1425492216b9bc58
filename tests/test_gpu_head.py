"""GPU parity of the client head: embedding lookup, final LN +
tied LM head, greedy next token (model.py:421-446), against the oracle and
the reference's golden generations.

Tolerances: embedding rows and greedy token ids bit-exact; logits <= 1e-5
relative (f64 accumulation vs the oracle's f32 numpy matmul)."""

import numpy as np
import pytest

import swarm_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = {
    "tiny": O.Shape(2, 8, 2, 32, 64),
    "small": O.Shape(4, 16, 2, 32, 128),
    "mid": O.Shape(3, 256, 4, 512, 256),
}


def cfg_of(shape):
    from paper_2209_01188_b200.model import ModelConfig

    return ModelConfig(shape.n_layers, shape.hidden, shape.n_heads, shape.vocab, shape.max_seq, shape.mlp_ratio)


def make_head(shape, **kw):
    from paper_2209_01188_b200.head import ClientHead

    head = ClientHead(cfg_of(shape), **kw)
    head.generate_weights(42)
    return head


@pytest.mark.parametrize("name", ["tiny", "small", "mid"])
def test_embed_rows_bit_exact(name):
    shape = SHAPES[name]
    head = make_head(shape)
    emb = O.make_embed(42, shape)
    toks = np.random.default_rng(1).integers(0, shape.vocab, 29)
    got = head.embed(toks).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), emb[toks].view(np.uint32))
    head.close()


def test_embed_rejects_out_of_range():
    from paper_2209_01188_b200.errors import InputError

    head = make_head(SHAPES["small"])
    with pytest.raises(InputError):
        head.embed([0, SHAPES["small"].vocab])
    with pytest.raises(InputError):
        head.embed([-1])
    head.close()


@pytest.mark.parametrize("name", ["small", "mid"])
def test_logits_match_oracle(name):
    import torch

    shape = SHAPES[name]
    head = make_head(shape)
    emb = O.make_embed(42, shape)
    h = np.random.default_rng(2).normal(size=(7, shape.hidden)).astype(np.float32)
    got = head.lm_head(torch.from_numpy(h)).cpu().numpy()
    want = O.final_logits(emb, h)
    err = np.max(np.abs(got.astype(np.float64) - want)) / np.max(np.abs(want))
    assert err <= 1e-5, err
    head.close()


@pytest.mark.parametrize("name", ["tiny", "small", "mid"])
def test_greedy_matches_oracle_argmax(name):
    import torch

    shape = SHAPES[name]
    head = make_head(shape)
    emb = O.make_embed(42, shape)
    rng = np.random.default_rng(3)
    for t in (1, 5, 32):
        h = rng.normal(size=(t, shape.hidden)).astype(np.float32) * rng.uniform(0.1, 10)
        got = head.greedy(torch.from_numpy(h))
        hn = O.layer_norm(h, np.ones(shape.hidden, np.float32), np.zeros(shape.hidden, np.float32))
        exact = hn.astype(np.float64) @ emb.T.astype(np.float64)
        assert got == [int(np.argmax(r)) for r in exact]
    head.close()


def test_greedy_tie_and_overflow_path():
    """A constant hidden row normalizes to beta = 0: every logit is 0, more
    than HEAD_CAP candidates qualify, every row is rescored, index 0 wins
    (numpy argmax's lowest-index rule, model.py:445)."""
    import torch

    from paper_2209_01188_b200.model import ModelConfig

    cfg = ModelConfig(1, 64, 2, 40000, 64)
    from paper_2209_01188_b200.head import ClientHead

    head = ClientHead(cfg)
    head.generate_weights(42)
    assert head.greedy(torch.full((2, 64), 3.0)) == [0, 0]
    head.close()


def test_greedy_nonfinite_raises():
    import torch

    from paper_2209_01188_b200.errors import InputError

    head = make_head(SHAPES["small"])
    h = torch.zeros(1, 16)
    h[0, 3] = float("nan")
    with pytest.raises(InputError):
        head.greedy(h)
    head.close()


def test_greedy_bloom_vocab_matches_exact_logits():
    """BLOOM vocabulary (250880) at h=1024: the int8 candidate pass picks the
    argmax of the head's own exact (f64-accumulated) logits."""
    import torch

    from paper_2209_01188_b200.head import ClientHead
    from paper_2209_01188_b200.model import SHAPES as S

    head = ClientHead(S["bloom-560m"])
    head.generate_weights(42)
    h = torch.randn(8, 1024, generator=torch.Generator().manual_seed(5))
    exact = head.lm_head(h).cpu().numpy()
    assert head.greedy(h) == [int(np.argmax(r)) for r in exact]
    head.close()


@pytest.mark.parametrize("name", ["tiny", "small", "mid"])
def test_generate_on_gpu_matches_golden(golden, name):
    """SwarmClient.generate with the head and two block spans on the GPU:
    token ids equal the reference's int8-weights generation."""
    from paper_2209_01188_b200.head import generate
    from paper_2209_01188_b200.span import BlockSpan

    g = golden("blocks")
    shape = SHAPES[name]
    cfg = cfg_of(shape)
    cut = shape.n_layers // 2
    spans = [BlockSpan(cfg, 0, cut, page_tokens=16), BlockSpan(cfg, cut, shape.n_layers, page_tokens=16)]
    for s in spans:
        s.generate_weights(42)
    head = make_head(shape)
    assert generate(spans, head, [1, 2, 3], 16) == g[f"{name}_gen_qw"].tolist()
    for s in spans:
        s.close()
    head.close()
