"""GPU parity of the training path: FORWARD with a tape of block
inputs and the exact BACKWARD of block_forward (model.py:383-418), against the
reference's FORWARD/BACKWARD golden fixtures (tests/golden/train.npz, f32
weights), the oracle's restatement with the int8 span's dequantized weights,
and a float64 torch autograd restatement at the 7B1 shape.

Tolerance: max-abs error relative to max |reference| <= 1e-3 (the FORWARD
itself carries the fp16 KV cache of the span; BACKWARD recomputes in f32)."""

import numpy as np
import pytest

import swarm_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-3

SHAPES = {
    "tiny": O.Shape(2, 8, 2, 32, 64),
    "small": O.Shape(4, 16, 2, 32, 128),
    "mid": O.Shape(3, 256, 4, 512, 256),
}


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def cfg_of(shape):
    from paper_2209_01188_b200.model import ModelConfig

    return ModelConfig(shape.n_layers, shape.hidden, shape.n_heads, shape.vocab, shape.max_seq, shape.mlp_ratio)


@pytest.mark.parametrize("name", ["tiny", "small", "mid"])
def test_f32_span_forward_backward_matches_reference(golden, name):
    import torch

    from paper_2209_01188_b200.span import BlockSpan

    g = golden("train")
    shape = SHAPES[name]
    span = BlockSpan(cfg_of(shape), 0, shape.n_layers, int8=False, page_tokens=16)
    span.load_weights([O.make_block(42, shape, i) for i in range(shape.n_layers)])
    batch = torch.from_numpy(g[f"{name}_batch"]).cuda()
    out, tape = span.forward(batch, tape=True)
    assert rel_err(out.cpu().numpy(), g[f"{name}_fwd"]) <= TOL
    # tape row 0 of block 0 is the input itself
    assert np.array_equal(tape[:, 0].cpu().numpy(), g[f"{name}_batch"])
    gin = span.backward(tape, torch.from_numpy(g[f"{name}_grad"]).cuda())
    assert rel_err(gin.cpu().numpy(), g[f"{name}_grad_in"]) <= TOL
    span.close()


@pytest.mark.parametrize("name", ["small", "mid"])
def test_int8_span_backward_matches_oracle(name):
    import torch

    from paper_2209_01188_b200.span import BlockSpan

    shape = SHAPES[name]
    span = BlockSpan(cfg_of(shape), 0, shape.n_layers, page_tokens=16)
    span.generate_weights(42)
    blocks = [O.dequantized_block(O.make_block(42, shape, i)) for i in range(shape.n_layers)]
    rng = np.random.default_rng(11)
    t = 9
    x = rng.normal(size=(2, t, shape.hidden)).astype(np.float32)
    gr = rng.uniform(-1, 1, (2, t, shape.hidden)).astype(np.float32)
    out, tape = span.forward(torch.from_numpy(x).cuda(), tape=True)
    gin = span.backward(tape, torch.from_numpy(gr).cuda()).cpu().numpy()
    for r in range(2):
        h, xs = x[r], []
        for blk in blocks:
            xs.append(h)
            h = O.block_step(blk, h, O.KV(shape), 0, shape)
        assert rel_err(out[r].cpu().numpy(), h) <= TOL
        want = gr[r]
        for blk, xin in zip(reversed(blocks), reversed(xs)):
            want = O.block_backward(blk, xin, want, shape)
        assert rel_err(gin[r], want) <= TOL, (name, r, rel_err(gin[r], want))
    span.close()


def test_backward_zero_grad_is_zero():
    """tests/test_server.py:224-236: a zero upstream gradient gives exactly zero."""
    import torch

    from paper_2209_01188_b200.span import BlockSpan

    shape = SHAPES["small"]
    span = BlockSpan(cfg_of(shape), 0, shape.n_layers, page_tokens=16)
    span.generate_weights(42)
    x = torch.randn(1, 5, shape.hidden, device="cuda")
    _, tape = span.forward(x, tape=True)
    gin = span.backward(tape, torch.zeros_like(x))
    assert bool((gin == 0).all())
    span.close()


@pytest.mark.parametrize("t", [48, 161])
def test_bloom7b1_block_backward_vs_f64_autograd(t):
    """One 7B1-shape block (h=4096, H=32), a 48-token row (one tcgen05
    token tile) and a 161-token row (three, the last one padded): the span's
    BACKWARD vs float64 torch autograd of the same dequantized block."""
    import torch

    from paper_2209_01188_b200.model import SHAPES as S
    from paper_2209_01188_b200.span import BlockSpan
    from torch_ref import RefBlock

    cfg = S["bloom-7b1"]
    span = BlockSpan(cfg, 0, 1, int8=True, page_tokens=64, max_tokens=64, n_pages=4)
    span.generate_weights(42)
    ref = RefBlock(span, 0)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(1, t, cfg.hidden, device="cuda", generator=g) * 0.05
    gr = torch.rand(1, t, cfg.hidden, device="cuda", generator=g) * 2 - 1
    _, tape = span.forward(x, tape=True)
    got = span.backward(tape, gr)[0].double()
    xd = x[0].double().requires_grad_(True)
    y = ref.step(xd, [None, None], 0)
    (y * gr[0].double()).sum().backward()
    want = xd.grad
    err = float((got - want).abs().max() / want.abs().max())
    assert err <= TOL, err
    span.close()
