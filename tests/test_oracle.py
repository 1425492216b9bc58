"""Pin the CPU oracle against the reference's golden vectors (no GPU).

The fixtures in tests/golden were produced by running the reference itself
(tests/golden/make_golden.py); the known-answer constants below are the
reference's own test vectors (tests/test_model.py:38,72-88 and
tests/test_quant.py:27-70 in /root/reference/pkg).
"""

import numpy as np
import pytest

import swarm_oracle as O


def test_splitmix_known_answers(golden):
    w = O.splitmix_words(0, 3)
    assert [int(v) for v in w] == [0x21EC192A9FB89B01, 0x5193D2334EDC103D, 0x30A9E36EB8C43980]
    g = golden("weights")
    assert np.array_equal(O.splitmix_words(0, 8), g["sm64_state0"])


def test_fnv_known_answers(golden):
    assert O.fnv1a_64(b"") == 0xCBF29CE484222325
    assert O.fnv1a_64(b"a") == 0xAF63DC4C8601EC8C
    g = golden("weights")
    for p, h in zip(g["paths"], g["fnv_paths"]):
        assert O.fnv1a_64(str(p).encode()) == int(h)


def test_frozen_embed_weights():
    # tests/test_model.py:38 (seed 42, first four embed weights)
    frozen = [-0.012020314112305641, -0.03984982892870903, -0.01412433385848999, 0.006638171151280403]
    assert O.named_tensor(42, "embed", 4).tolist() == pytest.approx(frozen, abs=0.0)


def test_tensor_streams_bit_exact(golden):
    g = golden("weights")
    for seed in (42, 7):
        for i, p in enumerate(g["paths"]):
            want = g[f"stream_{seed}_{i}"]
            got = O.named_tensor(seed, str(p), want.size)
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
            # offset access (counter form) agrees with the prefix
            assert np.array_equal(O.named_tensor(seed, str(p), 100, first=1000), want[1000:1100])


def _codec_cases(g):
    xo, so = g["x_off"], g["s_off"]
    for i, b in enumerate(g["block"]):
        yield (g["x"][xo[i]:xo[i + 1]], int(b), g["scales"][so[i]:so[i + 1]],
               g["codes"][xo[i]:xo[i + 1]], g["deq"][xo[i]:xo[i + 1]])


def test_wire_codec_bit_exact(golden):
    g = golden("codec")
    n = 0
    for x, b, scales, codes, deq in _codec_cases(g):
        s, c = O.wire_quantize(x, b)
        assert np.array_equal(s.view(np.uint32), scales.view(np.uint32))
        assert np.array_equal(c, codes)
        d = O.wire_dequantize(s, c, b)
        assert np.array_equal(d.view(np.uint32), deq.view(np.uint32))
        n += 1
    assert n >= 39


def test_wire_codec_known_answers():
    s, c = O.wire_quantize(np.array([1.0, -2.0, 0.5, 4.0], np.float32), 4)
    assert c.tolist() == [32, -64, 16, 127]
    assert s[0] == np.float32(4.0) / np.float32(127.0)
    s, c = O.wire_quantize(np.zeros(8, np.float32), 4)
    assert not s.any() and not c.any()


def test_wire_codec_fixed_point():
    rng = np.random.default_rng(0)
    x = rng.normal(size=300).astype(np.float32)
    once = O.wire_dequantize(*O.wire_quantize(x))
    twice = O.wire_dequantize(*O.wire_quantize(once))
    assert np.array_equal(once, twice)


def test_weight_quantizer_bit_exact(golden):
    g = golden("weights")
    for j in range(int(g["n_mats"][0])):
        wq = O.Int8Matrix(g[f"wq{j}_w"])
        assert np.array_equal(wq.codes, g[f"wq{j}_codes"])
        assert np.array_equal(wq.scales.view(np.uint32), g[f"wq{j}_scales"].view(np.uint32))
        assert np.array_equal(wq.outlier_idx, g[f"wq{j}_outl"])
        assert np.array_equal(wq.outlier_rows.T, g[f"wq{j}_outl_data"])
        got = wq.apply(g[f"wq{j}_x"].T).T
        want = g[f"wq{j}_mm"]
        assert np.max(np.abs(got - want)) <= 1e-5 * max(1.0, np.abs(want).max())


SHAPES = {
    "tiny": O.Shape(2, 8, 2, 32, 64),
    "small": O.Shape(4, 16, 2, 32, 128),
    "mid": O.Shape(3, 256, 4, 512, 256),
}


@pytest.mark.parametrize("name", ["tiny", "small", "mid"])
def test_block_forward_matches_reference(golden, name):
    g = golden("blocks")
    shape = SHAPES[name]
    blocks = [O.make_block(42, shape, i) for i in range(shape.n_layers)]
    emb = O.make_embed(42, shape)
    x = emb[g[f"{name}_tokens"]]
    f32 = O.forward_span(blocks, x, shape, quantized=False)
    qw = O.forward_span(blocks, x, shape, quantized=True)
    tol = 1e-5 * max(1.0, float(np.abs(g[f"{name}_fwd_f32"]).max()))
    assert np.max(np.abs(f32 - g[f"{name}_fwd_f32"])) <= tol
    assert np.max(np.abs(qw - g[f"{name}_fwd_qw"])) <= tol
    # incremental (prefill 5 + 4 single steps) through block 0, int8 path
    kv = O.KV(shape)
    qb = O.QuantBlock(blocks[0])
    outs = [O.block_step(blocks[0], x[:5], kv, 0, shape, qb)]
    for i in range(5, 9):
        outs.append(O.block_step(blocks[0], x[i:i + 1], kv, i, shape, qb))
    assert np.max(np.abs(np.concatenate(outs) - g[f"{name}_blk0_inc_qw"])) <= tol


@pytest.mark.parametrize("name", ["tiny", "small", "mid"])
def test_generate_tokens_match_reference(golden, name):
    g = golden("blocks")
    shape = SHAPES[name]
    assert O.generate(42, shape, [1, 2, 3], 16, quantized=False) == g[f"{name}_gen_f32"].tolist()
    assert O.generate(42, shape, [1, 2, 3], 16, quantized=True) == g[f"{name}_gen_qw"].tolist()


def test_oracle_backward_matches_reference_golden(golden):
    """oracle.block_backward (recompute from the tape) == the reference's
    FORWARD/BACKWARD (server.py:411-450) on the same rows (f32; tolerance for
    numpy summation order only)."""
    g = golden("train")
    for name, shape in (("tiny", O.Shape(2, 8, 2, 32, 64)), ("small", O.Shape(4, 16, 2, 32, 128)),
                        ("mid", O.Shape(3, 256, 4, 512, 256))):
        blocks = [O.make_block(42, shape, i) for i in range(shape.n_layers)]
        for r in range(g[f"{name}_batch"].shape[0]):
            h, tapes = g[f"{name}_batch"][r], []
            for blk in blocks:
                tapes.append(h)
                h = O.block_step(blk, h, O.KV(shape), 0, shape)
            np.testing.assert_allclose(h, g[f"{name}_fwd"][r], rtol=1e-5, atol=1e-5)
            gr = g[f"{name}_grad"][r]
            for blk, x in zip(reversed(blocks), reversed(tapes)):
                gr = O.block_backward(blk, x, gr, shape)
            want = g[f"{name}_grad_in"][r]
            assert np.max(np.abs(gr - want)) <= 1e-5 * max(np.max(np.abs(want)), 1.0), name
