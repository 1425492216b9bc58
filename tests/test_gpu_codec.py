"""GPU parity of the wire codec and the deterministic weight generator
(bit-exact against the reference's golden vectors and the oracle)."""

import numpy as np
import pytest

import swarm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    return torch


def _cases(g):
    xo, so = g["x_off"], g["s_off"]
    for i, b in enumerate(g["block"]):
        yield (g["x"][xo[i]:xo[i + 1]], int(b), g["scales"][so[i]:so[i + 1]],
               g["codes"][xo[i]:xo[i + 1]], g["deq"][xo[i]:xo[i + 1]])


def test_codec_golden_bit_exact(torch_cuda, golden):
    from paper_2209_01188_b200 import codec

    g = golden("codec")
    for x, b, scales, codes, deq in _cases(g):
        q = codec.quantize_blockwise(torch_cuda.from_numpy(x.copy()).cuda(), b)
        assert np.array_equal(q.scales.cpu().numpy().view(np.uint32), scales.view(np.uint32)), (x.size, b)
        assert np.array_equal(q.codes.cpu().numpy(), codes), (x.size, b)
        d = codec.dequantize_blockwise(q).cpu().numpy().reshape(-1)
        assert np.array_equal(d.view(np.uint32), deq.view(np.uint32))


def test_codec_random_sweep_bit_exact(torch_cuda):
    """10^4 tensors' worth of blocks with per-block magnitudes from 1e-30 to 1e30,
    ties and near-ties, vs the oracle (itself pinned to the reference)."""
    from paper_2209_01188_b200 import codec

    rng = np.random.default_rng(11)
    nb = 10000 * 4
    mags = 10.0 ** rng.uniform(-30, 30, size=(nb, 1))
    x = (rng.normal(size=(nb, 64)) * mags).astype(np.float32)
    # plant exact ties k+1/2 of the block scale in a quarter of the blocks
    tb = rng.choice(nb, nb // 4, replace=False)
    amax = np.abs(x[tb]).max(axis=1)
    sc = (amax / np.float32(127)).astype(np.float32)
    k = rng.integers(-126, 126, size=(tb.size, 8))
    ties = ((k + 0.5) * sc[:, None].astype(np.float64)).astype(np.float32)
    x[tb, 0] = amax  # keep the block absmax (hence the scale) fixed
    x[tb[:, None], np.arange(1, 9)[None, :]] = np.where(np.abs(ties) <= amax[:, None], ties, 0)
    x = x.reshape(-1)
    x[-37:] = 0  # ragged tail handled below
    for n in (x.size, x.size - 13):
        xs = x[:n]
        s_ref, c_ref = O.wire_quantize(xs, 64)
        q = codec.quantize_blockwise(torch_cuda.from_numpy(xs.copy()).cuda(), 64)
        assert np.array_equal(q.scales.cpu().numpy().view(np.uint32), s_ref.view(np.uint32))
        assert np.array_equal(q.codes.cpu().numpy(), c_ref)


def test_codec_fixed_point_on_device(torch_cuda):
    from paper_2209_01188_b200 import codec

    x = torch_cuda.randn(1 << 20, device="cuda")
    once = codec.dequantize_blockwise(codec.quantize_blockwise(x))
    twice = codec.dequantize_blockwise(codec.quantize_blockwise(once))
    assert torch_cuda.equal(once, twice)


def test_codec_empty_and_errors(torch_cuda):
    from paper_2209_01188_b200 import codec
    from paper_2209_01188_b200.errors import InputError

    q = codec.quantize_blockwise(torch_cuda.zeros(0, device="cuda"))
    assert codec.dequantize_blockwise(q).shape == (0,)
    with pytest.raises(InputError):
        codec.quantize_blockwise(torch_cuda.tensor([1.0, float("inf")], device="cuda"))
    with pytest.raises(InputError):
        codec.quantize_blockwise(torch_cuda.ones(4, device="cuda"), 0)


def test_wire_bytes_match_reference(torch_cuda, golden):
    from paper_2209_01188_b200 import codec

    g = golden("codec")
    got = codec.encode_tensor(g["wire_tensor"], codec.ENC_INT8)
    assert got == g["wire_int8"].tobytes()
    assert codec.encode_tensor(np.array([1.0, -1.0], np.float32), codec.ENC_F32) == g["wire_f32"].tobytes()
    back = codec.decode_tensor(got).cpu().numpy()
    s, c = O.wire_quantize(g["wire_tensor"])
    assert np.array_equal(back.reshape(-1), O.wire_dequantize(s, c))


def test_gen_tensor_bit_exact(torch_cuda, golden):
    from paper_2209_01188_b200 import codec

    g = golden("weights")
    for seed in (42, 7):
        for i, p in enumerate(g["paths"]):
            want = g[f"stream_{seed}_{i}"]
            got = codec.gen_tensor(seed, str(p), want.size).cpu().numpy()
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    # far offsets (counter form) vs the oracle
    for first in (0, 123456789, (1 << 33) + 5):
        got = codec.gen_tensor(42, "blocks.69.wmlp_out", 4096, first=first).cpu().numpy()
        want = O.named_tensor(42, "blocks.69.wmlp_out", 4096, first=first)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
