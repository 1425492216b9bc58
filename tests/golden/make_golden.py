"""Generate golden fixtures by running the REFERENCE implementation (swarmlm).

Run in the build container only (it imports /root/reference/pkg/src, which does
not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/{codec,weights,blocks,generate}.npz. Every array is the
reference's own output on seeded inputs; tests compare both the oracle
(oracle/swarm_oracle.py) and the CUDA path against them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("SWARMLM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from swarmlm import model as M  # noqa: E402
from swarmlm import quant as Q  # noqa: E402
from swarmlm.transport import wire as W  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def codec_cases():
    rng = np.random.default_rng(2209)
    cases = []
    # reference known answers (tests/test_quant.py:27-53)
    cases.append((np.array([1.0, -2.0, 0.5, 4.0], np.float32), 4))
    cases.append((np.zeros(8, np.float32), 4))
    cases.append((np.array([0.3, -9.0, 0.1], np.float32), 4))
    s = np.float32(2.0 / 127.0)
    cases.append((np.array([2.0, s * 0.5, -s * 0.5], np.float32), 4))
    # ragged lengths, partial last block, zero blocks, both block sizes
    for n in (1, 5, 63, 64, 65, 127, 130, 1000, 4097):
        x = rng.normal(size=n).astype(np.float32) * np.float32(rng.uniform(0.01, 100))
        if n > 70:
            x[64:128] = 0.0
        cases.append((x, 64))
    for bs in (1, 3, 7, 16, 33):
        cases.append((rng.normal(size=200).astype(np.float32), bs))
    # exact ties: x = (k + 0.5) * scale for many k, with absmax pinned
    for trial in range(8):
        amax = np.float32(rng.uniform(0.1, 10))
        sc = np.float32(amax / np.float32(127.0))
        k = rng.integers(-126, 126, size=63)
        x = ((k + 0.5) * sc.astype(np.float64)).astype(np.float32)
        cases.append((np.concatenate([[amax], x]).astype(np.float32), 64))
    # near-ties: neighbours of half-integers in f32
    for trial in range(8):
        amax = np.float32(rng.uniform(0.5, 3))
        sc = np.float32(amax / np.float32(127.0))
        k = rng.integers(-126, 126, size=63)
        x = ((k + 0.5) * sc.astype(np.float64)).astype(np.float32)
        x = np.nextafter(x, np.where(rng.random(63) < 0.5, -np.inf, np.inf).astype(np.float32)).astype(np.float32)
        cases.append((np.concatenate([[amax], x]).astype(np.float32), 64))
    # subnormal and tiny scales, huge magnitudes
    cases.append((np.array([1e-44, 0.0, -1e-44, 5e-45], np.float32), 4))
    cases.append((np.array([3e-43, 0.0, -1e-44, 5e-45], np.float32), 4))
    cases.append(((rng.normal(size=256) * 1e-39).astype(np.float32), 64))
    cases.append(((rng.normal(size=256) * 3e37).astype(np.float32), 64))
    # a larger random sweep: 2^16 elements, mixed per-block magnitudes
    big = rng.normal(size=(1024, 64)).astype(np.float32) * rng.uniform(1e-3, 1e3, size=(1024, 1)).astype(np.float32)
    cases.append((big.reshape(-1), 64))
    return cases


def make_codec():
    xs, bs, scales, codes, deq, wire = [], [], [], [], [], []
    with np.errstate(all="ignore"):
        for x, b in codec_cases():
            q = Q.quantize_blockwise(x, b)
            xs.append(x)
            bs.append(b)
            scales.append(q.scales.astype(np.float32))
            codes.append(q.codes.astype(np.int8))
            deq.append(Q.dequantize_blockwise(q))
    # int8 wire bytes for a [3, 100] tensor (transport/wire.py:87-106)
    rng = np.random.default_rng(5)
    t = rng.normal(size=(3, 100)).astype(np.float32)
    wire = np.frombuffer(W.encode_tensor(t, W.ENC_INT8), np.uint8)
    wire_f32 = np.frombuffer(W.encode_tensor(np.array([1.0, -1.0], np.float32), W.ENC_F32), np.uint8)

    def pack(arrs, dtype):
        off = np.cumsum([0] + [a.size for a in arrs]).astype(np.int64)
        return np.concatenate([a.astype(dtype) for a in arrs]) if arrs else np.zeros(0, dtype), off

    x_all, x_off = pack(xs, np.float32)
    s_all, s_off = pack(scales, np.float32)
    c_all, _ = pack(codes, np.int8)
    d_all, _ = pack(deq, np.float32)
    np.savez_compressed(
        os.path.join(OUT, "codec.npz"),
        x=x_all, x_off=x_off, block=np.array(bs, np.int64), scales=s_all, s_off=s_off,
        codes=c_all, deq=d_all, wire_tensor=t, wire_int8=wire, wire_f32=wire_f32,
    )


def make_weights():
    rng = np.random.default_rng(1188)
    out = {}
    out["sm64_state0"] = M.splitmix64_array(0, 8)
    out["fnv_empty"] = np.array([M.fnv1a64(b"")], np.uint64)
    out["fnv_a"] = np.array([M.fnv1a64(b"a")], np.uint64)
    paths = ["embed", "blocks.0.wqkv", "blocks.3.wmlp_out", "blocks.69.wo", "final_ln.gamma"]
    out["paths"] = np.array(paths)
    out["fnv_paths"] = np.array([M.fnv1a64(p.encode()) for p in paths], np.uint64)
    for seed in (42, 7):
        for i, p in enumerate(paths):
            out[f"stream_{seed}_{i}"] = M.tensor_stream(seed, p, 4096)
    # weight quantizer, quant.py:81-108 via from_block's transpose (quant.py:142-149)
    mats = []
    w = rng.uniform(-0.05, 0.05, (48, 80)).astype(np.float32)  # [in, out]
    mats.append(w)
    w = rng.normal(size=(64, 96)).astype(np.float32)
    w[[3, 17, 40], :] *= 9.0  # outlier input features
    w[5, :] = 0.0  # all-zero feature
    mats.append(w)
    w = (np.eye(16) * 10).astype(np.float32)  # all-outlier (tests/test_quant.py:122-129)
    mats.append(w)
    w = rng.uniform(-2, 2, (32, 16)).astype(np.float32)
    w[:, :] = np.round(w * 127 / 2) * np.float32(2 / 127)  # many exact-tie candidates
    mats.append(w)
    for j, w in enumerate(mats):
        wq = Q.quantize_weights_int8(w.T)
        out[f"wq{j}_w"] = w
        out[f"wq{j}_codes"] = wq.regular_codes
        out[f"wq{j}_scales"] = wq.col_scales
        out[f"wq{j}_outl"] = wq.outlier_cols.astype(np.int64)
        out[f"wq{j}_outl_data"] = wq.outlier_data
        x = rng.normal(size=(w.shape[0], 5)).astype(np.float32)
        out[f"wq{j}_x"] = x
        out[f"wq{j}_mm"] = Q.matmul_mixed(wq, x)
    out["n_mats"] = np.array([len(mats)])
    np.savez_compressed(os.path.join(OUT, "weights.npz"), **out)


SMALL = dict(n_layers=4, hidden=16, n_heads=2, vocab=32, max_seq=128)
TINY = dict(n_layers=2, hidden=8, n_heads=2, vocab=32, max_seq=64)
# a mid shape exercising dh=64 and the generic GEMV tiling (not a BLOOM shape)
MID = dict(n_layers=3, hidden=256, n_heads=4, vocab=512, max_seq=256)


def qw_generate(ckpt, prompt, n):
    cfg = ckpt.config
    qws = [Q.QuantizedBlockWeights.from_block(b) for b in ckpt.blocks]
    caches = [M.KvCache.empty(cfg) for _ in range(cfg.n_layers)]
    pend, pos, out, hid = list(prompt), 0, [], []
    for step in range(n):
        h = M.embed(ckpt, pend)
        for i in range(cfg.n_layers):
            h, caches[i], _ = M.block_forward(ckpt.blocks[i], h, caches[i], pos, cfg, qw=qws[i])
        hid.append(h[-1].copy())
        nxt = M.sample_next(M.lm_head(ckpt, h)[-1])
        pos += len(pend)
        pend = [nxt]
        out.append(nxt)
    return out, np.stack(hid)


def make_blocks():
    out = {}
    for name, kw in (("tiny", TINY), ("small", SMALL), ("mid", MID)):
        cfg = M.ModelConfig(**kw)
        ckpt = M.gen_checkpoint(42, cfg)
        rng = np.random.default_rng(len(name))
        tokens = rng.integers(0, cfg.vocab, 9)
        x = M.embed(ckpt, tokens)
        out[f"{name}_tokens"] = tokens
        # one-shot full forward, fp32 and int8-weights
        out[f"{name}_fwd_f32"] = M.forward_blocks(ckpt, x)
        h = x
        for b in ckpt.blocks:
            h, _, _ = M.block_forward(b, h, M.KvCache.empty(cfg), 0, cfg, qw=Q.QuantizedBlockWeights.from_block(b))
        out[f"{name}_fwd_qw"] = h
        # incremental: prefill 5, then 4 single steps through block 0 only (qw)
        qw0 = Q.QuantizedBlockWeights.from_block(ckpt.blocks[0])
        cache = M.KvCache.empty(cfg)
        o, cache, _ = M.block_forward(ckpt.blocks[0], x[:5], cache, 0, cfg, qw=qw0)
        steps = [o]
        for i in range(5, 9):
            o, cache, _ = M.block_forward(ckpt.blocks[0], x[i:i + 1], cache, i, cfg, qw=qw0)
            steps.append(o)
        out[f"{name}_blk0_inc_qw"] = np.concatenate(steps)
        out[f"{name}_gen_f32"] = np.array(M.reference_generate(ckpt, [1, 2, 3], 16))
        toks, hid = qw_generate(ckpt, [1, 2, 3], 16)
        out[f"{name}_gen_qw"] = np.array(toks)
        out[f"{name}_gen_qw_hidden"] = hid
    np.savez_compressed(os.path.join(OUT, "blocks.npz"), **out)


def make_train():
    """FORWARD tapes + BACKWARD (server.py:411-450): per row, block_forward with
    want_tape over every block (fp32 weights, empty cache), then block_backward
    in reverse (model.py:383-418) for a random upstream gradient."""
    out = {}
    for name, kw in (("tiny", TINY), ("small", SMALL), ("mid", MID)):
        cfg = M.ModelConfig(**kw)
        ckpt = M.gen_checkpoint(42, cfg)
        rng = np.random.default_rng(100 + len(name))
        B, t = 2, 7
        batch = np.stack([M.embed(ckpt, rng.integers(0, cfg.vocab, t)) for _ in range(B)])
        grad = rng.uniform(-1, 1, (B, t, cfg.hidden)).astype(np.float32)
        fwd = np.empty_like(batch)
        gin = np.empty_like(batch)
        for r in range(B):
            h, tapes = batch[r], []
            for b in ckpt.blocks:
                h, _, tape = M.block_forward(b, h, M.KvCache.empty(cfg), 0, cfg, want_tape=True)
                tapes.append(tape)
            fwd[r] = h
            g = grad[r]
            for b, tape in zip(reversed(ckpt.blocks), reversed(tapes)):
                g = M.block_backward(b, tape, g, cfg)
            gin[r] = g
        out[f"{name}_batch"], out[f"{name}_grad"] = batch, grad
        out[f"{name}_fwd"], out[f"{name}_grad_in"] = fwd, gin
    np.savez_compressed(os.path.join(OUT, "train.npz"), **out)


def make_c2():
    """Config 2 (BLOOM-560M shape, 24 blocks, h=1024, H=16): int8-weights
    greedy generation with a 128-token prefix then 128 decode steps (SURVEY
    §8: C2 T0=128, then 128 decode steps), reference qw semantics. Expensive on
    CPU (several minutes); stores tokens and last-position hiddens."""
    cfg = M.ModelConfig(n_layers=24, hidden=1024, n_heads=16, vocab=250880, max_seq=2048)
    ckpt = M.gen_checkpoint(42, cfg)
    prompt = np.random.default_rng(7).integers(0, cfg.vocab, 128).tolist()
    toks, hid = qw_generate(ckpt, prompt, 129)
    np.savez_compressed(os.path.join(OUT, "c2.npz"), prompt=np.array(prompt), tokens=np.array(toks), hidden=hid)


if __name__ == "__main__":
    what = sys.argv[1:] or ["codec", "weights", "blocks", "train", "c2"]
    for w in what:
        print("making", w, flush=True)
        globals()[f"make_{w}"]()
