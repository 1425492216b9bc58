"""Box front end (paper_2209_01188_b200.box): ONE span server for [0, L)
executed by two sub-span processes whose hop is a peer-memory mailbox
(pb_hop.cu). On a one-GPU box both ranks share the device (same IPC mailbox,
wait/signal kernels and control plane; no NVLink). The client makes a single
hop; tokens must equal the reference's goldens (f32 hops: what one reference
server hosting [0, L) computes) or the oracle relay that quantizes at every
hop (int8 hops, quantize='both').
"""

import numpy as np
import pytest

import swarm_oracle as O  # checker / client head only
from conftest import load_golden

pytestmark = pytest.mark.gpu

SMALL = (4, 16, 2, 32, 128)
MID = (3, 256, 4, 512, 256)


def _box(shape, quantize="none", world=2, **kw):
    from paper_2209_01188_b200.box import LocalBox
    from paper_2209_01188_b200.model import ModelConfig
    from paper_2209_01188_b200.server import ServerConfig

    cfg = ServerConfig(seed=42, model=ModelConfig(*shape), quantize=quantize, measure_steps=3, page_tokens=16, **kw)
    return LocalBox(cfg, world)


def _generate(address, shape, prompt, n, encoding=0):
    from paper_2209_01188_b200.client import SpanClient

    sh = O.Shape(*shape)
    emb = O.make_embed(42, sh)
    c = SpanClient(address, encoding)
    try:
        sid = c.open_session(sh.max_seq)
        pending, pos, out = list(prompt), 0, []
        for _ in range(n):
            h = c.step(sid, pos, emb[np.asarray(pending)].astype(np.float32))
            nxt = O.greedy(O.final_logits(emb, h)[-1])
            pos += len(pending)
            pending = [nxt]
            out.append(nxt)
        c.close_session(sid)
        return out
    finally:
        c.close()


@pytest.mark.parametrize("quantize,key", [("none", "gen_f32"), ("weights", "gen_qw")])
def test_box_one_hop_generation_equals_reference(quantize, key):
    box = _box(SMALL, quantize)
    try:
        assert _generate(box.address, SMALL, [1, 2, 3], 16) == load_golden("blocks")[f"small_{key}"].tolist()
    finally:
        assert box.stop() == [0, 0]


def test_box_int8_hops_equal_oracle_relay_and_concurrent_sessions():
    """quantize='both': the client sends int8, the in-box hop carries the
    wire codec, the reply is int8. Equals the oracle relay quantizing at each
    of those three points; eight concurrent sessions give the same tokens."""
    from concurrent.futures import ThreadPoolExecutor

    shape = O.Shape(*MID)
    blocks = [O.make_block(42, shape, i) for i in range(3)]
    emb = O.make_embed(42, shape)
    kvs = [O.KV(shape) for _ in blocks]
    qb = [O.QuantBlock(b) for b in blocks]
    q = lambda h: O.wire_dequantize(*O.wire_quantize(h.reshape(-1))).reshape(h.shape)  # noqa: E731
    pending, pos, want = [1, 2, 3], 0, []
    for _ in range(10):
        h = q(emb[np.asarray(pending)].astype(np.float32))
        for lo, hi in ((0, 2), (2, 3)):  # split_blocks(3, 2)
            for i in range(lo, hi):
                h = O.block_step(blocks[i], h, kvs[i], pos, shape, qb[i])
            h = q(h)
        nxt = O.greedy(O.final_logits(emb, h)[-1])
        pos += len(pending)
        pending = [nxt]
        want.append(nxt)
    box = _box(MID, "both")
    try:
        assert _generate(box.address, MID, [1, 2, 3], 10, encoding=1) == want
        with ThreadPoolExecutor(8) as ex:
            outs = list(ex.map(lambda _: _generate(box.address, MID, [1, 2, 3], 10, encoding=1), range(8)))
        assert all(o == want for o in outs)
    finally:
        assert box.stop() == [0, 0]


def test_box_long_prompt_forward_backward():
    """A prompt longer than the token workspace (causal chunk jobs through the
    ring), and FORWARD / BACKWARD through the box == the reference train
    goldens (tapes kept per rank, BACKWARD walked in reverse)."""
    from paper_2209_01188_b200.client import SpanClient
    from paper_2209_01188_b200.errors import ERR_UNKNOWN_TAPE, RemoteError

    g = load_golden("train")
    box = _box(SMALL, "none", max_batch_tokens=16)
    c = SpanClient(box.address)
    try:
        shape = O.Shape(*SMALL)
        blocks = [O.make_block(42, shape, i) for i in range(4)]
        x = O.make_embed(42, shape)[np.random.default_rng(5).integers(0, 32, 40)].astype(np.float32)
        sid = c.open_session(64)
        got = c.step(sid, 0, x)
        want = O.forward_span(blocks, x, shape, quantized=False)
        assert float(np.abs(got - want).max()) <= 1e-3 * float(np.abs(want).max())
        out, parts = c.forward(g["small_batch"])
        assert float(np.abs(out - g["small_fwd"]).max()) <= 1e-3 * float(np.abs(g["small_fwd"]).max())
        gin = c.backward(parts, g["small_grad"])
        assert float(np.abs(gin - g["small_grad_in"]).max()) <= 1e-3 * float(np.abs(g["small_grad_in"]).max())
        with pytest.raises(RemoteError) as ei:
            c.backward(parts, g["small_grad"])
        assert ei.value.code == ERR_UNKNOWN_TAPE
    finally:
        c.close()
        assert box.stop() == [0, 0]


def test_box_concurrent_long_prompts():
    """Eight sessions send prompts longer than the token workspace at once:
    every prompt runs as causal chunk jobs whose outputs come off the egress
    stream while other sessions' jobs are in flight (the cross-stream buffer
    lifetimes of BoxScheduler.run / BoxFrontEnd._run_step), and each reply
    equals the span forward of its own prompt. (At this size it did not
    reproduce the 7B1-scale race those lifetimes fixed; it guards the path.)"""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2209_01188_b200.client import SpanClient

    shape = O.Shape(*SMALL)
    blocks = [O.make_block(42, shape, i) for i in range(4)]
    emb = O.make_embed(42, shape)
    prompts = [emb[np.random.default_rng(100 + i).integers(0, 32, 40)].astype(np.float32) for i in range(8)]
    box = _box(SMALL, "none", max_batch_tokens=16, capacity=8)

    def one(i):
        c = SpanClient(box.address)
        try:
            sid = c.open_session(64)
            got = c.step(sid, 0, prompts[i])
            c.close_session(sid)
            return got
        finally:
            c.close()

    try:
        for _ in range(3):
            with ThreadPoolExecutor(8) as ex:
                outs = list(ex.map(one, range(8)))
            for x, got in zip(prompts, outs):
                want = O.forward_span(blocks, x, shape, quantized=False)
                assert np.isfinite(got).all()
                assert float(np.abs(got - want).max()) <= 1e-3 * float(np.abs(want).max())
    finally:
        assert box.stop() == [0, 0]
