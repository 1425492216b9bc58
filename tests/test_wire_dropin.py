"""Reference-free drop-in tests: OPEN / STEP / CLOSE / FORWARD / BACKWARD
frames built with this repo's own wire + codec (paper_2209_01188_b200.client)
against running span servers, checked against the golden fixtures the
REFERENCE produced (tests/golden/make_golden.py) and the pinned oracle. They
need nothing from baseline/_ref, so the handlers get hardware evidence on any
GPU box. Mirrors /root/reference/pkg/tests/test_server.py:80-236 and
tests/test_client.py:167-175.
"""

import os
import struct

import numpy as np
import pytest

import swarm_oracle as O  # checker / client head only
from conftest import load_golden

pytestmark = pytest.mark.gpu

SMALL = (4, 16, 2, 32, 128)
MID = (3, 256, 4, 512, 256)


def _server(shape, blocks, quantize="none", **kw):
    from paper_2209_01188_b200.model import ModelConfig
    from paper_2209_01188_b200.server import ServerConfig, ServerNode

    cfg = ServerConfig(seed=42, model=ModelConfig(*shape), blocks=blocks, quantize=quantize, measure_steps=5,
                       page_tokens=16, **kw)
    return ServerNode(cfg).start()


class _Chain:
    """The reference client's remote sequential chain (client.py:290-331) with
    the client head (embed + final LN + tied head + greedy) from the oracle."""

    def __init__(self, shape, spans, quantize="none", encoding=0, **kw):
        from paper_2209_01188_b200.client import SpanClient

        self.shape = O.Shape(*shape)
        self.nodes = [_server(shape, s, quantize, **kw) for s in spans]
        self.clients = [SpanClient(n.address, encoding) for n in self.nodes]
        self.embed = O.make_embed(42, self.shape)

    def generate(self, prompt, n):
        sids = [c.open_session(self.shape.max_seq) for c in self.clients]
        pending, pos, out = list(prompt), 0, []
        for _ in range(n):
            h = self.embed[np.asarray(pending)].astype(np.float32)
            for c, sid in zip(self.clients, sids):
                h = c.step(sid, pos, h)
            nxt = O.greedy(O.final_logits(self.embed, h)[-1])
            pos += len(pending)
            pending = [nxt]
            out.append(nxt)
        for c, sid in zip(self.clients, sids):
            c.close_session(sid)
        return out

    def close(self):
        for c in self.clients:
            c.close()
        for n in self.nodes:
            n.stop()


@pytest.mark.parametrize("name,shape,spans", [("small", SMALL, [(0, 2), (2, 4)]), ("mid", MID, [(0, 1), (1, 3)])])
@pytest.mark.parametrize("quantize,key", [("none", "gen_f32"), ("weights", "gen_qw")])
def test_two_span_generation_equals_reference_goldens(name, shape, spans, quantize, key):
    """C1-style: two span servers, prompt [1,2,3], 16 greedy tokens == the
    reference's own tokens (reference_generate / qw loop)."""
    want = load_golden("blocks")[f"{name}_{key}"].tolist()
    ch = _Chain(shape, spans, quantize)
    try:
        assert ch.generate([1, 2, 3], 16) == want
    finally:
        ch.close()


def test_int8_wire_generation_matches_oracle_relay():
    """quantize='both' + int8 client encoding: every hop's hidden state travels
    as the blockwise int8 codec. Tokens equal the oracle relay that quantizes
    each hop's input and output the same way (bit-exact codec)."""
    shape = O.Shape(*MID)
    blocks = [O.make_block(42, shape, i) for i in range(shape.n_layers)]
    emb = O.make_embed(42, shape)
    spans = [(0, 1), (1, 3)]
    kvs = [O.KV(shape) for _ in blocks]
    qb = [O.QuantBlock(b) for b in blocks]
    pending, pos, want = [1, 2, 3], 0, []
    for _ in range(10):
        h = emb[np.asarray(pending)].astype(np.float32)
        for s, e in spans:
            h = O.wire_dequantize(*O.wire_quantize(h.reshape(-1))).reshape(h.shape)  # client -> server
            for i in range(s, e):
                h = O.block_step(blocks[i], h, kvs[i], pos, shape, qb[i])
            h = O.wire_dequantize(*O.wire_quantize(h.reshape(-1))).reshape(h.shape)  # server reply
        nxt = O.greedy(O.final_logits(emb, h)[-1])
        pos += len(pending)
        pending = [nxt]
        want.append(nxt)
    ch = _Chain(MID, spans, "both", encoding=1)
    try:
        assert ch.generate([1, 2, 3], 10) == want
    finally:
        ch.close()


def test_long_prompt_beyond_batch_workspace():
    """A STEP longer than the server's per-launch token workspace runs as
    causal chunks (t > max_batch_tokens used to fail with BUSY).
    Output equals the one-shot oracle forward."""
    from paper_2209_01188_b200.client import SpanClient

    shape = O.Shape(*MID)
    blocks = [O.make_block(42, shape, i) for i in range(3)]
    x = O.make_embed(42, shape)[np.random.default_rng(3).integers(0, shape.vocab, 100)].astype(np.float32)
    want = O.forward_span(blocks, x, shape, quantized=True)
    node = _server(MID, (0, 3), "weights", max_batch_tokens=32)
    c = SpanClient(node.address)
    try:
        sid = c.open_session(200)
        got = c.step(sid, 0, x)
        assert float(np.abs(got - want).max()) <= 2e-3 * float(np.abs(want).max())
        nxt = c.step(sid, 100, x[:1])  # the session continues at position 100
        assert nxt.shape == (1, shape.hidden)
    finally:
        c.close()
        node.stop()


def test_step_protocol_semantics_and_error_codes():
    """test_server.py:80-189 semantics over raw frames: idempotent retry,
    DESYNC, UNKNOWN_SESSION, duplicate id, capacity BUSY, CLOSE frees a slot,
    max_len CAPACITY, malformed tensor / wrong width -> ERR_GENERIC (the
    reference's decode_tensor / block_forward exceptions escape its handler)."""
    from paper_2209_01188_b200.client import SpanClient, _np_tensor_msg
    from paper_2209_01188_b200.errors import (ERR_BAD_REQUEST, ERR_BUSY, ERR_CAPACITY, ERR_DESYNC, ERR_GENERIC,
                                              ERR_UNKNOWN_SESSION, RemoteError)
    from paper_2209_01188_b200.wire import MSG

    shape = O.Shape(*SMALL)
    emb = O.make_embed(42, shape)
    blocks = [O.make_block(42, shape, i) for i in range(4)]
    node = _server(SMALL, (0, 4), capacity=3)
    c = SpanClient(node.address)

    def code(fn, *a):
        with pytest.raises(RemoteError) as ei:
            fn(*a)
        return ei.value.code

    try:
        sid = c.open_session(8)
        h = emb[[1, 2, 3]].astype(np.float32)
        out = c.step(sid, 0, h)
        want = O.forward_span(blocks, h, shape, quantized=False)
        assert float(np.abs(out - want).max()) <= 1e-3 * float(np.abs(want).max())
        assert np.array_equal(c.step(sid, 0, h), out)  # idempotent retry (server.py:374-377)
        assert code(c.step, sid, 5, emb[[2]]) == ERR_DESYNC
        assert code(c.step, sid, 0, emb[[4, 4, 4]]) == ERR_DESYNC  # retry with another payload
        c.step(sid, 3, emb[[4]])
        assert code(c.step, sid, 4, emb[[1, 1, 1, 1, 1]]) == ERR_CAPACITY  # past max_len 8
        assert code(c.step, os.urandom(16), 0, emb[[1]]) == ERR_UNKNOWN_SESSION
        assert code(c.step_raw, sid, 4, b"\x00\x02\x00") == ERR_GENERIC  # truncated TensorMsg
        assert code(c.step, sid, 4, np.zeros((1, 8), np.float32)) == ERR_GENERIC  # wrong hidden width
        assert code(c.step_raw, sid, 4, _np_tensor_msg(np.zeros(16, np.float32), 0)) == ERR_BAD_REQUEST  # 1-D
        assert code(c.open_session, 8, sid) == ERR_BAD_REQUEST  # duplicate id
        assert code(c.open_session, 100000) == ERR_BAD_REQUEST  # max_len > max_seq
        c.open_session(8)
        c.open_session(8)
        assert code(c.open_session, 8) == ERR_BUSY
        c.close_session(sid)
        c.open_session(8)
        assert c.call(MSG.PING, b"") == b""
        import json

        info = json.loads(c.call(MSG.INFO, b"").decode())
        assert info["range"] == [0, 4] and info["throughput"] > 0 and info["quantize"] == "none"
        assert code(c.call, 0x55, b"") == ERR_BAD_REQUEST  # unknown message type
        assert code(c.call, MSG.OPEN_SESSION, os.urandom(16) + struct.pack(">I", 0)) == ERR_BAD_REQUEST
        assert code(c.call, MSG.STEP, b"short") == ERR_BAD_REQUEST
    finally:
        c.close()
        node.stop()


def test_cache_budget_lru_eviction():
    """server.py:397-407: after a step pushes sum(position x blocks) past the
    budget, least-recently-active sessions are evicted."""
    from paper_2209_01188_b200.client import SpanClient
    from paper_2209_01188_b200.errors import ERR_DESYNC, ERR_UNKNOWN_SESSION, RemoteError

    emb = O.make_embed(42, O.Shape(*SMALL))
    node = _server(SMALL, (0, 4), cache_budget_tokens=8 * 4)
    c = SpanClient(node.address)
    try:
        a = c.open_session(64)
        for i in range(5):
            c.step(a, i, emb[[1]])
        b = c.open_session(64)
        for i in range(5):
            c.step(b, i, emb[[2]])  # 10 positions x 4 blocks > 32: a (LRU) goes
        with pytest.raises(RemoteError) as ei:
            c.step(a, 5, emb[[1]])
        assert ei.value.code in (ERR_UNKNOWN_SESSION, ERR_DESYNC)
        c.step(b, 5, emb[[2]])
    finally:
        c.close()
        node.stop()


def test_forward_backward_equal_reference_goldens():
    """FORWARD tapes + BACKWARD over one [0, 4) span == the reference's
    block_forward(want_tape) / block_backward goldens (f32 weights, 1e-3
    relative: the span carries fp16 KV); a tape is consumed once."""
    from paper_2209_01188_b200.client import SpanClient
    from paper_2209_01188_b200.errors import ERR_UNKNOWN_TAPE, RemoteError

    g = load_golden("train")
    node = _server(SMALL, (0, 4))
    c = SpanClient(node.address)
    try:
        out, parts = c.forward(g["small_batch"])
        assert float(np.abs(out - g["small_fwd"]).max()) <= 1e-3 * float(np.abs(g["small_fwd"]).max())
        gin = c.backward(parts, g["small_grad"])
        assert float(np.abs(gin - g["small_grad_in"]).max()) <= 1e-3 * float(np.abs(g["small_grad_in"]).max())
        with pytest.raises(RemoteError) as ei:
            c.backward(parts, g["small_grad"])
        assert ei.value.code == ERR_UNKNOWN_TAPE
    finally:
        c.close()
        node.stop()


def test_forward_chunked_past_frame_cap():
    """A FORWARD batch larger than the 64 MiB frame cap (transport/wire.py:93)
    goes as row groups, each with its own tape; rows equal the oracle."""
    from paper_2209_01188_b200.client import SpanClient
    from paper_2209_01188_b200.wire import MAX_PAYLOAD

    shape = O.Shape(*MID)
    blocks = [O.make_block(42, shape, 0)]
    rng = np.random.default_rng(11)
    B, t = 270, 256
    batch = (rng.standard_normal((B, t, shape.hidden)) * 0.05).astype(np.float32)
    assert batch.nbytes > MAX_PAYLOAD
    node = _server(MID, (0, 1), "weights")
    c = SpanClient(node.address)
    try:
        out, parts = c.forward(batch)
        assert len(parts) >= 2 and sum(len(p.rows) for p in parts) == B
        for r in (0, 133, 269):
            want = O.forward_span(blocks, batch[r], shape, quantized=True)
            assert float(np.abs(out[r] - want).max()) <= 2e-3 * float(np.abs(want).max())
        gin = c.backward(parts, np.zeros_like(batch))
        assert not gin.any()
    finally:
        c.close()
        node.stop()


def test_concurrent_sessions_coalesced():
    """Eight concurrent chains through one span == single-chain tokens, with
    STEPs of different sessions coalesced into batched span steps."""
    from concurrent.futures import ThreadPoolExecutor

    want = load_golden("blocks")["small_gen_f32"].tolist()[:12]
    ch = _Chain(SMALL, [(0, 4)])
    try:
        def one(_):
            from paper_2209_01188_b200.client import SpanClient

            sub = _Chain.__new__(_Chain)
            sub.shape, sub.embed, sub.nodes = ch.shape, ch.embed, []
            sub.clients = [SpanClient(ch.nodes[0].address)]
            try:
                return sub.generate([1, 2, 3], 12)
            finally:
                sub.clients[0].close()

        with ThreadPoolExecutor(8) as ex:
            outs = list(ex.map(one, range(8)))
        assert all(o == want for o in outs)
        assert ch.nodes[0].sched.batched_steps >= ch.nodes[0].sched.batches
    finally:
        ch.close()
