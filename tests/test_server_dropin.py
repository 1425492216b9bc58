"""Drop-in tests: the REFERENCE client (swarmlm, installed into baseline/_ref by
`pip install --target baseline/_ref`) drives the B200 span server over TCP.

The reference package is the client and the registry seed here, never the
checker of numerics: token oracles are reference_generate / the reference's
own servers run side by side on the same checkpoint. Mirrors
/root/reference/pkg/tests/test_server.py and test_client.py:167-175.
"""

import os
import struct
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "swarmlm")):
        # a failure, not a skip: a silent skip once hid every drop-in test on
        # hardware (round 1). `__graft_entry__.build()` installs it.
        pytest.fail("reference client not installed in baseline/_ref (run __graft_entry__.build())")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import swarmlm.client  # noqa: F401
    import swarmlm.model  # noqa: F401
    import swarmlm.registry  # noqa: F401

    return sys.modules["swarmlm"]


@pytest.fixture(scope="module")
def small_ckpt(ref):
    from swarmlm.model import ModelConfig, gen_checkpoint

    return gen_checkpoint(42, ModelConfig(n_layers=4, hidden=16, n_heads=2, vocab=32, max_seq=128))


class Swarm:
    def __init__(self, ckpt):
        from swarmlm.registry import RegistrySeed

        self.ckpt = ckpt
        self.seed = RegistrySeed("127.0.0.1", 0, n_blocks=ckpt.config.n_layers).start()
        self.nodes = []

    def b200(self, blocks, quantize="none", **kw):
        from paper_2209_01188_b200.server import ServerConfig, ServerNode

        cfg = ServerConfig(blocks=blocks, quantize=quantize, bootstrap=[self.seed.address], measure_steps=5,
                           page_tokens=16, **kw)
        node = ServerNode(cfg, checkpoint=self.ckpt).start()
        self.nodes.append(node)
        return node

    def reference(self, blocks, quantize="none"):
        from swarmlm.server import ServerConfig, ServerNode

        cfg = ServerConfig(checkpoint_path="", host="127.0.0.1", port=0, blocks=blocks, quantize=quantize,
                           bootstrap=[self.seed.address], measure_steps=5)
        node = ServerNode(cfg, checkpoint=self.ckpt).start()
        self.nodes.append(node)
        return node

    def client(self, **kw):
        from swarmlm.client import SwarmClient

        return SwarmClient(self.ckpt, [self.seed.address], **kw)

    def close(self):
        for n in self.nodes:
            try:
                n.stop()
            except Exception:  # noqa: BLE001
                pass
        self.seed.stop()


@pytest.fixture
def swarm(small_ckpt):
    s = Swarm(small_ckpt)
    yield s
    s.close()


def _gen(swarm, n=16, **kw):
    c = swarm.client(**kw)
    try:
        return c.generate([1, 2, 3], n)
    finally:
        c.close()


def test_c1_two_span_generation_equals_reference_generate(swarm):
    """Config 1: two block-span servers, greedy 16 tokens, fp32 weights."""
    from swarmlm.model import reference_generate

    swarm.b200((0, 2))
    swarm.b200((2, 4))
    assert _gen(swarm) == reference_generate(swarm.ckpt, [1, 2, 3], 16)


@pytest.mark.parametrize("quantize", ["weights", "both"])
def test_int8_spans_equal_reference_servers(small_ckpt, quantize):
    """int8 weights (and int8 wire for 'both'): B200 spans vs the reference's
    own servers with the same quantize mode give identical greedy tokens."""
    from swarmlm.transport import ENC_INT8

    want_sw = Swarm(small_ckpt)
    try:
        want_sw.reference((0, 2), quantize)
        want_sw.reference((2, 4), quantize)
        want = _gen(want_sw, encoding=ENC_INT8) if quantize == "both" else _gen(want_sw)
    finally:
        want_sw.close()
    got_sw = Swarm(small_ckpt)
    try:
        got_sw.b200((0, 2), quantize)
        got_sw.b200((2, 4), quantize)
        got = _gen(got_sw, encoding=ENC_INT8) if quantize == "both" else _gen(got_sw)
    finally:
        got_sw.close()
    assert got == want


def _open(address, sid=None, max_len=64):
    from swarmlm.transport import MSG, rpc_call

    sid = sid or os.urandom(16)
    rpc_call(address, MSG.OPEN_SESSION, sid + struct.pack(">I", max_len), 5000.0)
    return sid


def _step(address, sid, pos, h):
    from swarmlm.transport import ENC_F32, MSG, decode_tensor, encode_tensor, rpc_call

    return decode_tensor(rpc_call(address, MSG.STEP, sid + struct.pack(">I", pos) + encode_tensor(h, ENC_F32), 10000.0))


def test_step_semantics(swarm):
    """test_server.py:80-189 semantics over the wire."""
    from swarmlm.errors import ERR_BUSY, ERR_DESYNC, ERR_UNKNOWN_SESSION, RemoteError
    from swarmlm.model import embed, forward_blocks
    from swarmlm.transport import MSG, rpc_call

    node = swarm.b200((0, 4), capacity=3)
    ck = swarm.ckpt
    sid = _open(node.address)
    h = embed(ck, [1, 2, 3])
    out = _step(node.address, sid, 0, h)
    want = forward_blocks(ck, h)
    # fp32 weights here, but the KV cache is fp16: 1e-3 relative (reference: exact f32)
    assert float(np.max(np.abs(out - want))) <= 1e-3 * float(np.abs(want).max())
    again = _step(node.address, sid, 0, h)  # idempotent retry of the previous step
    assert np.array_equal(out, again)
    with pytest.raises(RemoteError) as ei:
        _step(node.address, sid, 5, embed(ck, [2]))
    assert ei.value.code == ERR_DESYNC
    with pytest.raises(RemoteError) as ei:
        _step(node.address, sid, 0, embed(ck, [4, 4, 4]))  # retry with a different payload
    assert ei.value.code == ERR_DESYNC
    _step(node.address, sid, 3, embed(ck, [4]))
    with pytest.raises(RemoteError) as ei:
        _step(node.address, os.urandom(16), 0, embed(ck, [1]))
    assert ei.value.code == ERR_UNKNOWN_SESSION
    with pytest.raises(RemoteError):
        _open(node.address, sid=sid)  # duplicate id
    _open(node.address)
    _open(node.address)
    with pytest.raises(RemoteError) as ei:
        _open(node.address)
    assert ei.value.code == ERR_BUSY
    rpc_call(node.address, MSG.CLOSE_SESSION, sid, 5000.0)
    _open(node.address)  # close freed a slot
    info = __import__("json").loads(rpc_call(node.address, MSG.INFO, b"", 5000.0).decode())
    assert info["range"] == [0, 4] and info["throughput"] > 0 and len(info["weights_hash"]) == 64


def test_weights_hash_equals_reference(swarm):
    import json

    from swarmlm.transport import MSG, rpc_call

    a = swarm.b200((0, 2))
    b = swarm.reference((0, 2))
    ha = json.loads(rpc_call(a.address, MSG.INFO, b"", 5000.0).decode())["weights_hash"]
    hb = json.loads(rpc_call(b.address, MSG.INFO, b"", 5000.0).decode())["weights_hash"]
    assert ha == hb


def test_cache_budget_eviction(swarm):
    from swarmlm.errors import ERR_DESYNC, ERR_UNKNOWN_SESSION, RemoteError
    from swarmlm.model import embed

    node = swarm.b200((0, 4), cache_budget_tokens=8)
    ck = swarm.ckpt
    a = _open(node.address)
    for i in range(3):
        _step(node.address, a, i, embed(ck, [1]))
    b = _open(node.address)
    for i in range(3):
        _step(node.address, b, i, embed(ck, [2]))
    with pytest.raises(RemoteError) as ei:
        _step(node.address, a, 3, embed(ck, [1]))
    assert ei.value.code in (ERR_UNKNOWN_SESSION, ERR_DESYNC)


def test_concurrent_sessions_batched_and_isolated(swarm):
    """Eight clients generate concurrently through one span; every stream
    equals the single-client result (sessions coalesced into batched steps)."""
    from concurrent.futures import ThreadPoolExecutor

    from swarmlm.model import reference_generate

    node = swarm.b200((0, 4))
    want = reference_generate(swarm.ckpt, [1, 2, 3], 12)
    with ThreadPoolExecutor(8) as ex:
        outs = list(ex.map(lambda _: _gen(swarm, n=12), range(8)))
    assert all(o == want for o in outs)
    assert node.sched.batched_steps >= node.sched.batches


def test_forward_rpc_matches_block_forward(swarm):
    from swarmlm.model import KvCache, block_forward
    from swarmlm.transport import ENC_F32, MSG, decode_tensor, encode_tensor, rpc_call

    node = swarm.b200((1, 2))
    rng = np.random.default_rng(0)
    batch = rng.uniform(-0.5, 0.5, (3, 5, 16)).astype(np.float32)
    reply = rpc_call(node.address, MSG.FORWARD, encode_tensor(batch, ENC_F32), 10000.0)
    acts = decode_tensor(reply[16:])
    cfg = swarm.ckpt.config
    for r in range(3):
        want, _, _ = block_forward(swarm.ckpt.blocks[1], batch[r], KvCache.empty(cfg), 0, cfg)
        assert float(np.max(np.abs(acts[r] - want))) <= 1e-3 * float(np.abs(want).max())


def test_nonfinite_step_matches_reference(swarm):
    """A NaN hidden state: the reference computes NaN, fails to encode the reply
    (transport/wire.py:89-90 -> ERR_GENERIC) after advancing the position, and
    every later step of that session fails the same way. Same codes here."""
    from swarmlm.errors import RemoteError
    from swarmlm.model import embed
    from swarmlm.transport import MSG, rpc_call

    ck = swarm.ckpt

    def raw_step(address, sid, pos, arr):
        arr = np.asarray(arr, "<f4")
        msg = struct.pack(">BB", 0, 2) + struct.pack(">II", *arr.shape) + arr.tobytes()
        try:
            rpc_call(address, MSG.STEP, sid + struct.pack(">I", pos) + msg, 10000.0)
            return 0
        except RemoteError as e:
            return e.code

    codes = {}
    for kind, node in (("ref", swarm.reference((0, 4))), ("b200", swarm.b200((0, 4)))):
        sid = _open(node.address)
        bad = embed(ck, [2]).copy()
        bad[0, 3] = np.nan
        codes[kind] = [raw_step(node.address, sid, 0, embed(ck, [1, 2, 3])), raw_step(node.address, sid, 3, bad),
                       raw_step(node.address, sid, 3, bad), raw_step(node.address, sid, 4, embed(ck, [5]))]
    assert codes["b200"] == codes["ref"], codes
    assert codes["ref"][0] == 0 and codes["ref"][1] != 0


def test_forward_backward_matches_reference_server(swarm):
    """tests/test_server.py:195-210 over the wire, B200 server vs the
    reference server on the same checkpoint (f32 weights): activations and
    input gradients within 1e-3 (the reference pins numpy's own arithmetic
    bit-exactly; the span carries an fp16 KV cache in FORWARD)."""
    from swarmlm.transport import ENC_F32, MSG, decode_tensor, encode_tensor, rpc_call

    rng = np.random.default_rng(0)
    batch = rng.uniform(-0.5, 0.5, (2, 3, 16)).astype(np.float32)
    grad = rng.uniform(-1, 1, (2, 3, 16)).astype(np.float32)
    res = {}
    for kind, node in (("ref", swarm.reference((1, 3))), ("b200", swarm.b200((1, 3)))):
        reply = rpc_call(node.address, MSG.FORWARD, encode_tensor(batch, ENC_F32), 10000.0)
        tape_id, acts = reply[:16], decode_tensor(reply[16:])
        gin = decode_tensor(rpc_call(node.address, MSG.BACKWARD, tape_id + encode_tensor(grad, ENC_F32), 10000.0))
        res[kind] = (acts, gin)
    for a, b in zip(res["b200"], res["ref"]):
        assert float(np.max(np.abs(a - b))) <= 1e-3 * float(np.abs(b).max())


def test_backward_consume_once_and_zero_grad(swarm):
    """tests/test_server.py:212-236: a tape serves one BACKWARD
    (ERR_UNKNOWN_TAPE after), a zero gradient gives an exactly zero reply."""
    from swarmlm.errors import ERR_UNKNOWN_TAPE, RemoteError
    from swarmlm.transport import ENC_F32, MSG, decode_tensor, encode_tensor, rpc_call

    node = swarm.b200((0, 4))
    rng = np.random.default_rng(1)
    batch = rng.uniform(-0.5, 0.5, (1, 2, 16)).astype(np.float32)
    reply = rpc_call(node.address, MSG.FORWARD, encode_tensor(batch, ENC_F32), 10000.0)
    zero = encode_tensor(np.zeros_like(batch), ENC_F32)
    gin = decode_tensor(rpc_call(node.address, MSG.BACKWARD, reply[:16] + zero, 10000.0))
    assert np.array_equal(gin, np.zeros_like(batch))
    with pytest.raises(RemoteError) as ei:
        rpc_call(node.address, MSG.BACKWARD, reply[:16] + zero, 10000.0)
    assert ei.value.code == ERR_UNKNOWN_TAPE
    with pytest.raises(RemoteError) as ei:
        rpc_call(node.address, MSG.BACKWARD, os.urandom(16) + zero, 10000.0)
    assert ei.value.code == ERR_UNKNOWN_TAPE


def test_distributed_backward_matches_reference_client(small_ckpt):
    """The reference client's DistributedModel.forward/backward (client.py:417-498)
    over two B200 spans equals the same calls over two reference servers."""
    from swarmlm.client import DistributedModel

    rng = np.random.default_rng(5)
    batch = rng.uniform(-0.5, 0.5, (2, 4, 16)).astype(np.float32)
    grad = rng.uniform(-1, 1, (2, 4, 16)).astype(np.float32)
    outs = {}
    for kind in ("ref", "b200"):
        sw = Swarm(small_ckpt)
        try:
            for r in ((0, 2), (2, 4)):
                (sw.reference if kind == "ref" else sw.b200)(r)
            cl = sw.client()
            try:
                dm = DistributedModel(cl)
                h, handles = dm.forward(batch)
                outs[kind] = (h, dm.backward(handles, grad))
            finally:
                cl.close()
        finally:
            sw.close()
    for a, b in zip(outs["b200"], outs["ref"]):
        assert float(np.max(np.abs(a - b))) <= 1e-3 * float(np.abs(b).max())


def test_box_serves_reference_client_in_one_hop(small_ckpt):
    """The box front end (two sub-span processes, peer-memory hop) announces
    ONE ServerEntry [0, 4) to the reference registry; the reference client's
    plan is a single hop, and its generate() equals reference_generate
    (client.py:230-257, registry.py:40)."""
    from swarmlm.model import reference_generate

    from paper_2209_01188_b200.box import LocalBox
    from paper_2209_01188_b200.model import ModelConfig
    from paper_2209_01188_b200.server import ServerConfig

    sw = Swarm(small_ckpt)
    box = None
    try:
        cfg = ServerConfig(seed=42, model=ModelConfig(4, 16, 2, 32, 128), bootstrap=[sw.seed.address],
                           measure_steps=3, page_tokens=16)
        box = LocalBox(cfg, 2)
        c = sw.client()
        try:
            plan = c.plan()
            assert len(plan) == 1 and (plan[0].entry.range.start, plan[0].entry.range.end) == (0, 4)
            assert c.generate([1, 2, 3], 16) == reference_generate(small_ckpt, [1, 2, 3], 16)
        finally:
            c.close()
    finally:
        if box is not None:
            assert box.stop() == [0, 0]
        sw.close()
