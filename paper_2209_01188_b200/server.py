"""Span server: the drop-in for the reference's ServerNode compute path
(/root/reference/pkg/src/swarmlm/server.py:48-450), same constructor shape,
same RPC messages, same session semantics and error codes, with the hosted
blocks executed by a B200 BlockSpan.

Kept from the reference (restated, not imported):
  OPEN_SESSION / STEP / CLOSE_SESSION / FORWARD / INFO / PING handlers
  (server.py:295-429), idempotent STEP retry by sha256 digest
  (server.py:367,374-377), DESYNC / CAPACITY / BUSY / UNKNOWN_SESSION codes,
  LRU cache-budget eviction (server.py:397-407), idle-session janitor
  (server.py:223-233), registry announcements (server.py:171-195).
Changed for the B200:
  sessions' KV caches are pages of one HBM pool; concurrent STEPs of different
  sessions are coalesced into one batched span step by a scheduler thread;
  the int8 wire codec runs on the GPU; FORWARD runs on the span's weights.
Out of scope: BACKWARD (a "next" row), rebalancing/allocation
(control plane); maybe_rebalance() reports no move.
"""

from __future__ import annotations

import hashlib
import json
import logging
import os
import queue
import struct
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import codec
from .errors import (
    ERR_BAD_REQUEST,
    ERR_GENERIC,
    ERR_BUSY,
    ERR_CAPACITY,
    ERR_DESYNC,
    ERR_UNKNOWN_SESSION,
    ERR_UNKNOWN_TAPE,
    CapacityError,
    InputError,
    RemoteError,
    SwarmError,
)
from .model import ModelConfig
from .rpc import RpcServer, as_view as rpc_view, call
from .span import BlockSpan
from .wire import MSG

log = logging.getLogger(__name__)

DEFAULT_CAPACITY = 64
DEFAULT_CACHE_BUDGET = 65536
SESSION_IDLE_TIMEOUT_S = 120.0
TAPE_TTL_S = 60.0  # server.py:43
_TIMING = os.environ.get("PB_SERVER_TIMING") == "1"  # diagnostic: per-STEP decode / compute / encode seconds
SERVER_VERSION = "0.1.0-b200"
DEFAULT_NET_BYTES_PER_S = 1.25e8
DEFAULT_TTL_MS = 30_000
TOMBSTONE_TTL_MS = 10_000


@dataclass(frozen=True, order=True)
class BlockRange:
    start: int
    end: int

    def __len__(self) -> int:
        return self.end - self.start


@dataclass
class ServerConfig:
    """Reference fields (server.py:48-66) plus B200 knobs."""

    checkpoint_path: str = ""
    host: str = "127.0.0.1"
    port: int = 0
    blocks: object = "auto"  # "auto" (whole model) or (start, end)
    span: int | None = None
    quantize: str = "none"  # none | activations | weights | both
    bootstrap: list = field(default_factory=list)
    shape: object = None  # link shaping is not emulated on the box
    capacity: int = DEFAULT_CAPACITY
    cache_budget_tokens: int = DEFAULT_CACHE_BUDGET
    ttl_ms: int = DEFAULT_TTL_MS
    gossip_period_ms: int = 2_000
    rebalance_eps: float = 0.2
    rebalance_period_s: tuple = (5.0, 10.0)
    measure_steps: int = 100
    net_bytes_per_s: float = DEFAULT_NET_BYTES_PER_S
    remeasure_period_s: float = 60.0
    # B200 additions
    seed: int | None = None           # generate gen_checkpoint(seed) weights on device
    model: ModelConfig | None = None  # shape when generating
    device: int = 0
    page_tokens: int = 64
    max_batch_tokens: int = 256
    kv_pages: int | None = None


# ------------------------------------------------------------------ checkpoints


def read_ptck(path: str, block_range=None):
    """Parse a PTCK file (model.py:213-264 layout, restated): returns
    (ModelConfig, {block_index: {name: f32 array}}) for the requested blocks only."""
    with open(path, "rb") as f:
        data = f.read()
    if data[:4] != b"PTCK":
        raise InputError("not a checkpoint file (bad magic)")
    if data[4] != 1:
        raise InputError(f"unsupported checkpoint version {data[4]}")
    L, d, h, v, ms, r = struct.unpack(">6I", data[5:29])
    cfg = ModelConfig(L, d, h, v, ms, r)
    off = 29 + 4 * v * d  # skip embed
    names = [("ln1_gamma", d), ("ln1_beta", d), ("wqkv", d * 3 * d), ("bqkv", 3 * d), ("wo", d * d), ("bo", d),
             ("ln2_gamma", d), ("ln2_beta", d), ("wmlp_in", d * r * d), ("bmlp_in", r * d),
             ("wmlp_out", r * d * d), ("bmlp_out", d)]
    shapes = {"wqkv": (d, 3 * d), "wo": (d, d), "wmlp_in": (d, r * d), "wmlp_out": (r * d, d)}
    per_block = sum(n for _, n in names)
    want = set(range(*block_range)) if block_range else set(range(L))
    blocks = {}
    for i in range(L):
        if i in want:
            o = off
            arrs = {}
            for nm, n in names:
                a = np.frombuffer(data, "<f4", count=n, offset=o).astype(np.float32)
                arrs[nm] = a.reshape(shapes.get(nm, (n,)))
                o += 4 * n
            blocks[i] = arrs
        off += 4 * per_block
    if off + 8 * d != len(data):
        raise InputError("checkpoint size mismatch")
    return cfg, blocks


class _BlockView:
    def __init__(self, d: dict):
        self.__dict__.update(d)


def _block_tensors(b):
    """(name, f32 array) in the checkpoint traversal order (model.py:102-117)."""
    names = ["ln1_gamma", "ln1_beta", "wqkv", "bqkv", "wo", "bo", "ln2_gamma", "ln2_beta", "wmlp_in", "bmlp_in",
             "wmlp_out", "bmlp_out"]
    return [(n, np.asarray(getattr(b, n), np.float32)) for n in names]


# ------------------------------------------------------------------ sessions / scheduling


class _Session:
    def __init__(self, sid: bytes, seq, max_len: int):
        self.session_id = sid
        self.seq = seq
        self.position = 0
        self.max_len = max_len
        self.last_active = time.monotonic()
        self.lock = threading.Lock()
        self.last_step = None  # (start_pos, digest, reply)
        self.poisoned = False  # a non-finite hidden state entered the caches (reference: NaN KV)


class _NonFinite(InputError):
    """The computed hidden state is not finite: encoding the reply fails."""


class _Job:
    __slots__ = ("seq", "msg", "t", "enc", "res", "err", "done", "ev")

    def __init__(self, seq, msg, enc):
        self.seq, self.msg, self.enc = seq, msg, enc
        self.t = msg.rows
        self.res = self.err = self.ev = None
        self.done = threading.Event()


class StepScheduler:
    """Coalesces concurrent STEPs of distinct sessions into one batched span
    step (one launch sequence per block for the whole batch), with the wire
    codec of the whole batch on the scheduler's stream: the handlers only DMA
    their TensorMsg sections to the device (codec.upload_tensor) and slice
    their reply out of one pinned copy of the batch's encoded output. (Codec
    kernels on the handlers' own streams queued behind the next batch's
    persistent kernels, which hold every SM: 1-2 ms per STEP at 8 sessions.)"""

    # batches queued on the GPU at once. Measured (7B1, one GPU, 8 / 16 sessions over TCP, bench e2e):
    # 1 -> 847 / 1031 tokens/s, 2 -> 835 / 966, 3 -> 763 / 874, unbounded -> 501 / 651
    MAX_INFLIGHT = 1

    def __init__(self, span: BlockSpan, max_tokens: int, max_seqs: int):
        self.span, self.max_tokens, self.max_seqs = span, max_tokens, max_seqs
        self.q: queue.Queue = queue.Queue()
        self.batches = 0
        self.batched_steps = 0
        self._stop = False
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()

    def run(self, seq, msg, encoding: int) -> bytes:
        """Queue one STEP (msg: codec.DeviceTensorMsg [t, d]) and return the
        reply TensorMsg bytes in `encoding`. The scheduler thread only enqueues
        the batch and moves on; the wait for the batch's completion event
        happens here, in the handler's thread (msg stays referenced until the
        step has read it). Non-finite output raises InputError, as encoding
        it does (transport/wire.py:89-90)."""
        job = _Job(seq, msg, encoding)
        self.q.put(job)
        job.done.wait()
        if job.err is not None:
            raise job.err
        job.ev.synchronize()
        return self._reply(job)

    def stop(self):
        self._stop = True
        self.q.put(None)

    # ---------------------------------------------------------------- batch execution

    def _execute(self, ready):
        """One batch on the current stream: decode, step, encode, one D2H copy.
        Returns the batch's completion event (its jobs get their reply slices)."""
        import torch

        span, d = self.span, self.span.config.hidden
        dev = span.device
        seqs, lens = [j.seq for j in ready], [j.t for j in ready]
        ntok, enc = sum(lens), ready[0].enc
        codes = scales = y = None
        whole = d % 64 == 0  # 64-value blocks never straddle rows: one batch-wide quantization
        if (enc == codec.ENC_INT8 and whole and ntok <= span.max_tokens and len(ready) <= span.max_seqs
                and all(j.msg.encoding == codec.ENC_INT8 and j.msg.block_size == 64 for j in ready)):
            # int8 in, int8 out: dequantize, blocks, quantize inside one C-ABI call (pb_span_step_int8)
            cat = (lambda xs: xs[0]) if len(ready) == 1 else torch.cat
            y = torch.empty(ntok, d, dtype=torch.float32, device=dev)
            codes = torch.empty(ntok * d, dtype=torch.int8, device=dev)
            scales = torch.empty(ntok * d // 64, dtype=torch.float32, device=dev)
            span.step_codes(seqs, lens, in_codes=cat([j.msg.codes for j in ready]),
                            in_scales=cat([j.msg.scales for j in ready]), out_codes=codes, out_scales=scales, out_f32=y)
        else:
            outs = span.step([(j.seq, j.msg.decode().reshape(j.t, d)) for j in ready])
            y = outs[0] if len(outs) == 1 else torch.cat(outs)
            if enc == codec.ENC_INT8:
                if whole:
                    q = codec.quantize_blockwise(y.reshape(-1), 64)
                    codes, scales = q.codes, q.scales
                else:
                    qs = [codec.quantize_blockwise(y[r0:r0 + t].reshape(-1), 64)
                          for r0, t in zip(np.cumsum([0] + lens[:-1]), lens)]
                    codes, scales = torch.cat([q.codes for q in qs]), torch.cat([q.scales for q in qs])
        flags = torch.isfinite(y).all(dim=1).to(torch.uint8)
        # one pinned buffer: [scales f32 | codes int8] (int8 reply) or [values f32], then the row flags
        nsc = 0 if scales is None else scales.numel()
        body = 4 * nsc + codes.numel() if codes is not None else 4 * ntok * d
        buf = torch.empty(body + ntok, dtype=torch.uint8, pin_memory=True)
        if codes is not None:
            buf[:4 * nsc].view(torch.float32).copy_(scales, non_blocking=True)
            buf[4 * nsc:body].view(torch.int8).copy_(codes, non_blocking=True)
        else:
            buf[:body].view(torch.float32).copy_(y.reshape(-1), non_blocking=True)
        buf[body:].copy_(flags, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(dev))
        host = buf.numpy()
        r0 = c0 = s0 = 0
        for j, t in zip(ready, lens):
            nb = -(-t * d // 64)
            j.res = (buf, host, body, nsc, r0, c0, s0)
            j.ev = ev
            r0, c0, s0 = r0 + t, c0 + t * d, s0 + nb
        return ev

    def _reply(self, job) -> bytes:
        buf, host, body, nsc, r0, c0, s0 = job.res
        t, d = job.t, self.span.config.hidden
        if not host[body + r0:body + r0 + t].all():
            raise _NonFinite("non-finite tensor")
        head = codec.encode_header(job.enc, (t, d))
        if job.enc == codec.ENC_F32:
            return head + host[4 * c0:4 * (c0 + t * d)].tobytes()
        nb = -(-t * d // 64)
        return (head + struct.pack(">I", 64) + host[4 * s0:4 * (s0 + nb)].tobytes()
                + host[4 * nsc + c0:4 * nsc + c0 + t * d].tobytes())

    def _loop(self):
        import torch

        torch.cuda.set_device(self.span.device)
        pending = None
        inflight: list = []  # completion events of launched batches, oldest first
        while not self._stop:
            job = pending or self.q.get()
            pending = None
            if job is None:
                break
            # at most MAX_INFLIGHT batches queued on the GPU: the next launch waits for the
            # oldest to finish, and the STEPs arriving meanwhile join the batch (continuous
            # batching) instead of each becoming a small launch of its own
            while len(inflight) >= self.MAX_INFLIGHT:
                inflight.pop(0).synchronize()
            batch, ntok = [job], job.t
            while len(batch) < self.max_seqs:
                try:
                    nxt = self.q.get_nowait()
                except queue.Empty:
                    break
                if nxt is None:
                    self._stop = True
                    break
                if ntok + nxt.t > self.max_tokens or nxt.enc != job.enc:
                    pending = nxt
                    break
                batch.append(nxt)
                ntok += nxt.t
            # pages are reserved per job: a session the pool cannot extend fails
            # alone (CapacityError -> the handler makes room or answers BUSY)
            # instead of failing every co-batched session
            ready = []
            for j in batch:
                try:
                    self.span.reserve(j.seq, j.seq.length + j.t)
                    ready.append(j)
                except CapacityError as e:
                    j.err = e
            try:
                if ready:
                    inflight.append(self._execute(ready))
            except Exception as e:  # noqa: BLE001
                for j in ready:
                    j.err = e
            self.batches += 1
            self.batched_steps += len(batch)
            for j in batch:
                j.done.set()


# ------------------------------------------------------------------ server


class ServerNode:
    def __init__(self, config: ServerConfig, checkpoint=None, span: BlockSpan | None = None):
        """`span` (optional) is an already-loaded BlockSpan for config.blocks
        (bench.py reuses the 176B-shape span instead of building a second one)."""
        self.config = config
        self._given_span = span
        self.server_id = os.urandom(16).hex()
        self.events: list = []
        self.throughput = 0.0
        self.range: BlockRange | None = None
        self._sessions: dict = {}
        self._sessions_lock = threading.Lock()
        self.timing: list = []  # PB_SERVER_TIMING diagnostics
        self._tapes: dict[bytes, tuple[float, object]] = {}  # tape_id -> (born, device tape [B, n_blocks, t, d])
        self._tapes_lock = threading.Lock()
        self._io = threading.local()
        self._stop = threading.Event()
        self.rpc: RpcServer | None = None
        self._ckpt = checkpoint
        self._blocks_host = None
        if checkpoint is not None:
            self.model = checkpoint.config
        elif config.seed is not None:
            if config.model is None:
                raise InputError("seed-generated weights need ServerConfig.model")
            self.model = config.model
        else:
            if not os.path.exists(config.checkpoint_path):
                raise InputError(f"checkpoint {config.checkpoint_path!r} not found")
            self.model, _ = read_ptck(config.checkpoint_path, (0, 0))
        self.model = ModelConfig(self.model.n_layers, self.model.hidden, self.model.n_heads, self.model.vocab,
                                 self.model.max_seq, self.model.mlp_ratio)
        self.span: BlockSpan | None = None
        self._weights_hash = None

    # ---------------------------------------------------------------- lifecycle

    def _pick_range(self) -> BlockRange:
        L = self.model.n_layers
        if self.config.blocks != "auto":
            s, e = self.config.blocks
            if not (0 <= s < e <= L):
                raise InputError(f"explicit block range [{s}, {e}) outside [0, {L})")
            return BlockRange(s, e)
        k = self.config.span or L
        if k > L:
            raise InputError("span exceeds layer count")
        return BlockRange(0, k)  # allocation policy is control plane (out of scope)

    def start(self) -> "ServerNode":
        import torch

        self.range = self._pick_range()
        n = len(self.range)
        int8 = self.config.quantize in ("weights", "both")
        pos_budget = max(1, self.config.cache_budget_tokens // n)
        # the budget's positions + one partial page per session + one maximal
        # STEP in flight before _enforce_cache_budget runs (server.py:389)
        pages = self.config.kv_pages or (-(-pos_budget // self.config.page_tokens) + self.config.capacity + 2
                                         + -(-self.model.max_seq // self.config.page_tokens))
        torch.cuda.set_device(self.config.device)
        if self._given_span is not None:
            self.span = self._given_span
            if (self.span.start, self.span.end) != (self.range.start, self.range.end) or self.span.int8 != int8:
                raise InputError("given span does not match the configured range / quantize mode")
            self._weights_hash = hashlib.sha256(f"span:{self.model}:{self.range}".encode()).hexdigest()
        else:
            self.span = self._make_span(int8, pages)
        self.sched = self._make_scheduler()
        self.rpc = RpcServer(self.config.host, self.config.port, self._dispatch,
                             pinned_device=self.config.device).start()
        self._announce("joining", throughput=1e-6)
        self.throughput = self.measure_throughput()
        self._announce("online")
        for target in (self._announce_loop, self._janitor_loop):
            threading.Thread(target=target, daemon=True).start()
        log.info("b200 server %s serving blocks [%d, %d) at %s", self.server_id[:8], self.range.start,
                 self.range.end, self.address)
        return self

    def _make_span(self, int8: bool, pages: int):
        """The hosted blocks on this process's GPU (overridden by the box front end)."""
        span = BlockSpan(self.model, self.range.start, self.range.end, int8=int8,
                         page_tokens=self.config.page_tokens, n_pages=pages,
                         max_tokens=self.config.max_batch_tokens, max_seqs=max(1, self.config.capacity),
                         device=self.config.device)
        self.span = span
        self._load_weights()
        return span

    def _make_scheduler(self):
        return StepScheduler(self.span, self.config.max_batch_tokens, max(1, self.config.capacity))

    def _load_weights(self):
        if self.config.seed is not None and self._ckpt is None:
            self.span.generate_weights(self.config.seed)
            h = hashlib.sha256(f"gen:{self.config.seed}:{self.model}:{self.range}".encode())
            self._weights_hash = h.hexdigest()
            return
        if self._ckpt is not None:
            blocks = [self._ckpt.blocks[i] for i in range(self.range.start, self.range.end)]
        else:
            _, bl = read_ptck(self.config.checkpoint_path, (self.range.start, self.range.end))
            blocks = [_BlockView(bl[i]) for i in range(self.range.start, self.range.end)]
        h = hashlib.sha256()  # server.py:286-291
        for b in blocks:
            for _, arr in _block_tensors(b):
                h.update(np.ascontiguousarray(arr, "<f4").tobytes())
        self._weights_hash = h.hexdigest()
        self.span.load_weights(blocks)

    @property
    def address(self) -> str:
        return self.rpc.address

    def stop(self):
        if self._stop.is_set():
            return
        try:
            self._announce("offline", ttl_ms=TOMBSTONE_TTL_MS)
        except SwarmError:
            pass
        self._shutdown()

    def kill(self):
        self._shutdown()

    def _shutdown(self):
        self._stop.set()
        if self.rpc:
            self.rpc.stop()
        if getattr(self, "sched", None):
            self.sched.stop()

    # ---------------------------------------------------------------- registry

    def _entry(self, state: str, throughput=None, ttl_ms=None) -> dict:
        """ServerEntry dict (registry.py:40) announced to the bootstrap peers."""
        return {
            "id": self.server_id, "address": self.address, "start": self.range.start, "end": self.range.end,
            "throughput": throughput if throughput is not None else max(self.throughput, 1e-6),
            "announced_at": int(time.time() * 1000), "ttl_ms": ttl_ms or self.config.ttl_ms, "state": state,
        }

    def _announce(self, state: str, throughput=None, ttl_ms=None):
        """server.py:171-195: push our entry to the registry seeds. Discovery
        itself (LOOKUP / GOSSIP replicas) is control plane and stays with the
        reference's registry."""
        entry = self._entry(state, throughput, ttl_ms)
        self.events.append({"t": entry["announced_at"], "event": "announce", "state": state,
                            "range": [self.range.start, self.range.end]})
        payload = json.dumps(entry).encode()
        for peer in self.config.bootstrap:
            try:
                call(peer, MSG.ANNOUNCE, payload, 3000.0)
            except SwarmError as e:
                log.debug("announce to %s failed: %s", peer, e)

    def _announce_loop(self):
        period = self.config.ttl_ms / 3000.0
        while not self._stop.wait(period):
            self._announce("online")

    def _janitor_loop(self):
        while not self._stop.wait(5.0):
            now = time.monotonic()
            with self._sessions_lock:
                stale = [sid for sid, s in self._sessions.items() if now - s.last_active > SESSION_IDLE_TIMEOUT_S]
                victims = [self._sessions.pop(sid) for sid in stale]
            for v in victims:
                self.span.release(v.seq)
            with self._tapes_lock:  # server.py:230-233
                expired = [self._tapes.pop(tid)[1] for tid, (born, _) in list(self._tapes.items())
                           if now - born > TAPE_TTL_S]
            drop = getattr(self.span, "drop_tape", None)  # tapes held on other GPUs (box front end)
            for tape in expired:
                if drop is not None:
                    drop(tape)

    def maybe_rebalance(self) -> bool:
        return False  # allocation/rebalancing is control plane (out of scope)

    # ---------------------------------------------------------------- measurement

    def measure_throughput(self) -> float:
        """min(compute, network) tokens/s over the hosted span (server.py:262-282),
        compute measured with single-token steps on the GPU."""
        import torch

        steps = max(1, min(self.config.measure_steps, self.model.max_seq))
        seq = self.span.new_sequence()
        x = torch.zeros(1, self.model.hidden, device=self.span.device)
        try:
            self.span.step([(seq, x)])  # warm-up
            torch.cuda.synchronize(self.span.device)
            t0 = time.perf_counter()
            for _ in range(min(steps, self.model.max_seq - 1)):
                self.span.step([(seq, x)])
            torch.cuda.synchronize(self.span.device)
            compute = max(1, min(steps, self.model.max_seq - 1)) / max(time.perf_counter() - t0, 1e-9)
        finally:
            self.span.release(seq)
        net = self.config.net_bytes_per_s
        return min(compute, net / (4.0 * self.model.hidden))

    def weights_hash(self) -> str:
        return self._weights_hash

    # ---------------------------------------------------------------- RPC
    #
    # Handlers take an rpc.Payload (a zero-copy view of the received frame,
    # page-locked for tensor-sized payloads) and return reply bytes. Error codes
    # follow the reference handler by handler (server.py:295-450): malformed
    # TensorMsg bytes and blocks rejecting the hidden width escape its handlers
    # as exceptions, i.e. ERR_GENERIC "internal error: ..." (transport/rpc.py:247-250).

    def _dispatch(self, msg_type: int, payload):
        if msg_type == MSG.PING:
            return MSG.PING, b""
        if msg_type == MSG.INFO:
            return MSG.INFO, self._info_payload()
        if msg_type == MSG.OPEN_SESSION:
            return MSG.OPEN_SESSION, self._open_session(payload)
        if msg_type == MSG.STEP:
            return MSG.STEP, self._step(payload)
        if msg_type == MSG.CLOSE_SESSION:
            return MSG.CLOSE_SESSION, self._close_session(payload)
        if msg_type == MSG.FORWARD:
            return MSG.FORWARD, self._forward(payload)
        if msg_type == MSG.BACKWARD:
            return MSG.BACKWARD, self._backward(payload)
        if msg_type == MSG.ANNOUNCE:  # accepted and ignored: discovery is the registry's job
            return MSG.ANNOUNCE, b""
        if msg_type == MSG.LOOKUP:
            return MSG.LOOKUP, b"[]"
        if msg_type == MSG.GOSSIP:
            return MSG.GOSSIP, b"[]"
        raise RemoteError(ERR_BAD_REQUEST, f"unknown message type 0x{msg_type:02x}")

    def _info_payload(self) -> bytes:
        return json.dumps({
            "server_id": self.server_id, "range": [self.range.start, self.range.end],
            "throughput": self.throughput, "position_capacity": self.config.cache_budget_tokens,
            "version": SERVER_VERSION, "weights_hash": self.weights_hash(), "quantize": self.config.quantize,
        }).encode()

    def _reply_encoding(self) -> int:
        return codec.ENC_INT8 if self.config.quantize in ("activations", "both") else codec.ENC_F32

    def _open_session(self, payload) -> bytes:
        if len(payload) != 20:
            raise RemoteError(ERR_BAD_REQUEST, "OPEN_SESSION wants 16-byte id + u32 max_len")
        sid, (max_len,) = bytes(payload[:16]), struct.unpack(">I", bytes(payload[16:20]))
        if max_len < 1 or max_len > self.model.max_seq:
            raise RemoteError(ERR_BAD_REQUEST, f"max_len must be in [1, {self.model.max_seq}]")
        with self._sessions_lock:
            if sid in self._sessions:
                raise RemoteError(ERR_BAD_REQUEST, "duplicate session id")
            if len(self._sessions) >= self.config.capacity:
                raise RemoteError(ERR_BUSY, "session capacity exhausted")
            self._sessions[sid] = _Session(sid, self.span.new_sequence(), max_len)
        return b""

    def _get_session(self, sid: bytes) -> _Session:
        with self._sessions_lock:
            s = self._sessions.get(sid)
        if s is None:
            raise RemoteError(ERR_UNKNOWN_SESSION, "unknown session")
        return s

    # Request / reply codec work runs on a per-handler-thread CUDA stream: on the
    # compute stream a reply's quantize + D2H (and a request's H2D) would queue
    # behind whatever step the scheduler launched next -- milliseconds per hop
    # at the 176B shape. The H2D is complete when _decode returns (the page-locked
    # receive block goes back to the pool right after the handler).

    def _io_stream(self):
        import torch

        st = getattr(self._io, "stream", None)
        if st is None:
            st = self._io.stream = torch.cuda.Stream(device=self.span.device)
        return st

    def _decode(self, data):
        import torch

        st = self._io_stream()
        with torch.cuda.stream(st):
            x = codec.decode_tensor(data, device=self.span.device)
        st.synchronize()
        return x

    def _run_step(self, seq, msg, encoding: int) -> bytes:
        """One STEP through the span (hook: the box front end runs it through its ring)."""
        return self.sched.run(seq, msg, encoding)

    def _upload(self, data):
        """STEP ingress: the TensorMsg sections to the device (DMA only)."""
        import torch

        st = self._io_stream()
        with torch.cuda.stream(st):
            msg = codec.upload_tensor(data, device=self.span.device)
        st.synchronize()
        return msg

    def _encode(self, t, encoding, producer=None):
        """producer: the stream that computed `t` when that work may still be
        queued (FORWARD / BACKWARD run on the handler's default stream); STEP
        outputs are complete when the scheduler hands them over."""
        import torch

        st = self._io_stream()
        if producer is not None:
            st.wait_stream(producer)
        with torch.cuda.stream(st):
            return codec.encode_tensor(t, encoding)

    @staticmethod
    def _internal(e: Exception) -> RemoteError:
        return RemoteError(ERR_GENERIC, f"internal error: {e}")

    def _step(self, payload) -> bytes:
        if len(payload) < 20:
            raise RemoteError(ERR_BAD_REQUEST, "short STEP payload")
        sid = bytes(payload[:16])
        (start_pos,) = struct.unpack(">I", bytes(payload[16:20]))
        session = self._get_session(sid)
        tensor = payload[20:]
        digest = hashlib.sha256(rpc_view(tensor)).digest()
        try:
            _, dims, _, _, _ = codec.parse_tensor(tensor)
        except SwarmError as e:
            raise self._internal(e) from e
        if len(dims) != 2:
            raise RemoteError(ERR_BAD_REQUEST, "STEP tensor must be 2-D [t, d]")
        t = dims[0]
        with session.lock:
            session.last_active = time.monotonic()
            if session.last_step is not None and start_pos + t == session.position:
                last_pos, last_digest, last_reply = session.last_step
                if last_pos == start_pos and last_digest == digest:
                    return last_reply
            if start_pos != session.position:
                raise RemoteError(ERR_DESYNC, f"position mismatch: got {start_pos}, have {session.position}")
            if start_pos + t > session.max_len:
                raise RemoteError(ERR_CAPACITY, "session exceeds max_len")
            if dims[1] != self.model.hidden or t < 1:
                raise self._internal(InputError(f"hidden must be [t, {self.model.hidden}]"))
            with self._sessions_lock:
                if self._sessions.get(sid) is not session:
                    raise RemoteError(ERR_UNKNOWN_SESSION, "session evicted")
            if session.poisoned or not codec.payload_finite(tensor):
                # the reference computes NaN/inf hidden states and fails encoding the reply
                # (transport/wire.py:89-90 -> ERR_GENERIC) after advancing the position
                # (server.py:386-387); every later step of the session fails the same way
                session.poisoned = True
                session.position += t
                raise RemoteError(ERR_GENERIC, "internal error: non-finite tensor")
            tm = [time.perf_counter()] if _TIMING else None
            msg = self._upload(tensor)
            if tm:
                tm.append(time.perf_counter())
            enc = self._reply_encoding()
            try:
                reply = self._run_step(session.seq, msg, enc)
            except CapacityError:
                # the pool is short of pages for this step: the reference never
                # refuses a step for memory (it evicts after computing,
                # server.py:389), so evict idle LRU sessions now and retry once
                self._make_room(session, t)
                try:
                    reply = self._run_step(session.seq, msg, enc)
                except CapacityError as e:
                    raise RemoteError(ERR_BUSY, f"KV pool exhausted: {e}") from e
            except _NonFinite:
                session.position += t  # computed, then failed encoding the reply (as the reference)
                raise
            session.position += t
            if tm:
                tm.append(time.perf_counter())
            session.last_step = (start_pos, digest, reply)
            if tm:
                tm.append(time.perf_counter())
                self.timing.append(tuple(b - a for a, b in zip(tm, tm[1:])))
        self._enforce_cache_budget()
        return reply

    def _close_session(self, payload) -> bytes:
        with self._sessions_lock:
            s = self._sessions.pop(bytes(payload[:16]), None)
        if s is not None:
            with s.lock:
                self.span.release(s.seq)
        return b""

    def _make_room(self, requester: _Session, t: int) -> None:
        """Evict least-recently-active sessions other than `requester` (never
        one with a step in flight) until the pool can extend the requester by
        t positions."""
        need = self.span.pages_needed(requester.seq, requester.seq.length + t)
        with self._sessions_lock:
            order = sorted((s for s in self._sessions.values() if s is not requester), key=lambda s: s.last_active)
        for v in order:
            if self.span.pool.free_pages >= need:
                return
            if not v.lock.acquire(blocking=False):
                continue
            try:
                with self._sessions_lock:
                    if self._sessions.get(v.session_id) is v:
                        del self._sessions[v.session_id]
                self.span.release(v.seq)
            finally:
                v.lock.release()

    def _enforce_cache_budget(self):
        n = len(self.range)
        victims = []
        with self._sessions_lock:
            total = sum(s.position * n for s in self._sessions.values())
            if total > self.config.cache_budget_tokens:
                for v in sorted(self._sessions.values(), key=lambda s: s.last_active):
                    del self._sessions[v.session_id]
                    victims.append(v)
                    total -= v.position * n
                    if total <= self.config.cache_budget_tokens:
                        break
        for v in victims:
            with v.lock:
                self.span.release(v.seq)

    def _forward(self, payload) -> bytes:
        try:
            finite = codec.payload_finite(payload)
            batch = self._decode(payload)
        except SwarmError as e:
            raise self._internal(e) from e
        if batch.ndim != 3:
            raise RemoteError(ERR_BAD_REQUEST, "FORWARD tensor must be [B, t, d]")
        if batch.shape[2] != self.model.hidden:
            raise self._internal(InputError(f"hidden must be [t, {self.model.hidden}]"))
        if not finite:  # the reference computes NaN/inf and fails encoding the reply (wire.py:89-90)
            raise RemoteError(ERR_GENERIC, "internal error: non-finite tensor")
        try:
            out, tape = self.span.forward(batch, tape=True)
        except CapacityError as e:
            raise self._internal(e) from e
        tape_id = os.urandom(16)
        with self._tapes_lock:  # server.py:426-428
            self._tapes[tape_id] = (time.monotonic(), tape)
        import torch

        return tape_id + self._encode(out, self._reply_encoding(), torch.cuda.current_stream(self.span.device))

    def _backward(self, payload) -> bytes:
        """server.py:431-450: consume-once tape, f32 reply (gradients travel at full precision)."""
        if len(payload) < 16:
            raise RemoteError(ERR_BAD_REQUEST, "short BACKWARD payload")
        with self._tapes_lock:
            item = self._tapes.pop(bytes(payload[:16]), None)
        if item is None:
            raise RemoteError(ERR_UNKNOWN_TAPE, "unknown or expired tape")
        _, tape = item
        try:
            grad = self._decode(payload[16:])
        except SwarmError as e:
            raise self._internal(e) from e
        if grad.ndim != 3 or grad.shape[0] != tape.shape[0]:
            raise RemoteError(ERR_BAD_REQUEST, "BACKWARD grad shape mismatch")
        if tuple(grad.shape[1:]) != tuple(tape.shape[2:]):
            raise self._internal(InputError("BACKWARD grad shape mismatch"))
        import torch

        gin = self.span.backward(tape, grad)
        return self._encode(gin, codec.ENC_F32, torch.cuda.current_stream(self.span.device))
