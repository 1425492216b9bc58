"""Box front end: ONE span server for blocks [s, e) executed by N GPUs of
one box, one process per GPU.

The reference relays every hop through the client (client.py:312-331: decode
the server's reply, re-encode, send to the next server over TCP). Here the
registry sees a single ServerEntry [s, e) (registry.py:40, announced by rank
0), the client makes one STEP, and the hops between the consecutive sub-spans
(split_blocks: 70 blocks over 8 GPUs -> 9,9,9,9,9,9,8,8) never leave the
box: sub-span r's last kernel stores the hidden state straight into sub-span
r+1's mailbox in that GPU's HBM (CUDA IPC over NVLink, pb_hop.cu), a
one-thread kernel publishes the job, and r+1's stream waits on it. The last
sub-span writes the result into rank 0's mailbox; rank 0 encodes the reply.

Hop payload: the wire codec (int8 codes + f32 scales, 15 232 B per token at
h=14336) when the server compresses activations (quantize in {activations,
both}: the exact bytes a reference client would relay between servers of
that mode), f32 otherwise (then the box computes what ONE reference server
hosting [s, e) computes).

Control plane (rank 0 -> ranks 1..N-1, gloo over loopback): one fixed-size
int64 descriptor per job, sent before rank 0 launches its own part so the
other ranks enqueue their wait/step/signal ahead of the data. Every rank
applies the same descriptors in the same order, so:
  * causality: jobs of one session (e.g. the causal chunks of a long prompt)
    run in submission order on every GPU;
  * KV pages: each rank's pool sees the identical alloc/free sequence, so a
    reservation that succeeds on rank 0 succeeds everywhere (rank 0 decides);
  * mailbox slots: job j uses slot j % (D + 1) and at most D jobs are in
    flight between rank 0's submit and rank 0's completion, so a slot is
    never overwritten before every rank consumed it.
FORWARD rows travel the same ring with each rank keeping its own tape piece;
BACKWARD walks the ranks in reverse over the control plane (f32 gradients,
not a hot path).
"""

from __future__ import annotations

import itertools
import logging
import os
import queue
import struct
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import codec

from .errors import CapacityError, InputError
from .pipeline import DevPtr, P2PRing, dev_view, split_blocks
from .server import ServerConfig, ServerNode, _NonFinite
from .span import BlockSpan, Sequence

log = logging.getLogger(__name__)

OP_STEP, OP_RELEASE, OP_FORWARD, OP_BACKWARD, OP_DROP, OP_STOP = 1, 2, 3, 4, 5, 6
_TIMING = os.environ.get("PB_SERVER_TIMING") == "1"
HEAD = 12  # op, job, n_seq, fmt, key, B, t, r0, c0, c, tape, (reserved); then (slot, t) pairs
FMT_F32, FMT_INT8 = 0, 1


def desc_len(max_seqs: int) -> int:
    return HEAD + 2 * max_seqs


def payload_bytes(n_tok: int, d: int, fmt: int) -> int:
    n = n_tok * d
    if fmt == FMT_F32:
        return 4 * n
    return -(-n // 16) * 16 + 4 * (-(-n // 64))


def sub_ranges(start: int, end: int, world: int):
    return [(start + a, start + b) for a, b in split_blocks(end - start, world)]


@dataclass
class BoxPlan:
    """Everything every rank derives identically from the server config."""

    config: ServerConfig
    world: int

    @property
    def int8_weights(self) -> bool:
        return self.config.quantize in ("weights", "both")

    @property
    def fmt(self) -> int:
        return FMT_INT8 if self.config.quantize in ("activations", "both") else FMT_F32

    @property
    def in_flight(self) -> int:
        return max(2, min(2 * self.world, 16))

    @property
    def max_seqs(self) -> int:
        return max(1, self.config.capacity)

    def pages(self, n_blocks_total: int) -> int:
        c = self.config
        pos_budget = max(1, c.cache_budget_tokens // n_blocks_total)
        return c.kv_pages or (-(-pos_budget // c.page_tokens) + c.capacity + 2 + -(-c.model.max_seq // c.page_tokens))


# ---------------------------------------------------------------------- per-rank data path


class RankState:
    """One rank's sub-span, its mailbox ring and its session / tape tables.
    `apply` executes a descriptor (ranks 1..N-1 and, through BoxScheduler, rank 0)."""

    def __init__(self, plan: BoxPlan, rank: int, span: BlockSpan, ring: P2PRing, dist, group=None,
                 owns_span: bool = True):
        """dist: torch.distributed; group: the (gloo) process group of the
        control plane, None for the default group; owns_span: close the
        sub-span on shutdown (False when the caller keeps using it)."""
        self.plan, self.rank, self.world = plan, rank, plan.world
        self.span, self.ring, self.dist, self.group = span, ring, dist, group
        self.owns_span = owns_span
        self.d = span.config.hidden
        self.seqs: dict[int, Sequence] = {}
        self.fwd: dict[tuple, Sequence] = {}
        self.tapes: dict[int, object] = {}

    def finish(self) -> None:
        import torch

        torch.cuda.synchronize(self.span.device)

    def close(self) -> None:
        self.ring.close()
        if self.owns_span:
            self.span.close()

    def seq(self, slot: int) -> Sequence:
        s = self.seqs.get(slot)
        if s is None:
            s = self.seqs[slot] = Sequence()
        return s

    def _views(self, base: int, n_tok: int, fmt: int):
        if fmt == FMT_F32:
            return dict(f32=DevPtr(base))
        n = n_tok * self.d
        return dict(codes=DevPtr(base), scales=DevPtr(base + -(-n // 16) * 16))

    def hop(self, j: int, seqs, lens, x=None, tape=None) -> None:
        """Enqueue job j on this rank's stream: (wait for the predecessor's
        payload), run the sub-span, store the result into the successor's
        mailbox slot j % slots and publish it."""
        import torch

        from . import _lib

        st = _lib.stream_ptr(torch.cuda.current_stream())
        n_tok, fmt = int(sum(lens)), self.plan.fmt
        kw = {}
        if self.rank == 0:
            kw["in_f32"] = x
        else:
            self.ring.wait(j, st)
            v = self._views(self.ring.local_slot(j), n_tok, fmt)
            kw.update(in_f32=v.get("f32"), in_codes=v.get("codes"), in_scales=v.get("scales"))
        v = self._views(self.ring.peer_slot(j), n_tok, fmt)
        kw.update(out_f32=v.get("f32"), out_codes=v.get("codes"), out_scales=v.get("scales"))
        self.span.step_codes(seqs, lens, tape=tape, **kw)
        self.ring.signal(j, st)

    def bind_thread(self) -> None:
        import torch

        torch.cuda.set_device(self.span.device)

    def new_stream(self):
        import torch

        return torch.cuda.Stream(device=self.span.device)

    def egress(self, j: int, n_tok: int, stream):
        """Rank 0: on `stream`, wait until the last sub-span published job j
        into our mailbox, then copy (f32) or dequantize (int8) it out.
        Returns (event, output [n_tok, d])."""
        import torch

        from . import _lib, codec

        d = self.d
        with torch.cuda.stream(stream):
            self.ring.wait(j, _lib.stream_ptr(stream))
            slot = dev_view(self.ring.local_slot(j), payload_bytes(n_tok, d, self.plan.fmt), self.span.device)
            if self.plan.fmt == FMT_F32:
                out = slot.view(torch.float32).view(n_tok, d).clone()
            else:
                n = n_tok * d
                off = -(-n // 16) * 16
                q = codec.QuantizedBlockwise(64, slot[off:off + 4 * (-(-n // 64))].view(torch.float32),
                                             slot[:n].view(torch.int8), (n_tok, d))
                out = codec.dequantize_blockwise(q)
            ev = torch.cuda.Event()
            ev.record(stream)
        return ev, out

    def egress_codes(self, j: int, n_tok: int, stream):
        """Rank 0, int8 ring: on `stream`, wait for job j's result in our mailbox
        and copy its wire codes + block scales (the last sub-span's own
        quantization of its f32 output, i.e. exactly the int8 reply) to one
        pinned buffer [scales f32 | codes]. Returns (event, buffer)."""
        import torch

        from . import _lib

        d, n = self.d, n_tok * self.d
        nb = -(-n // 64)
        with torch.cuda.stream(stream):
            self.ring.wait(j, _lib.stream_ptr(stream))
            slot = dev_view(self.ring.local_slot(j), payload_bytes(n_tok, d, self.plan.fmt), self.span.device)
            off = -(-n // 16) * 16
            buf = torch.empty(4 * nb + n, dtype=torch.uint8, pin_memory=True)
            buf[:4 * nb].copy_(slot[off:off + 4 * nb], non_blocking=True)
            buf[4 * nb:].copy_(slot[:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        return ev, buf

    def apply(self, desc, x=None):
        op = int(desc[0])
        if op == OP_STEP:
            j, n = int(desc[1]), int(desc[2])
            pairs = desc[HEAD:HEAD + 2 * n].view(n, 2).tolist()
            seqs = [self.seq(slot) for slot, _ in pairs]
            lens = [t for _, t in pairs]
            for s, t in zip(seqs, lens):
                self.span.reserve(s, s.length + t)
            self.hop(j, seqs, lens, x)
        elif op == OP_RELEASE:
            s = self.seqs.pop(int(desc[4]), None)
            if s is not None:
                self.span.release(s)
        elif op == OP_FORWARD:
            self._forward(desc, x)
        elif op == OP_BACKWARD:
            return self._backward(desc)
        elif op == OP_DROP:
            self.tapes.pop(int(desc[4]), None)
        return None

    def _forward(self, desc, x=None):
        """Rows r0 .. r0+n, positions c0 .. c0+c of FORWARD request `key`
        (B rows of t tokens): cache-less rows (server.py:418-425) whose
        temporary KV pages persist across the causal chunks of a long row."""
        import torch

        j, n, key, B, t, r0, c0, c, want_tape = (int(desc[i]) for i in (1, 2, 4, 5, 6, 7, 8, 9, 10))
        seqs = []
        for r in range(r0, r0 + n):
            s = self.fwd.get((key, r))
            if s is None:
                s = self.fwd[(key, r)] = Sequence()
            self.span.reserve(s, c0 + c)
            seqs.append(s)
        tp = None
        if want_tape:
            tape = self.tapes.get(key)
            if tape is None:
                tape = self.tapes[key] = torch.empty(B, self.span.n_blocks, t, self.d, device=self.span.device)
            tp = torch.empty(self.span.n_blocks, n * c, self.d, device=self.span.device)
        self.hop(j, seqs, [c] * n, x, tape=tp)
        if tp is not None:
            self.tapes[key][r0:r0 + n, :, c0:c0 + c] = tp.view(self.span.n_blocks, n, c, self.d).transpose(0, 1)
        if c0 + c == t:  # last chunk: the rows' pages go back (later kernels on this stream reuse them in order)
            for r in range(r0, r0 + n):
                self.span.release(self.fwd.pop((key, r)))

    def _backward(self, desc):
        """Reverse walk (model.py:383-418 per hosted block): rank N-1 takes
        dL/d(out) from rank 0, every rank passes dL/d(its input) to rank-1;
        rank 0 returns dL/d(box input)."""
        import torch

        key, B, t = int(desc[4]), int(desc[5]), int(desc[6])
        tape = self.tapes.pop(key)
        src = 0 if self.rank == self.world - 1 else self.rank + 1
        g = torch.empty(B, t, self.d)
        self.dist.recv(g, src=src, group=self.group)
        gin = self.span.backward(tape, g.to(self.span.device))
        if self.rank > 0:
            self.dist.send(gin.cpu(), dst=self.rank - 1, group=self.group)
            return None
        return gin


def serve_rank(plan: BoxPlan, rank: int, dist, state=None) -> None:
    """Ranks 1..N-1: build the sub-span and the ring (or use `state`), then
    apply descriptors from rank 0 until OP_STOP."""
    import torch

    state = state or _build_rank(plan, rank, dist)
    buf = torch.empty(desc_len(plan.max_seqs), dtype=torch.int64)
    try:
        while True:
            dist.recv(buf, src=0, group=state.group)
            if int(buf[0]) == OP_STOP:
                break
            state.apply(buf.clone())
        state.finish()
    finally:
        state.close()


def _build_rank(plan: BoxPlan, rank: int, dist) -> RankState:
    import torch

    c = plan.config
    start, end = c.blocks
    lo, hi = sub_ranges(start, end, plan.world)[rank]
    torch.cuda.set_device(c.device)
    span = BlockSpan(c.model, lo, hi, int8=plan.int8_weights, page_tokens=c.page_tokens,
                     n_pages=plan.pages(end - start), max_tokens=c.max_batch_tokens, max_seqs=plan.max_seqs,
                     device=c.device)
    if c.seed is None:
        from .server import _BlockView, read_ptck

        _, bl = read_ptck(c.checkpoint_path, (lo, hi))
        span.load_weights([_BlockView(bl[i]) for i in range(lo, hi)])
    else:
        span.generate_weights(c.seed)
    torch.cuda.synchronize()
    ring = P2PRing(rank, plan.world, plan.in_flight, payload_bytes(c.max_batch_tokens, c.model.hidden, FMT_F32),
                   c.device, dist)
    return RankState(plan, rank, span, ring, dist)


# ---------------------------------------------------------------------- rank 0: scheduler


class _Fwd:
    __slots__ = ("batch", "out", "key", "done", "err")

    def __init__(self, batch, out, key):
        self.batch, self.out, self.key = batch, out, key
        self.done = threading.Event()
        self.err = None


class _BoxJob:
    __slots__ = ("seq", "x", "msg", "enc", "t", "out", "err", "done")

    def __init__(self, seq, x=None, msg=None, enc=None):
        self.seq, self.x, self.msg, self.enc = seq, x, msg, enc
        self.t = int(x.shape[0]) if x is not None else msg.rows
        self.out = self.err = None
        self.done = threading.Event()


class BoxScheduler:
    """Rank 0's single control thread: coalesces concurrent STEPs of distinct
    sessions into ring jobs (StepScheduler's batching), reserves rank 0's
    pages (mirrored everywhere by descriptor order), sends each descriptor,
    launches rank 0's part and the egress (wait for the ring to close, copy
    or dequantize the result), and keeps up to D jobs in flight; a completion
    thread hands results back in order."""

    def __init__(self, state: RankState, plan: BoxPlan):
        import torch

        self.state, self.plan = state, plan
        self.span = state.span
        self.max_tokens = plan.config.max_batch_tokens
        self.max_seqs = plan.max_seqs
        self.q: queue.Queue = queue.Queue()
        self.done_q: queue.Queue = queue.Queue()
        self.slots_free = threading.Semaphore(plan.in_flight)
        self.busy = 0  # jobs launched and not yet completed
        self._busy_lock = threading.Lock()
        self.job_ids = itertools.count()
        self.batches = self.batched_steps = 0
        self.egress = state.new_stream()
        self._pending_sends = []
        self.timing = []  # PB_SERVER_TIMING: (send, rank-0 launch, egress launch, done) per job
        self._stop = False
        self._t = threading.Thread(target=self._loop, name="box-sched", daemon=True)
        self._c = threading.Thread(target=self._complete_loop, name="box-done", daemon=True)
        self._t.start()
        self._c.start()

    # ------------------------------------------------------------ API (handler threads)

    def run(self, seq, x):
        """One session's STEP through the ring. A step longer than the token
        workspace goes as consecutive causal chunk jobs (every rank runs them
        in order); its pages are reserved up front so no chunk can fail
        half-way (ranks other than 0 reserve lazily, never more than rank 0)."""
        import torch

        t = x.shape[0]
        if t > self.max_tokens:
            self.call("reserve", seq, seq.length + t)
            parts = [self.run(seq, x[c0:c0 + self.max_tokens]) for c0 in range(0, t, self.max_tokens)]
            out = torch.cat(parts)
            # the parts were allocated on the egress stream: keep their memory from being reused there
            # (the next job's egress) before this stream's concatenation has read them
            for p in parts:
                if p.is_cuda:
                    p.record_stream(torch.cuda.current_stream(p.device))
            return out
        job = _BoxJob(seq, x)
        self.q.put(("step", job))
        job.done.wait()
        if job.err is not None:
            raise job.err
        return job.out

    def run_msg(self, seq, msg, encoding: int) -> bytes:
        """One session's STEP as wire bytes in and out (t <= max_tokens): the
        scheduler decodes the batch on rank 0's stream, and with an int8 ring
        and an int8 reply the reply is the last sub-span's own codes, copied
        once per job from the mailbox (no decode / re-encode on the handler)."""
        job = _BoxJob(seq, msg=msg, enc=encoding)
        self.q.put(("step", job))
        job.done.wait()
        if job.err is not None:
            raise job.err
        if job.enc is None:  # f32 result (the ring or the reply is not int8): encoded by the caller
            return job.out
        buf, host, sbytes, r0, t = job.out
        d = self.span.config.hidden
        s0, nb = r0 * d // 64, -(-t * d // 64)
        sc = host[4 * s0:4 * (s0 + nb)]
        if not np.isfinite(sc.view(np.float32)).all():
            raise _NonFinite("non-finite tensor")
        codes = host[sbytes + r0 * d:sbytes + (r0 + t) * d]
        return codec.encode_header(codec.ENC_INT8, (t, d)) + struct.pack(">I", 64) + sc.tobytes() + codes.tobytes()

    def call(self, kind, *args):
        """Run a control operation (release / forward / backward / drop) in order."""
        ev = _Fwd(None, None, 0)
        self.q.put((kind, ev, args))
        ev.done.wait()
        if ev.err is not None:
            raise ev.err
        return ev.out

    def stop(self):
        self.q.put(("stop", None))
        self._t.join(timeout=30)

    # ------------------------------------------------------------ control thread

    def _send(self, desc):
        import torch.distributed as dist

        for r in range(1, self.plan.world):
            self._pending_sends.append(dist.isend(desc, dst=r, group=self.state.group))
        if len(self._pending_sends) > 256:
            for w in self._pending_sends:
                w.wait()
            self._pending_sends.clear()

    def _flush_sends(self):
        for w in self._pending_sends:
            w.wait()
        self._pending_sends.clear()

    def _desc(self, op, **f):
        import torch

        d = torch.zeros(desc_len(self.max_seqs), dtype=torch.int64)
        d[0] = op
        for i, name in ((1, "job"), (2, "n"), (3, "fmt"), (4, "key"), (5, "B"), (6, "t"), (7, "r0"), (8, "c0"),
                        (9, "c"), (10, "tape")):
            if name in f:
                d[i] = int(f[name])
        return d

    def _loop(self):
        self.state.bind_thread()
        pending = None
        while True:
            item = pending or self.q.get()
            pending = None
            kind = item[0]
            if kind == "stop":
                self._send(self._desc(OP_STOP))
                self._flush_sends()
                self.done_q.put(None)
                return
            if kind == "step":
                batch, ntok = [item[1]], item[1].t
                key = (item[1].msg is None, item[1].enc)
                while len(batch) < self.max_seqs and ntok < self.max_tokens:
                    try:
                        nxt = self.q.get_nowait()
                    except queue.Empty:
                        break
                    if (nxt[0] != "step" or ntok + nxt[1].t > self.max_tokens
                            or (nxt[1].msg is None, nxt[1].enc) != key):
                        pending = nxt
                        break
                    batch.append(nxt[1])
                    ntok += nxt[1].t
                # spread concurrent sessions over the idle pipeline stages instead of coalescing
                # them into one job that would leave the other stages idle (measured: 2 sessions on
                # a 2-GPU box arrive together and ran as one 2-token job per period)
                parts = min(len(batch), max(1, self.plan.world - self.busy))
                per = -(-len(batch) // parts)
                for i in range(0, len(batch), per):
                    self._submit_steps(batch[i:i + per])
                continue
            ev, args = item[1], item[2]
            try:
                if kind == "reserve":
                    self.span.reserve(*args)
                elif kind == "release":
                    (seq,) = args
                    self.state.seqs.pop(seq.slot, None)
                    self.span.release(seq)
                    self._send(self._desc(OP_RELEASE, key=seq.slot))
                elif kind == "drop":
                    self._send(self._desc(OP_DROP, key=args[0]))
                    self.state.tapes.pop(args[0], None)
                elif kind == "forward":
                    self._submit_forward(*args, ev)
                    continue  # completed by the completion thread
                elif kind == "backward":
                    key, grad = args
                    desc = self._desc(OP_BACKWARD, key=key, B=grad.shape[0], t=grad.shape[1])
                    self._send(desc)
                    self._flush_sends()
                    import torch.distributed as dist

                    dist.send(grad.detach().cpu().contiguous(), dst=self.plan.world - 1, group=self.state.group)
                    ev.out = self.state.apply(desc)
            except Exception as e:  # noqa: BLE001
                ev.err = e
            ev.done.set()

    def _launch(self, desc, x, n_tok, place, codes=False):
        """Send job desc, launch rank 0's part and the egress; `place(out)`
        runs on the completion thread once the ring closed (codes: the int8
        result copied out as wire codes + scales, RankState.egress_codes)."""
        t0 = time.perf_counter()
        self._send(desc)
        t1 = time.perf_counter()
        self.state.apply(desc, x)
        t2 = time.perf_counter()
        egress = self.state.egress_codes if codes else self.state.egress
        waitable, out = egress(int(desc[1]), n_tok, self.egress)
        t3 = time.perf_counter()
        with self._busy_lock:
            self.busy += 1
        self.done_q.put((waitable, out, place, (t0, t1, t2, t3)))

    def _submit_steps(self, batch):
        import torch

        ready = []
        for job in batch:
            try:
                if job.t > self.max_tokens:
                    raise InputError("internal: oversized job reached the box scheduler")
                self.span.reserve(job.seq, job.seq.length + job.t)
                ready.append(job)
            except (CapacityError, InputError) as e:
                job.err = e
                job.done.set()
        if not ready:
            return
        self.slots_free.acquire()
        try:
            j = next(self.job_ids)
            desc = self._desc(OP_STEP, job=j, n=len(ready), fmt=self.plan.fmt)
            for i, job in enumerate(ready):
                desc[HEAD + 2 * i] = job.seq.slot
                desc[HEAD + 2 * i + 1] = job.t
                self.state.seqs[job.seq.slot] = job.seq
            d = self.span.config.hidden
            # wire inputs are decoded here, on rank 0's stream, in order with the hop
            xs = [jb.x if jb.x is not None else jb.msg.decode().reshape(jb.t, d) for jb in ready]
            x = xs[0] if len(xs) == 1 else torch.cat(xs)
            x = x.to(device=self.span.device, dtype=torch.float32).contiguous()
            lens = [jb.t for jb in ready]
            codes = (self.plan.fmt == FMT_INT8 and d % 64 == 0
                     and all(jb.msg is not None and jb.enc == codec.ENC_INT8 for jb in ready))

            def place(out, ready=ready, lens=lens, codes=codes, d=d):
                if codes:
                    host = out.numpy()
                    sbytes = 4 * -(-sum(lens) * d // 64)
                    r0 = 0
                    for jb, t in zip(ready, lens):
                        jb.out = (out, host, sbytes, r0, t)
                        r0 += t
                        jb.done.set()
                    return
                for jb, o in zip(ready, torch.split(out, lens)):
                    jb.out = o
                    jb.enc = None  # an f32 result: the handler encodes it
                    jb.done.set()

            self._launch(desc, x, x.shape[0], place, codes=codes)
            self.batches += 1
            self.batched_steps += len(ready)
        except Exception as e:  # noqa: BLE001
            self.slots_free.release()
            for job in ready:
                job.err = e
                job.done.set()

    def _submit_forward(self, batch, out, key, want_tape, ev):
        import torch

        B, t, d = batch.shape
        if t <= self.max_tokens:
            per = max(1, min(self.max_seqs, self.max_tokens // t))
            plan = [(r0, min(per, B - r0), 0, t) for r0 in range(0, B, per)]
        else:
            plan = [(r, 1, c0, min(self.max_tokens, t - c0)) for r in range(B) for c0 in range(0, t, self.max_tokens)]
        remaining = [len(plan)]
        lock = threading.Lock()
        for r0, n, c0, c in plan:
            self.slots_free.acquire()
            j = next(self.job_ids)
            desc = self._desc(OP_FORWARD, job=j, n=n, key=key, B=B, t=t, r0=r0, c0=c0, c=c, tape=want_tape)
            x = batch[r0:r0 + n, c0:c0 + c].reshape(n * c, d).to(device=self.span.device,
                                                                  dtype=torch.float32).contiguous()

            def place(o, r0=r0, n=n, c0=c0, c=c):
                out[r0:r0 + n, c0:c0 + c] = o.view(n, c, d)
                if o.is_cuda:  # o lives in the egress stream's pool: not reused before this copy ran
                    o.record_stream(torch.cuda.current_stream(o.device))
                with lock:
                    remaining[0] -= 1
                    last = remaining[0] == 0
                if last:
                    ev.done.set()

            try:
                self._launch(desc, x, n * c, place)
            except Exception as e:  # noqa: BLE001
                self.slots_free.release()
                ev.err = e
                ev.done.set()
                return

    # ------------------------------------------------------------ completion thread

    def _complete_loop(self):
        self.state.bind_thread()
        while True:
            item = self.done_q.get()
            if item is None:
                return
            ev, out, place, ts = item
            ev.synchronize()
            if _TIMING:
                self.timing.append((*ts, time.perf_counter()))
            with self._busy_lock:
                self.busy -= 1
            self.slots_free.release()
            place(out)


# ---------------------------------------------------------------------- rank 0: what ServerNode sees


class BoxSequence(Sequence):
    """A session's KV state; `slot` names it in descriptors on every rank."""

    _ids = itertools.count(1)

    def __init__(self):
        super().__init__()
        self.slot = next(BoxSequence._ids)


class TapeHandle:
    """FORWARD tape held piecewise on every rank; `shape` is what the
    BACKWARD handler validates against ([B, n_blocks, t, d])."""

    _ids = itertools.count(1)

    def __init__(self, shape):
        self.key = next(TapeHandle._ids)
        self.shape = shape


class BoxSpan:
    """The BlockSpan interface ServerNode uses (sessions, step, forward,
    backward, pool accounting), implemented over the ring of sub-spans."""

    def __init__(self, plan: BoxPlan, state: RankState, start: int, end: int):
        self.plan, self.state = plan, state
        self.config = state.span.config
        self.start, self.end = start, end
        self.n_blocks = end - start
        self.int8 = plan.int8_weights
        self.device = state.span.device
        self.pool = state.span.pool
        self.sched = BoxScheduler(state, plan)

    def new_sequence(self) -> BoxSequence:
        return BoxSequence()

    def pages_needed(self, seq, new_len: int) -> int:
        return self.state.span.pages_needed(seq, new_len)

    def release(self, seq) -> None:
        self.sched.call("release", seq)

    def step(self, items):
        return [self.sched.run(seq, x) for seq, x in items]

    def forward(self, batch, tape: bool = False):
        import torch

        B, t, d = batch.shape
        if t > self.config.max_seq:
            raise CapacityError(f"t={t} exceeds max_seq")
        out = torch.empty(B, t, d, device=self.device)
        handle = TapeHandle((B, self.n_blocks, t, d))  # its key also names the rows' temporary sequences
        self.sched.call("forward", batch, out, handle.key, int(tape))
        return (out, handle) if tape else out

    def backward(self, tape: TapeHandle, grad):
        return self.sched.call("backward", tape.key, grad)

    def drop_tape(self, tape: TapeHandle) -> None:
        self.sched.call("drop", tape.key)

    def close(self):
        self.sched.stop()
        self.state.ring.close()
        self.state.span.close()


class BoxFrontEnd(ServerNode):
    """Rank 0 of the box: the reference ServerNode protocol (sessions, STEP
    semantics, budget, FORWARD/BACKWARD, announcements) over a BoxSpan."""

    def __init__(self, config: ServerConfig, world: int, dist, state: RankState | None = None):
        """state: rank 0's prebuilt RankState (sub-span + ring + control group),
        e.g. the bench reusing its resident spans; None builds it."""
        if state is None and config.seed is None and not config.checkpoint_path:
            raise InputError("the box front end loads weights per GPU: give a seed or a checkpoint path")
        super().__init__(config)
        self.world, self.dist, self._state = world, dist, state
        self.step_timing: list = []  # PB_SERVER_TIMING: (decode, ring, encode) seconds per STEP

    def _pick_range(self):
        r = super()._pick_range()
        self.config.blocks = (r.start, r.end)
        return r

    def _make_span(self, int8: bool, pages: int):
        import hashlib

        plan = BoxPlan(self.config, self.world)
        state = self._state or _build_rank(plan, 0, self.dist)
        h = hashlib.sha256(f"box:{self.config.seed}:{self.model}:{self.range}:{self.config.checkpoint_path}".encode())
        self._weights_hash = h.hexdigest()
        return BoxSpan(plan, state, self.range.start, self.range.end)

    def _make_scheduler(self):
        return self.span.sched

    def _run_step(self, seq, msg, encoding: int) -> bytes:
        import torch

        t0 = time.perf_counter()
        t1 = t0
        out = None
        if msg.rows <= self.sched.max_tokens:
            res = self.sched.run_msg(seq, msg, encoding)
            if isinstance(res, bytes):
                if _TIMING:
                    self.step_timing.append((0.0, time.perf_counter() - t0, 0.0))
                return res
            out = res
        else:
            st = self._io_stream()
            with torch.cuda.stream(st):
                x = msg.decode()
            st.synchronize()
            t1 = time.perf_counter()
            out = self.sched.run(seq, x)  # (a long step: concatenated on this thread's current stream)
        t2 = time.perf_counter()
        try:
            reply = self._encode(out, encoding, producer=torch.cuda.current_stream(self.span.device))
        except InputError as e:
            raise _NonFinite(str(e)) from e  # computed, then failed encoding (position advances)
        if _TIMING:
            self.step_timing.append((t1 - t0, t2 - t1, time.perf_counter() - t2))
        return reply

    def _shutdown(self):
        super()._shutdown()
        if isinstance(self.span, BoxSpan):
            self.span.state.ring.close()


def run_box(config: ServerConfig, rank: int, world: int, dist, ready=None, stop_event=None):
    """Entry for one box process (rank r of N, already in a gloo process
    group; config.device = this rank's GPU). Rank 0 serves until stop_event
    is set (or forever) and calls ready(address) once online."""
    plan = BoxPlan(config, world)
    if rank > 0:
        if config.blocks == "auto":
            config.blocks = (0, config.span or config.model.n_layers)
        serve_rank(plan, rank, dist)
        return
    node = BoxFrontEnd(config, world, dist).start()
    if ready is not None:
        ready(node.address)
    try:
        if stop_event is not None:
            stop_event.wait()
        else:
            threading.Event().wait()
    finally:
        node.stop()


def _box_child(rank, world, port, config, q, stop_ev, devices):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        config.device = devices[rank] if devices else rank % torch.cuda.device_count()
        run_box(config, rank, world, dist, ready=lambda a: q.put(("ok", a)), stop_event=stop_ev)
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001 - reported to the launcher
        q.put(("error", f"rank {rank}: {type(e).__name__}: {e}"))
        raise


class LocalBox:
    """A box started from Python: N spawned processes (rank r on GPU
    devices[r], default r mod device count). `address` is rank 0's server."""

    def __init__(self, config: ServerConfig, world: int, devices=None, timeout_s: float = 600.0):
        import socket

        import torch.multiprocessing as mp

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        ctx = mp.get_context("spawn")
        self._q, self._stop = ctx.Queue(), ctx.Event()
        self.procs = [ctx.Process(target=_box_child, args=(r, world, port, config, self._q, self._stop, devices),
                                  daemon=True) for r in range(world)]
        for p in self.procs:
            p.start()
        kind, val = self._q.get(timeout=timeout_s)
        if kind != "ok":
            self.stop()
            raise RuntimeError(f"box failed to start: {val}")
        self.address = val

    def stop(self, timeout_s: float = 60.0):
        self._stop.set()
        for p in self.procs:
            p.join(timeout=timeout_s)
        for p in self.procs:
            if p.is_alive():
                p.kill()
        return [p.exitcode for p in self.procs]


def main(argv=None):
    """python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
         -m paper_2209_01188_b200.box --shape bloom-176b --seed 42 --quantize both --port 31337"""
    import argparse

    import torch
    import torch.distributed as dist

    from .model import SHAPES

    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--checkpoint", default="")
    p.add_argument("--blocks", type=int, nargs=2, default=None)
    p.add_argument("--quantize", default="both")
    p.add_argument("--host", default="127.0.0.1")
    p.add_argument("--port", type=int, default=0)
    p.add_argument("--bootstrap", nargs="*", default=[])
    p.add_argument("--capacity", type=int, default=64)
    p.add_argument("--max-batch-tokens", type=int, default=256)
    a = p.parse_args(argv)
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    dist.init_process_group("gloo")
    dev = local % torch.cuda.device_count()
    cfg = ServerConfig(checkpoint_path=a.checkpoint, host=a.host, port=a.port,
                       blocks=tuple(a.blocks) if a.blocks else "auto", quantize=a.quantize, bootstrap=a.bootstrap,
                       capacity=a.capacity, seed=None if a.checkpoint else a.seed, model=SHAPES[a.shape],
                       device=dev, max_batch_tokens=a.max_batch_tokens)
    run_box(cfg, rank, world, dist, ready=lambda addr: print(f"box serving at {addr}", flush=True))


if __name__ == "__main__":
    main()
