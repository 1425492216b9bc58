"""Span-to-span hop schedule for one box: consecutive block spans pinned to
consecutive GPUs (one process per GPU), the hidden state of every hop carried
as the reference's int8 wire codec (codes + scales) over NCCL send/recv.

This replaces the reference client's relay (client.py:312-331: the client
receives each server's reply, decodes it, re-encodes it and sends it to the
next hop). Because quantize(dequantize(quantize(x))) == quantize(x)
(SURVEY §0.6), forwarding the codes directly is bit-identical to that relay.

Ring schedule with S sessions in flight (S = number of spans keeps every GPU
busy): job j is session j % S; span r receives job j from span r-1, runs it,
and sends it to span r+1; the last span hands the result back to span 0 (the
stand-in for the client's LM head + next-token embedding), which starts the
session's next step. NCCL matches send/recv in issue order per peer pair, and
every rank issues the same job order, so the schedule cannot deadlock.
"""

from __future__ import annotations


class RingSchedule:
    """Jobs first .. total_jobs-1 (job ids keep increasing across phases: the
    peer-memory flags are monotonic)."""

    def __init__(self, rank: int, world: int, sessions: int, total_jobs: int, first: int = 0):
        self.rank, self.world, self.sessions, self.total_jobs = rank, world, sessions, total_jobs
        self.first = first

    def recv_from(self, j: int):
        """Peer to receive job j's hidden from, or None (span 0 starting a session)."""
        if self.world == 1:
            return None
        if self.rank > 0:
            return self.rank - 1
        return self.world - 1 if j >= self.first + self.sessions else None

    def send_to(self, j: int):
        """Peer to send job j's output to, or None (session finished / single span)."""
        if self.world == 1:
            return None
        if self.rank < self.world - 1:
            return self.rank + 1
        return 0 if j + self.sessions < self.total_jobs else None


def split_blocks(n_layers: int, n_spans: int):
    """Contiguous, balanced spans: 70 blocks over 8 GPUs -> 9,9,9,9,9,9,8,8."""
    base, extra = divmod(n_layers, n_spans)
    out, s = [], 0
    for r in range(n_spans):
        k = base + (1 if r < extra else 0)
        out.append((s, s + k))
        s += k
    return out


def run_jobs(sched: RingSchedule, jobs, step, exchange, inbox):
    """Run `jobs` (increasing job ids) on this span.

    step(j, payload | None) -> outbox (payload sent downstream);
    exchange(ops) runs [(op, buffer, peer)] with op in {"send", "recv"} as ONE
    group (NCCL group / batch_isend_irecv) so the send of job j and the receive
    of job j+1 progress together. With S = world sessions every group lies on
    an anti-diagonal (rank + job = const) of the pipeline, which is what keeps
    the ring deadlock-free even when sends do not complete eagerly.
    inbox: receive buffer, or a callable job -> buffer (sized per job); it is
    reused: the group only starts after the step that read it, by stream order."""
    if not jobs:
        return
    box = inbox if callable(inbox) else (lambda j: inbox)
    src = sched.recv_from(jobs[0])
    if src is not None:
        exchange([("recv", box(jobs[0]), src)])
    have_input = src is not None
    for i, j in enumerate(jobs):
        out = step(j, box(j) if have_input else None)
        ops = []
        dst = sched.send_to(j)
        if dst is not None:
            ops.append(("send", out, dst))
        have_input = False
        if i + 1 < len(jobs):
            nsrc = sched.recv_from(jobs[i + 1])
            if nsrc is not None:
                ops.append(("recv", box(jobs[i + 1]), nsrc))
                have_input = True
        if ops:
            exchange(ops)


def torch_exchange(ops):
    """exchange() over torch.distributed (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist

    p2p = [dist.P2POp(dist.isend if op == "send" else dist.irecv, buf, peer) for op, buf, peer in ops]
    for w in dist.batch_isend_irecv(p2p):
        w.wait()


class DevPtr:
    """A raw device address where the span API expects a tensor (data_ptr())."""

    def __init__(self, addr: int):
        self.addr = int(addr)

    def data_ptr(self) -> int:
        return self.addr


class _CudaArray:
    __slots__ = ("__cuda_array_interface__",)

    def __init__(self, addr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (int(addr), False),
                                         "version": 3, "strides": None}


def dev_view(addr: int, nbytes: int, device):
    """A torch uint8 tensor aliasing `nbytes` of device memory at `addr`
    (e.g. a mailbox slot allocated by pb_hop_alloc); no copy, no ownership."""
    import torch

    return torch.as_tensor(_CudaArray(addr, nbytes), device=device)


class P2PRing:
    """The RingSchedule's hops over NVLink peer memory (pb_hop.cu) instead of
    NCCL: every rank exports one mailbox (u64 flags + `slots` payload slots)
    by CUDA IPC handle and maps its successor's. Job j's payload goes to slot
    j % slots of the receiver; its flag there is set to j + 1 (monotonic per
    slot). slots = sessions + 1 is enough without flow control: only
    `sessions` jobs are in flight around the ring, so job j + slots cannot be
    sent before job j was consumed."""

    FLAGS = 64

    def __init__(self, rank: int, world: int, sessions: int, slot_bytes: int, device: int, dist, timeout_ms=120000):
        import ctypes as C

        from . import _lib

        self.rank, self.world, self.S = rank, world, sessions
        self.slots = sessions + 1
        assert self.slots <= self.FLAGS
        self.slot_bytes = -(-slot_bytes // 256) * 256
        self.timeout_ms = timeout_ms
        self.L = _lib.lib()
        total = 8 * self.FLAGS + self.slots * self.slot_bytes
        base, handle = C.c_void_p(), (C.c_char * 64)()
        self.base = self.peer = None
        rc = self.L.pb_hop_alloc(total, device, C.byref(base), handle)
        if rc == 0:
            self.base = base.value
        handles = [None] * world  # collective on every rank, even after a local failure
        dist.all_gather_object(handles, bytes(handle) if rc == 0 else None)
        if any(h is None for h in handles):
            self.close()
            raise RuntimeError("mailbox allocation failed on a rank")
        peer = C.c_void_p()
        succ = (rank + 1) % world
        _lib.check(self.L.pb_hop_open(C.create_string_buffer(handles[succ], 64), device, C.byref(peer)))
        self.peer = peer.value
        # Ranks sharing one physical GPU must not spin on each other's flags in
        # kernels (separate contexts time-slice; a spinning kernel can stall the
        # context switch): there the receiver polls its flag from the host.
        import torch

        self.device = device
        uuids = [None] * world
        dist.all_gather_object(uuids, str(torch.cuda.get_device_properties(device).uuid))
        self.host_wait = len(set(uuids)) < world
        if self.host_wait:
            self._poll_stream = torch.cuda.Stream(device=device)
            self._poll_host = torch.zeros(1, dtype=torch.int64).pin_memory()

    def _slot(self, base: int, j: int) -> int:
        return base + 8 * self.FLAGS + (j % self.slots) * self.slot_bytes

    def local_slot(self, j: int) -> int:
        return self._slot(self.base, j)

    def peer_slot(self, j: int) -> int:
        return self._slot(self.peer, j)

    def wait(self, j: int, stream: int) -> None:
        """Order `stream`'s next work after job j's payload arrived: a one-thread
        acquire-spin kernel on that stream (GPUs of their own), or a host poll
        when ranks share a GPU (the caller's thread blocks until the flag is set)."""
        from . import _lib

        if self.host_wait:
            return self._poll(j)
        _lib.check(self.L.pb_hop_wait(self.base + 8 * (j % self.slots), j + 1, self.timeout_ms, stream))

    def _poll(self, j: int) -> None:
        import time

        import torch

        flag = dev_view(self.base + 8 * (j % self.slots), 8, torch.device("cuda", self.device)).view(torch.int64)
        deadline = time.monotonic() + self.timeout_ms / 1000.0
        with torch.cuda.stream(self._poll_stream):
            while True:
                self._poll_host.copy_(flag, non_blocking=True)
                self._poll_stream.synchronize()
                if int(self._poll_host[0]) >= j + 1:
                    return
                if time.monotonic() > deadline:
                    raise TimeoutError(f"hop: no signal for job {j} after {self.timeout_ms} ms")
                time.sleep(20e-6)

    def signal(self, j: int, stream: int) -> None:
        """Publish job j (payload already stored in the successor's slot j % slots)."""
        from . import _lib

        _lib.check(self.L.pb_hop_signal(self.peer + 8 * (j % self.slots), j + 1, stream))

    def close(self) -> None:
        if getattr(self, "peer", None):
            self.L.pb_hop_close(self.peer)
            self.peer = None
        if getattr(self, "base", None):
            self.L.pb_hop_free(self.base)
            self.base = None
