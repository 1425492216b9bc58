"""Framed-RPC ingress/egress of the span server.

Wire contract (what a drop-in must speak, restated from
/root/reference/pkg/src/swarmlm/transport/rpc.py:35-43,178-274 and
transport/wire.py:52-84): 16-byte frame header, `handler(msg_type, payload)
-> (reply_type, reply)`, a `RemoteError` becomes an ERROR frame with its code,
any other exception an ERR_GENERIC frame "internal error: ...", replies are
matched to requests by id (so they may leave out of order), and a malformed
frame drops only its connection.

Design (B200 server side, not the reference's thread-per-connection reader):
one selector thread owns every socket and fills each frame directly into its
final buffer with `recv_into` -- no per-chunk `bytes` concatenation. Payloads
of TensorMsg size are received into page-locked host blocks from a reusable
pool (`PinnedPool`), so the STEP / FORWARD tensors reach HBM by one DMA
(`codec.decode_tensor(..., pinned)`) without a pageable bounce buffer. Complete
frames are served on a worker pool; a worker writes its reply with one
`sendall` under the connection's send lock and then returns the payload block
to the pool.
"""

from __future__ import annotations

import itertools
import logging
import selectors
import socket
import threading
from concurrent.futures import ThreadPoolExecutor

from .errors import ERR_GENERIC, ProtocolError, RemoteError, TimeoutError_, TransportError
from .wire import FRAME_HEADER_LEN, MSG, _parse_header, decode_error, encode_error, encode_frame, read_frame

log = logging.getLogger(__name__)

PIN_MIN_BYTES = 4096  # smaller payloads (session ids, decode headers) stay in ordinary memory


class PinnedPool:
    """Page-locked host blocks in power-of-two size classes, reused across
    frames (cudaHostAlloc costs far more than a frame). Blocks are torch uint8
    tensors. A handler that DMAs from its payload must have completed the copy
    before it returns (the server's _decode synchronizes its copy stream): the
    block is refilled by the next frame right after."""

    def __init__(self, device: int, max_cached_bytes: int = 1 << 30):
        self.device = device
        self._free: dict[int, list] = {}
        self._lock = threading.Lock()
        self._cached = 0
        self.max_cached = max_cached_bytes

    @staticmethod
    def _cls(n: int) -> int:
        return max(PIN_MIN_BYTES, 1 << (n - 1).bit_length())

    def take(self, n: int):
        import torch

        c = self._cls(n)
        with self._lock:
            lst = self._free.get(c)
            if lst:
                self._cached -= c
                return lst.pop()
        return torch.empty(c, dtype=torch.uint8).pin_memory()

    def give(self, block) -> None:
        c = block.numel()
        with self._lock:
            if self._cached + c <= self.max_cached:
                self._free.setdefault(c, []).append(block)
                self._cached += c


class Payload:
    """Read-only view of one request payload. `view` is a memoryview of the
    received bytes; `pinned` (or None) is the page-locked torch tensor holding
    the same bytes, sliced alongside. Slicing returns a Payload; bytes(p)
    copies."""

    __slots__ = ("view", "pinned")

    def __init__(self, view, pinned=None):
        self.view = view if isinstance(view, memoryview) else memoryview(view)
        self.pinned = pinned

    def __len__(self) -> int:
        return len(self.view)

    def __bytes__(self) -> bytes:
        return self.view.tobytes()

    def __getitem__(self, k):
        if isinstance(k, slice):
            a, b, step = k.indices(len(self.view))
            if step != 1:
                raise ValueError("strided payload slice")
            return Payload(self.view[a:b], self.pinned[a:b] if self.pinned is not None else None)
        return self.view[k]


def as_view(data) -> memoryview:
    return data.view if isinstance(data, Payload) else memoryview(data)


class _Conn:
    __slots__ = ("sock", "send_lock", "hdr", "hdr_got", "buf", "got", "block", "msg_type", "rid")

    def __init__(self, sock):
        self.sock = sock
        self.send_lock = threading.Lock()
        self.hdr = bytearray(FRAME_HEADER_LEN)
        self.hdr_got = 0
        self.buf = None
        self.got = 0
        self.block = None
        self.msg_type = self.rid = 0


class RpcServer:
    def __init__(self, host: str, port: int, handler, max_workers: int = 64, pinned_device: int | None = None):
        """pinned_device: CUDA device whose transfers read the payloads (page-locked
        receive buffers), or None for ordinary memory (no CUDA needed)."""
        self.handler = handler
        self._listener = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        self._listener.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        self._listener.bind((host, port))
        self._listener.listen(128)
        self._listener.setblocking(False)
        self.host = host
        self.port = self._listener.getsockname()[1]
        self.pool = PinnedPool(pinned_device) if pinned_device is not None else None
        self._workers = ThreadPoolExecutor(max_workers=max_workers, thread_name_prefix="rpc-worker")
        self._sel = selectors.DefaultSelector()
        self._wake_r, self._wake_w = socket.socketpair()
        self._wake_r.setblocking(False)
        self._conns: dict[int, _Conn] = {}
        self._stopping = False
        self._thread = None
        self.frames = 0

    @property
    def address(self) -> str:
        return f"{self.host}:{self.port}"

    def start(self) -> "RpcServer":
        self._sel.register(self._listener, selectors.EVENT_READ, "accept")
        self._sel.register(self._wake_r, selectors.EVENT_READ, "wake")
        self._thread = threading.Thread(target=self._loop, name="rpc-loop", daemon=True)
        self._thread.start()
        return self

    # ------------------------------------------------------------------ selector loop

    def _loop(self):
        while not self._stopping:
            try:
                events = self._sel.select(timeout=1.0)
            except (OSError, ValueError):
                break
            for key, _ in events:
                tag = key.data
                if tag == "accept":
                    self._accept()
                elif tag == "wake":
                    try:
                        self._wake_r.recv(64)
                    except OSError:
                        pass
                else:
                    self._readable(tag)
        for c in list(self._conns.values()):
            self._drop(c)

    def _accept(self):
        while True:
            try:
                sock, _ = self._listener.accept()
            except (BlockingIOError, InterruptedError):
                return
            except OSError:
                return
            sock.setblocking(True)  # reads happen only on readiness; worker replies use blocking sendall
            sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            c = _Conn(sock)
            self._conns[sock.fileno()] = c
            self._sel.register(sock, selectors.EVENT_READ, c)

    def _readable(self, c: _Conn):
        try:
            if c.buf is None:
                n = c.sock.recv_into(memoryview(c.hdr)[c.hdr_got:])
                if n == 0:
                    return self._drop(c)
                c.hdr_got += n
                if c.hdr_got == FRAME_HEADER_LEN:
                    self._begin_payload(c)
            else:
                n = c.sock.recv_into(c.buf[c.got:])
                if n == 0:
                    return self._drop(c)
                c.got += n
                if c.got == len(c.buf):
                    self._dispatch(c)
        except ProtocolError as e:
            log.warning("dropping connection on a malformed frame: %s", e)
            self._drop(c)
        except OSError:
            self._drop(c)

    def _begin_payload(self, c: _Conn):
        c.msg_type, c.rid, plen = _parse_header(bytes(c.hdr))
        c.got = 0
        if plen >= PIN_MIN_BYTES and self.pool is not None:
            c.block = self.pool.take(plen)
            c.buf = memoryview(c.block.numpy())[:plen]
        else:
            c.block = None
            c.buf = memoryview(bytearray(plen))
        if plen == 0:
            self._dispatch(c)

    def _dispatch(self, c: _Conn):
        pinned = c.block[:len(c.buf)] if c.block is not None else None
        payload = Payload(c.buf, pinned)
        job = (c, c.msg_type, c.rid, payload, c.block)
        c.buf, c.block, c.hdr_got, c.got = None, None, 0, 0
        self.frames += 1
        try:
            self._workers.submit(self._serve, *job)
        except RuntimeError:  # shutting down
            pass

    def _drop(self, c: _Conn):
        self._conns.pop(c.sock.fileno(), None)
        try:
            self._sel.unregister(c.sock)
        except (KeyError, ValueError, OSError):
            pass
        try:
            c.sock.close()
        except OSError:
            pass
        if c.block is not None and self.pool is not None:
            self.pool.give(c.block)
            c.block = None

    # ------------------------------------------------------------------ workers

    def _serve(self, c: _Conn, msg_type: int, rid: int, payload: Payload, block):
        try:
            try:
                rtype, reply = self.handler(msg_type, payload)
            except RemoteError as e:
                rtype, reply = MSG.ERROR, encode_error(e.code, e.message)
            except Exception as e:  # noqa: BLE001 - reported to the caller as ERR_GENERIC
                log.exception("rpc handler raised (type 0x%02x)", msg_type)
                rtype, reply = MSG.ERROR, encode_error(ERR_GENERIC, f"internal error: {e}")
            frame = encode_frame(rtype, rid, reply)
            with c.send_lock:
                c.sock.sendall(frame)
        except OSError:
            pass
        finally:
            if block is not None and self.pool is not None:
                self.pool.give(block)

    def stop(self):
        if self._stopping:
            return
        self._stopping = True
        try:
            self._wake_w.send(b"x")
        except OSError:
            pass
        if self._thread is not None:
            self._thread.join(timeout=5)
        for s in (self._listener, self._wake_r, self._wake_w):
            try:
                s.close()
            except OSError:
                pass
        try:
            self._sel.close()
        except (OSError, ValueError):
            pass
        self._workers.shutdown(wait=False, cancel_futures=True)


# ------------------------------------------------------------------ client side


_ids = itertools.count(1)


def _recv_exact(sock, n: int) -> bytes:
    buf = bytearray(n)
    view, got = memoryview(buf), 0
    while got < n:
        try:
            k = sock.recv_into(view[got:])
        except socket.timeout as e:
            raise TimeoutError_("rpc timed out") from e
        except OSError as e:
            raise TransportError(f"recv failed: {e}") from e
        if k == 0:
            raise TransportError("connection closed by peer")
        got += k
    return bytes(buf)


class Connection:
    """One persistent request/response connection (sequential calls)."""

    def __init__(self, address: str, timeout_ms: float = 5000.0):
        host, port = address.rsplit(":", 1)
        self.address = address
        try:
            self.sock = socket.create_connection((host, int(port)), timeout=timeout_ms / 1000.0)
        except OSError as e:
            raise TransportError(f"connect to {address} failed: {e}") from e
        self.sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)

    def call(self, msg_type: int, payload: bytes = b"", deadline_ms: float = 5000.0) -> bytes:
        self.sock.settimeout(deadline_ms / 1000.0)
        rid = next(_ids)
        try:
            self.sock.sendall(encode_frame(msg_type, rid, payload))
        except OSError as e:
            raise TransportError(f"send to {self.address} failed: {e}") from e
        frame = read_frame(lambda n: _recv_exact(self.sock, n))
        if frame.request_id != rid:
            raise ProtocolError(f"reply id {frame.request_id} for request {rid}")
        if frame.msg_type == MSG.ERROR:
            raise decode_error(frame.payload)
        return frame.payload

    def close(self):
        try:
            self.sock.close()
        except OSError:
            pass


def call(address: str, msg_type: int, payload: bytes = b"", deadline_ms: float = 5000.0) -> bytes:
    """One request on a fresh connection (registry announcements)."""
    conn = Connection(address, deadline_ms)
    try:
        return conn.call(msg_type, payload, deadline_ms)
    finally:
        conn.close()


__all__ = ["RpcServer", "PinnedPool", "Payload", "Connection", "call", "as_view"]
