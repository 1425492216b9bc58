"""TCP ingress for the span server: the reference's handler contract
(/root/reference/pkg/src/swarmlm/transport/rpc.py:178-274): framed requests on
a thread pool, `handler(msg_type, payload) -> (reply_type, reply)`, RemoteError
-> ERROR frame, any other exception -> ERR_GENERIC, out-of-order replies matched
by request id. Plus a minimal client `call()` used to announce to the registry.

The compute path never runs on these threads' critical section beyond
submitting work: the STEP handler hands tensors to the span scheduler.
"""

from __future__ import annotations

import itertools
import logging
import socket
import threading
from concurrent.futures import ThreadPoolExecutor

from .errors import ERR_GENERIC, ProtocolError, RemoteError, TimeoutError_, TransportError
from .wire import MSG, encode_error, encode_frame, read_frame, decode_error

log = logging.getLogger(__name__)


def _recv_exact(sock, n: int) -> bytes:
    buf = bytearray()
    while len(buf) < n:
        try:
            chunk = sock.recv(n - len(buf))
        except OSError as e:
            raise TransportError(f"recv failed: {e}") from e
        if not chunk:
            raise TransportError("connection closed by peer")
        buf.extend(chunk)
    return bytes(buf)


class RpcServer:
    def __init__(self, host: str, port: int, handler, max_workers: int = 64):
        self.handler = handler
        self._listener = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        self._listener.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        self._listener.bind((host, port))
        self._listener.listen(128)
        self.host = host
        self.port = self._listener.getsockname()[1]
        self._pool = ThreadPoolExecutor(max_workers=max_workers)
        self._conns: set = set()
        self._lock = threading.Lock()
        self._stopping = False

    @property
    def address(self) -> str:
        return f"{self.host}:{self.port}"

    def start(self) -> "RpcServer":
        threading.Thread(target=self._accept_loop, daemon=True).start()
        return self

    def _accept_loop(self):
        while not self._stopping:
            try:
                sock, _ = self._listener.accept()
            except OSError:
                return
            sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            with self._lock:
                self._conns.add(sock)
            threading.Thread(target=self._conn_loop, args=(sock,), daemon=True).start()

    def _conn_loop(self, sock):
        send_lock = threading.Lock()
        try:
            while True:
                frame = read_frame(lambda n: _recv_exact(sock, n))
                self._pool.submit(self._handle, frame, sock, send_lock)
        except ProtocolError as e:
            log.warning("protocol error, dropping connection: %s", e)
        except (TransportError, OSError, RuntimeError):
            pass
        finally:
            with self._lock:
                self._conns.discard(sock)
            try:
                sock.close()
            except OSError:
                pass

    def _handle(self, frame, sock, send_lock):
        try:
            rtype, reply = self.handler(frame.msg_type, frame.payload)
        except RemoteError as e:
            rtype, reply = MSG.ERROR, encode_error(e.code, e.message)
        except Exception as e:  # noqa: BLE001 - a handler bug must not kill the server
            log.exception("handler failed for msg_type 0x%02x", frame.msg_type)
            rtype, reply = MSG.ERROR, encode_error(ERR_GENERIC, f"internal error: {e}")
        try:
            with send_lock:
                sock.sendall(encode_frame(rtype, frame.request_id, reply))
        except OSError:
            pass

    def stop(self):
        self._stopping = True
        try:
            self._listener.close()
        except OSError:
            pass
        with self._lock:
            conns = list(self._conns)
        for c in conns:
            try:
                c.close()
            except OSError:
                pass
        self._pool.shutdown(wait=False, cancel_futures=True)


_ids = itertools.count(1)


def call(address: str, msg_type: int, payload: bytes = b"", deadline_ms: float = 5000.0) -> bytes:
    """One request on a fresh connection (registry announce/gossip)."""
    host, port = address.rsplit(":", 1)
    try:
        sock = socket.create_connection((host, int(port)), timeout=deadline_ms / 1000.0)
    except OSError as e:
        raise TransportError(f"connect to {address} failed: {e}") from e
    try:
        sock.settimeout(deadline_ms / 1000.0)
        rid = next(_ids)
        sock.sendall(encode_frame(msg_type, rid, payload))
        try:
            frame = read_frame(lambda n: _recv_exact(sock, n))
        except socket.timeout as e:
            raise TimeoutError_(f"rpc to {address} timed out") from e
        if frame.msg_type == MSG.ERROR:
            raise decode_error(frame.payload)
        return frame.payload
    finally:
        sock.close()
