"""CPU tests of the framed-RPC layer (paper_2209_01188_b200.rpc): the
reference's handler contract (transport/rpc.py:178-274) over the selector
reactor -- replies matched by id, RemoteError -> ERROR frame with its code,
other exceptions -> ERR_GENERIC, a malformed frame drops only its
connection, large payloads received whole, concurrent connections."""

import socket
import struct
import threading
import time

import pytest

from paper_2209_01188_b200.errors import ERR_BUSY, ERR_GENERIC, ProtocolError, RemoteError
from paper_2209_01188_b200.rpc import Connection, Payload, RpcServer, call
from paper_2209_01188_b200.wire import MSG, decode_frame, encode_frame, read_frame


def handler(msg_type, payload):
    assert isinstance(payload, Payload)
    if msg_type == MSG.PING:
        return MSG.PING, bytes(payload)
    if msg_type == 0x40:  # slow echo: replies may overtake each other
        time.sleep(struct.unpack(">d", bytes(payload[:8]))[0])
        return 0x40, bytes(payload)
    if msg_type == 0x41:
        raise RemoteError(ERR_BUSY, "busy now")
    if msg_type == 0x42:
        raise ValueError("boom")
    if msg_type == 0x43:  # length + checksum of a large payload, sliced without copies
        v = payload[4:]
        return 0x43, struct.pack(">QQ", len(v), sum(v.view[::4096]))
    raise RemoteError(6, "unknown")


@pytest.fixture
def server():
    s = RpcServer("127.0.0.1", 0, handler).start()
    yield s
    s.stop()


def test_ping_and_error_frames(server):
    assert call(server.address, MSG.PING, b"hello") == b"hello"
    with pytest.raises(RemoteError) as ei:
        call(server.address, 0x41)
    assert ei.value.code == ERR_BUSY and ei.value.message == "busy now"
    with pytest.raises(RemoteError) as ei:
        call(server.address, 0x42)
    assert ei.value.code == ERR_GENERIC and ei.value.message == "internal error: boom"


def test_large_payload_received_whole(server):
    data = bytes(range(256)) * (1 << 16)  # 16 MiB
    c = Connection(server.address)
    try:
        n, chk = struct.unpack(">QQ", c.call(0x43, b"abcd" + data, 30000.0))
    finally:
        c.close()
    assert n == len(data) and chk == sum(memoryview(data)[::4096])


def test_out_of_order_replies_matched_by_id(server):
    sock = socket.create_connection(("127.0.0.1", server.port))
    try:
        sock.sendall(encode_frame(0x40, 1, struct.pack(">d", 0.3) + b"slow"))
        sock.sendall(encode_frame(0x40, 2, struct.pack(">d", 0.0) + b"fast"))

        def rx(n):
            buf = b""
            while len(buf) < n:
                buf += sock.recv(n - len(buf))
            return buf

        first, second = read_frame(rx), read_frame(rx)
        assert (first.request_id, second.request_id) == (2, 1)
        assert first.payload.endswith(b"fast") and second.payload.endswith(b"slow")
    finally:
        sock.close()


def test_malformed_frame_drops_only_that_connection(server):
    bad = socket.create_connection(("127.0.0.1", server.port))
    good = Connection(server.address)
    try:
        bad.sendall(b"XX" + bytes(14))  # bad magic
        bad.settimeout(5)
        assert bad.recv(16) == b""  # closed by the server
        assert good.call(MSG.PING, b"still here") == b"still here"
    finally:
        bad.close()
        good.close()


def test_concurrent_connections(server):
    errs = []

    def worker(i):
        try:
            c = Connection(server.address)
            for k in range(20):
                msg = f"{i}:{k}".encode() * 100
                assert c.call(MSG.PING, msg) == msg
            c.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(16)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs


def test_frame_codec_roundtrip():
    f = encode_frame(MSG.STEP, 7, b"xyz")
    fr = decode_frame(f)
    assert (fr.msg_type, fr.request_id, fr.payload) == (MSG.STEP, 7, b"xyz")
    with pytest.raises(ProtocolError):
        decode_frame(f[:-1])
