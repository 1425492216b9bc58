"""Frame codec of the reference wire protocol, restated byte for byte
(/root/reference/pkg/src/swarmlm/transport/wire.py:1-84): magic 0x50 0x54,
version 1, msg_type u8, request_id u64 BE, payload_len u32 BE, payload.
The TensorMsg codec lives in codec.py (GPU int8 path)."""

from __future__ import annotations

import struct
from dataclasses import dataclass

from .errors import InputError, ProtocolError

MAGIC = b"\x50\x54"
VERSION = 1
FRAME_HEADER_LEN = 16
MAX_PAYLOAD = 64 * 1024 * 1024


class MSG:
    PING = 0x01
    INFO = 0x02
    OPEN_SESSION = 0x10
    STEP = 0x11
    CLOSE_SESSION = 0x12
    FORWARD = 0x20
    BACKWARD = 0x21
    ANNOUNCE = 0x30
    LOOKUP = 0x31
    GOSSIP = 0x32
    ERROR = 0x7F


@dataclass(frozen=True)
class Frame:
    msg_type: int
    request_id: int
    payload: bytes


def encode_frame(msg_type: int, request_id: int, payload: bytes) -> bytes:
    if len(payload) >= MAX_PAYLOAD:
        raise InputError(f"payload {len(payload)} exceeds {MAX_PAYLOAD} byte cap")
    return MAGIC + struct.pack(">BBQI", VERSION, msg_type, request_id, len(payload)) + payload


def _parse_header(header: bytes):
    if header[:2] != MAGIC:
        raise ProtocolError("bad magic")
    version, msg_type, request_id, plen = struct.unpack(">BBQI", header[2:FRAME_HEADER_LEN])
    if version != VERSION:
        raise ProtocolError(f"unknown protocol version {version}")
    if plen > MAX_PAYLOAD:
        raise ProtocolError("oversized payload")
    return msg_type, request_id, plen


def decode_frame(data: bytes) -> Frame:
    if len(data) < FRAME_HEADER_LEN:
        raise ProtocolError("truncated frame header")
    msg_type, request_id, plen = _parse_header(data[:FRAME_HEADER_LEN])
    if len(data) != FRAME_HEADER_LEN + plen:
        raise ProtocolError("payload length mismatch")
    return Frame(msg_type, request_id, data[FRAME_HEADER_LEN:])


def read_frame(recv_exact) -> Frame:
    msg_type, request_id, plen = _parse_header(recv_exact(FRAME_HEADER_LEN))
    return Frame(msg_type, request_id, recv_exact(plen) if plen else b"")


def encode_error(code: int, message: str) -> bytes:
    """ERROR payload: u16 code BE + UTF-8 message (transport/rpc.py:35-36)."""
    return struct.pack(">H", code) + message.encode()


def decode_error(payload: bytes):
    from .errors import RemoteError

    if len(payload) < 2:
        return RemoteError(0, "malformed error payload")
    (code,) = struct.unpack(">H", payload[:2])
    return RemoteError(code, payload[2:].decode(errors="replace"))
