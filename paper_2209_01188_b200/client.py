"""Per-hop client calls against a span server, in the reference's wire
vocabulary (client.py:290-331 STEP chain, client.py:442-498 FORWARD /
BACKWARD parts), used by the box front end, the bench's end-to-end leg and
the reference-free drop-in tests.

FORWARD chunking: one frame carries at most 64 MiB (transport/wire.py:93),
so a [B, t, d] batch larger than that (the C5 shape [32, 512, 14336] f32 is
939 MB) is sent as consecutive row groups, each its own FORWARD with its own
tape -- the same per-part tapes the reference's DistributedModel keeps when it
splits rows over servers (client.py:452-468, `_StagePart`).
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

from . import codec
from .rpc import Connection
from .wire import MAX_PAYLOAD, MSG


def _np_tensor_msg(x: np.ndarray, encoding: int) -> bytes:
    """TensorMsg bytes of a host array (transport/wire.py:87-106 layout)."""
    x = np.ascontiguousarray(x, np.float32)
    if encoding == codec.ENC_F32:
        return codec.encode_header(codec.ENC_F32, x.shape) + x.astype("<f4").tobytes()
    return codec.encode_tensor(x, encoding)


def _np_decode(data: bytes) -> np.ndarray:
    enc, dims, bs, scales, payload = codec.parse_tensor(data)
    if enc == codec.ENC_F32:
        return payload.reshape(dims).copy()
    return codec.decode_tensor(data).cpu().numpy()


@dataclass
class ForwardPart:
    tape_id: bytes
    rows: range


class SpanClient:
    """One persistent connection to one span server."""

    def __init__(self, address: str, encoding: int = codec.ENC_F32, timeout_ms: float = 60_000.0):
        self.address, self.encoding, self.timeout_ms = address, encoding, timeout_ms
        self.conn = Connection(address, timeout_ms)

    def close(self):
        self.conn.close()

    def call(self, msg_type: int, payload: bytes = b"") -> bytes:
        return self.conn.call(msg_type, payload, self.timeout_ms)

    # ---------------------------------------------------------------- sessions

    def open_session(self, max_len: int, sid: bytes | None = None) -> bytes:
        sid = sid or os.urandom(16)
        self.call(MSG.OPEN_SESSION, sid + struct.pack(">I", max_len))
        return sid

    def close_session(self, sid: bytes) -> None:
        self.call(MSG.CLOSE_SESSION, sid)

    def step_raw(self, sid: bytes, start_pos: int, tensor_msg: bytes) -> bytes:
        return self.call(MSG.STEP, sid + struct.pack(">I", start_pos) + tensor_msg)

    def step(self, sid: bytes, start_pos: int, hidden: np.ndarray) -> np.ndarray:
        return _np_decode(self.step_raw(sid, start_pos, _np_tensor_msg(hidden, self.encoding)))

    # ---------------------------------------------------------------- FORWARD / BACKWARD

    def forward(self, batch: np.ndarray):
        """FORWARD of [B, t, d] in row groups of at most MAX_PAYLOAD bytes per
        frame; returns (outputs [B, t, d], [ForwardPart])."""
        batch = np.asarray(batch, np.float32)
        B, t, d = batch.shape
        row_bytes = 4 * t * d
        per = max(1, (MAX_PAYLOAD - 64) // max(row_bytes, 1))
        out = np.empty_like(batch)
        parts = []
        for r0 in range(0, B, per):
            rows = range(r0, min(B, r0 + per))
            reply = self.call(MSG.FORWARD, _np_tensor_msg(batch[r0:rows.stop], self.encoding))
            out[r0:rows.stop] = _np_decode(reply[16:])
            parts.append(ForwardPart(reply[:16], rows))
        return out, parts

    def backward(self, parts, grad: np.ndarray) -> np.ndarray:
        grad = np.asarray(grad, np.float32)
        out = np.empty_like(grad)
        for p in parts:
            reply = self.call(MSG.BACKWARD, p.tape_id + _np_tensor_msg(grad[p.rows.start:p.rows.stop], codec.ENC_F32))
            out[p.rows.start:p.rows.stop] = _np_decode(reply)
        return out
