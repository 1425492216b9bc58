"""Device-side codecs behind the reference's quant/wire API.

quantize_blockwise / dequantize_blockwise mirror
/root/reference/pkg/src/swarmlm/quant.py:33-66 (same names, argument meaning
and errors) on CUDA tensors; encode_tensor / decode_tensor mirror
transport/wire.py:87-138 byte for byte, running the int8 codec on the GPU.
gen_tensor mirrors model.py:60-62 tensor_stream.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InputError, ProtocolError
from .model import stream_key

DEFAULT_BLOCK_SIZE = 64
ENC_F32 = 0
ENC_INT8 = 1
MAX_PAYLOAD = 64 * 1024 * 1024


@dataclass
class QuantizedBlockwise:
    block_size: int
    scales: object  # torch f32 [n_blocks] (device)
    codes: object   # torch int8 [n] (device)
    shape: tuple


def _dev():
    import torch

    return torch.device("cuda", torch.cuda.current_device())


def quantize_blockwise(x, block_size: int = DEFAULT_BLOCK_SIZE) -> QuantizedBlockwise:
    import torch

    if block_size < 1:
        raise InputError("block_size must be >= 1")
    x = torch.as_tensor(x)
    if not x.is_cuda:
        x = x.to(_dev())
    x = x.to(torch.float32).contiguous()
    if not bool(torch.isfinite(x).all()):
        raise InputError("non-finite input tensor")
    n = x.numel()
    nb = max(1, math.ceil(n / block_size)) if n else 0
    scales = torch.empty(nb, dtype=torch.float32, device=x.device)
    codes = torch.empty(n, dtype=torch.int8, device=x.device)
    _lib.check(_lib.lib().pb_quantize_blockwise(_lib.ptr(x), n, block_size, _lib.ptr(codes), _lib.ptr(scales),
                                                _lib.stream_ptr(torch.cuda.current_stream(x.device))))
    return QuantizedBlockwise(block_size, scales, codes, tuple(x.shape))


def dequantize_blockwise(q: QuantizedBlockwise):
    import torch

    n = int(np.prod(q.shape)) if q.shape else 1
    expected = max(1, math.ceil(n / q.block_size)) if n else 0
    if q.codes.numel() != n or q.scales.numel() != expected:
        raise InputError("corrupt quantized tensor: size/scale count mismatch")
    out = torch.empty(n, dtype=torch.float32, device=q.codes.device)
    _lib.check(_lib.lib().pb_dequantize_blockwise(_lib.ptr(q.codes.contiguous()), _lib.ptr(q.scales.contiguous()),
                                                  n, q.block_size, _lib.ptr(out),
                                                  _lib.stream_ptr(torch.cuda.current_stream(out.device))))
    return out.reshape(q.shape)


def gen_tensor(seed: int, path: str, n: int, first: int = 0):
    """tensor_stream(seed, path, n) on the device (elements [first, first+n))."""
    import torch

    out = torch.empty(n, dtype=torch.float32, device=_dev())
    _lib.check(_lib.lib().pb_gen_tensor(stream_key(seed, path), first, n, _lib.ptr(out),
                                        _lib.stream_ptr(torch.cuda.current_stream(out.device))))
    return out


# ------------------------------------------------------------------ wire TensorMsg


def encode_header(encoding: int, shape) -> bytes:
    return struct.pack(">BB", encoding, len(shape)) + b"".join(struct.pack(">I", d) for d in shape)


_PINNED: dict = {}


def _pinned(nbytes: int):
    """Reusable pinned host staging buffer (one per thread, grown on demand)."""
    import threading

    import torch

    key = threading.get_ident()
    buf = _PINNED.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8).pin_memory()
        _PINNED[key] = buf
    return buf


def encode_tensor(t, encoding: int = ENC_F32, block_size: int = 64) -> bytes:
    """TensorMsg bytes (transport/wire.py:87-106). `t` may be a numpy array or a
    CUDA tensor; int8 encoding runs on the GPU. A CUDA tensor leaves the device
    in one pinned copy (codes, scales and the finiteness flag together, one
    stream synchronization)."""
    import torch

    if encoding not in (ENC_F32, ENC_INT8):
        raise InputError(f"unknown tensor encoding {encoding}")
    if isinstance(t, np.ndarray):
        arr = np.asarray(t, np.float32)
        shape = arr.shape
        if not np.all(np.isfinite(arr)):
            raise InputError("non-finite tensor")
    else:
        arr = None
        shape = tuple(t.shape)
    if len(shape) > 255:
        raise InputError("too many dimensions")
    n = int(np.prod(shape)) if shape else 1
    if n and n * 4 > MAX_PAYLOAD:
        raise InputError("tensor exceeds frame cap")
    head = encode_header(encoding, shape)
    if arr is not None:
        if encoding == ENC_F32:
            return head + np.ascontiguousarray(arr, "<f4").tobytes()
        q = quantize_blockwise(torch.as_tensor(arr), block_size)
        return (head + struct.pack(">I", block_size) + q.scales.cpu().numpy().astype("<f4").tobytes()
                + q.codes.cpu().numpy().tobytes())
    x = t.detach().to(torch.float32).contiguous()
    stream = torch.cuda.current_stream(x.device)
    flag = (~torch.isfinite(x)).any().to(torch.uint8).reshape(1)
    if encoding == ENC_F32:
        buf = _pinned(4 * n + 1)
        buf[:4 * n].view(torch.float32).copy_(x.reshape(-1), non_blocking=True)
        buf[4 * n:4 * n + 1].copy_(flag, non_blocking=True)
        stream.synchronize()
        if buf[4 * n].item():
            raise InputError("non-finite tensor")
        return head + buf[:4 * n].numpy().tobytes()
    if block_size < 1:
        raise InputError("block_size must be >= 1")
    nb = max(1, math.ceil(n / block_size)) if n else 0
    scales = torch.empty(nb, dtype=torch.float32, device=x.device)
    codes = torch.empty(n, dtype=torch.int8, device=x.device)
    _lib.check(_lib.lib().pb_quantize_blockwise(_lib.ptr(x), n, block_size, _lib.ptr(codes), _lib.ptr(scales),
                                                _lib.stream_ptr(stream)))
    buf = _pinned(4 * nb + n + 1)
    buf[:4 * nb].view(torch.float32).copy_(scales, non_blocking=True)
    buf[4 * nb:4 * nb + n].view(torch.int8).copy_(codes, non_blocking=True)
    buf[4 * nb + n:4 * nb + n + 1].copy_(flag, non_blocking=True)
    stream.synchronize()
    if buf[4 * nb + n].item():
        raise InputError("non-finite tensor")
    return head + struct.pack(">I", block_size) + buf[:4 * nb + n].numpy().tobytes()


def _buf(data):
    """(memoryview, pinned torch uint8 tensor | None) of bytes / memoryview / rpc.Payload."""
    if hasattr(data, "pinned") and hasattr(data, "view"):
        return data.view, data.pinned
    return memoryview(data), None


def parse_tensor(data):
    """Split TensorMsg bytes into (encoding, dims, block_size, scales np, codes np | f32 np)
    without decoding (transport/wire.py:109-138 validation). `data` may be
    bytes, a memoryview or an rpc.Payload (zero-copy numpy views)."""
    return _parse(_buf(data)[0])[:5]


def _parse(data):
    if len(data) < 2:
        raise ProtocolError("truncated tensor header")
    encoding, ndim = struct.unpack(">BB", data[:2])
    off = 2
    if len(data) < off + 4 * ndim:
        raise ProtocolError("truncated tensor dims")
    dims = struct.unpack(f">{ndim}I", data[off:off + 4 * ndim]) if ndim else ()
    off += 4 * ndim
    n = int(math.prod(dims)) if ndim else 1
    if encoding == ENC_F32:
        if len(data) != off + 4 * n:
            raise ProtocolError("f32 tensor size mismatch")
        return encoding, dims, 0, None, np.frombuffer(data, "<f4", count=n, offset=off), (off, None)
    if encoding == ENC_INT8:
        if len(data) < off + 4:
            raise ProtocolError("truncated int8 tensor")
        (block_size,) = struct.unpack(">I", data[off:off + 4])
        off += 4
        if block_size < 1:
            raise ProtocolError("bad block size")
        nb = math.ceil(n / block_size) if n else 0
        if len(data) != off + 4 * nb + n:
            raise ProtocolError("int8 tensor size mismatch")
        scales = np.frombuffer(data, "<f4", count=nb, offset=off)
        codes = np.frombuffer(data, np.int8, count=n, offset=off + 4 * nb)
        return encoding, dims, block_size, scales, codes, (off + 4 * nb, off)
    raise ProtocolError(f"unknown tensor encoding {encoding}")


def payload_finite(data) -> bool:
    """True iff the TensorMsg's values are finite (f32 values, or int8 scales:
    int8 codes times finite scales are finite)."""
    enc, _, _, scales, payload = parse_tensor(data)
    vals = payload if enc == ENC_F32 else scales
    return bool(np.isfinite(vals).all()) if vals.size else True


def _h2d(arr, pinned, off, nbytes, dtype, dev):
    """Host -> device copy of one TensorMsg section: straight from the
    page-locked receive buffer when there is one (asynchronous DMA, ordered on
    the current stream before any kernel that reads it), else via a copy of
    the pageable bytes."""
    import torch

    if pinned is not None and nbytes:
        dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)  # aligned: sections start at any byte offset
        dst.copy_(pinned[off:off + nbytes], non_blocking=True)
        return dst.view(dtype)
    return torch.from_numpy(arr.copy()).to(dev)


class DeviceTensorMsg:
    """A TensorMsg's sections on the device, not decoded: f32 values, or int8
    codes + block scales (upload_tensor)."""

    __slots__ = ("encoding", "dims", "block_size", "values", "codes", "scales")

    def __init__(self, encoding, dims, block_size=0, values=None, codes=None, scales=None):
        self.encoding, self.dims, self.block_size = encoding, tuple(dims), block_size
        self.values, self.codes, self.scales = values, codes, scales

    @property
    def rows(self) -> int:
        return int(self.dims[0]) if self.dims else 1

    def decode(self):
        """-> CUDA f32 tensor of dims (int8: one dequantize kernel on the current stream)."""
        if self.encoding == ENC_F32:
            return self.values
        return dequantize_blockwise(QuantizedBlockwise(self.block_size, self.scales, self.codes, self.dims))


def upload_tensor(data, device=None) -> DeviceTensorMsg:
    """TensorMsg -> its sections on the device (DMA only, no kernel: the
    STEP scheduler decodes a whole batch on its own stream)."""
    import torch

    dev = device or _dev()
    view, pinned = _buf(data)
    enc, dims, bs, scales, payload, (poff, soff) = _parse(view)
    if enc == ENC_F32:
        return DeviceTensorMsg(enc, dims, values=_h2d(payload, pinned, poff, 4 * payload.size, torch.float32,
                                                      dev).reshape(dims))
    return DeviceTensorMsg(enc, dims, bs, codes=_h2d(payload, pinned, poff, payload.size, torch.int8, dev),
                           scales=_h2d(scales, pinned, soff, 4 * scales.size, torch.float32, dev))


def decode_tensor(data, device=None):
    """TensorMsg -> CUDA f32 tensor (int8 decoded on the GPU)."""
    import torch

    dev = device or _dev()
    view, pinned = _buf(data)
    enc, dims, bs, scales, payload, (poff, soff) = _parse(view)
    if enc == ENC_F32:
        return _h2d(payload, pinned, poff, 4 * payload.size, torch.float32, dev).reshape(dims)
    q = QuantizedBlockwise(bs, _h2d(scales, pinned, soff, 4 * scales.size, torch.float32, dev),
                           _h2d(payload, pinned, poff, payload.size, torch.int8, dev), tuple(dims))
    return dequantize_blockwise(q)
