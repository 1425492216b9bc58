"""ctypes binding of libpetals_b200.so (include/petals_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises. Call `build.build()` (or
`__graft_entry__.build()`) to compile it in-tree.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import RemoteError, raise_for

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PB_LIB") or os.path.join(HERE, "libpetals_b200.so")  # PB_LIB: A/B builds

# every symbol declared in include/petals_b200.h
EXPORTS = [
    "pb_last_error", "pb_version", "pb_quantize_blockwise", "pb_dequantize_blockwise", "pb_gen_tensor",
    "pb_span_create", "pb_span_destroy", "pb_span_device_bytes", "pb_span_gen_block", "pb_span_load_block",
    "pb_span_outliers", "pb_span_read_codes", "pb_span_step", "pb_span_step_int8", "pb_span_last_launches",
    "pb_span_profile", "pb_span_profile_read", "pb_head_create", "pb_head_destroy", "pb_head_device_bytes",
    "pb_head_gen", "pb_head_load", "pb_head_embed", "pb_head_embed_device", "pb_head_logits", "pb_head_greedy",
    "pb_span_step_tape", "pb_span_backward", "pb_trace_set", "pb_trace_meta",
    "pb_hop_alloc", "pb_hop_free", "pb_hop_open", "pb_hop_close", "pb_hop_wait", "pb_hop_signal",
]


class SpanConfig(C.Structure):
    _fields_ = [
        ("hidden", C.c_int32), ("n_heads", C.c_int32), ("mlp_ratio", C.c_int32), ("max_seq", C.c_int32),
        ("n_blocks", C.c_int32), ("first_block", C.c_int32), ("weights", C.c_int32), ("page_tokens", C.c_int32),
        ("n_pages", C.c_int32), ("max_tokens", C.c_int32), ("max_seqs", C.c_int32),
        ("outlier_threshold", C.c_float), ("device", C.c_int32), ("tc_min_tokens", C.c_int32),
        ("graphs", C.c_int32), ("operand_kernel", C.c_int32),
    ]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2209_01188_b200.build`")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, U64, F, VP = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_void_p
    L.pb_last_error.restype = C.c_char_p
    L.pb_version.restype = C.c_int
    sig = {
        "pb_quantize_blockwise": [P, I64, I32, P, P, VP],
        "pb_dequantize_blockwise": [P, P, I64, I32, P, VP],
        "pb_gen_tensor": [U64, I64, I64, P, VP],
        "pb_span_create": [C.POINTER(SpanConfig), C.POINTER(C.c_void_p)],
        "pb_span_destroy": [P],
        "pb_span_gen_block": [P, I32, U64, U64, U64, U64, F, I32, VP],
        "pb_span_load_block": [P, I32] + [P] * 12 + [VP],
        "pb_span_outliers": [P, I32, I32, P, I32, C.POINTER(C.c_int32)],
        "pb_span_read_codes": [P, I32, I32, P, P],
        "pb_span_step": [P, I32, I32, P, P, P, P, P, VP],
        "pb_span_step_int8": [P, I32, I32, P, P, P, P, P, P, P, P, P, P, VP],
        "pb_span_step_tape": [P, I32, I32, P, P, P, P, P, P, VP],
        "pb_span_backward": [P, P, I32, P, P, VP],
        "pb_span_profile": [P, I32],
        "pb_trace_set": [P, I64],
        "pb_hop_alloc": [I64, I32, C.POINTER(C.c_void_p), P],
        "pb_hop_free": [P],
        "pb_hop_open": [P, I32, C.POINTER(C.c_void_p)],
        "pb_hop_close": [P],
        "pb_hop_wait": [P, U64, I64, VP],
        "pb_hop_signal": [P, U64, VP],
        "pb_span_profile_read": [P, I32, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double)],
        "pb_head_create": [I32, I32, I32, I32, C.POINTER(C.c_void_p)],
        "pb_head_destroy": [P],
        "pb_head_gen": [P, U64, VP],
        "pb_head_load": [P, P, P, P, VP],
        "pb_head_embed": [P, P, I32, P, VP],
        "pb_head_embed_device": [P, P, I32, P, VP],
        "pb_head_logits": [P, P, I32, P, VP],
        "pb_head_greedy": [P, P, I32, P, P, VP],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.pb_span_device_bytes.argtypes = [P]
    L.pb_span_device_bytes.restype = C.c_int64
    L.pb_head_device_bytes.argtypes = [P]
    L.pb_head_device_bytes.restype = C.c_int64
    L.pb_trace_meta.argtypes = [P, I64]
    L.pb_trace_meta.restype = C.c_int64
    L.pb_span_last_launches.argtypes = [P]
    L.pb_span_last_launches.restype = C.c_int32
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        raise_for(rc, lib().pb_last_error().decode(errors="replace"))


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0


__all__ = ["lib", "check", "SpanConfig", "EXPORTS", "LIB_PATH", "ptr", "stream_ptr", "RemoteError"]
