"""Host-side block span: the Python mirror of the reference's per-server
compute (block_forward looped over a hosted range, server.py:383-385) on top
of the C-ABI span (include/petals_b200.h).

A `BlockSpan` owns the int8 (or f32) weights of blocks [start, end), a paged
fp16 KV pool shared by all sessions, and the workspaces; `step()` runs one
batched inference step for any number of sequences (each with t >= 1 new
positions), `forward()` the cache-less parallel forward of server.py:411-429.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import CapacityError, InputError
from .model import ModelConfig, block_keys


class PagePool:
    """Free list of KV pages; one page = page_tokens positions of every hosted block."""

    def __init__(self, n_pages: int):
        self.n_pages = n_pages
        self._free = list(range(n_pages - 1, -1, -1))
        self._lock = threading.Lock()

    @property
    def free_pages(self) -> int:
        return len(self._free)

    def alloc(self, n: int) -> list[int]:
        with self._lock:
            if n > len(self._free):
                raise CapacityError(f"KV pool exhausted: need {n} pages, {len(self._free)} free")
            return [self._free.pop() for _ in range(n)]

    def free(self, pages: list[int]) -> None:
        with self._lock:
            self._free.extend(reversed(pages))


@dataclass
class Sequence:
    """KV state of one session on this span (server.py:69-77 _Session.caches)."""

    pages: list = field(default_factory=list)
    length: int = 0


class BlockSpan:
    def __init__(self, config: ModelConfig, start: int, end: int, *, int8: bool = True, page_tokens: int = 64,
                 n_pages: int | None = None, max_tokens: int = 256, max_seqs: int = 64, device: int = 0,
                 outlier_threshold: float = 6.0, tc_min_tokens: int = 0, graphs: bool = True,
                 operand_kernel: bool = False):
        """operand_kernel: batch-1 decode builds its operands in k_fragwrite instead of the
        GEMV's operand warps (bit-identical; the A/B of tests/test_gpu_fused.py)."""
        import torch

        if not (0 <= start < end <= config.n_layers):
            raise InputError(f"block range [{start}, {end}) outside [0, {config.n_layers})")
        self.config, self.start, self.end = config, start, end
        self.n_blocks = end - start
        self.int8 = int8
        self.device = torch.device("cuda", device)
        self.page_tokens = page_tokens
        self.max_pages = -(-config.max_seq // page_tokens)
        if n_pages is None:
            n_pages = max(self.max_pages * 4, 8)
        self.max_tokens, self.max_seqs = max_tokens, max_seqs
        cfg = _lib.SpanConfig(
            hidden=config.hidden, n_heads=config.n_heads, mlp_ratio=config.mlp_ratio, max_seq=config.max_seq,
            n_blocks=self.n_blocks, first_block=start, weights=1 if int8 else 0, page_tokens=page_tokens,
            n_pages=n_pages, max_tokens=max_tokens, max_seqs=max_seqs, outlier_threshold=outlier_threshold,
            device=device, tc_min_tokens=tc_min_tokens, graphs=1 if graphs else 0,
            operand_kernel=1 if operand_kernel else 0,
        )
        handle = C.c_void_p()
        torch.cuda.init()
        _lib.check(_lib.lib().pb_span_create(C.byref(cfg), C.byref(handle)))
        self._h = handle
        self.pool = PagePool(n_pages)
        self._lock = threading.Lock()

    # ------------------------------------------------------------------ lifecycle

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().pb_span_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().pb_span_device_bytes(self._h))

    @property
    def last_launches(self) -> int:
        return int(_lib.lib().pb_span_last_launches(self._h))

    PROF_GEMV, PROF_ATTN, PROF_PROLOGUE, PROF_GEMM_F32, PROF_CODEC, PROF_TC_GEMM, PROF_TC_DECODE = range(7)

    def profile(self, on: bool) -> None:
        """Bracket every launch with CUDA events (resets previous records)."""
        _lib.check(_lib.lib().pb_span_profile(self._h, 1 if on else 0))

    def profile_read(self, kind: int):
        """(device ms, launches, algorithmic bytes) summed over one kernel kind."""
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        _lib.check(_lib.lib().pb_span_profile_read(self._h, kind, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    # ------------------------------------------------------------------ weights

    def generate_weights(self, seed: int, outlier_boost: float = 0.0, boost_every: int = 0) -> None:
        """gen_checkpoint(seed) weights for the hosted blocks, generated and
        quantized on the device (model.py:176-209; quant.py:142-149)."""
        import torch

        st = _lib.stream_ptr(torch.cuda.current_stream(self.device))
        for j in range(self.n_blocks):
            k = block_keys(seed, self.start + j)
            _lib.check(_lib.lib().pb_span_gen_block(self._h, j, *k, float(outlier_boost), int(boost_every), st))

    def load_weights(self, blocks) -> None:
        """Load reference-layout f32 blocks (objects with ln1_gamma, ..., or
        the oracle's Block fields) for the hosted range, then quantize."""
        import torch

        st = _lib.stream_ptr(torch.cuda.current_stream(self.device))
        for j, b in enumerate(blocks):
            def t(*names):
                for n in names:
                    if hasattr(b, n):
                        return torch.as_tensor(np.ascontiguousarray(getattr(b, n), np.float32), device=self.device)
                raise AttributeError(names)

            ts = [t("ln1_gamma", "ln1_g"), t("ln1_beta", "ln1_b"), t("wqkv"), t("bqkv"), t("wo"), t("bo"),
                  t("ln2_gamma", "ln2_g"), t("ln2_beta", "ln2_b"), t("wmlp_in"), t("bmlp_in"), t("wmlp_out"),
                  t("bmlp_out")]
            _lib.check(_lib.lib().pb_span_load_block(self._h, j, *[_lib.ptr(x) for x in ts], st))

    def read_codes(self, j: int, m: int):
        """Reference-layout codes [out, in] int8 and scales [in] of matrix m
        (0 wqkv, 1 wo, 2 wmlp_in, 3 wmlp_out) of hosted block j."""
        d, r = self.config.hidden, self.config.mlp_ratio
        K, M = [(d, 3 * d), (d, d), (d, r * d), (r * d, d)][m]
        codes = np.empty((M, K), np.int8)
        scales = np.empty(K, np.float32)
        _lib.check(_lib.lib().pb_span_read_codes(self._h, j, m, codes.ctypes.data, scales.ctypes.data))
        return codes, scales

    def outliers(self, j: int, m: int) -> np.ndarray:
        cap = 1 << 16
        buf = np.empty(cap, np.int32)
        n = C.c_int32()
        _lib.check(_lib.lib().pb_span_outliers(self._h, j, m, buf.ctypes.data, cap, C.byref(n)))
        return buf[: n.value].copy()

    # ------------------------------------------------------------------ sequences

    def new_sequence(self) -> Sequence:
        return Sequence()

    def release(self, seq: Sequence) -> None:
        if seq.pages:
            self.pool.free(seq.pages)
        seq.pages = []
        seq.length = 0

    def pages_needed(self, seq: Sequence, new_len: int) -> int:
        return max(0, -(-new_len // self.page_tokens) - len(seq.pages))

    def reserve(self, seq: Sequence, new_len: int) -> None:
        """Give `seq` KV pages for positions [0, new_len) (CapacityError when the
        pool is short; the sequence keeps what it had)."""
        need = self.pages_needed(seq, new_len)
        if need > 0:
            seq.pages.extend(self.pool.alloc(need))

    _reserve = reserve

    def _meta(self, seqs, lens):
        n_tok = int(sum(lens))
        tok_seq = np.empty(n_tok, np.int32)
        tok_pos = np.empty(n_tok, np.int32)
        pages = np.zeros((len(seqs), self.max_pages), np.int32)
        o = 0
        for i, (s, t) in enumerate(zip(seqs, lens)):
            tok_seq[o:o + t] = i
            tok_pos[o:o + t] = np.arange(s.length, s.length + t, dtype=np.int32)
            pages[i, : len(s.pages)] = s.pages
            o += t
        return n_tok, tok_seq, tok_pos, pages

    def step(self, items, out=None):
        """One batched step. items: [(Sequence, hidden [t, d] cuda f32)];
        returns the outputs in order (views of one [n_tok, d] tensor).

        A step larger than the span's workspace (more than max_tokens new
        positions or max_seqs sequences) runs as consecutive causal chunks;
        the reference accepts any t <= max_seq in one STEP (server.py:361-390).
        It is all-or-nothing: if a chunk fails, every sequence is rolled back
        to its length before the call."""
        import torch

        seqs = [s for s, _ in items]
        lens = [int(h.shape[0]) for _, h in items]
        if len(set(map(id, seqs))) != len(seqs):
            raise InputError("a sequence may appear once per step")
        d = self.config.hidden
        for s, t in zip(seqs, lens):
            if t < 1:
                raise InputError("empty step")
            if s.length + t > self.config.max_seq:
                raise CapacityError(f"position {s.length + t} exceeds max_seq {self.config.max_seq}")
        if sum(lens) > self.max_tokens or len(items) > self.max_seqs:
            return self._step_chunked(items, lens)
        with self._lock:
            for s, t in zip(seqs, lens):
                self._reserve(s, s.length + t)
            n_tok, tok_seq, tok_pos, pages = self._meta(seqs, lens)
            x = items[0][1] if len(items) == 1 else torch.cat([h for _, h in items])
            x = x.to(device=self.device, dtype=torch.float32).contiguous()
            if x.shape != (n_tok, d):
                raise InputError(f"hidden must be [t, {d}]")
            y = out if out is not None else torch.empty_like(x)
            st = _lib.stream_ptr(torch.cuda.current_stream(self.device))
            _lib.check(_lib.lib().pb_span_step(self._h, n_tok, len(seqs), tok_seq.ctypes.data, tok_pos.ctypes.data,
                                               pages.ctypes.data, _lib.ptr(x), _lib.ptr(y), st))
            for s, t in zip(seqs, lens):
                s.length += t
        return list(torch.split(y, lens))

    def _step_chunked(self, items, lens):
        """Each sequence's new positions in causal chunks of at most max_tokens,
        up to max_seqs sequences per launch sequence."""
        import torch

        start = [s.length for s, _ in items]
        outs = [[] for _ in items]
        done = [0] * len(items)
        try:
            while True:
                group, budget = [], self.max_tokens
                for i, ((s, h), t) in enumerate(zip(items, lens)):
                    if done[i] < t and budget > 0 and len(group) < self.max_seqs:
                        c = min(t - done[i], budget)
                        group.append((i, c))
                        budget -= c
                if not group:
                    break
                res = self.step([(items[i][0], items[i][1][done[i]:done[i] + c]) for i, c in group])
                for (i, c), y in zip(group, res):
                    outs[i].append(y)
                    done[i] += c
        except Exception:
            for (s, _), L in zip(items, start):
                s.length = L
            raise
        return [o[0] if len(o) == 1 else torch.cat(o) for o in outs]

    def step_codes(self, seqs, lens, in_codes=None, in_scales=None, in_f32=None, out_codes=None, out_scales=None,
                   out_f32=None, tape=None):
        """Batched step whose input and/or output hidden states are the wire
        codec (codes [n_tok*d] int8, scales [ceil(n_tok*d/64)] f32) on the
        device (pb_span_step_int8): the span-to-span hop payload. Sequences'
        tokens are concatenated in `seqs` order (lens[i] new positions each).
        tape (nullable, [n_blocks, n_tok, d] f32): record the FORWARD tape."""
        import torch

        with self._lock:
            for s, t in zip(seqs, lens):
                self._reserve(s, s.length + t)
            n_tok, tok_seq, tok_pos, pages = self._meta(seqs, lens)
            st = _lib.stream_ptr(torch.cuda.current_stream(self.device))
            _lib.check(_lib.lib().pb_span_step_int8(
                self._h, n_tok, len(seqs), tok_seq.ctypes.data, tok_pos.ctypes.data, pages.ctypes.data,
                _lib.ptr(in_codes), _lib.ptr(in_scales), _lib.ptr(in_f32), _lib.ptr(out_codes), _lib.ptr(out_scales),
                _lib.ptr(out_f32), _lib.ptr(tape), st))
            for s, t in zip(seqs, lens):
                s.length += t

    def forward(self, batch, tape: bool = False):
        """Cache-less forward of independent rows (server.py:411-429 semantics):
        batch [B, t, d] -> [B, t, d]. Rows are packed into steps of up to
        max_tokens positions with temporary KV pages. With tape=True also
        returns the FORWARD tape [B, n_blocks, t, d] (each hosted block's input
        rows) that `backward` consumes."""
        import torch

        B, t, d = batch.shape
        if t > self.config.max_seq:
            raise CapacityError(f"t={t} exceeds max_seq")
        out = torch.empty_like(batch)
        # rows packed per launch sequence; a row longer than the workspace runs
        # alone in causal chunks of max_tokens positions (its KV pages persist
        # across the chunks)
        per = max(1, min(self.max_seqs, self.max_tokens // t)) if t <= self.max_tokens else 1
        tp = torch.empty(B, self.n_blocks, t, d, device=self.device) if tape else None
        for r0 in range(0, B, per):
            rows = range(r0, min(B, r0 + per))
            seqs = [Sequence() for _ in rows]
            try:
                if tape:
                    n = len(rows)
                    step_t = min(t, self.max_tokens)
                    for c0 in range(0, t, step_t):
                        c = min(step_t, t - c0)
                        x = batch[r0:r0 + n, c0:c0 + c].reshape(n * c, d).to(device=self.device,
                                                                              dtype=torch.float32).contiguous()
                        y = torch.empty_like(x)
                        buf = torch.empty(self.n_blocks, n * c, d, device=self.device)
                        with self._lock:
                            for s in seqs:
                                self._reserve(s, c0 + c)
                            n_tok, tok_seq, tok_pos, pages = self._meta(seqs, [c] * n)
                            st = _lib.stream_ptr(torch.cuda.current_stream(self.device))
                            _lib.check(_lib.lib().pb_span_step_tape(
                                self._h, n_tok, n, tok_seq.ctypes.data, tok_pos.ctypes.data, pages.ctypes.data,
                                _lib.ptr(x), _lib.ptr(y), _lib.ptr(buf), st))
                            for s in seqs:
                                s.length += c
                        out[r0:r0 + n, c0:c0 + c] = y.view(n, c, d)
                        tp[r0:r0 + n, :, c0:c0 + c] = buf.view(self.n_blocks, n, c, d).transpose(0, 1)
                else:
                    res = self.step([(s, batch[r]) for s, r in zip(seqs, rows)])
                    for r, y in zip(rows, res):
                        out[r] = y
            finally:
                for s in seqs:
                    self.release(s)
        return (out, tp) if tape else out

    def backward(self, tape, grad):
        """BACKWARD (server.py:431-450): dL/d(span input) [B, t, d] from the
        FORWARD tape [B, n_blocks, t, d] and dL/d(span output) [B, t, d], one
        row at a time through the hosted blocks in reverse (model.py:383-418)."""
        import torch

        B, nb, t, d = tape.shape
        if nb != self.n_blocks or grad.shape != (B, t, d):
            raise InputError("BACKWARD grad shape mismatch")
        g = grad.to(device=self.device, dtype=torch.float32).contiguous()
        tape = tape.contiguous()
        out = torch.empty_like(g)
        st = _lib.stream_ptr(torch.cuda.current_stream(self.device))
        for r in range(B):
            _lib.check(_lib.lib().pb_span_backward(self._h, _lib.ptr(tape[r]), t, _lib.ptr(g[r]), _lib.ptr(out[r]),
                                                   st))
        return out
