"""Client-side head on the GPU: the reference client's
`embed` (model.py:421-425), `lm_head` (model.py:428-433) and greedy
`sample_next` (model.py:437-446), as used by `SwarmClient.generate`
(client.py:247-250), over the C-ABI head (include/petals_b200.h pb_head_*).

Greedy decoding streams an int8 copy of the tied embedding (the block
matrices' LLM.int8 layout) and rescoring its candidates exactly, so the
chosen token is the argmax of the exact logits (pb_head.cu header).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import InputError
from .model import ModelConfig, stream_key


class ClientHead:
    def __init__(self, config: ModelConfig, *, max_tokens: int = 32, device: int = 0):
        import torch

        self.config = config
        self.device = torch.device("cuda", device)
        self.max_tokens = max_tokens
        h = C.c_void_p()
        torch.cuda.init()
        _lib.check(_lib.lib().pb_head_create(config.vocab, config.hidden, max_tokens, device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().pb_head_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    @property
    def device_bytes(self) -> int:
        return int(_lib.lib().pb_head_device_bytes(self._h))

    def _stream(self):
        import torch

        return _lib.stream_ptr(torch.cuda.current_stream(self.device))

    # ------------------------------------------------------------------ weights

    def generate_weights(self, seed: int) -> None:
        """gen_checkpoint's embed (model.py:190) and final LN (gamma 1, beta 0)."""
        _lib.check(_lib.lib().pb_head_gen(self._h, stream_key(seed, "embed"), self._stream()))

    def load_weights(self, embed, final_ln_gamma, final_ln_beta) -> None:
        import torch

        d, V = self.config.hidden, self.config.vocab
        e = torch.as_tensor(np.asarray(embed, np.float32)).reshape(V, d).to(self.device)
        g = torch.as_tensor(np.asarray(final_ln_gamma, np.float32)).to(self.device)
        b = torch.as_tensor(np.asarray(final_ln_beta, np.float32)).to(self.device)
        _lib.check(_lib.lib().pb_head_load(self._h, _lib.ptr(e), _lib.ptr(g), _lib.ptr(b), self._stream()))

    # ------------------------------------------------------------------ compute

    def _rows(self, hidden):
        import torch

        x = torch.as_tensor(hidden).to(device=self.device, dtype=torch.float32)
        if x.ndim != 2 or x.shape[1] != self.config.hidden:
            raise InputError("hidden must be [t, d]")
        if x.shape[0] > self.max_tokens:
            raise InputError(f"at most {self.max_tokens} rows per call")
        return x.contiguous()

    def embed(self, tokens):
        """model.py:421-425: [t, d] f32 rows of the embedding (InputError if out of range)."""
        import torch

        tok = np.ascontiguousarray(np.asarray(tokens, np.int64).reshape(-1))
        if tok.size and (tok.min() < 0 or tok.max() >= self.config.vocab):
            raise InputError("token out of range")
        out = torch.empty(tok.size, self.config.hidden, device=self.device)
        for i in range(0, tok.size, self.max_tokens):
            part = np.ascontiguousarray(tok[i:i + self.max_tokens], np.int32)
            _lib.check(_lib.lib().pb_head_embed(self._h, part.ctypes.data, part.size, _lib.ptr(out[i:]),
                                                self._stream()))
        return out

    def lm_head(self, hidden):
        """model.py:428-433: logits [t, V] f32 of the final LN'd rows (f64 accumulation)."""
        import torch

        x = self._rows(hidden)
        out = torch.empty(x.shape[0], self.config.vocab, device=self.device)
        _lib.check(_lib.lib().pb_head_logits(self._h, _lib.ptr(x), x.shape[0], _lib.ptr(out), self._stream()))
        return out

    def greedy_device(self, hidden, tokens_out, next_embed=None) -> None:
        """Greedy token of every row into the int32 device tensor `tokens_out`
        (-1 = non-finite logits), optionally writing their embedding rows."""
        x = self._rows(hidden)
        _lib.check(_lib.lib().pb_head_greedy(self._h, _lib.ptr(x), x.shape[0], _lib.ptr(tokens_out),
                                             _lib.ptr(next_embed), self._stream()))

    def greedy(self, hidden) -> list[int]:
        """sample_next(lm_head(hidden)[i], "greedy") for every row i (model.py:437-446)."""
        import torch

        x = self._rows(hidden)
        tok = torch.empty(x.shape[0], dtype=torch.int32, device=self.device)
        self.greedy_device(x, tok)
        out = tok.cpu().tolist()
        if any(t < 0 for t in out):
            raise InputError("non-finite logits")
        return out


def generate(spans, head: ClientHead, prompt_tokens, max_new_tokens: int) -> list[int]:
    """SwarmClient.generate (client.py:230-257) with every hop local: the
    prompt is prefilled through the spans in order, then one greedy token per
    step; the hidden state stays on the device between spans."""
    prompt = list(prompt_tokens)
    if not prompt:
        raise InputError("empty prompt")
    seqs = [s.new_sequence() for s in spans]
    try:
        out: list[int] = []
        pending = prompt
        for _ in range(max_new_tokens):
            h = head.embed(pending)
            for span, seq in zip(spans, seqs):
                h = span.step([(seq, h)])[0]
            nxt = head.greedy(h[-1:])[0]
            out.append(nxt)
            pending = [nxt]
        return out
    finally:
        for span, seq in zip(spans, seqs):
            span.release(seq)
