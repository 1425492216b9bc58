"""Model shape and deterministic-weight addressing.

ModelConfig restates /root/reference/pkg/src/swarmlm/model.py:65-84 (same
fields, same validation); stream keys restate model.py:47-51,60-62 so that the
on-device generator (pb_gen_tensor / pb_span_gen_block) reproduces
gen_checkpoint (model.py:176-209) bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import InputError

LN_EPS = 1e-5
MASK64 = (1 << 64) - 1
MATRICES = ("wqkv", "wo", "wmlp_in", "wmlp_out")


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int
    hidden: int
    n_heads: int
    vocab: int
    max_seq: int
    mlp_ratio: int = 4

    def __post_init__(self):
        if self.n_layers < 1 or self.hidden < 1 or self.n_heads < 1:
            raise InputError("layers, hidden and heads must be positive")
        if self.vocab < 1 or self.max_seq < 1 or self.mlp_ratio < 1:
            raise InputError("vocab, max_seq and mlp_ratio must be positive")
        if self.hidden % self.n_heads != 0:
            raise InputError("hidden must be a multiple of n_heads")

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & MASK64
    return h


def stream_key(seed: int, path: str) -> int:
    """SplitMix64 key of tensor `path` (model.py:62): seed ^ fnv1a64(path)."""
    return (seed ^ fnv1a64(path.encode())) & MASK64


def block_keys(seed: int, block: int) -> tuple[int, int, int, int]:
    return tuple(stream_key(seed, f"blocks.{block}.{m}") for m in MATRICES)


# Named shapes of BASELINE.json's configs.
SHAPES = {
    "tiny": ModelConfig(n_layers=2, hidden=8, n_heads=2, vocab=32, max_seq=64),
    "small": ModelConfig(n_layers=4, hidden=16, n_heads=2, vocab=32, max_seq=128),
    "bloom-560m": ModelConfig(n_layers=24, hidden=1024, n_heads=16, vocab=250880, max_seq=2048),
    "bloom-7b1": ModelConfig(n_layers=30, hidden=4096, n_heads=32, vocab=250880, max_seq=2048),
    "bloom-176b": ModelConfig(n_layers=70, hidden=14336, n_heads=112, vocab=250880, max_seq=2048),
}
