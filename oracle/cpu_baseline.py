"""CPU baseline sample for bench.py (TEST/BENCH INFRASTRUCTURE ONLY).

Times the oracle's restatement of the reference int8 decode step
(swarm_oracle.block_step with the quantize='weights' path: full-matrix
dequantization + f32 matmul, exactly what quant.py:117-129 does) for ONE block
of a given shape at a given context length, on the host cores, and
extrapolates to the full model. Codes are random (the arithmetic, not the
values, is being timed), which skips the reference's slow Python quantizer.
"""

from __future__ import annotations

import os
import time

import numpy as np

import swarm_oracle as O


def _random_int8_matrix(rng, k_in: int, m_out: int) -> O.Int8Matrix:
    m = object.__new__(O.Int8Matrix)
    m.codes = rng.integers(-127, 128, size=(m_out, k_in), dtype=np.int8)
    m.scales = (rng.uniform(0.03, 0.05, size=k_in) / 127).astype(np.float32)
    m.outlier = np.zeros(k_in, bool)
    m.outlier_idx = np.zeros(0, np.int64)
    m.outlier_rows = np.zeros((0, m_out), np.float32)
    m.shape_in_out = (k_in, m_out)
    return m


class BlockSample:
    def __init__(self, hidden: int, n_heads: int, ctx: int, mlp_ratio: int = 4, seed: int = 0):
        rng = np.random.default_rng(seed)
        d, r = hidden, mlp_ratio
        self.shape = O.Shape(1, d, n_heads, 8, max(ctx + 1, 2), r)
        self.block = O.Block(None, None, None, None, d, r)
        q = object.__new__(O.QuantBlock)
        q.wqkv = _random_int8_matrix(rng, d, 3 * d)
        q.wo = _random_int8_matrix(rng, d, d)
        q.wmlp_in = _random_int8_matrix(rng, d, r * d)
        q.wmlp_out = _random_int8_matrix(rng, r * d, d)
        self.qblock = q
        self.ctx = ctx
        dh = d // n_heads
        self.k0 = rng.normal(size=(ctx - 1, n_heads, dh)).astype(np.float32)
        self.v0 = rng.normal(size=(ctx - 1, n_heads, dh)).astype(np.float32)
        self.x = rng.normal(size=(1, d)).astype(np.float32)

    def step_seconds(self) -> float:
        kv = O.KV(self.shape)
        kv.k, kv.v = self.k0, self.v0
        t0 = time.perf_counter()
        O.block_step(self.block, self.x, kv, self.ctx - 1, self.shape, self.qblock)
        return time.perf_counter() - t0


def cores() -> int:
    return os.cpu_count() or 1
