"""BACKWARD time per block and row, with the matmul share as
useful tensor TFLOP/s: per block and row of t positions the recompute runs
qkv, wo, mlp_in (8 h^2 weights) and the backward all four matrices
(12 h^2), 2 t 20 h^2 useful flops.

  python tools/backward_probe.py --shape bloom-176b --blocks 2 --rows 128,512,2048
  PB_LIB=paper_2209_01188_b200/build/bwd_old/libpetals_b200.so python tools/backward_probe.py ...  (A/B)
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--blocks", type=int, default=2)
    p.add_argument("--rows", default="128,512,2048")
    p.add_argument("--reps", type=int, default=3)
    args = p.parse_args()
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[args.shape]
    h, L = cfg.hidden, args.blocks
    rows = [int(r) for r in args.rows.split(",")]
    span = BlockSpan(cfg, 0, L, int8=True, page_tokens=64, n_pages=max(rows) // 64 + 4, max_tokens=256, max_seqs=8)
    span.generate_weights(42)
    g = torch.Generator(device="cuda").manual_seed(1)
    for t in rows:
        x = torch.randn(1, t, h, device="cuda", generator=g) * 0.05
        gr = torch.rand(1, t, h, device="cuda", generator=g) * 2 - 1
        _, tape = span.forward(x, tape=True)
        span.backward(tape, gr)  # warm-up (allocations, kernel setup)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            out = span.backward(tape, gr)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps / L
        flops = 2.0 * t * 20 * h * h
        print(f"{args.shape} t={t:5d}: {ms:9.2f} ms per block  {t / ms * 1e3:9.0f} positions/s per block  "
              f"{flops / (ms / 1e3) / 1e12:7.1f} useful matmul TFLOP/s  finite={bool(torch.isfinite(out).all())}",
              flush=True)
        del tape, out
        torch.cuda.empty_cache()
    span.close()


if __name__ == "__main__":
    main()
