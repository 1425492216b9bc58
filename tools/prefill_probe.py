"""Prefill / FORWARD probe: one block of a named shape, a fresh sequence
prefilled in chunks of --chunk tokens; prints the live tcgen05 GEMM time and
rate (CUDA events, profile kind 5) and the wall tokens/s.

  python tools/prefill_probe.py [--chunk 256] [--tokens 1024] [--blocks 1]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--chunk", type=int, default=256)
    p.add_argument("--tokens", type=int, default=1024)
    p.add_argument("--blocks", type=int, default=1)
    p.add_argument("--rows", type=int, default=1, help="independent sequences per step")
    args = p.parse_args()
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[args.shape]
    per = -(-args.tokens // 64) + 1
    span = BlockSpan(cfg, 0, args.blocks, int8=True, page_tokens=64, n_pages=args.rows * per + 2,
                     max_tokens=args.chunk * args.rows, max_seqs=args.rows)
    span.generate_weights(42)
    x = torch.randn(args.chunk * args.rows, cfg.hidden, device="cuda") * 0.05

    def run(profile):
        seqs = [span.new_sequence() for _ in range(args.rows)]
        span.profile(profile)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(0, args.tokens, args.chunk):
            span.step([(s, x[i * args.chunk:(i + 1) * args.chunk]) for i, s in enumerate(seqs)])
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        for s in seqs:
            span.release(s)
        return wall

    run(False)
    wall = run(False)
    run(True)
    ms, n, ops = span.profile_read(5)
    att_ms, att_n, _ = span.profile_read(span.PROF_ATTN)
    tok = args.tokens * args.rows
    print(f"{args.shape} x{args.blocks} blocks, {args.rows} rows x {args.tokens} tokens in chunks of {args.chunk}: "
          f"{tok / wall:.0f} tokens/s wall | tcgen05: {n} launches {ms:.2f} ms, {ops / ms / 1e9:.0f} int8 TOPS issued, "
          f"{ops / 3 / ms / 1e9:.0f} useful TFLOP/s | attention {att_ms:.2f} ms over {att_n} launches")


if __name__ == "__main__":
    main()
