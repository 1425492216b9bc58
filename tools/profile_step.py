"""Small driver for ncu: a span of a named shape decoding batch-1 steps at a
synthetic context (KV pages reserved, not prefilled — timing of the decode
kernels does not depend on KV values).

  python tools/profile_step.py --shape bloom-176b --blocks 2 --ctx 2048 --steps 3
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--blocks", type=int, default=2)
    p.add_argument("--ctx", type=int, default=2048)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--batch", type=int, default=1)
    args = p.parse_args()
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[args.shape]
    span = BlockSpan(cfg, 0, args.blocks, int8=True, page_tokens=64, n_pages=args.batch * 32 + 2, max_tokens=64,
                     max_seqs=max(args.batch, 1))
    span.generate_weights(42)
    seqs = [span.new_sequence() for _ in range(args.batch)]
    for s in seqs:
        span._reserve(s, args.ctx - args.steps - 1)
        s.length = args.ctx - args.steps - 1
    x = torch.randn(args.batch, cfg.hidden, device="cuda") * 0.05
    for _ in range(args.steps):
        span.step([(s, x[i:i + 1]) for i, s in enumerate(seqs)])
    torch.cuda.synchronize()
    print("ok", span.last_launches, "launches per step")


if __name__ == "__main__":
    main()
