"""Attention-only timing probe: one block of a named shape, batch decode at a
synthetic context; prints the live per-launch device time of the attention
kernel (CUDA events, PROF_ATTN) and of the GEMVs.

  python tools/attn_probe.py [--ctx 2048] [--steps 20] [--batch 1]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--ctx", type=int, default=2048)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--batch", type=int, default=1)
    args = p.parse_args()
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[args.shape]
    span = BlockSpan(cfg, 0, 1, int8=True, page_tokens=64, n_pages=args.batch * 33 + 2, max_tokens=64,
                     max_seqs=max(args.batch, 1))
    span.generate_weights(42)
    seqs = [span.new_sequence() for _ in range(args.batch)]
    for s in seqs:
        span._reserve(s, args.ctx - args.steps - 4)
        s.length = args.ctx - args.steps - 4
    x = torch.randn(args.batch, cfg.hidden, device="cuda") * 0.05
    for _ in range(3):
        span.step([(s, x[i:i + 1]) for i, s in enumerate(seqs)])
    span.profile(True)
    for _ in range(args.steps):
        span.step([(s, x[i:i + 1]) for i, s in enumerate(seqs)])
    torch.cuda.synchronize()
    ms, n, b = span.profile_read(span.PROF_ATTN)
    gms, gn, gb = span.profile_read(span.PROF_GEMV)
    print(f"batch {args.batch} ctx {args.ctx}: attention {1e3 * ms / n:.1f} us/launch, {b / n / 1e6:.1f} MB/launch, "
          f"{b / (ms / 1e3) / 1e9:.0f} GB/s | gemv {1e3 * gms / gn:.1f} us/launch, {gb / (gms / 1e3) / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main()
